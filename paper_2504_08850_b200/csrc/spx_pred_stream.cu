// Translation unit of the STREAM fused predictor kernel family (K <= 8, bf16
// head, d in {2048, 4096, 8192}); dispatched by spx_predictor.cu.
#include "spx_pred_common.cuh"
namespace spx {
#include "spx_pred_fast.cuh"
#include "spx_pred_stream.cuh"

int launch_stream_bf16(const PredParams &p, const StreamPlan &sp, int grid, cudaStream_t stream,
                       int smem_optin, bool ldgx) {
  StreamLaunch<__nv_bfloat16> L{p, sp, grid, stream, smem_optin, ldgx};
  if (p.d == 2048) L.template operator()<4>();
  else if (p.d == 4096) L.template operator()<8>();
  else L.template operator()<16>();
  return spx_launch_status("spx_predictor_eval");
}
}  // namespace spx
