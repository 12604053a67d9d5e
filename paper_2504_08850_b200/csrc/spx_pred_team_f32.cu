// Translation unit of the TEAM fused predictor kernel family (any K <= 64,
// any d): f32 head; dispatched by spx_predictor.cu.
#include "spx_pred_common.cuh"
namespace spx {
#include "spx_pred_fast.cuh"

template <typename TW, int CPL>
int launch_team_cpl(const PredParams &p, const SmemPlan &sp, int grid, cudaStream_t stream,
                    int smem_optin) {
  FastLaunch<TW>{p, sp, grid, stream, smem_optin}.template operator()<CPL>();
  return spx_launch_status("spx_predictor_eval");
}
template int launch_team_cpl<float, 1>(const PredParams &, const SmemPlan &, int, cudaStream_t, int);
template int launch_team_cpl<float, 2>(const PredParams &, const SmemPlan &, int, cudaStream_t, int);
template int launch_team_cpl<float, 4>(const PredParams &, const SmemPlan &, int, cudaStream_t, int);
template int launch_team_cpl<float, 8>(const PredParams &, const SmemPlan &, int, cudaStream_t, int);
template int launch_team_cpl<float, 16>(const PredParams &, const SmemPlan &, int, cudaStream_t, int);
}  // namespace spx
