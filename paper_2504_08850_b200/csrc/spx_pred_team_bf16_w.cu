// Translation unit of the WIDE-ROW team kernel variant: the TEAM fused
// predictor kernel (spx_pred_fast.cuh) with 2 DOT teams instead of 4, for bf16
// heads whose rows are too wide for the 4-team ring (d = 8192 with K > 8:
// 4 teams x 2 units x 2 rows x 16 KB do not fit in shared memory).  Same
// arithmetic (canonical CDOT, FAST certification); only the team count
// differs.  Lives in namespace spx::wide so its constants and kernels do not
// collide with the 4-team family.
#include "spx_pred_common.cuh"
#define SPX_FAST_NTEAM 2
namespace spx {
namespace wide {
#include "spx_pred_fast.cuh"
}  // namespace wide

// Plan + launch (CPL 16: 4096 < d <= 8192); SPX_EINVAL when it does not fit.
int launch_team_wide_bf16(const PredParams &p0, int smem_optin, int sms, cudaStream_t stream,
                          bool &inline_rc) {
  using namespace wide;
  PredParams p = p0;
  if (p.d <= 4096 || p.d > 8192) return SPX_EINVAL;
  SmemPlan sp = plan_smem<__nv_bfloat16>(p.d, p.K, p.H, smem_optin);
  if (sp.bytes == 0) return SPX_EINVAL;
  const size_t rscr = recheck_scratch_bytes(p.d, p.K);
  inline_rc = p.recheck && rscr <= sp.off_bar;
  p.recheck_inline = inline_rc ? 1 : 0;
  const long long need = (p.B + NTEAM - 1) / NTEAM;
  const int grid = (int)(need < sms ? need : sms);
  FastLaunch<__nv_bfloat16>{p, sp, grid > 0 ? grid : 1, stream, smem_optin}.template operator()<16>();
  return spx_launch_status("spx_predictor_eval");
}

bool team_wide_fits(int d, int K, int H, int smem_optin) {
  return d > 4096 && d <= 8192 &&
         wide::plan_smem<__nv_bfloat16>(d, K, H, smem_optin).bytes != 0;
}
}  // namespace spx
