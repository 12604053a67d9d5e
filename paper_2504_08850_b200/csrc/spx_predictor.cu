#include "spx_pred_common.cuh"
namespace spx {
#include "spx_pred_fast.cuh"
#include "spx_pred_stream.cuh"
}  // namespace spx

namespace spx {

// the wide-row (2-team) variant, spx_pred_team_bf16_w.cu
int launch_team_wide_bf16(const PredParams &p, int smem_optin, int sms, cudaStream_t stream,
                          bool &inline_rc);
bool team_wide_fits(int d, int K, int H, int smem_optin);

// FAST kernel families, one translation unit each (spx_pred_stream.cu,
// spx_pred_team.cu)
int launch_stream_bf16(const PredParams &p, const StreamPlan &sp, int grid, cudaStream_t stream,
                       int smem_optin, bool ldgx);
template <typename TW, int CPL>
int launch_team_cpl(const PredParams &p, const SmemPlan &sp, int grid, cudaStream_t stream,
                    int smem_optin);
template <typename TW>
int launch_team(const PredParams &p, const SmemPlan &sp, int grid, cudaStream_t stream,
                int smem_optin) {
  const int nchunk = p.d / CHUNK;
  if (nchunk <= NPART * 1) return launch_team_cpl<TW, 1>(p, sp, grid, stream, smem_optin);
  if (nchunk <= NPART * 2) return launch_team_cpl<TW, 2>(p, sp, grid, stream, smem_optin);
  if (nchunk <= NPART * 4) return launch_team_cpl<TW, 4>(p, sp, grid, stream, smem_optin);
  if (nchunk <= NPART * 8) return launch_team_cpl<TW, 8>(p, sp, grid, stream, smem_optin);
  if (nchunk <= NPART * 16) return launch_team_cpl<TW, 16>(p, sp, grid, stream, smem_optin);
  return SPX_EINVAL;
}

template <typename TW>
__global__ void __launch_bounds__(STRICT_THREADS)
predictor_strict_kernel(PredParams p) {
  const int row = blockIdx.x;
  if (row >= p.B) return;
  if (row_skipped(p, row)) {
    if (threadIdx.x == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  __shared__ int ids_s[MAXK];
  __shared__ float s_stat[2];
  __shared__ int s_flag;
  strict_row<TW>(p, row, dsm, feats, hs, ids_s, s_stat, &s_flag);
  if (threadIdx.x == 0 && p.prev_err) p.prev_err[row] = 0.f;
}

// STRICT re-evaluation of deferred rows as its own launch: used when the
// FAST kernel's shared memory cannot hold the re-evaluation scratch (its
// epilogue then leaves the flagged rows).  Scans the row flags.
template <typename TW>
__global__ void __launch_bounds__(STRICT_THREADS)
predictor_recheck_kernel(PredParams p) {
  if (p.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  extern __shared__ __align__(16) uint8_t dsm[];
  float *scr = reinterpret_cast<float *>(dsm);
  for (int row = blockIdx.x; row < p.B; row += gridDim.x) {
    if (*(volatile int *)(p.recheck + 5 + row)) {
      __syncthreads();
      if (threadIdx.x == 0) p.recheck[5 + row] = 0;
      recheck_row<TW>(p, row, scr);
    }
  }
}

// spx_predictor_cert: per-layer constants of the bound (see certify_row).
__global__ void predictor_cert_kernel(const float *w1, const float *b1, const float *w2, int K,
                                      int H, float *cert) {
  const int i = blockIdx.x, lane = threadIdx.x;   // one warp per output
  const int n = 3 * K;
  float s = 0.f;
  if (i < n) {
    for (int j = lane; j < H; j += 32) s = fmaf(fabsf(w2[j]), fabsf(w1[(size_t)i * H + j]), s);
  } else if (i == n) {
    for (int j = lane; j < H; j += 32) s = fmaf(fabsf(w2[j]), fabsf(b1[j]), s);
  } else {
    for (int j = lane; j < H; j += 32) s += fabsf(w2[j]);
  }
  s = warp_butterfly_sum(s);
  if (lane == 0) cert[i] = s * 1.0001f;            // rounded up past the sum's own error
}

// ---------------------------------------------------------------------------
// Function-level operators (the reference's extract_features and
// predictor_forward called on their own, predictor.py:42-52 / :97-103).  They
// run the same warp code as the fused kernel, so results are identical.

__global__ void features_kernel(const float *logits, float *prev, float *feats_out, int *err,
                                int B, int K) {
  const int row = blockIdx.x;
  if (row >= B) return;
  __shared__ float feats[3 * MAXK];
  PredParams p{};
  p.prev = prev; p.err = err; p.K = K;
  for (int i = threadIdx.x; i < K; i += 32) feats[i] = logits[(size_t)row * K + i];
  __syncwarp();
  if (!warp_softmax_features(p, row, feats, threadIdx.x)) return;
  for (int i = threadIdx.x; i < 3 * K; i += 32) feats_out[(size_t)row * 3 * K + i] = feats[i];
}

// extract_features for wide speculative sets (K > MAXK: the spec_full_vocab
// ablation, engine.py:166-168).  One CTA per row, working in feats_out; the
// two sums stay the reference's strict left-to-right chains (thread 0).
__global__ void features_wide_kernel(const float *logits, const float *prev, float *feats_out,
                                     int *err, int K) {
  const int row = blockIdx.x, tid = threadIdx.x;
  const float *x = logits + (size_t)row * K, *pv = prev + (size_t)row * K;
  float *f = feats_out + (size_t)row * 3 * K;
  __shared__ float s_red[32];
  __shared__ int s_bad;
  __shared__ float s_esum;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  float m = -INFINITY;
  for (int i = tid; i < K; i += blockDim.x) {
    const float v = x[i];
    if (!is_finite(v)) s_bad = 1;
    m = fmaxf(m, v);
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((tid & 31) == 0) s_red[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    float mm = s_red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmaxf(mm, s_red[w]);
    s_red[0] = mm;
  }
  __syncthreads();
  m = s_red[0];
  for (int i = tid; i < K; i += blockDim.x) {
    f[i] = x[i];
    f[K + i] = np_expf(__fsub_rn(x[i], m));
  }
  __syncthreads();
  // the softmax denominator stays the strict left-to-right chain on thread 0
  // (operands staged through shared memory in chunks so the chain never waits
  // on HBM); the prev check is numpy's pairwise sum (predictor.py:49)
  constexpr int WCH = 2048;
  __shared__ float s_e[WCH];
  float esum = 0.f;
  for (int c0 = 0; c0 < K; c0 += WCH) {
    const int n = K - c0 < WCH ? K - c0 : WCH;
    for (int i = tid; i < n; i += blockDim.x) s_e[i] = f[K + c0 + i];
    __syncthreads();
    if (tid == 0) {
#pragma unroll 8
      for (int c = 0; c < n; ++c) esum = __fadd_rn(esum, s_e[c]);
    }
    __syncthreads();
  }
  constexpr int MAXLEAF = 2560;                 // K <= ~150k without the serial fallback
  __shared__ int2 s_leaf[MAXLEAF];
  __shared__ float s_lsum[MAXLEAF];
  __shared__ int s_nleaf;
  __shared__ float s_psum;
  const float psum = np_pairwise_sum_cta(0, K, [&](int i) { return pv[i]; }, s_leaf, s_lsum,
                                         MAXLEAF, &s_nleaf, &s_psum);
  if (tid == 0) {
    int e = 0;
    if (s_bad) e |= ERR_LOGIT_NONFINITE;
    if (fabs((double)psum - 1.0) > 1e-5) e |= ERR_PREV_SUM;
    if (e) atomicOr(err, e);
    s_bad = e;
    s_esum = esum;
  }
  __syncthreads();
  if (s_bad) return;
  for (int i = tid; i < K; i += blockDim.x) {
    const float pr = __fdiv_rn(f[K + i], s_esum);
    f[K + i] = pr;
    f[2 * K + i] = __fsub_rn(pr, pv[i]);
  }
}

// softmax_1d (model.py:149-152) of each row of n logits, evaluated only at K
// requested ids (the draft proposal's probabilities, speculation.py:80-84):
// the same max, np_expf and strict left-to-right denominator as
// features_wide_kernel -- bit-identical probabilities -- without the
// prev-sum check and the 3n feature writes.  The chain runs on thread 0 over
// shared-memory chunks that warps 1.. fill one chunk ahead.
__global__ void __launch_bounds__(256) softmax_pick_kernel(const float *logits, int n,
                                                           const int32_t *ids, int K,
                                                           float *probs_out, int mode, int *err) {
  constexpr int WCH = 2048;
  __shared__ __align__(16) float s_e[2][WCH];
  __shared__ float s_red[8];
  __shared__ int s_bad;
  __shared__ float s_sum;
  const int row = blockIdx.x, tid = threadIdx.x;
  const float *x = logits + (size_t)row * n;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  float m = -INFINITY;
  for (int i = tid; i < n; i += blockDim.x) {
    const float v = x[i];
    if (!is_finite(v)) s_bad = 1;
    m = fmaxf(m, v);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) s_red[tid >> 5] = m;
  __syncthreads();
  m = s_red[0];
  for (int w = 1; w < 8; ++w) m = fmaxf(m, s_red[w]);
  if (mode != SPX_MODE_STRICT) {
    // FAST: the denominator as a fixed-order block sum (each thread's strided
    // share, then the warp and CTA trees) -- the FAST contract's tolerance,
    // not the reference's left-to-right chain
    float part = 0.f;
    for (int i = tid; i < n; i += blockDim.x) part += np_expf(__fsub_rn(x[i], m));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __syncthreads();
    if ((tid & 31) == 0) s_red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t += s_red[w];
      s_sum = t;
      if (s_bad) atomicOr(err, ERR_LOGIT_NONFINITE);
    }
    __syncthreads();
    for (int j = tid; j < K; j += blockDim.x) {
      const int id = ids[(size_t)row * K + j];
      if (id < 0 || id >= n) {
        atomicOr(err, ERR_ID_RANGE);
        probs_out[(size_t)row * K + j] = 0.f;
        continue;
      }
      probs_out[(size_t)row * K + j] = __fdiv_rn(np_expf(__fsub_rn(x[id], m)), s_sum);
    }
    return;
  }
  const int nch = (n + WCH - 1) / WCH;
  for (int i = tid; i < (n < WCH ? n : WCH); i += blockDim.x) s_e[0][i] = np_expf(__fsub_rn(x[i], m));
  __syncthreads();
  float esum = 0.f;
  for (int c = 0; c < nch; ++c) {
    if (tid == 0) {
      const int len = n - c * WCH < WCH ? n - c * WCH : WCH;
      const float *e = s_e[c & 1];
      const float4 *e4 = reinterpret_cast<const float4 *>(e);
      int j = 0;
#pragma unroll 4
      for (; j + 4 <= len; j += 4) {                // 16-byte loads, the chain stays sequential
        const float4 q = e4[j >> 2];
        esum = __fadd_rn(esum, q.x);
        esum = __fadd_rn(esum, q.y);
        esum = __fadd_rn(esum, q.z);
        esum = __fadd_rn(esum, q.w);
      }
      for (; j < len; ++j) esum = __fadd_rn(esum, e[j]);
    } else if (tid >= 32 && c + 1 < nch) {
      const int b = (c + 1) * WCH, len = n - b < WCH ? n - b : WCH;
      for (int j = tid - 32; j < len; j += blockDim.x - 32)
        s_e[(c + 1) & 1][j] = np_expf(__fsub_rn(x[b + j], m));
    }
    __syncthreads();
  }
  if (tid == 0) {
    s_sum = esum;
    if (s_bad) atomicOr(err, ERR_LOGIT_NONFINITE);
  }
  __syncthreads();
  for (int j = tid; j < K; j += blockDim.x) {
    const int id = ids[(size_t)row * K + j];
    if (id < 0 || id >= n) {                         // model.py:307-308
      atomicOr(err, ERR_ID_RANGE);
      probs_out[(size_t)row * K + j] = 0.f;
      continue;
    }
    probs_out[(size_t)row * K + j] = __fdiv_rn(np_expf(__fsub_rn(x[id], m)), s_sum);
  }
}

__global__ void mlp_kernel(PredParams p, const float *feats_in) {
  const int row = blockIdx.x;
  if (row >= p.B) return;
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  const int lane = threadIdx.x;
  for (int i = lane; i < 3 * p.K; i += 32) feats[i] = feats_in[(size_t)row * 3 * p.K + i];
  __syncwarp();
  const float z2 = warp_mlp(feats, p.w1, p.b1, p.w2, p.b2, p.K, p.H, hs, lane);
  if (lane == 0) {
    if (p.z_out) p.z_out[row] = z2;
    if (p.prob_out) p.prob_out[row] = sigmoid64(z2);
    write_fired(p, row, z2 >= p.z_cut);
  }
}

}  // namespace spx

using namespace spx;

static int g_sms = 0, g_smem_optin = 0;
static unsigned long long *g_debug_trace = nullptr;

// Debug hook (not part of the ABI contract): per-row globaltimer stamps of the
// fast predictor kernel, 8 u64 per row: issue(5) wait-start(0) data(1)
// pass1(2) dots(3) tail-done(4).  NULL disables.
extern "C" void spx_debug_trace(void *buf) {
  g_debug_trace = reinterpret_cast<unsigned long long *>(buf);
}
static void device_limits() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (g_sms <= 0) g_sms = 148;
    if (g_smem_optin <= 0) g_smem_optin = 227 * 1024;
  }
}

template <typename TW>
static int launch_fast(const PredParams &p, const spx_predictor_args *a, cudaStream_t stream,
                       bool &inline_rc);

template <typename TW>
static int launch_predictor(const PredParams &p, const spx_predictor_args *a, cudaStream_t stream) {
  device_limits();
  bool strict = a->mode == SPX_MODE_STRICT;
  if (!strict) {
    // FAST shapes that neither the stream nor the team kernel can stage in shared
    // memory (e.g. d = 8192 with K > 8) take the reference-order kernel: exact,
    // one CTA per request
    const bool stream_ok = std::is_same<TW, __nv_bfloat16>::value && p.K <= SKMAX &&
                           (p.d == 2048 || p.d == 4096 || p.d == 8192);
    const bool wide_ok = std::is_same<TW, __nv_bfloat16>::value &&
                         team_wide_fits(p.d, p.K, p.H, g_smem_optin);
    if (!stream_ok && !wide_ok && plan_smem<TW>(p.d, p.K, p.H, g_smem_optin).bytes == 0)
      strict = true;
  }
  if (strict) {
    const size_t smem = strict_smem_bytes(p.d, p.K);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(predictor_strict_kernel<TW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    predictor_strict_kernel<TW><<<(unsigned)a->B, STRICT_THREADS, smem, stream>>>(p);
  } else {
    bool inline_rc = false;
    const int rc = launch_fast<TW>(p, a, stream, inline_rc);
    if (rc) return rc;
    if (p.recheck && !inline_rc) {
      // STRICT re-evaluation of deferred rows as a separate launch (the FAST
      // kernel's shared memory could not hold its scratch)
      const size_t smem = recheck_scratch_bytes(p.d, p.K);
      static bool configured = false;
      if (!configured) {
        cudaFuncSetAttribute(predictor_recheck_kernel<TW>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        configured = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(p.B < g_sms ? p.B : g_sms));
      cfg.blockDim = dim3(STRICT_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = p.pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, predictor_recheck_kernel<TW>, p);
    }
  }
  return spx_launch_status("spx_predictor_eval");
}

template <typename TW>
static int launch_fast(const PredParams &p0, const spx_predictor_args *a, cudaStream_t stream,
                       bool &inline_rc) {
  PredParams p = p0;
  const size_t rscr = recheck_scratch_bytes(p.d, p.K);
  {
    if (((size_t)p.d * sizeof(TW)) % 16) return SPX_EINVAL;   // TMA bulk: 16-byte rows
    static const int env_stream = getenv("SPX_PRED_STREAM") ? atoi(getenv("SPX_PRED_STREAM")) : 3;
    if (std::is_same<TW, __nv_bfloat16>::value && env_stream && p.K <= SKMAX &&
        (p.d == 2048 || p.d == 4096 || p.d == 8192) && (p.policy != SPX_POLICY_MLP || p.H <= 1024)) {
      // env_stream: 1 = ring of whole evaluations, one CTA/SM; 2 = hidden rows by
      // ld.global, LM-head ring, two CTAs/SM
      // Two CTAs per SM whenever a 2-slot ring + W1 fit in half the shared
      // memory: hidden rows staged with the LM-head rows when the slot is small
      // (K <= 2 at d = 4096), else hidden rows by ld.global (LDGX, K <= 4);
      // otherwise one CTA per SM with the whole budget.  SPX_PRED_STREAM: 1 /
      // 2 force the staged / LDGX variant (sweeps), 3 = automatic.
      // (measured: with two CTAs per SM the ld.global hidden rows win; with one
      // CTA per SM staging the hidden rows in the slot wins, e.g. d = 8192)
      const int half = 113 * 1024;
      bool ldgx = env_stream != 1;
      int per_sm = 2;
      StreamPlan st = plan_stream<TW>(p.d, p.K, p.H, half, ldgx);
      if ((!st.bytes || st.S < 2) && env_stream == 3) {
        ldgx = false;
        st = plan_stream<TW>(p.d, p.K, p.H, half, false);
      }
      if (!st.bytes || st.S < 2) {
        ldgx = env_stream == 2;
        st = plan_stream<TW>(p.d, p.K, p.H, g_smem_optin, ldgx);
        per_sm = 1;
      }
      if (st.bytes) {
        inline_rc = p.recheck && rscr <= st.off_bar;   // epilogue re-evaluates deferred rows
        p.recheck_inline = inline_rc ? 1 : 0;
        // SPX_PRED_CTAS_PER_SM (sweeps): 1 leaves the second CTA slot of every SM
        // free for the next (programmatic dependent) launch's prefetch
        static const int env_cps = getenv("SPX_PRED_CTAS_PER_SM") ? atoi(getenv("SPX_PRED_CTAS_PER_SM")) : 2;
        if (env_cps == 1) per_sm = 1;
        const long long cap = (long long)per_sm * g_sms;
        const int grid = (int)(a->B < cap ? a->B : cap);
        if constexpr (std::is_same<TW, __nv_bfloat16>::value)
          return launch_stream_bf16(p, st, grid, stream, g_smem_optin, ldgx);
      }
    }
    // tuning overrides (benchmark sweeps only)
    static const int env_w1 = getenv("SPX_PRED_W1SMEM") ? atoi(getenv("SPX_PRED_W1SMEM")) : -1;
    static const int env_ring = getenv("SPX_PRED_RING") ? atoi(getenv("SPX_PRED_RING")) : -1;
    SmemPlan sp = plan_smem<TW>(p.d, p.K, p.H, g_smem_optin, env_w1, env_ring);
    if (sp.bytes == 0) {
      // rows too wide for the 4-team ring (d = 8192, K > 8): the 2-team variant
      if constexpr (std::is_same<TW, __nv_bfloat16>::value)
        return launch_team_wide_bf16(p, g_smem_optin, g_sms, stream, inline_rc);
      return SPX_EINVAL;
    }
    inline_rc = p.recheck && rscr <= sp.off_bar;
    p.recheck_inline = inline_rc ? 1 : 0;
    const long long need = (a->B + NTEAM - 1) / NTEAM;
    const int grid = (int)(need < g_sms ? need : g_sms);
    return launch_team<TW>(p, sp, grid > 0 ? grid : 1, stream, g_smem_optin);
  }
  return spx_launch_status("spx_predictor_eval");
}

static int params_from_args(const spx_predictor_args *a, PredParams &p) {
  if (!a) return SPX_EINVAL;
  if (a->B < 0 || a->d <= 0 || a->d % CHUNK || a->V <= 0 || a->K < 1 || a->K > MAXK ||
      (a->policy == SPX_POLICY_MLP && (a->H < 1 || a->H > MAXH)))
    return SPX_EINVAL;
  if (!a->hidden || !a->norm_g || !a->norm_b || !a->head || !a->ids || !a->prev || !a->err)
    return SPX_EINVAL;
  if (a->policy == SPX_POLICY_MLP && (!a->w1 || !a->b1 || !a->w2)) return SPX_EINVAL;
  if (a->hidden_stride % CHUNK) return SPX_EINVAL;
  p = PredParams{};
  p.hidden = a->hidden; p.hidden_stride = a->hidden_stride ? a->hidden_stride : a->d;
  p.norm_g = a->norm_g; p.norm_b = a->norm_b;
  p.head = a->head; p.head_bw = a->head_bw;
  p.ids = a->ids; p.prev = a->prev;
  p.w1 = a->w1; p.b1 = a->b1; p.w2 = a->w2; p.b2 = a->b2; p.z_cut = a->z_cut;
  p.policy = a->policy; p.const_prob = a->const_prob; p.threshold = a->threshold;
  p.logits_out = a->logits_out; p.feat_out = a->feat_out; p.z_out = a->z_out;
  p.prob_out = a->prob_out; p.fired = a->fired;
  p.row_layer_mask = a->row_layer_mask; p.row_done = a->row_done; p.evals = a->evals;
  p.layer = a->layer; p.err = a->err; p.trace = g_debug_trace;
  p.pdl = a->pdl == 2 ? 2 : a->pdl ? 1 : 0;
  p.B = (int)a->B; p.d = (int)a->d; p.V = (int)a->V; p.K = (int)a->K;
  p.H = a->policy == SPX_POLICY_MLP ? (int)a->H : 0;
  p.head_wmax = a->head_wmax; p.cert = a->cert;
  p.cert_kappa = a->cert_kappa; p.cert_hnorm = a->cert_hnorm;
  p.prev_err = a->prev_err;
  p.recheck = a->mode == SPX_MODE_FAST ? a->recheck : nullptr;
  p.recheck_inline = 0;
  p.fired_any = a->fired_any;
  if (p.recheck && (!a->head_wmax || !a->prev_err ||
                    (a->policy == SPX_POLICY_MLP && !a->cert)))
    return SPX_EINVAL;
  return 0;
}

extern "C" int spx_predictor_eval(const spx_predictor_args *a, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  PredParams p;
  const int rc = params_from_args(a, p);
  if (rc) return rc;
  if (a->B == 0) return 0;
  if (a->head_dtype == SPX_DTYPE_F32) return launch_predictor<float>(p, a, stream);
  if (a->head_dtype == SPX_DTYPE_BF16) return launch_predictor<__nv_bfloat16>(p, a, stream);
  return SPX_EINVAL;
}

// SPLIT path (spx_pred_split.cu): K1 gather -> inter, then K2+K3 tail.
namespace spx {
bool split_supported(const PredParams &p, int head_dtype);
int launch_split_gather(const PredParams &p, float *inter, const PredParams *pt,
                        const float *inter_t, cudaStream_t s);
int launch_split_tail(const PredParams &p, const float *inter, cudaStream_t s);
}  // namespace spx

extern "C" int spx_predictor_split_ok(const spx_predictor_args *a) {
  PredParams p;
  if (params_from_args(a, p)) return 0;
  return a->mode == SPX_MODE_FAST && split_supported(p, a->head_dtype) ? 1 : 0;
}

extern "C" int spx_predictor_gather(const spx_predictor_args *a, float *inter, void *stream) {
  PredParams p;
  const int rc = params_from_args(a, p);
  if (rc) return rc;
  if (!inter || a->mode != SPX_MODE_FAST || !split_supported(p, a->head_dtype)) return SPX_EINVAL;
  if (a->B == 0) return 0;
  p.pdl = a->pdl < 0 || a->pdl > 3 ? 0 : a->pdl;
  const int r = launch_split_gather(p, inter, nullptr, nullptr, (cudaStream_t)stream);
  if (r) return r;
  return spx_launch_status("spx_predictor_gather");
}

extern "C" int spx_predictor_gather_tail(const spx_predictor_args *a, float *inter,
                                         const spx_predictor_args *t, const float *inter_t,
                                         void *stream) {
  PredParams p, pt;
  int rc = params_from_args(a, p);
  if (rc) return rc;
  rc = params_from_args(t, pt);
  if (rc) return rc;
  if (!inter || !inter_t || a->mode != SPX_MODE_FAST || t->mode != SPX_MODE_FAST ||
      !split_supported(p, a->head_dtype) || !split_supported(pt, t->head_dtype) || p.B != pt.B)
    return SPX_EINVAL;
  if (a->B == 0) return 0;
  p.pdl = 3;
  const int r = launch_split_gather(p, inter, &pt, inter_t, (cudaStream_t)stream);
  if (r) return r;
  return spx_launch_status("spx_predictor_gather_tail");
}

extern "C" int spx_predictor_tail_pipelined(const spx_predictor_args *t, const float *inter_t,
                                            void *stream) {
  PredParams pt;
  const int rc = params_from_args(t, pt);
  if (rc) return rc;
  if (!inter_t || t->mode != SPX_MODE_FAST || !split_supported(pt, t->head_dtype))
    return SPX_EINVAL;
  if (t->B == 0) return 0;
  PredParams p = pt;                 // an empty gather of the same shape: tail warps only
  p.B = 0;
  p.pdl = 3;
  const int r = launch_split_gather(p, nullptr, &pt, inter_t, (cudaStream_t)stream);
  if (r) return r;
  return spx_launch_status("spx_predictor_tail_pipelined");
}

extern "C" int spx_predictor_tail(const spx_predictor_args *a, const float *inter, void *stream) {
  PredParams p;
  const int rc = params_from_args(a, p);
  if (rc) return rc;
  if (!inter || a->mode != SPX_MODE_FAST || !split_supported(p, a->head_dtype)) return SPX_EINVAL;
  if (a->B == 0) return 0;
  p.pdl = 0;
  const int r = launch_split_tail(p, inter, (cudaStream_t)stream);
  if (r) return r;
  return spx_launch_status("spx_predictor_tail");
}

extern "C" int spx_extract_features(const float *logits, const float *prev, float *feats_out,
                                    int32_t *err, int64_t B, int64_t K, void *stream) {
  if (!logits || !prev || !feats_out || !err || B < 0 || K < 1 || K > (1 << 24)) return SPX_EINVAL;
  if (B == 0) return 0;
  if (K > MAXK) {
    features_wide_kernel<<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>(logits, prev, feats_out,
                                                                       err, (int)K);
    return spx_launch_status("spx_extract_features");
  }
  features_kernel<<<(unsigned)B, 32, 0, (cudaStream_t)stream>>>(
      logits, const_cast<float *>(prev), feats_out, err, (int)B, (int)K);
  return spx_launch_status("spx_extract_features");
}

extern "C" int spx_softmax_pick(const float *logits, int64_t rows, int64_t n,
                                const int32_t *ids, int32_t K, float *probs_out, int32_t mode,
                                int32_t *err, void *stream) {
  if (!logits || !ids || !probs_out || !err || rows < 0 || n < 1 || n > (1 << 30) || K < 1)
    return SPX_EINVAL;
  if (rows == 0) return 0;
  softmax_pick_kernel<<<(unsigned)rows, 256, 0, (cudaStream_t)stream>>>(logits, (int)n, ids, K,
                                                                         probs_out, mode, err);
  return spx_launch_status("spx_softmax_pick");
}

extern "C" int spx_predictor_mlp(const float *feats, const float *w1, const float *b1,
                                 const float *w2, float b2, float z_cut, float *z_out,
                                 double *prob_out, uint8_t *fired_out, int64_t B, int64_t K,
                                 int64_t H, void *stream) {
  if (!feats || !w1 || !b1 || !w2 || B < 0 || K < 1 || K > MAXK || H < 1 || H > MAXH)
    return SPX_EINVAL;
  if (B == 0) return 0;
  PredParams p{};
  p.w1 = w1; p.b1 = b1; p.w2 = w2; p.b2 = b2; p.z_cut = z_cut;
  p.z_out = z_out; p.prob_out = prob_out; p.fired = fired_out;
  p.B = (int)B; p.K = (int)K; p.H = (int)H;
  mlp_kernel<<<(unsigned)B, 32, 0, (cudaStream_t)stream>>>(p, feats);
  return spx_launch_status("spx_predictor_mlp");
}

// Tree-node evaluation (tree.py:213-220): live node i's K merged logits (K6
// output, live order) -> features against that node's carried probabilities
// prev[node] (updated in place) -> MLP / constant policy -> fired[node],
// prob[node].  One warp per live node; the per-node gather/scatter by
// live_idx is fused so the tree engine needs no index kernels.
namespace spx {
__global__ void tree_node_eval_kernel(PredParams p, const float *logits, const int32_t *live_idx,
                                      int n_live) {
  const int i = blockIdx.x;
  if (i >= n_live) return;
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  const int lane = threadIdx.x, node = live_idx[i];
  for (int c = lane; c < p.K; c += 32) feats[c] = logits[(size_t)i * p.K + c];
  __syncwarp();
  warp_row_tail(p, node, feats, p.w1, p.b1, p.w2, hs, lane);
}
}  // namespace spx

extern "C" int spx_tree_node_eval(const float *logits, const int32_t *live_idx, int64_t n_live,
                                  float *prev, const float *w1, const float *b1, const float *w2,
                                  float b2, float z_cut, int32_t policy, double const_prob,
                                  double threshold, double *prob_out, uint8_t *fired,
                                  int32_t *err, int64_t K, int64_t H, void *stream) {
  if (!logits || !live_idx || !prev || !fired || !err || n_live < 0 || K < 1 || K > MAXK)
    return SPX_EINVAL;
  if (policy == SPX_POLICY_MLP && (!w1 || !b1 || !w2 || H < 1 || H > MAXH)) return SPX_EINVAL;
  if (policy != SPX_POLICY_MLP && policy != SPX_POLICY_CONST) return SPX_EINVAL;
  if (n_live == 0) return 0;
  PredParams p{};
  p.prev = prev; p.w1 = w1; p.b1 = b1; p.w2 = w2; p.b2 = b2; p.z_cut = z_cut;
  p.policy = policy; p.const_prob = const_prob; p.threshold = threshold;
  p.prob_out = prob_out; p.fired = fired; p.err = err;
  p.K = (int)K; p.H = policy == SPX_POLICY_MLP ? (int)H : 0;
  tree_node_eval_kernel<<<(unsigned)n_live, 32, 0, (cudaStream_t)stream>>>(p, logits, live_idx,
                                                                          (int)n_live);
  return spx_launch_status("spx_tree_node_eval");
}

extern "C" int spx_predictor_cert(const float *w1, const float *b1, const float *w2, int64_t K,
                                  int64_t H, float *cert, void *stream) {
  if (!w1 || !b1 || !w2 || !cert || K < 1 || K > MAXK || H < 1 || H > MAXH) return SPX_EINVAL;
  predictor_cert_kernel<<<(unsigned)(3 * K + 2), 32, 0, (cudaStream_t)stream>>>(w1, b1, w2, (int)K,
                                                                               (int)H, cert);
  return spx_launch_status("spx_predictor_cert");
}

namespace spx {
template <typename TW>
__global__ void head_stats_kernel(const TW *head, int64_t V, int d, float *wmax) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < V; v += warps) {
    float m = 0.f;
    for (int j = lane * CHUNK; j < d; j += 32 * CHUNK) {
      float w[4];
      load4_f32<TW>(head + (size_t)v * d + j, w);
#pragma unroll
      for (int e = 0; e < CHUNK; ++e) m = fmaxf(m, fabsf(w[e]));
    }
    m = warp_max_f(m);
    if (lane == 0) wmax[v] = m;
  }
}
}  // namespace spx

extern "C" int spx_head_stats(const void *head, int32_t head_dtype, int64_t V, int64_t d,
                              float *wmax, void *stream) {
  if (!head || !wmax || V < 1 || d < CHUNK || d % CHUNK) return SPX_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dtype == SPX_DTYPE_BF16)
    head_stats_kernel<__nv_bfloat16><<<592, 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16 *>(head), V, (int)d, wmax);
  else if (head_dtype == SPX_DTYPE_F32)
    head_stats_kernel<float><<<592, 256, 0, st>>>(reinterpret_cast<const float *>(head), V, (int)d,
                                                  wmax);
  else
    return SPX_EINVAL;
  return spx_launch_status("spx_head_stats");
}
