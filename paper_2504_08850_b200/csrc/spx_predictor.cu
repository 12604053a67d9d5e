// K1+K2+K3: fused speculative early-exit predictor evaluation (sm_100a).
//
// One launch evaluates one decoder layer's exit predictor for B rows
// (independent requests, or tree nodes).  Per row it does, in one CTA:
//   final LayerNorm of the hidden row        reference model.py:140-146, :312
//   gather of the K speculative LM-head rows reference model.py:313 (our head
//     is stored (V, d) bf16 so a gather is K contiguous 8 KiB rows)
//   K local logits                          reference model.py:314
//   softmax over the K ids + delta vs prev  reference predictor.py:42-52,
//                                           model.py:149-152
//   2-layer MLP + bias, ReLU                reference predictor.py:97-103
//   f64 sigmoid + strict threshold          reference predictor.py:87-94,
//                                           :106-109
// and writes prob / fired / the updated local probs (the next layer's
// "prev", engine.py:196) to device memory.  Rows whose engine state says
// "already exited" or "layer not scheduled" return at entry: that is how the
// device exit flag gates later launches without a host sync.
//
// MLP arithmetic reproduces the reference's numpy/OpenBLAS (SkylakeX
// kernels) order exactly: z1 = ascending FMA chain from 0 (3K <= 48) or
// 8/4/2/1-column blocks each chained from 0 and added (3K >= 51), then + b1;
// z2 = the AVX-512 sdot tree.  The decision is
// z2 >= z_cut with z_cut the smallest f32 whose f64 sigmoid exceeds the
// threshold, so the decision is exactly the reference's `prob > threshold`.
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"

namespace spx {

constexpr int PRED_THREADS = 128;     // 4 warps == the 128 canonical partials
constexpr int MAXK = 64;
constexpr int MAXH = 1024;

struct PredParams {
  const float *hidden; int64_t hidden_stride;
  const float *norm_g, *norm_b;
  const void *head;            // (V, d) bf16 or f32
  const int32_t *ids;          // (B, K)
  float *prev;                 // (B, K) in: previous local probs; out: new
  const float *w1, *b1, *w2;   // (3K, H), (H), (H)
  float b2, z_cut;
  int policy;                  // 0 = MLP, 1 = constant probability
  double const_prob, threshold;
  float *logits_out;           // (B, K) optional
  float *feat_out;             // (B, 3K) optional
  float *z_out;                // (B) optional
  double *prob_out;            // (B) optional
  uint8_t *fired;              // (B) optional
  const uint64_t *row_layer_mask;  // (B) optional: bit `layer` must be set
  const uint8_t *row_done;         // (B) optional: nonzero -> skip row
  int32_t *evals;                  // (B) optional: += 1 per evaluated row
  int layer;
  int *err;
  int B, d, V, K, H;
};

template <int G>
__device__ __forceinline__ void cta_canon_reduce(float (&v)[G], float *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < G; ++g) v[g] = warp_butterfly_sum(v[g]);
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) red[g * 4 + warp] = v[g];
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g)
    v[g] = canon_combine(red[g * 4 + 0], red[g * 4 + 1], red[g * 4 + 2], red[g * 4 + 3]);
  __syncthreads();
}

// ---------------------------------------------------------------- MLP tail
// Shared by both reduction policies; runs after feats[0..3K) are in smem.
__device__ void mlp_and_decide(const PredParams &p, int row, const float *feats, float *hs,
                               float *as, bool row_ok) {
  const int tid = threadIdx.x;
  const int n = 3 * p.K, H = p.H;
  // z1 / ReLU for units j = tid + 128 m
  for (int j = tid; j < H; j += PRED_THREADS) {
    float y;
    if (n <= 48) {
      float acc = 0.0f;
      for (int i = 0; i < n; ++i) acc = __fmaf_rn(feats[i], __ldg(p.w1 + (size_t)i * H + j), acc);
      y = acc;
    } else {
      y = 0.0f;
      int i = 0;
      const int blocks[4] = {8, 4, 2, 1};
      for (int bi = 0; bi < 4; ++bi) {
        const int bs = blocks[bi];
        while (n - i >= bs) {
          float t = 0.0f;
          for (int q = 0; q < bs; ++q)
            t = __fmaf_rn(feats[i + q], __ldg(p.w1 + (size_t)(i + q) * H + j), t);
          y = __fadd_rn(y, t);
          i += bs;
          if (bs != 8) break;
        }
      }
    }
    const float z1 = __fadd_rn(y, __ldg(p.b1 + j));
    hs[j] = z1 > 0.0f ? z1 : 0.0f;
  }
  __syncthreads();
  // z2: OpenBLAS SkylakeX sdot order (sdot.c + sdot_microk_skylakex-2.c)
  const int n1 = H & ~31, n64 = n1 & ~63;
  if (tid < 64) {
    float a = 0.0f;
    for (int b = 0; b < n64; b += 64) a = __fmaf_rn(hs[b + tid], __ldg(p.w2 + b + tid), a);
    as[tid] = a;
  }
  __syncthreads();
  if (tid == 0) {
    float dot = 0.0f;
    if (n1) {
      float s[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        float acc[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          acc[a] = __fadd_rn(as[16 * a + m], as[16 * a + m + 8]);
          if (n1 > n64) acc[a] = __fmaf_rn(hs[n64 + 8 * a + m], __ldg(p.w2 + n64 + 8 * a + m), acc[a]);
        }
        s[m] = __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), acc[2]), acc[3]);
      }
      float hh[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) hh[m] = __fadd_rn(s[m], s[m + 4]);
      dot = __fadd_rn(__fadd_rn(hh[0], hh[1]), __fadd_rn(hh[2], hh[3]));
    }
    for (int i = n1; i < H; ++i) dot = __fadd_rn(dot, __fmul_rn(hs[i], __ldg(p.w2 + i)));
    const float z2 = __fadd_rn(dot, p.b2);
    // predictor.py:87-94 in float64
    const double z = (double)z2;
    double prob;
    if (z >= 0.0) prob = 1.0 / (1.0 + exp(-z));
    else { const double ez = exp(z); prob = ez / (1.0 + ez); }
    const bool fire = row_ok && (z2 >= p.z_cut);
    if (p.z_out) p.z_out[row] = z2;
    if (p.prob_out) p.prob_out[row] = prob;
    if (p.fired) p.fired[row] = fire ? 1 : 0;
  }
}

// Softmax over the K logits (model.py:149-152), features (predictor.py:51-52),
// validation (predictor.py:45-50).  logits in feats[0..K); writes feats[K..3K).
__device__ bool softmax_features(const PredParams &p, int row, float *feats, float *scratch) {
  const int tid = threadIdx.x, K = p.K;
  __shared__ float s_max, s_sum;
  __shared__ int s_bad;
  if (tid == 0) {
    float m = feats[0];
    bool bad = false;
    double ps = 0.0;
    float psf = 0.0f;
    for (int c = 0; c < K; ++c) {
      const float x = feats[c];
      bad |= !is_finite(x);
      m = fmaxf(m, x);
      psf = __fadd_rn(psf, p.prev[(size_t)row * K + c]);
    }
    ps = (double)psf;
    int e = 0;
    if (bad) e |= ERR_LOGIT_NONFINITE;
    if (fabs(ps - 1.0) > 1e-5) e |= ERR_PREV_SUM;
    s_bad = e;
    s_max = m;
    if (e) atomicOr(p.err, e);
  }
  __syncthreads();
  if (s_bad) return false;
  if (tid < K) scratch[tid] = np_expf(__fsub_rn(feats[tid], s_max));
  __syncthreads();
  if (tid == 0) {
    float acc = 0.0f;
    for (int c = 0; c < K; ++c) acc = __fadd_rn(acc, scratch[c]);   // seq_sum
    s_sum = acc;
  }
  __syncthreads();
  if (tid < K) {
    const float pr = __fdiv_rn(scratch[tid], s_sum);
    const float pv = p.prev[(size_t)row * K + tid];
    feats[K + tid] = pr;
    feats[2 * K + tid] = __fsub_rn(pr, pv);
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ bool row_skipped(const PredParams &p, int row) {
  if (p.row_done && p.row_done[row]) return true;
  if (p.row_layer_mask && !((p.row_layer_mask[row] >> p.layer) & 1ull)) return true;
  return false;
}

__device__ void finish_row(const PredParams &p, int row, float *feats, float *hs, float *as,
                           float *scratch) {
  const int tid = threadIdx.x, K = p.K;
  const bool ok = softmax_features(p, row, feats, scratch);
  if (tid < K) {
    if (p.logits_out) p.logits_out[(size_t)row * K + tid] = feats[tid];
  }
  if (!ok) {
    if (tid == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  if (p.feat_out)
    for (int i = tid; i < 3 * K; i += PRED_THREADS) p.feat_out[(size_t)row * 3 * K + i] = feats[i];
  if (tid < K) p.prev[(size_t)row * K + tid] = feats[K + tid];   // engine.py:196
  if (tid == 0 && p.evals) p.evals[row] += 1;
  if (p.policy == 0) {
    mlp_and_decide(p, row, feats, hs, as, true);
  } else if (tid == 0) {
    const bool fire = p.const_prob > p.threshold;
    if (p.prob_out) p.prob_out[row] = p.const_prob;
    if (p.z_out) p.z_out[row] = 0.0f;
    if (p.fired) p.fired[row] = fire ? 1 : 0;
  }
}

// ------------------------------------------------------------ FAST (CDOT)
// CPT = canonical chunks per thread (d <= 1024*CPT).
template <typename TW, int CPT>
__global__ void __launch_bounds__(PRED_THREADS)
predictor_fast_kernel(PredParams p) {
  const int row = blockIdx.x;
  if (row >= p.B) return;
  if (row_skipped(p, row)) {
    if (threadIdx.x == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  __shared__ float red[4 * 4];
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  __shared__ float as[64];
  __shared__ float scratch[MAXK];
  __shared__ int s_flag;
  const int tid = threadIdx.x;
  const int nchunk = p.d / CHUNK;
  const float *x = p.hidden + (size_t)row * p.hidden_stride;
  if (tid == 0) s_flag = 0;
  __syncthreads();

  // ---- load the hidden row and the norm params (canonical chunk ownership)
  float xv[CPT][CHUNK];
#pragma unroll
  for (int s = 0; s < CPT; ++s) {
    const int c = tid + NPART * s;
    if (c < nchunk) {
      const float4 a = ldg_f4(x + CHUNK * c), b = ldg_f4(x + CHUNK * c + 4);
      xv[s][0] = a.x; xv[s][1] = a.y; xv[s][2] = a.z; xv[s][3] = a.w;
      xv[s][4] = b.x; xv[s][5] = b.y; xv[s][6] = b.z; xv[s][7] = b.w;
    } else {
#pragma unroll
      for (int e = 0; e < CHUNK; ++e) xv[s][e] = 0.0f;
    }
  }
  // ---- LayerNorm stats (model.py:140-146) in canonical order
  float part[1] = {0.0f};
  bool finite = true;
#pragma unroll
  for (int s = 0; s < CPT; ++s)
#pragma unroll
    for (int e = 0; e < CHUNK; ++e) {
      part[0] = __fadd_rn(part[0], xv[s][e]);
      finite &= is_finite(xv[s][e]);
    }
  if (!finite) { atomicOr(p.err, ERR_HIDDEN_NONFINITE); s_flag = 1; }
  cta_canon_reduce<1>(part, red);
  const float df = (float)p.d;
  const float mean = __fdiv_rn(part[0], df);
  float sq[1] = {0.0f};
#pragma unroll
  for (int s = 0; s < CPT; ++s)
#pragma unroll
    for (int e = 0; e < CHUNK; ++e) {
      const int c = tid + NPART * s;
      if (c < nchunk) {
        xv[s][e] = __fsub_rn(xv[s][e], mean);
        sq[0] = __fmaf_rn(xv[s][e], xv[s][e], sq[0]);
      }
    }
  cta_canon_reduce<1>(sq, red);
  const float var = __fdiv_rn(sq[0], df);
  const float denom = __fsqrt_rn(__fadd_rn(var, 1e-5f));
#pragma unroll
  for (int s = 0; s < CPT; ++s) {
    const int c = tid + NPART * s;
    if (c < nchunk) {
      const float4 g0 = ldg_f4(p.norm_g + CHUNK * c), g1 = ldg_f4(p.norm_g + CHUNK * c + 4);
      const float4 b0 = ldg_f4(p.norm_b + CHUNK * c), b1 = ldg_f4(p.norm_b + CHUNK * c + 4);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int e = 0; e < CHUNK; ++e)
        xv[s][e] = __fadd_rn(__fmul_rn(__fdiv_rn(xv[s][e], denom), gg[e]), bb[e]);
    }
  }
  // ---- K speculative logits, 4 ids per pass
  const int K = p.K;
  for (int c0 = 0; c0 < K; c0 += 4) {
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    Chunk<TW> wv[4][CPT];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int id = (c0 + q < K) ? p.ids[(size_t)row * K + c0 + q] : 0;
      if (id < 0 || id >= p.V) {
        if (tid == 0) atomicOr(p.err, ERR_ID_RANGE);
        s_flag = 1;
        id = 0;
      }
      const TW *wr = reinterpret_cast<const TW *>(p.head) + (size_t)id * p.d;
#pragma unroll
      for (int s = 0; s < CPT; ++s) {
        const int c = tid + NPART * s;
        if (c0 + q < K && c < nchunk) wv[q][s].load(wr + CHUNK * c);
        else wv[q][s].zero();
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int s = 0; s < CPT; ++s) {
        float w[8];
        wv[q][s].to_f32(w);
#pragma unroll
        for (int e = 0; e < CHUNK; ++e) acc[q] = __fmaf_rn(xv[s][e], w[e], acc[q]);
      }
    cta_canon_reduce<4>(acc, red);
    if (tid < 4 && c0 + tid < K) feats[c0 + tid] = acc[tid];
  }
  __syncthreads();
  if (s_flag) {
    if (tid == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  finish_row(p, row, feats, hs, as, scratch);
}

// ----------------------------------------------------------- STRICT (parity)
// The reference's own operation sequence: every sum a left-to-right chain of
// separately rounded adds from 0, every product rounded (no FMA).  Uses
// dynamic smem of d floats.
template <typename TW>
__global__ void __launch_bounds__(PRED_THREADS)
predictor_strict_kernel(PredParams p) {
  const int row = blockIdx.x;
  if (row >= p.B) return;
  if (row_skipped(p, row)) {
    if (threadIdx.x == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  extern __shared__ float hn[];   // d floats
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  __shared__ float as[64];
  __shared__ float scratch[MAXK];
  __shared__ float s_mean, s_denom;
  __shared__ int s_flag;
  const int tid = threadIdx.x, d = p.d;
  const float *x = p.hidden + (size_t)row * p.hidden_stride;
  if (tid == 0) s_flag = 0;
  __syncthreads();
  bool finite = true;
  for (int j = tid; j < d; j += PRED_THREADS) { hn[j] = x[j]; finite &= is_finite(hn[j]); }
  if (!finite) { atomicOr(p.err, ERR_HIDDEN_NONFINITE); s_flag = 1; }
  __syncthreads();
  const float df = (float)d;
  if (tid == 0) {
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, hn[j]);
    s_mean = __fdiv_rn(acc, df);
  }
  __syncthreads();
  const float mean = s_mean;
  for (int j = tid; j < d; j += PRED_THREADS) hn[j] = __fsub_rn(hn[j], mean);
  __syncthreads();
  if (tid == 0) {
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, __fmul_rn(hn[j], hn[j]));
    s_denom = __fsqrt_rn(__fadd_rn(__fdiv_rn(acc, df), 1e-5f));
  }
  __syncthreads();
  const float denom = s_denom;
  for (int j = tid; j < d; j += PRED_THREADS)
    hn[j] = __fadd_rn(__fmul_rn(__fdiv_rn(hn[j], denom), p.norm_g[j]), p.norm_b[j]);
  __syncthreads();
  const int K = p.K;
  if (tid < K) {
    int id = p.ids[(size_t)row * K + tid];
    if (id < 0 || id >= p.V) { atomicOr(p.err, ERR_ID_RANGE); s_flag = 1; id = 0; }
    const TW *wr = reinterpret_cast<const TW *>(p.head) + (size_t)id * d;
    float acc = 0.0f;
    for (int j = 0; j < d; j += CHUNK) {
      float w[8];
      load8_f32<TW>(wr + j, w);
#pragma unroll
      for (int e = 0; e < CHUNK; ++e) acc = __fadd_rn(acc, __fmul_rn(hn[j + e], w[e]));
    }
    feats[tid] = acc;
  }
  __syncthreads();
  if (s_flag) {
    if (tid == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  finish_row(p, row, feats, hs, as, scratch);
}

}  // namespace spx

using namespace spx;

template <typename TW>
static int launch_predictor(const PredParams &p, const spx_predictor_args *a, dim3 grid,
                            dim3 block, cudaStream_t stream) {
  if (a->mode == SPX_MODE_STRICT) {
    const size_t smem = (size_t)a->d * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(predictor_strict_kernel<TW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    predictor_strict_kernel<TW><<<grid, block, smem, stream>>>(p);
  } else {
    const int nchunk = (int)(a->d / CHUNK);
    if (nchunk <= NPART * 1) predictor_fast_kernel<TW, 1><<<grid, block, 0, stream>>>(p);
    else if (nchunk <= NPART * 2) predictor_fast_kernel<TW, 2><<<grid, block, 0, stream>>>(p);
    else if (nchunk <= NPART * 4) predictor_fast_kernel<TW, 4><<<grid, block, 0, stream>>>(p);
    else if (nchunk <= NPART * 8) predictor_fast_kernel<TW, 8><<<grid, block, 0, stream>>>(p);
    else return SPX_EINVAL;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}

extern "C" int spx_predictor_eval(const spx_predictor_args *a, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!a) return SPX_EINVAL;
  if (a->B < 0 || a->d <= 0 || a->d % CHUNK || a->V <= 0 || a->K < 1 || a->K > MAXK ||
      (a->policy == SPX_POLICY_MLP && (a->H < 1 || a->H > MAXH)))
    return SPX_EINVAL;
  if (!a->hidden || !a->norm_g || !a->norm_b || !a->head || !a->ids || !a->prev || !a->err)
    return SPX_EINVAL;
  if (a->policy == SPX_POLICY_MLP && (!a->w1 || !a->b1 || !a->w2)) return SPX_EINVAL;
  if (a->B == 0) return 0;
  PredParams p;
  p.hidden = a->hidden; p.hidden_stride = a->hidden_stride ? a->hidden_stride : a->d;
  p.norm_g = a->norm_g; p.norm_b = a->norm_b;
  p.head = a->head;
  p.ids = a->ids; p.prev = a->prev;
  p.w1 = a->w1; p.b1 = a->b1; p.w2 = a->w2; p.b2 = a->b2; p.z_cut = a->z_cut;
  p.policy = a->policy; p.const_prob = a->const_prob; p.threshold = a->threshold;
  p.logits_out = a->logits_out; p.feat_out = a->feat_out; p.z_out = a->z_out;
  p.prob_out = a->prob_out; p.fired = a->fired;
  p.row_layer_mask = a->row_layer_mask; p.row_done = a->row_done; p.evals = a->evals;
  p.layer = a->layer; p.err = a->err;
  p.B = (int)a->B; p.d = (int)a->d; p.V = (int)a->V; p.K = (int)a->K; p.H = (int)a->H;
  const dim3 grid((unsigned)a->B), block(PRED_THREADS);
  if (a->head_dtype == SPX_DTYPE_F32) return launch_predictor<float>(p, a, grid, block, stream);
  if (a->head_dtype == SPX_DTYPE_BF16)
    return launch_predictor<__nv_bfloat16>(p, a, grid, block, stream);
  return SPX_EINVAL;
}

// ---------------------------------------------------------------------------
// Function-level operators (the reference's extract_features and
// predictor_forward called on their own, predictor.py:42-52 / :97-103).  They
// run the same device code as the fused kernel, so results are identical.

namespace spx {

__global__ void __launch_bounds__(PRED_THREADS)
features_kernel(const float *logits, float *prev, float *feats_out, int *err, int B, int K) {
  const int row = blockIdx.x;
  if (row >= B) return;
  __shared__ float feats[3 * MAXK];
  __shared__ float scratch[MAXK];
  PredParams p{};
  p.prev = prev; p.err = err; p.K = K;
  if (threadIdx.x < K) feats[threadIdx.x] = logits[(size_t)row * K + threadIdx.x];
  __syncthreads();
  if (!softmax_features(p, row, feats, scratch)) return;
  for (int i = threadIdx.x; i < 3 * K; i += PRED_THREADS) feats_out[(size_t)row * 3 * K + i] = feats[i];
}

__global__ void __launch_bounds__(PRED_THREADS)
mlp_kernel(PredParams p, const float *feats_in) {
  const int row = blockIdx.x;
  if (row >= p.B) return;
  __shared__ float feats[3 * MAXK];
  __shared__ float hs[MAXH];
  __shared__ float as[64];
  for (int i = threadIdx.x; i < 3 * p.K; i += PRED_THREADS) feats[i] = feats_in[(size_t)row * 3 * p.K + i];
  __syncthreads();
  mlp_and_decide(p, row, feats, hs, as, true);
}

}  // namespace spx

extern "C" int spx_extract_features(const float *logits, const float *prev, float *feats_out,
                                    int32_t *err, int64_t B, int64_t K, void *stream) {
  if (!logits || !prev || !feats_out || !err || B < 0 || K < 1 || K > MAXK) return SPX_EINVAL;
  if (B == 0) return 0;
  features_kernel<<<(unsigned)B, PRED_THREADS, 0, (cudaStream_t)stream>>>(
      logits, const_cast<float *>(prev), feats_out, err, (int)B, (int)K);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
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
  mlp_kernel<<<(unsigned)B, PRED_THREADS, 0, (cudaStream_t)stream>>>(p, feats);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}
