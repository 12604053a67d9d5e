#include <type_traits>
// K1+K2+K3: fused speculative early-exit predictor evaluation (sm_100a).
//
// One launch evaluates one decoder layer's exit predictor for B rows
// (independent requests, or tree nodes).  Per row:
//   final LayerNorm of the hidden row        reference model.py:140-146, :312
//   gather of the K speculative LM-head rows reference model.py:313 (our head
//     is stored (V, d) so the gather is K contiguous rows, fetched by TMA)
//   K local logits                          reference model.py:314
//   softmax over the K ids + delta vs prev  reference predictor.py:42-52,
//                                           model.py:149-152
//   2-layer MLP + bias, ReLU                reference predictor.py:97-103
//   f64 sigmoid + strict threshold          reference predictor.py:87-94,
//                                           :106-109
// and writes prob / fired / the updated local probs (the next layer's
// "prev", engine.py:196) to device memory.  Rows whose engine state says
// "already exited" or "layer not scheduled" are skipped at entry: that is how
// the device exit flag gates later launches without a host sync.
//
// FAST kernel (production): persistent, one CTA per SM, one WARP per row.
// Each warp owns a shared-memory stage (hidden row + G LM-head rows) filled by
// 1-D TMA bulk copies (cp.async.bulk, mbarrier completion); the next row's
// copies are issued as soon as the current row's dot products are done, so
// HBM traffic overlaps the softmax/MLP tail.  The predictor weights (W1, b1,
// w2) and the final-norm params are staged in shared memory once per CTA.
// Every reduction is the canonical CDOT order (spx_common.cuh).
//
// MLP arithmetic reproduces the reference's numpy/OpenBLAS (SkylakeX
// kernels) order exactly: z1 = ascending FMA chain from 0 (3K <= 48) or
// 8/4/2/1-column blocks each chained from 0 and added (3K >= 51), then + b1;
// z2 = the AVX-512 sdot tree.  The decision is z2 >= z_cut with z_cut the
// smallest f32 whose f64 sigmoid exceeds the threshold, i.e. exactly the
// reference's `prob > threshold`.
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"
#include <cstdlib>

namespace spx {

constexpr int MAXK = 64;
constexpr int MAXH = 1024;
constexpr int GROUP = 4;              // LM-head rows per TMA stage

struct PredParams {
  const float *hidden; int64_t hidden_stride;
  const float *norm_g, *norm_b;
  const void *head;            // (V, d) bf16 or f32
  const float *head_bw;        // (V) CDOT(final_norm.b, head_v) (FAST path), may be null
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
  unsigned long long *trace;       // debug: per-row globaltimer stamps (8 per row)
  int pdl;                         // launched with programmatic stream serialization
  int B, d, V, K, H;
};

__device__ __forceinline__ bool row_skipped(const PredParams &p, int row) {
  if (p.row_done && p.row_done[row]) return true;
  if (p.row_layer_mask && !((p.row_layer_mask[row] >> p.layer) & 1ull)) return true;
  return false;
}

// ---------------------------------------------------------------- warp tail
// Softmax over the K logits in feats[0..K) (model.py:149-152), features
// (predictor.py:51-52) into feats[K..3K), validation (predictor.py:45-50).
// Whole warp; returns false (and flags err) on invalid input.
__device__ bool warp_softmax_features(const PredParams &p, int row, float *feats, int lane) {
  const int K = p.K;
  const bool v0 = lane < K, v1 = lane + 32 < K;
  const float x0 = v0 ? feats[lane] : 0.f, x1 = v1 ? feats[lane + 32] : 0.f;
  const float pv0 = v0 ? p.prev[(size_t)row * K + lane] : 0.f;
  const float pv1 = v1 ? p.prev[(size_t)row * K + lane + 32] : 0.f;
  bool bad = (v0 && !is_finite(x0)) || (v1 && !is_finite(x1));
  bad = __any_sync(0xffffffffu, bad);
  float m = v0 ? x0 : -INFINITY;
  if (v1) m = fmaxf(m, x1);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
  const float e0 = v0 ? np_expf(__fsub_rn(x0, m)) : 0.f;
  const float e1 = v1 ? np_expf(__fsub_rn(x1, m)) : 0.f;
  // strict left-to-right sums (seq_sum) over c = 0..K-1, replicated per lane
  float esum = 0.f, psum = 0.f;
  for (int c = 0; c < K; ++c) {
    const float ec = __shfl_sync(0xffffffffu, c < 32 ? e0 : e1, c & 31);
    const float pc = __shfl_sync(0xffffffffu, c < 32 ? pv0 : pv1, c & 31);
    esum = __fadd_rn(esum, ec);
    psum = __fadd_rn(psum, pc);
  }
  int e = 0;
  if (bad) e |= ERR_LOGIT_NONFINITE;
  if (fabs((double)psum - 1.0) > 1e-5) e |= ERR_PREV_SUM;
  if (e) {
    if (lane == 0) atomicOr(p.err, e);
    return false;
  }
  if (v0) {
    const float pr = __fdiv_rn(e0, esum);
    feats[K + lane] = pr;
    feats[2 * K + lane] = __fsub_rn(pr, pv0);
  }
  if (v1) {
    const float pr = __fdiv_rn(e1, esum);
    feats[K + lane + 32] = pr;
    feats[2 * K + lane + 32] = __fsub_rn(pr, pv1);
  }
  __syncwarp();
  return true;
}

// z1 of one unit j (scalar path; ragged H tails).
__device__ __forceinline__ float z1_unit(const float *feats, const float *w1, int n, int H,
                                         int j) {
  float acc = 0.f;
  if (n <= 48) {
    for (int i = 0; i < n; ++i) acc = __fmaf_rn(feats[i], w1[(size_t)i * H + j], acc);
    return acc;
  }
  int i = 0;
  const int blocks[4] = {8, 4, 2, 1};
  for (int bi = 0; bi < 4; ++bi) {
    const int bs = blocks[bi];
    while (n - i >= bs) {
      float t = 0.f;
      for (int q = 0; q < bs; ++q) t = __fmaf_rn(feats[i + q], w1[(size_t)(i + q) * H + j], t);
      acc = __fadd_rn(acc, t);
      i += bs;
      if (bs != 8) break;
    }
  }
  return acc;
}

// z1 = feats @ W1 + b1 and ReLU into hs, for the units owned by this warp:
// j = jb + 4*lane + 128*(u0 + u) + e (jb over 512-blocks, u < NU, e < 4),
// i.e. NU*4 independent FMA chains per lane with 16-byte conflict-free W1
// reads.  NU = 4, u0 = 0: one warp does all units; NU = 1, u0 = w: warp w of
// a 4-warp team does a quarter.  Per-unit arithmetic is identical.
template <bool G>
__device__ __forceinline__ float4 ld_w1(const float *p) {
  if (G) return __ldg(reinterpret_cast<const float4 *>(p));
  return *reinterpret_cast<const float4 *>(p);
}

template <int NU, bool W1G = false>
__device__ __forceinline__ void mlp_z1(const float *feats, const float *w1, const float *b1, int n, int H,
                       float *hs, int lane, int u0) {
  if ((H % 4) == 0) {
    for (int jb = 0; jb < H; jb += 512) {
      float y[NU][4];
#pragma unroll
      for (int u = 0; u < NU; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) y[u][e] = 0.f;
      if (n <= 48) {
#pragma unroll 12
        for (int i = 0; i < n; ++i) {
          const float f = feats[i];
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int j0 = jb + 4 * lane + 128 * (u0 + u);
            if (j0 < H) {
              const float4 w = ld_w1<W1G>(w1 + (size_t)i * H + j0);
              const float2 ff = make_float2(f, f);
              const float2 a = ffma2(ff, make_float2(w.x, w.y), make_float2(y[u][0], y[u][1]));
              const float2 b = ffma2(ff, make_float2(w.z, w.w), make_float2(y[u][2], y[u][3]));
              y[u][0] = a.x; y[u][1] = a.y; y[u][2] = b.x; y[u][3] = b.y;
            }
          }
        }
      } else {
        int i = 0;
        const int blocks[4] = {8, 4, 2, 1};
        for (int bi = 0; bi < 4; ++bi) {
          const int bs = blocks[bi];
          while (n - i >= bs) {
            float t[NU][4];
#pragma unroll
            for (int u = 0; u < NU; ++u)
#pragma unroll
              for (int e = 0; e < 4; ++e) t[u][e] = 0.f;
            for (int q = 0; q < bs; ++q) {
              const float f = feats[i + q];
#pragma unroll
              for (int u = 0; u < NU; ++u) {
                const int j0 = jb + 4 * lane + 128 * (u0 + u);
                if (j0 < H) {
                  const float4 w = ld_w1<W1G>(w1 + (size_t)(i + q) * H + j0);
                  const float2 ff = make_float2(f, f);
                  const float2 a = ffma2(ff, make_float2(w.x, w.y), make_float2(t[u][0], t[u][1]));
                  const float2 b = ffma2(ff, make_float2(w.z, w.w), make_float2(t[u][2], t[u][3]));
                  t[u][0] = a.x; t[u][1] = a.y; t[u][2] = b.x; t[u][3] = b.y;
                }
              }
            }
#pragma unroll
            for (int u = 0; u < NU; ++u)
#pragma unroll
              for (int e = 0; e < 4; ++e) y[u][e] = __fadd_rn(y[u][e], t[u][e]);
            i += bs;
            if (bs != 8) break;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int j0 = jb + 4 * lane + 128 * (u0 + u);
        if (j0 < H) {
          const float4 bb = *reinterpret_cast<const float4 *>(b1 + j0);
          float4 r;
          r.x = fmaxf(__fadd_rn(y[u][0], bb.x), 0.f); r.y = fmaxf(__fadd_rn(y[u][1], bb.y), 0.f);
          r.z = fmaxf(__fadd_rn(y[u][2], bb.z), 0.f); r.w = fmaxf(__fadd_rn(y[u][3], bb.w), 0.f);
          *reinterpret_cast<float4 *>(hs + j0) = r;
        }
      }
    }
  } else {
    // ragged H: scalar units, split over the same NU/u0 ownership by lanes
    for (int j = lane + 32 * u0; j < H; j += 32 * (NU == 4 ? 1 : 4)) {
      const float z1 = __fadd_rn(z1_unit(feats, w1, n, H, j), b1[j]);
      hs[j] = z1 > 0.f ? z1 : 0.f;
    }
  }
}

// sdot partial A[c] (c < 64) = FMA chain over the 64-element blocks.
__device__ __forceinline__ float z2_partial(const float *hs, const float *w2, int H, int c) {
  const int n64 = (H & ~31) & ~63;
  float a = 0.f;
  for (int b = 0; b < n64; b += 64) a = __fmaf_rn(hs[b + c], w2[b + c], a);
  return a;
}

// z2: OpenBLAS SkylakeX sdot order (sdot.c + sdot_microk_skylakex-2.c):
// 4 x 16-lane FMA accumulators over 64-element blocks (alo = A[lane], ahi =
// A[lane+32]), fold 16->8, optional 32-element AVX2 step, lane-wise
// ((a0+a1)+a2)+a3, 8->4, ((q0+q1)+(q2+q3)), scalar tail, + b2.  Whole warp.
__device__ __forceinline__ float z2_tree(float alo, float ahi, const float *hs, const float *w2, int H, float b2,
                         int lane) {
  const int n1 = H & ~31, n64 = n1 & ~63;
  float blo = __fadd_rn(alo, __shfl_down_sync(0xffffffffu, alo, 8));
  float bhi = __fadd_rn(ahi, __shfl_down_sync(0xffffffffu, ahi, 8));
  const int m = lane & 15;
  if (n1 > n64 && m < 8) {
    const int a = lane >> 4;                 // 0 or 1 (lo), 2 or 3 (hi)
    blo = __fmaf_rn(hs[n64 + 8 * a + m], w2[n64 + 8 * a + m], blo);
    bhi = __fmaf_rn(hs[n64 + 8 * (a + 2) + m], w2[n64 + 8 * (a + 2) + m], bhi);
  }
  const float b1v = __shfl_down_sync(0xffffffffu, blo, 16);   // B_1[m] for lanes 0..7
  const float b3v = __shfl_down_sync(0xffffffffu, bhi, 16);   // B_3[m]
  const float s = __fadd_rn(__fadd_rn(__fadd_rn(blo, b1v), bhi), b3v);
  const float q = __fadd_rn(s, __shfl_down_sync(0xffffffffu, s, 4));
  const float q0 = __shfl_sync(0xffffffffu, q, 0), q1 = __shfl_sync(0xffffffffu, q, 1);
  const float q2 = __shfl_sync(0xffffffffu, q, 2), q3 = __shfl_sync(0xffffffffu, q, 3);
  float dot = n1 ? __fadd_rn(__fadd_rn(q0, q1), __fadd_rn(q2, q3)) : 0.f;
  for (int i = n1; i < H; ++i) dot = __fadd_rn(dot, __fmul_rn(hs[i], w2[i]));
  __syncwarp();
  return __fadd_rn(dot, b2);
}

// MLP of one row by one warp.  w1/b1/w2 may point to shared or global memory;
// hs: scratch of H floats.  Returns z2 in every lane.
__device__ __forceinline__ float warp_mlp(const float *feats, const float *w1, const float *b1, const float *w2,
                          float b2, int K, int H, float *hs, int lane) {
  mlp_z1<4>(feats, w1, b1, 3 * K, H, hs, lane, 0);
  __syncwarp();
  return z2_tree(z2_partial(hs, w2, H, lane), z2_partial(hs, w2, H, lane + 32), hs, w2, H, b2,
                 lane);
}
// Same, W1 read from global memory through the read-only path.
__device__ __forceinline__ float warp_mlp_g(const float *feats, const float *w1, const float *b1, const float *w2,
                            float b2, int K, int H, float *hs, int lane) {
  mlp_z1<4, true>(feats, w1, b1, 3 * K, H, hs, lane, 0);
  __syncwarp();
  return z2_tree(z2_partial(hs, w2, H, lane), z2_partial(hs, w2, H, lane + 32), hs, w2, H, b2,
                 lane);
}

__device__ __forceinline__ float sigmoid32(float z) {     // predictor.py:87-94, in f32
  if (z >= 0.f) return 1.f / (1.f + __expf(-z));
  const float ez = __expf(z);
  return ez / (1.f + ez);
}

__device__ __forceinline__ double sigmoid64(float z2) {   // predictor.py:87-94
  const double z = (double)z2;
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double ez = exp(z);
  return ez / (1.0 + ez);
}

// Everything after the logits, for one row (whole warp).
__device__ void warp_row_tail(const PredParams &p, int row, float *feats, const float *w1,
                              const float *b1, const float *w2, float *hs, int lane) {
  const int K = p.K;
  const bool ok = warp_softmax_features(p, row, feats, lane);
  if (p.logits_out) {
    if (lane < K) p.logits_out[(size_t)row * K + lane] = feats[lane];
    if (lane + 32 < K) p.logits_out[(size_t)row * K + lane + 32] = feats[lane + 32];
  }
  if (!ok) {
    if (lane == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  if (p.feat_out)
    for (int i = lane; i < 3 * K; i += 32) p.feat_out[(size_t)row * 3 * K + i] = feats[i];
  if (lane < K) p.prev[(size_t)row * K + lane] = feats[K + lane];            // engine.py:196
  if (lane + 32 < K) p.prev[(size_t)row * K + lane + 32] = feats[K + lane + 32];
  if (lane == 0 && p.evals) p.evals[row] += 1;
  if (p.policy == SPX_POLICY_MLP) {
    const float z2 = warp_mlp(feats, w1, b1, w2, p.b2, K, p.H, hs, lane);
    if (lane == 0) {
      if (p.z_out) p.z_out[row] = z2;
      if (p.prob_out) p.prob_out[row] = sigmoid64(z2);
      if (p.fired) p.fired[row] = (z2 >= p.z_cut) ? 1 : 0;
    }
  } else if (lane == 0) {
    if (p.prob_out) p.prob_out[row] = p.const_prob;
    if (p.z_out) p.z_out[row] = 0.0f;
    if (p.fired) p.fired[row] = (p.const_prob > p.threshold) ? 1 : 0;
  }
}

// ------------------------------------------------------------ FAST
#include "spx_pred_fast.cuh"
#include "spx_pred_stream.cuh"

// ----------------------------------------------------------- STRICT (parity)
// The reference's own operation sequence: every sum a left-to-right chain of
// separately rounded adds from 0, every product rounded (no FMA).  One CTA
// per row; the softmax/MLP tail is the same warp code as the FAST kernel.
constexpr int STRICT_THREADS = 128;

template <typename TW>
__global__ void __launch_bounds__(STRICT_THREADS)
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
  __shared__ float s_mean, s_denom;
  __shared__ int s_flag;
  const int tid = threadIdx.x, d = p.d;
  const float *x = p.hidden + (size_t)row * p.hidden_stride;
  if (tid == 0) s_flag = 0;
  __syncthreads();
  bool finite = true;
  for (int j = tid; j < d; j += STRICT_THREADS) { hn[j] = x[j]; finite &= is_finite(hn[j]); }
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
  for (int j = tid; j < d; j += STRICT_THREADS) hn[j] = __fsub_rn(hn[j], mean);
  __syncthreads();
  if (tid == 0) {
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, __fmul_rn(hn[j], hn[j]));
    s_denom = __fsqrt_rn(__fadd_rn(__fdiv_rn(acc, df), 1e-5f));
  }
  __syncthreads();
  const float denom = s_denom;
  for (int j = tid; j < d; j += STRICT_THREADS) hn[j] = ln_elem(hn[j], denom, p.norm_g[j], p.norm_b[j]);
  __syncthreads();
  const int K = p.K;
  if (tid < K) {
    int id = p.ids[(size_t)row * K + tid];
    if (id < 0 || id >= p.V) { atomicOr(p.err, ERR_ID_RANGE); s_flag = 1; id = 0; }
    const TW *wr = reinterpret_cast<const TW *>(p.head) + (size_t)id * d;
    float acc = 0.0f;
    for (int j = 0; j < d; j += CHUNK) {
      float w[4];
      load4_f32<TW>(wr + j, w);
#pragma unroll
      for (int e = 0; e < CHUNK; ++e) acc = __fadd_rn(acc, __fmul_rn(hn[j + e], w[e]));
    }
    feats[tid] = acc;
  }
  __syncthreads();
  if (tid >= 32) return;
  if (s_flag) {
    if (tid == 0 && p.fired) p.fired[row] = 0;
    return;
  }
  warp_row_tail(p, row, feats, p.w1, p.b1, p.w2, hs, tid);
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
  // the two sums stay strict left-to-right chains on thread 0; the operands are
  // staged through shared memory in chunks so the chain never waits on HBM
  constexpr int WCH = 2048;
  __shared__ float s_e[WCH], s_p[WCH];
  float esum = 0.f, psum = 0.f;
  for (int c0 = 0; c0 < K; c0 += WCH) {
    const int n = K - c0 < WCH ? K - c0 : WCH;
    for (int i = tid; i < n; i += blockDim.x) { s_e[i] = f[K + c0 + i]; s_p[i] = pv[c0 + i]; }
    __syncthreads();
    if (tid == 0) {
#pragma unroll 8
      for (int c = 0; c < n; ++c) {
        esum = __fadd_rn(esum, s_e[c]);
        psum = __fadd_rn(psum, s_p[c]);
      }
    }
    __syncthreads();
  }
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
    if (p.fired) p.fired[row] = (z2 >= p.z_cut) ? 1 : 0;
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
static int launch_predictor(const PredParams &p, const spx_predictor_args *a, cudaStream_t stream) {
  device_limits();
  bool strict = a->mode == SPX_MODE_STRICT;
  if (!strict) {
    // FAST shapes that neither the stream nor the team kernel can stage in shared
    // memory (e.g. d = 8192 with K > 8) take the reference-order kernel: exact,
    // one CTA per request
    const bool stream_ok = std::is_same<TW, __nv_bfloat16>::value && p.K <= SKMAX &&
                           (p.d == 2048 || p.d == 4096 || p.d == 8192);
    if (!stream_ok && plan_smem<TW>(p.d, p.K, p.H, g_smem_optin).bytes == 0) strict = true;
  }
  if (strict) {
    const size_t smem = (size_t)a->d * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(predictor_strict_kernel<TW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    predictor_strict_kernel<TW><<<(unsigned)a->B, STRICT_THREADS, smem, stream>>>(p);
  } else {
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
        // SPX_PRED_CTAS_PER_SM (sweeps): 1 leaves the second CTA slot of every SM
        // free for the next (programmatic dependent) launch's prefetch
        static const int env_cps = getenv("SPX_PRED_CTAS_PER_SM") ? atoi(getenv("SPX_PRED_CTAS_PER_SM")) : 2;
        if (env_cps == 1) per_sm = 1;
        const long long cap = (long long)per_sm * g_sms;
        const int grid = (int)(a->B < cap ? a->B : cap);
        StreamLaunch<TW> L{p, st, grid, stream, g_smem_optin, ldgx};
        if (p.d == 2048) L.template operator()<4>();
        else if (p.d == 4096) L.template operator()<8>();
        else L.template operator()<16>();
        return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
      }
    }
    // tuning overrides (benchmark sweeps only)
    static const int env_w1 = getenv("SPX_PRED_W1SMEM") ? atoi(getenv("SPX_PRED_W1SMEM")) : -1;
    static const int env_ring = getenv("SPX_PRED_RING") ? atoi(getenv("SPX_PRED_RING")) : -1;
    SmemPlan sp = plan_smem<TW>(p.d, p.K, p.H, g_smem_optin, env_w1, env_ring);
    if (sp.bytes == 0) return SPX_EINVAL;
    const long long need = (a->B + NTEAM - 1) / NTEAM;
    const int grid = (int)(need < g_sms ? need : g_sms);
    if (!dispatch_cpl(p.d, FastLaunch<TW>{p, sp, grid > 0 ? grid : 1, stream, g_smem_optin}))
      return SPX_EINVAL;
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
  if (a->hidden_stride % CHUNK) return SPX_EINVAL;
  if (a->B == 0) return 0;
  PredParams p;
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
  if (a->head_dtype == SPX_DTYPE_F32) return launch_predictor<float>(p, a, stream);
  if (a->head_dtype == SPX_DTYPE_BF16) return launch_predictor<__nv_bfloat16>(p, a, stream);
  return SPX_EINVAL;
}

extern "C" int spx_extract_features(const float *logits, const float *prev, float *feats_out,
                                    int32_t *err, int64_t B, int64_t K, void *stream) {
  if (!logits || !prev || !feats_out || !err || B < 0 || K < 1 || K > (1 << 24)) return SPX_EINVAL;
  if (B == 0) return 0;
  if (K > MAXK) {
    features_wide_kernel<<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>(logits, prev, feats_out,
                                                                       err, (int)K);
    return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
  }
  features_kernel<<<(unsigned)B, 32, 0, (cudaStream_t)stream>>>(
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
  mlp_kernel<<<(unsigned)B, 32, 0, (cudaStream_t)stream>>>(p, feats);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
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
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}
