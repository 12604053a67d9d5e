// Shared device code of the fused predictor kernels (K1-K3): parameters,
// the warp tails (softmax / features / MLP), the certification of FAST
// decisions and the STRICT row.  Included by spx_predictor.cu (dispatch,
// STRICT / recheck / function-level kernels), spx_pred_stream.cu and
// spx_pred_team.cu (the FAST kernel families, one translation unit each so
// they compile in parallel).
#pragma once
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
  // FAST-mode decision certification; recheck == nullptr: off
  const float *head_wmax;          // (V) max_j |W_vj|
  const float *cert;               // (3K+2) per-layer MLP constants
  float cert_kappa, cert_hnorm;
  float *prev_err;                 // (B)
  int *recheck;                    // (5 + B): see spx_predictor_args.recheck
  int recheck_inline;              // the FAST kernel drains the list itself (epilogue)
  uint8_t *fired_any;              // (B) optional: |= the decision (the token's "fired")
};

// the decision of a row: fired[row], and fired_any[row] |= it (ExitRecord's
// predictor_fired accumulates over the token's layers, engine.py:199-200)
__device__ __forceinline__ void write_fired(const PredParams &p, int row, bool f) {
  if (p.fired) p.fired[row] = f ? 1 : 0;
  if (f && p.fired_any) p.fired_any[row] = 1;
}

__device__ __forceinline__ bool row_skipped(const PredParams &p, int row) {
  if (p.row_done && p.row_done[row]) return true;
  if (p.row_layer_mask && !((p.row_layer_mask[row] >> p.layer) & 1ull)) return true;
  return false;
}

// ---------------------------------------------------------------- warp tail
// Softmax over the K logits in feats[0..K) (model.py:149-152), features
// (predictor.py:51-52) into feats[K..3K), validation (predictor.py:45-50).
// Whole warp; returns false (and flags err) on invalid input.
static __device__ bool warp_softmax_features(const PredParams &p, int row, float *feats, int lane) {
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
  // softmax denominator: strict left-to-right seq_sum (model.py:151); prev
  // check: numpy's pairwise ndarray.sum (predictor.py:49); replicated per lane
  float esum = 0.f;
  for (int c = 0; c < K; ++c)
    esum = __fadd_rn(esum, __shfl_sync(0xffffffffu, c < 32 ? e0 : e1, c & 31));
  const float psum = np_pairwise_block(
      0, K, [&](int c) { return __shfl_sync(0xffffffffu, c < 32 ? pv0 : pv1, c & 31); });
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
static __device__ float warp_row_tail(const PredParams &p, int row, float *feats, const float *w1,
                               const float *b1, const float *w2, float *hs, int lane) {
  const int K = p.K;
  const bool ok = warp_softmax_features(p, row, feats, lane);
  if (p.logits_out) {
    if (lane < K) p.logits_out[(size_t)row * K + lane] = feats[lane];
    if (lane + 32 < K) p.logits_out[(size_t)row * K + lane + 32] = feats[lane + 32];
  }
  if (!ok) {
    if (lane == 0 && p.fired) p.fired[row] = 0;
    return __int_as_float(0x7fc00000);
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
      write_fired(p, row, z2 >= p.z_cut);
    }
    return z2;
  } else if (lane == 0) {
    if (p.prob_out) p.prob_out[row] = p.const_prob;
    if (p.z_out) p.z_out[row] = 0.0f;
    write_fired(p, row, p.const_prob > p.threshold);
  }
  return __int_as_float(0x7fc00000);
}

// ------------------------------------------------------------ certification
// FAST-mode decisions are held to the reference's bit for bit.
// A FAST row's logits differ from the reference's sequential-sum logits only
// by rounding; the bound below turns that into a bound on z2, and a row whose
// |z2 - z_cut| exceeds it provably (under the stated rounding model) gets the
// reference's decision.  The rest are re-evaluated by the STRICT chain
// (predictor_recheck_kernel) in a follow-up launch.
//   logit:    e_c = kappa * (hnorm * wmax[id_c] * (1 + lnf) + |l_c|)
//             kappa = 2 lambda u sqrt(d), lambda = 8, u = 2^-24 (probabilistic
//             rounding-error model of Higham & Mary for both sums; the (1+lnf)
//             term covers the mean / variance passes, lnf = sqrt(1+mean^2/var))
//   softmax:  dp_k = p_k (e_k + sum_c p_c e_c + 8u(K+4)) + 2 max(e)^2
//   feature:  df = [e | dp | dp + prev_err + 2u|p - prev|]
//   MLP:      loose  sum_i M_i df_i,  M_i = sum_j |w2_j||W1_ij|
//             tight  sum_i |g_i| df_i + sum_{|z1_j| <= dz1_j} |w2_j| dz1_j with
//                    g_i = sum_{z1_j > dz1_j} w2_j W1_ij (exactly linear there)
//             + the rounding slack of both MLP evaluations.
constexpr float CERT_LAMBDA = 8.f;
constexpr float U24 = 5.9604644775390625e-8f;    // 2^-24

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

// Is |z2 - z_cut| larger than the largest change of z2 under feature
// perturbations bounded by df (plus rounding slack)?  f, df: 3K floats; hs:
// the row's relu(z1) (H floats, overwritten).  Whole warp, uniform result.
static __device__ bool mlp_margin_ok(const PredParams &p, const float *f, const float *df, float *hs,
                              const float *w1, const float *b1, const float *w2, float z2, int K,
                              int H, int lane) {
  if (!(fabsf(p.z_cut) <= 3.0e38f)) return true;        // NaN / inf cut: decision constant
  const int n = 3 * K;
  const float *M = p.cert;
  float sm = 0.f, sfm = 0.f, shw = 0.f;
  for (int i = lane; i < n; i += 32) {
    sm = fmaf(M[i], df[i], sm);
    sfm = fmaf(fabsf(f[i]), M[i], sfm);
  }
  for (int j = lane; j < H; j += 32) shw = fmaf(hs[j], fabsf(w2[j]), shw);
  sm = warp_butterfly_sum(sm);
  sfm = warp_butterfly_sum(sfm);
  shw = warp_butterfly_sum(shw);
  const float lu = CERT_LAMBDA * U24;
  const float rz1 = lu * sqrtf((float)(n + 1));
  const float eps_r = 2.f * (rz1 * (sfm + M[n]) + lu * sqrtf((float)H / 64.f + 8.f) * shw) +
                      4.f * U24 * (fabsf(z2) + fabsf(p.b2));
  const float gap = fabsf(z2 - p.z_cut);
  if (gap > (sm + eps_r) * 1.0001f) return true;
  // tight pass: classify units, gradient of the surely-active part
  float bsum = 0.f;
  for (int j = lane; j < H; j += 32) {
    float z1 = 0.f, dz = 0.f, fa = 0.f;
    for (int i = 0; i < n; ++i) {
      const float w = w1[(size_t)i * H + j];
      z1 = fmaf(f[i], w, z1);
      dz = fmaf(fabsf(w), df[i], dz);
      fa = fmaf(fabsf(f[i]), fabsf(w), fa);
    }
    z1 += b1[j];
    dz = dz * 1.0001f + 2.f * rz1 * (fa + fabsf(b1[j])) + 4.f * U24 * fabsf(z1);
    float coef = 0.f;
    if (z1 > dz) coef = w2[j];
    else if (z1 >= -dz) bsum = fmaf(fabsf(w2[j]), dz, bsum);
    hs[j] = coef;
  }
  __syncwarp();
  bsum = warp_butterfly_sum(bsum);
  float gs = 0.f;
  for (int i = 0; i < n; ++i) {
    float g = 0.f;
    for (int j = lane; j < H; j += 32) g = fmaf(hs[j], w1[(size_t)i * H + j], g);
    g = warp_butterfly_sum(g);
    gs = fmaf(fabsf(g), df[i], gs);
  }
  __syncwarp();
  return gap > (gs + bsum + eps_r) * 1.0001f;
}

// Certify one FAST row.  feats = [x | p | p - prev] (3K, shared memory, the
// computed FAST features), df: 3K scratch, hs: relu(z1) of the row (H,
// overwritten), lnf = sqrt(1 + mean^2/var) of the hidden row.  perr: bound on
// |p - p_ref| (the next layer's prev_err).  Whole warp.
// wmax(c) = head_wmax[id_c] (the caller may have prefetched it).
template <class WM>
__device__ __forceinline__ bool certify_row(const PredParams &p, int row, const float *feats,
                                            float *df, float *hs, const float *w1, const float *b1,
                                            const float *w2, float z2, float lnf, int K, int H,
                                            bool mlp, int lane, float &perr, WM wmax) {
  const float *x = feats, *pr = feats + K, *dv = feats + 2 * K;
  auto ebound = [&](int c) {
    return p.cert_kappa * fmaf(p.cert_hnorm * wmax(c), 1.f + lnf, fabsf(x[c]));
  };
  const float e0 = lane < K ? ebound(lane) : 0.f;
  const float e1 = lane + 32 < K ? ebound(lane + 32) : 0.f;
  const float emax = warp_max_f(fmaxf(e0, e1));
  const float spe = warp_butterfly_sum((lane < K ? pr[lane] * e0 : 0.f) +
                                       (lane + 32 < K ? pr[lane + 32] * e1 : 0.f));
  const float slackp = 8.f * U24 * (float)(K + 4);
  const float dprev = p.prev_err ? p.prev_err[row] : 0.f;
  float pe = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (c < K) {
      const float e = h ? e1 : e0;
      const float dp = fmaf(pr[c], e + spe + slackp, 2.f * emax * emax);
      df[c] = e;
      df[K + c] = dp;
      df[2 * K + c] = dp + dprev + 2.f * U24 * fabsf(dv[c]);
      pe = fmaxf(pe, dp);
    }
  }
  perr = warp_max_f(pe);
  __syncwarp();
  if (!mlp) return true;
  return mlp_margin_ok(p, feats, df, hs, w1, b1, w2, z2, K, H, lane);
}

// Deferred rows (p.recheck, int32): [3] total re-evaluated, [4] unresolved
// (cumulative statistics), [5 + row] = 1 while `row` awaits its STRICT
// re-evaluation.  The CTA that defers a row re-evaluates it in its own
// epilogue, so the common case (nothing deferred) costs no global atomics.
__device__ __forceinline__ void defer_row(const PredParams &p, int row, int *s_defer) {
  p.recheck[5 + row] = 1;
  atomicAdd(s_defer, 1);
}

// ----------------------------------------------------------- STRICT (parity)
// The reference's own operation sequence: every sum a left-to-right chain of
// separately rounded adds from 0, every product rounded (no FMA).  One CTA
// per row; the softmax/MLP tail is the same warp code as the FAST kernel.
// The K LM-head rows are staged through shared memory in 128-column chunks
// (double-buffered, loaded by the threads that do not run a chain) so each
// dot chain is bound by the FADD latency, not by global-load latency.
constexpr int STRICT_THREADS = 128;
constexpr int SCH = 128;                      // staged columns per chunk
constexpr int SCH_LD = SCH + 1;               // padded row stride (conflict-free chains)

inline size_t strict_smem_bytes(int d, int K) {
  return (size_t)d * 4 + (size_t)2 * K * SCH_LD * 4;
}

template <typename TW>
__device__ float strict_row(const PredParams &p, int row, uint8_t *dsmem, float *feats, float *hs,
                            int *ids_s, float *s_stat, int *s_flag) {
  float *hn = reinterpret_cast<float *>(dsmem);
  float *wst = hn + p.d;                      // [2][K][SCH_LD]
  const int tid = threadIdx.x, NT = blockDim.x, d = p.d, K = p.K;
  const float *x = p.hidden + (size_t)row * p.hidden_stride;
  if (tid == 0) *s_flag = 0;
  __syncthreads();
  bool finite = true;
  for (int j = tid; j < d; j += NT) { hn[j] = x[j]; finite &= is_finite(hn[j]); }
  if (!finite) { atomicOr(p.err, ERR_HIDDEN_NONFINITE); *s_flag = 1; }
  for (int c = tid; c < K; c += NT) {
    int id = p.ids[(size_t)row * K + c];
    if (id < 0 || id >= p.V) { atomicOr(p.err, ERR_ID_RANGE); *s_flag = 1; id = 0; }
    ids_s[c] = id;
  }
  __syncthreads();
  const TW *head = reinterpret_cast<const TW *>(p.head);
  auto stage = [&](int c0, float *buf, int t0, int nt) {
    const int per = SCH / CHUNK;
    for (int q = tid - t0; q < K * per; q += nt) {
      const int k = q / per, e4 = (q % per) * CHUNK;
      if (c0 + e4 < d) {
        float w[4];
        load4_f32<TW>(head + (size_t)ids_s[k] * d + c0 + e4, w);
#pragma unroll
        for (int e = 0; e < CHUNK; ++e) buf[k * SCH_LD + e4 + e] = w[e];
      }
    }
  };
  stage(0, wst, 0, NT);           // first chunk: overlaps the LN chains
  const float df = (float)d;
  if (tid == 0) {
    float acc = 0.0f;
#pragma unroll 8
    for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, hn[j]);
    s_stat[0] = __fdiv_rn(acc, df);
  }
  __syncthreads();
  const float mean = s_stat[0];
  for (int j = tid; j < d; j += NT) hn[j] = __fsub_rn(hn[j], mean);
  __syncthreads();
  if (tid == 0) {
    float acc = 0.0f;
#pragma unroll 8
    for (int j = 0; j < d; ++j) acc = __fadd_rn(acc, __fmul_rn(hn[j], hn[j]));
    s_stat[1] = __fsqrt_rn(__fadd_rn(__fdiv_rn(acc, df), 1e-5f));
  }
  __syncthreads();
  const float denom = s_stat[1];
  for (int j = tid; j < d; j += NT) hn[j] = ln_elem(hn[j], denom, p.norm_g[j], p.norm_b[j]);
  __syncthreads();
  float acc = 0.0f;
  const int nchunks = (d + SCH - 1) / SCH;
  for (int ci = 0; ci < nchunks; ++ci) {
    const float *buf = wst + (size_t)(ci & 1) * K * SCH_LD;
    if (ci + 1 < nchunks) {
      if (K < NT) {
        if (tid >= K) stage((ci + 1) * SCH, wst + (size_t)((ci + 1) & 1) * K * SCH_LD, K, NT - K);
      }
    }
    if (tid < K) {
      const int c0 = ci * SCH, n = d - c0 < SCH ? d - c0 : SCH;
      const float *wr = buf + tid * SCH_LD;
#pragma unroll 8
      for (int e = 0; e < n; ++e) acc = __fadd_rn(acc, __fmul_rn(hn[c0 + e], wr[e]));
    }
    __syncthreads();
  }
  if (tid < K) feats[tid] = acc;
  __syncthreads();
  if (tid >= 32) return 0.f;
  if (*s_flag) {
    if (tid == 0 && p.fired) p.fired[row] = 0;
    return __int_as_float(0x7fc00000);
  }
  return warp_row_tail(p, row, feats, p.w1, p.b1, p.w2, hs, tid);
}


// ---------------------------------------------------------- inline recheck
// Scratch of one STRICT re-evaluation in dynamic shared memory (floats):
// hn[d] | staged head chunks [2][K][SCH_LD] (rounded to 16 B) | feats, df
// [3*MAXK] | hs[MAXH] | ids[MAXK] | stat[2] | flag
__host__ __device__ inline size_t recheck_wst_floats(int K) {
  return ((size_t)2 * K * SCH_LD + 3) / 4 * 4;
}
inline size_t recheck_scratch_bytes(int d, int K) {
  return 4 * (((size_t)d + 3) / 4 * 4 + recheck_wst_floats(K) + 6 * MAXK + MAXH + MAXK + 8);
}

// STRICT re-evaluation of one deferred row by the whole CTA; writes every
// output the FAST launch withheld, prev = the reference probabilities,
// prev_err = 0, and counts the row in recheck[4] when the carried prev bound
// still straddled the cut.
template <typename TW>
__device__ void recheck_row(const PredParams &p, int row, float *scr) {
  const int d = p.d, K = p.K;
  float *feats = scr + (d + 3) / 4 * 4 + recheck_wst_floats(K), *df = feats + 3 * MAXK;
  float *hs = df + 3 * MAXK;
  int *ids_s = reinterpret_cast<int *>(hs + MAXH);
  float *stat = reinterpret_cast<float *>(ids_s + MAXK);
  int *flag = reinterpret_cast<int *>(stat + 2);
  const float dprev = p.prev_err ? p.prev_err[row] : 0.f;
  __syncthreads();
  const float z2 = strict_row<TW>(p, row, reinterpret_cast<uint8_t *>(scr), feats, hs, ids_s,
                                  stat, flag);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (dprev > 0.f && z2 == z2 && p.policy == SPX_POLICY_MLP) {
      for (int c = lane; c < 3 * K; c += 32)
        df[c] = c < 2 * K ? 0.f : dprev + 2.f * U24 * fabsf(feats[c]);
      __syncwarp();
      if (!mlp_margin_ok(p, feats, df, hs, p.w1, p.b1, p.w2, z2, K, p.H, lane) && lane == 0)
        atomicAdd(p.recheck + 4, 1);
    }
    if (lane == 0) {
      if (p.prev_err) p.prev_err[row] = 0.f;
      atomicAdd(p.recheck + 3, 1);
    }
  }
  __syncthreads();
}

// Every CTA of a FAST launch ends here (all threads): the rows this CTA
// deferred (s_defer counts them; their flags are recheck[5 + row]) are
// re-evaluated by the STRICT chain.  Nothing deferred: one shared load.
template <typename TW, class RowOf>
__device__ void recheck_epilogue(const PredParams &p, uint8_t *smem, const int *s_defer,
                                 int rows_cta, RowOf row_of) {
  __syncthreads();                                    // every role is done with smem
  if (!p.recheck || !p.recheck_inline || *s_defer == 0) return;
  float *scr = reinterpret_cast<float *>(smem);
  for (int i = 0; i < rows_cta; ++i) {
    const int row = row_of(i);
    if (*(volatile int *)(p.recheck + 5 + row)) {
      __syncthreads();                                // every thread has read the flag
      if (threadIdx.x == 0) p.recheck[5 + row] = 0;
      recheck_row<TW>(p, row, scr);
    }
  }
}
}  // namespace spx
