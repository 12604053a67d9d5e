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
__device__ void mlp_z1(const float *feats, const float *w1, const float *b1, int n, int H,
                       float *hs, int lane, int u0) {
  if ((H % 4) == 0) {
    for (int jb = 0; jb < H; jb += 512) {
      float y[NU][4];
#pragma unroll
      for (int u = 0; u < NU; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) y[u][e] = 0.f;
      if (n <= 48) {
#pragma unroll 4
        for (int i = 0; i < n; ++i) {
          const float f = feats[i];
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int j0 = jb + 4 * lane + 128 * (u0 + u);
            if (j0 < H) {
              const float4 w = ld_w1<W1G>(w1 + (size_t)i * H + j0);
              y[u][0] = __fmaf_rn(f, w.x, y[u][0]); y[u][1] = __fmaf_rn(f, w.y, y[u][1]);
              y[u][2] = __fmaf_rn(f, w.z, y[u][2]); y[u][3] = __fmaf_rn(f, w.w, y[u][3]);
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
                  t[u][0] = __fmaf_rn(f, w.x, t[u][0]); t[u][1] = __fmaf_rn(f, w.y, t[u][1]);
                  t[u][2] = __fmaf_rn(f, w.z, t[u][2]); t[u][3] = __fmaf_rn(f, w.w, t[u][3]);
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
__device__ float z2_tree(float alo, float ahi, const float *hs, const float *w2, int H, float b2,
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
__device__ float warp_mlp(const float *feats, const float *w1, const float *b1, const float *w2,
                          float b2, int K, int H, float *hs, int lane) {
  mlp_z1<4>(feats, w1, b1, 3 * K, H, hs, lane, 0);
  __syncwarp();
  return z2_tree(z2_partial(hs, w2, H, lane), z2_partial(hs, w2, H, lane + 32), hs, w2, H, b2,
                 lane);
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

// ------------------------------------------------------------ FAST (TMA)
// One 4-warp TEAM per row: warp w of the team owns canonical partial group
// g = w (partials 32w..32w+31), so every per-row reduction is split four
// ways; teams synchronise with their own named barrier.  Each team owns a
// shared-memory stage (hidden row + GROUP LM-head rows) filled by 1-D TMA
// bulk copies; the next row's copies are issued as soon as the current row's
// dot products are done.  Fast-path algebra (canonical, shared with K4/K6):
//   mean = CSUM(x)/d ; xc = x - mean ; var = CSUM(xc*xc)/d ; r = 1/sqrt(var+eps)
//   logit_v = r * CDOT(xc*g, W_v) + bw_v      (bw_v = CDOT(b, W_v), per model)
// i.e. the LayerNorm is folded into the head dot (one pass over the row for
// the variance and all K dots).
constexpr int TEAM = 4;
constexpr int MAXT = 4;
constexpr int RED_FLOATS = 32;    // (GROUP + 2) * 4 used

struct SmemPlan {
  int nt;          // teams (= row stages) per CTA
  int w1_smem;     // W1 staged in shared memory?
  size_t bytes;
  size_t off_g, off_w2, off_b1, off_w1, off_team, team_bytes, scratch_bytes, off_bar;
};

template <typename TW>
inline SmemPlan plan_smem(int d, int K, int H, int max_bytes) {
  SmemPlan best{};
  const size_t stage = (size_t)d * 4 + (size_t)GROUP * d * sizeof(TW);
  const size_t scratch = ((size_t)(RED_FLOATS + 4 + 3 * MAXK + (H > 0 ? H : 4) + 64) * 4 + 127) /
                         128 * 128;
  const size_t per_team = scratch + (stage + 127) / 128 * 128;
  const size_t w1b = ((size_t)3 * K * H * 4 + 127) / 128 * 128;
  const size_t fixed0 = (((size_t)d + 2 * H) * 4 + 127) / 128 * 128;
  for (int w1 = 0; w1 <= (H > 0 ? 1 : 0); ++w1) {
    const size_t fixed = fixed0 + (w1 ? w1b : 0);
    int nt = 0;
    for (int t = MAXT; t >= 1; --t)
      if (fixed + (size_t)t * per_team + (MAXT + 1) * 8 <= (size_t)max_bytes) { nt = t; break; }
    if (nt > best.nt || (nt == best.nt && nt > 0 && w1)) {
      SmemPlan s{};
      s.nt = nt; s.w1_smem = w1;
      size_t o = 0;
      s.off_g = o; o += (size_t)d * 4;
      s.off_w2 = o; o += (size_t)H * 4;
      s.off_b1 = o; o += (size_t)H * 4;
      o = (o + 127) / 128 * 128;
      s.off_w1 = o; if (w1) o += w1b;
      s.off_team = o; s.team_bytes = per_team; s.scratch_bytes = scratch;
      o += (size_t)nt * per_team;
      s.off_bar = o; o += (size_t)(nt + 1) * 8;
      s.bytes = o;
      best = s;
    }
  }
  return best;
}

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
}

template <typename TW, int CPL, bool FULL>
__global__ void __launch_bounds__(32 * TEAM * MAXT)
predictor_team_kernel(PredParams p, SmemPlan sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = warp / TEAM, w = warp % TEAM, nt = sp.nt;
  const int d = p.d, K = p.K, H = p.H, nchunk = d / CHUNK;
  float *gs = reinterpret_cast<float *>(smem + sp.off_g);
  float *w2s = reinterpret_cast<float *>(smem + sp.off_w2);
  float *b1s = reinterpret_cast<float *>(smem + sp.off_b1);
  float *w1s = reinterpret_cast<float *>(smem + sp.off_w1);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + sp.off_bar) + team;
  uint64_t *setup_bar = reinterpret_cast<uint64_t *>(smem + sp.off_bar) + nt;
  uint8_t *tbase = smem + sp.off_team + (size_t)team * sp.team_bytes;
  float *red = reinterpret_cast<float *>(tbase);            // [GROUP+2][4]
  int *tflag = reinterpret_cast<int *>(red + RED_FLOATS);   // [4]
  float *feats = red + RED_FLOATS + 4;
  float *hs = feats + 3 * MAXK;
  float *as = hs + (H > 0 ? H : 4);
  float *sh = reinterpret_cast<float *>(tbase + sp.scratch_bytes);
  TW *sw = reinterpret_cast<TW *>(tbase + sp.scratch_bytes + (size_t)d * 4);
  const TW *head = reinterpret_cast<const TW *>(p.head);

  const bool mlp = p.policy == SPX_POLICY_MLP;
  const bool bulk_consts = (H % 4) == 0;
  if (w == 0 && lane == 0 && team < nt) mbar_init(bar, 1);
  if (threadIdx.x == 0) mbar_init(setup_bar, 1);
  fence_mbar_init();
  __syncthreads();
  if (threadIdx.x == 0) {            // per-CTA constants by TMA
    uint32_t bytes = (uint32_t)d * 4u;
    if (mlp && bulk_consts) bytes += 2u * H * 4u + (sp.w1_smem ? 3u * K * H * 4u : 0u);
    mbar_arrive_expect_tx(setup_bar, bytes);
    bulk_g2s(gs, p.norm_g, (uint32_t)d * 4u, setup_bar);
    if (mlp && bulk_consts) {
      bulk_g2s(w2s, p.w2, (uint32_t)H * 4u, setup_bar);
      bulk_g2s(b1s, p.b1, (uint32_t)H * 4u, setup_bar);
      if (sp.w1_smem) bulk_g2s(w1s, p.w1, 3u * K * H * 4u, setup_bar);
    }
  }
  if (mlp && !bulk_consts) {
    for (int i = threadIdx.x; i < H; i += blockDim.x) { w2s[i] = p.w2[i]; b1s[i] = p.b1[i]; }
    if (sp.w1_smem)
      for (int i = threadIdx.x; i < 3 * K * H; i += blockDim.x) w1s[i] = p.w1[i];
    __syncthreads();
  }
  const float *w1 = sp.w1_smem ? w1s : p.w1;
  const uint32_t wrow_bytes = (uint32_t)((size_t)d * sizeof(TW));
  const bool leader = (w == 0 && lane == 0);

  // leader: TMA copies for `row` (hidden row when with_hidden, W rows of ids
  // [c0, c0+ng)); returns nonzero if an id was out of range (clamped to 0).
  auto issue_group = [&](int row, int c0, int ng, bool with_hidden) -> int {
    int bad = 0;
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, (with_hidden ? (uint32_t)d * 4u : 0u) + (uint32_t)ng * wrow_bytes);
    if (with_hidden)
      bulk_g2s(sh, p.hidden + (size_t)row * p.hidden_stride, (uint32_t)d * 4u, bar);
    for (int q = 0; q < ng; ++q) {
      int id = p.ids[(size_t)row * K + c0 + q];
      if (id < 0 || id >= p.V) { bad = 1; id = 0; }
      bulk_g2s(sw + (size_t)q * d, head + (size_t)id * d, wrow_bytes, bar);
    }
    return bad;
  };

  const int stride = gridDim.x * nt;
  int row = blockIdx.x * nt + team;
  if (team >= nt) return;
  uint32_t phase = 0;
  int id_bad = 0;
  bool skip = row >= p.B || row_skipped(p, row);
  if (leader && !skip) id_bad = issue_group(row, 0, K < GROUP ? K : GROUP, true);
  mbar_wait(setup_bar, 0);

  while (row < p.B) {
    const int next = row + stride;
    if (skip) {
      if (leader && p.fired) p.fired[row] = 0;
      row = next;
      skip = row >= p.B || row_skipped(p, row);
      if (leader && !skip) id_bad = issue_group(row, 0, K < GROUP ? K : GROUP, true);
      continue;
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    // ---- pass 1: mean (this warp = canonical group w)
    float part = 0.f;
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int c = 32 * w + lane + NPART * s;
      if (FULL || c < nchunk) {
        const float4 v = *reinterpret_cast<const float4 *>(sh + CHUNK * c);
        part = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(part, v.x), v.y), v.z), v.w);
      }
    }
    part = warp_butterfly_sum(part);
    if (lane == 0) red[GROUP * 4 + w] = part;
    team_sync(team);
    const float total = canon_combine(red[GROUP * 4 + 0], red[GROUP * 4 + 1], red[GROUP * 4 + 2],
                                      red[GROUP * 4 + 3]);
    const float mean = __fdiv_rn(total, (float)d);
    bool hbad = false;
    if (!is_finite(total)) {            // rare: exact element scan (model.py:310-311)
      bool fin = true;
      for (int c = 32 * w + lane; c < nchunk; c += NPART) {
        const float4 v = *reinterpret_cast<const float4 *>(sh + CHUNK * c);
        fin &= is_finite(v.x) & is_finite(v.y) & is_finite(v.z) & is_finite(v.w);
      }
      const bool wbad = __any_sync(0xffffffffu, !fin);
      if (lane == 0) tflag[w] = wbad ? 1 : 0;
      team_sync(team);
      hbad = (tflag[0] | tflag[1] | tflag[2] | tflag[3]) != 0;
      team_sync(team);
    }
    float r = 0.f;
    const float2 nmean = make_float2(-mean, -mean);
    // ---- pass 2 (per id group): variance (first group) + GROUP dots, packed
    // FP32 (FADD2/FMUL2/FFMA2) with per-chain order identical to CDOT.
    for (int c0 = 0; c0 < K; c0 += GROUP) {
      const int ng = (K - c0) < GROUP ? (K - c0) : GROUP;
      if (c0 > 0) {
        team_sync(team);                       // everyone done with the W stage / red
        if (leader) id_bad |= issue_group(row, c0, ng, false);
        mbar_wait(bar, phase);
        phase ^= 1u;
      }
      float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
      float sq = 0.f;
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int c = 32 * w + lane + NPART * s;
        if (FULL || c < nchunk) {
          const float4 xv = *reinterpret_cast<const float4 *>(sh + CHUNK * c);
          const float4 gv = *reinterpret_cast<const float4 *>(gs + CHUNK * c);
          const float2 xc01 = fadd2(make_float2(xv.x, xv.y), nmean);
          const float2 xc23 = fadd2(make_float2(xv.z, xv.w), nmean);
          if (c0 == 0)
            sq = __fmaf_rn(xc23.y, xc23.y, __fmaf_rn(xc23.x, xc23.x,
                           __fmaf_rn(xc01.y, xc01.y, __fmaf_rn(xc01.x, xc01.x, sq))));
          const float2 xg01 = fmul2(xc01, make_float2(gv.x, gv.y));
          const float2 xg23 = fmul2(xc23, make_float2(gv.z, gv.w));
          float wv[GROUP][4];
#pragma unroll
          for (int q = 0; q < GROUP; ++q) {
            Chunk<TW> ch;
            ch.lds(sw + (size_t)q * d + CHUNK * c);
            ch.to_f32(wv[q]);
          }
          const float xe[4] = {xg01.x, xg01.y, xg23.x, xg23.y};
#pragma unroll
          for (int e = 0; e < CHUNK; ++e) {
            const float2 xx = make_float2(xe[e], xe[e]);
            acc01 = ffma2(xx, make_float2(wv[0][e], wv[1][e]), acc01);
            acc23 = ffma2(xx, make_float2(wv[2][e], wv[3][e]), acc23);
          }
        }
      }
      float acc[GROUP] = {acc01.x, acc01.y, acc23.x, acc23.y};
#pragma unroll
      for (int q = 0; q < GROUP; ++q) acc[q] = warp_butterfly_sum(acc[q]);
      if (c0 == 0) sq = warp_butterfly_sum(sq);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < GROUP; ++q) red[q * 4 + w] = acc[q];
        if (c0 == 0) red[(GROUP + 1) * 4 + w] = sq;
      }
      team_sync(team);
      if (c0 == 0) {
        const float var = __fdiv_rn(canon_combine(red[(GROUP + 1) * 4 + 0], red[(GROUP + 1) * 4 + 1],
                                                  red[(GROUP + 1) * 4 + 2], red[(GROUP + 1) * 4 + 3]),
                                    (float)d);
        r = __frcp_rn(__fsqrt_rn(__fadd_rn(var, 1e-5f)));
      }
      if (w == 0 && lane < ng) {
        const int q = lane;
        int id = p.ids[(size_t)row * K + c0 + q];
        id = (id < 0 || id >= p.V) ? 0 : id;
        const float dot = canon_combine(red[q * 4 + 0], red[q * 4 + 1], red[q * 4 + 2], red[q * 4 + 3]);
        feats[c0 + q] = __fadd_rn(__fmul_rn(r, dot), p.head_bw ? __ldg(p.head_bw + id) : 0.f);
      }
    }
    const int ibad = __shfl_sync(0xffffffffu, id_bad, 0);   // leader's lane is lane 0 of w0
    team_sync(team);                                       // stage free, feats complete
    // ---- prefetch the next row while this row's tail runs
    const int nrow = next;
    const bool nskip = nrow >= p.B || row_skipped(p, nrow);
    if (leader) id_bad = nskip ? 0 : issue_group(nrow, 0, K < GROUP ? K : GROUP, true);
    // ---- softmax / features (warp 0), error handling
    if (w == 0) {
      int ok = 0;
      if (ibad || hbad) {
        if (lane == 0) atomicOr(p.err, (ibad ? ERR_ID_RANGE : 0) | (hbad ? ERR_HIDDEN_NONFINITE : 0));
      } else {
        ok = warp_softmax_features(p, row, feats, lane) ? 1 : 0;
      }
      if (p.logits_out && !ibad && !hbad) {
        if (lane < K) p.logits_out[(size_t)row * K + lane] = feats[lane];
        if (lane + 32 < K) p.logits_out[(size_t)row * K + lane + 32] = feats[lane + 32];
      }
      if (ok) {
        if (p.feat_out)
          for (int i = lane; i < 3 * K; i += 32) p.feat_out[(size_t)row * 3 * K + i] = feats[i];
        if (lane < K) p.prev[(size_t)row * K + lane] = feats[K + lane];          // engine.py:196
        if (lane + 32 < K) p.prev[(size_t)row * K + lane + 32] = feats[K + lane + 32];
        if (lane == 0 && p.evals) p.evals[row] += 1;
      } else if (lane == 0 && p.fired) {
        p.fired[row] = 0;
      }
      if (lane == 0) tflag[0] = ok;
    }
    team_sync(team);
    const int ok = tflag[0];
    if (ok) {
      if (mlp) {
        if (sp.w1_smem) mlp_z1<1, false>(feats, w1, b1s, 3 * K, H, hs, lane, w);
        else mlp_z1<1, true>(feats, w1, b1s, 3 * K, H, hs, lane, w);
        team_sync(team);
        if (w < 2) as[32 * w + lane] = z2_partial(hs, w2s, H, 32 * w + lane);
        team_sync(team);
        if (w == 0) {
          const float z2 = z2_tree(as[lane], as[lane + 32], hs, w2s, H, p.b2, lane);
          if (lane == 0) {
            if (p.z_out) p.z_out[row] = z2;
            if (p.prob_out) p.prob_out[row] = sigmoid64(z2);
            if (p.fired) p.fired[row] = (z2 >= p.z_cut) ? 1 : 0;
          }
        }
      } else if (leader) {
        if (p.prob_out) p.prob_out[row] = p.const_prob;
        if (p.z_out) p.z_out[row] = 0.0f;
        if (p.fired) p.fired[row] = (p.const_prob > p.threshold) ? 1 : 0;
      }
    }
    team_sync(team);                      // feats/hs/as/tflag reused by the next row
    row = nrow;
    skip = nskip;
  }
}

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
struct TeamLaunch {
  const PredParams &p; const SmemPlan &sp; int grid; cudaStream_t stream;
  template <int CPL> void operator()() const {
    if (p.d == CHUNK * NPART * CPL) launch<CPL, true>();
    else launch<CPL, false>();
  }
  template <int CPL, bool FULL> void launch() const {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(predictor_team_kernel<TW, CPL, FULL>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, g_smem_optin);
      configured = true;
    }
    predictor_team_kernel<TW, CPL, FULL>
        <<<grid > 0 ? grid : 1, 32 * TEAM * sp.nt, sp.bytes, stream>>>(p, sp);
  }
};

template <typename TW>
static int launch_predictor(const PredParams &p, const spx_predictor_args *a, cudaStream_t stream) {
  device_limits();
  if (a->mode == SPX_MODE_STRICT) {
    const size_t smem = (size_t)a->d * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(predictor_strict_kernel<TW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    predictor_strict_kernel<TW><<<(unsigned)a->B, STRICT_THREADS, smem, stream>>>(p);
  } else {
    if (((size_t)p.d * sizeof(TW)) % 16) return SPX_EINVAL;   // TMA bulk: 16-byte rows
    SmemPlan sp = plan_smem<TW>(p.d, p.K, p.H, g_smem_optin);
    if (sp.nt == 0) return SPX_EINVAL;
    const long long need = (a->B + sp.nt - 1) / sp.nt;
    const int grid = (int)(need < g_sms ? need : g_sms);
    if (!dispatch_cpl(p.d, TeamLaunch<TW>{p, sp, grid, stream})) return SPX_EINVAL;
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
  p.layer = a->layer; p.err = a->err;
  p.B = (int)a->B; p.d = (int)a->d; p.V = (int)a->V; p.K = (int)a->K;
  p.H = a->policy == SPX_POLICY_MLP ? (int)a->H : 0;
  if (a->head_dtype == SPX_DTYPE_F32) return launch_predictor<float>(p, a, stream);
  if (a->head_dtype == SPX_DTYPE_BF16) return launch_predictor<__nv_bfloat16>(p, a, stream);
  return SPX_EINVAL;
}

extern "C" int spx_extract_features(const float *logits, const float *prev, float *feats_out,
                                    int32_t *err, int64_t B, int64_t K, void *stream) {
  if (!logits || !prev || !feats_out || !err || B < 0 || K < 1 || K > MAXK) return SPX_EINVAL;
  if (B == 0) return 0;
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
