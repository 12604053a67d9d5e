// K4: full-head verification GEMV + argmax + membership (sm_100a), and the
// final LayerNorm kernel shared with the tree path.
//
// Reference: verify_exit (engine.py:59-64) = argmax(full_head_logits) in the
// speculative set; full_head_logits (model.py:289-295); the fall-through
// final argmax (engine.py:208-210); TreeEngine._verify_path (tree.py:274-283).
//
// HBM-bound: one pass over the (V, d) bf16 head (262 MB at Llama2-7B shape)
// for up to VER_ROWS gated rows at once; each vocab row is read by one warp
// with 16-byte loads and dotted in the canonical CDOT order (4 partials per
// lane == the 128 partials of the predictor kernel), so logits are
// bit-identical to K1's speculative logits.  The argmax is reduced with a
// 64-bit (orderable value, ~index) atomicMax -- value first, lowest index on
// ties, as np.argmax -- and the last CTA to finish resolves membership and
// writes the device exit flag.
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"
#include <type_traits>
#include <cstdlib>

namespace spx {

constexpr int VER_THREADS = 256;
constexpr int VER_ROWS = 4;          // gated rows handled per pass

struct VerParams {
  const float *hidden; int64_t hidden_stride;
  const float *g, *b;
  const void *head;
  const float *head_bw;
  const uint8_t *gate, *row_done;
  const int32_t *spec_ptr, *spec_ids;
  int32_t *token_out; uint8_t *verified_out; float *maxlogit_out, *logits_out;
  uint8_t *done_out; int32_t *exit_layer_out, *full_heads;
  int layer;
  unsigned long long *scratch; unsigned int *counter;
  int mode; int *err;
  int B, d, V;
  int32_t *topk_out; int topk_k;
};

__device__ __forceinline__ bool ver_row_on(const VerParams &p, int r) {
  if (p.row_done && p.row_done[r]) return false;
  if (p.gate && !p.gate[r]) return false;
  return true;
}

// Head-side normalisation of one row into `hn` (shared or global) by one warp.
// FAST: hn = xg = (x - mean) * g with the canonical statistics and *r_out =
// 1/sqrt(var + eps) -- the folded form logit = r * CDOT(xg, W) + bw used by
// every fast head kernel (identical bits to the predictor kernel).  STRICT:
// the reference LayerNorm (sequential sums, division; model.py:140-146),
// *r_out = 1.  `layer_norm_out` (FAST only) writes the plain LayerNorm value
// (xg * r + b) instead, for the function-level layer_norm.
template <int CPL>
__device__ void warp_head_prep(const float *x, const float *g, const float *b, int d, float *hn,
                               int lane, bool strict, float *r_out, int *bad,
                               bool layer_norm_out = false) {
  const float df = (float)d;
  for (int j = lane; j < d; j += 32) hn[j] = x[j];
  __syncwarp();
  if (!strict) {
    float mean, denom;
    bool bb;
    warp_ln_stats<CPL>(hn, d, lane, mean, denom, bb);
    if (bb) *bad = 1;
    const float r = __frcp_rn(denom);
    for (int j = lane; j < d; j += 32) {
      const float xg = __fmul_rn(__fsub_rn(hn[j], mean), g[j]);
      hn[j] = layer_norm_out ? __fadd_rn(__fmul_rn(xg, r), b[j]) : xg;
    }
    *r_out = r;
  } else {
    float m = 0.f, v = 0.f;
    bool fin = true;
    if (lane == 0) {
      for (int j = 0; j < d; ++j) { m = __fadd_rn(m, hn[j]); fin &= is_finite(hn[j]); }
      m = __fdiv_rn(m, df);
      for (int j = 0; j < d; ++j) {
        const float xc = __fsub_rn(hn[j], m);
        v = __fadd_rn(v, __fmul_rn(xc, xc));
      }
      v = __fsqrt_rn(__fadd_rn(__fdiv_rn(v, df), 1e-5f));
      if (!fin) *bad = 1;
    }
    const float mean = __shfl_sync(0xffffffffu, m, 0);
    const float denom = __shfl_sync(0xffffffffu, v, 0);
    __syncwarp();
    for (int j = lane; j < d; j += 32) hn[j] = ln_elem(__fsub_rn(hn[j], mean), denom, g[j], b[j]);
    *r_out = 1.0f;
  }
  __syncwarp();
}

// Canonical dot of one vocab row with R normed rows (smem); warp-cooperative.
template <typename TW, int R, int CPL>
__device__ __forceinline__ void warp_cdot(const TW *wrow, const float *hn, int d,
                                          int nr, int lane, float *out) {
  const int nchunk = d / CHUNK;
  float acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[r][g] = 0.f;
  // CPL = chunk steps per partial (nchunk <= 128*CPL)
  Chunk<TW> w[4][CPL];
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int c = 32 * g + lane + NPART * s;
      if (c < nchunk) w[g][s].load(wrow + CHUNK * c);
      else w[g][s].zero();
    }
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int c = 32 * g + lane + NPART * s;
      if (c < nchunk) {
        float wf[4];
        w[g][s].to_f32(wf);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < nr) {
            const float4 h = *reinterpret_cast<const float4 *>(hn + (size_t)r * d + CHUNK * c);
            acc[r][g] = __fmaf_rn(h.x, wf[0], acc[r][g]);
            acc[r][g] = __fmaf_rn(h.y, wf[1], acc[r][g]);
            acc[r][g] = __fmaf_rn(h.z, wf[2], acc[r][g]);
            acc[r][g] = __fmaf_rn(h.w, wf[3], acc[r][g]);
          }
        }
      }
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float gs[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) gs[g] = warp_butterfly_sum(acc[r][g]);
    out[r] = canon_combine(gs[0], gs[1], gs[2], gs[3]);
  }
}

template <typename TW, int CPL, int VR>
__global__ void __launch_bounds__(VER_THREADS)
verify_kernel(VerParams p) {
  const TW *head = reinterpret_cast<const TW *>(p.head);
  extern __shared__ float hn[];           // VR * d
  __shared__ int s_rows[VR];
  __shared__ int s_nr, s_bad;
  __shared__ float s_r[VR];
  __shared__ unsigned long long s_best[VER_THREADS / 32][VR];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = VER_THREADS / 32;
  const bool strict = p.mode == SPX_MODE_STRICT;

  __shared__ int s_next;
  int r0 = 0;
  while (true) {
    // collect the next <= VR gated rows (same on every CTA)
    if (threadIdx.x == 0) {
      int nr = 0, r = r0;
      for (; r < p.B && nr < VR; ++r)
        if (ver_row_on(p, r)) s_rows[nr++] = r;
      s_nr = nr;
      s_bad = 0;
      s_next = r;
    }
    __syncthreads();
    r0 = s_next;
    const int nr = s_nr;
    if (nr == 0) break;
    if (warp < nr) {
      int bad = 0;
      float rr = 1.f;
      warp_head_prep<CPL>(p.hidden + (size_t)s_rows[warp] * p.hidden_stride, p.g, p.b, p.d,
                          hn + (size_t)warp * p.d, lane, strict, &rr, &bad);
      if (lane == 0) s_r[warp] = rr;
      if (bad && lane == 0) { atomicOr(p.err, ERR_HIDDEN_NONFINITE); s_bad = 1; }
    }
    __syncthreads();
    unsigned long long best[VR];
#pragma unroll
    for (int r = 0; r < VR; ++r) best[r] = 0ull;
    const int gw = blockIdx.x * nwarps + warp, tw = gridDim.x * nwarps;
    if (!strict) {
      float rs[VR];
#pragma unroll
      for (int r = 0; r < VR; ++r) rs[r] = s_r[r];
      for (int v = gw; v < p.V; v += tw) {
        float lg[VR];
        warp_cdot<TW, VR, CPL>(head + (size_t)v * p.d, hn, p.d, nr, lane, lg);
        const float bw = p.head_bw ? p.head_bw[v] : 0.f;
#pragma unroll
        for (int r = 0; r < VR; ++r) {
          lg[r] = __fadd_rn(__fmul_rn(rs[r], lg[r]), bw);
          if (r < nr) {
            const unsigned long long k = argmax_key(lg[r], (uint32_t)v);
            best[r] = k > best[r] ? k : best[r];
            if (p.logits_out && lane == 0) p.logits_out[(size_t)s_rows[r] * p.V + v] = lg[r];
          }
        }
      }
    } else {
      // STRICT: one thread per vocab row, sequential chain over d (no FMA)
      const int gt = blockIdx.x * VER_THREADS + threadIdx.x, tt = gridDim.x * VER_THREADS;
      for (int v = gt; v < p.V; v += tt) {
        const TW *wr = head + (size_t)v * p.d;
        float acc[VR] = {};
        for (int j = 0; j < p.d; j += CHUNK) {
          float wf[4];
          load4_f32<TW>(wr + j, wf);
#pragma unroll
          for (int r = 0; r < VR; ++r)
            if (r < nr)
#pragma unroll
              for (int e = 0; e < CHUNK; ++e)
                acc[r] = __fadd_rn(acc[r], __fmul_rn(hn[(size_t)r * p.d + j + e], wf[e]));
        }
#pragma unroll
        for (int r = 0; r < VR; ++r)
          if (r < nr) {
            const unsigned long long k = argmax_key(acc[r], (uint32_t)v);
            best[r] = k > best[r] ? k : best[r];
            if (p.logits_out) p.logits_out[(size_t)s_rows[r] * p.V + v] = acc[r];
          }
      }
#pragma unroll
      for (int r = 0; r < VR; ++r)
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, best[r], m);
          best[r] = o > best[r] ? o : best[r];
        }
    }
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < VR; ++r) s_best[warp][r] = best[r];
    __syncthreads();
    if (threadIdx.x < nr) {
      unsigned long long b = 0ull;
      for (int w = 0; w < nwarps; ++w) b = s_best[w][threadIdx.x] > b ? s_best[w][threadIdx.x] : b;
      atomicMax(p.scratch + s_rows[threadIdx.x], b);
    }
    __syncthreads();
    if (r0 >= p.B) break;
  }
  // ---- last CTA resolves argmax tokens, membership and the exit flag
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int r = threadIdx.x; r < p.B; r += VER_THREADS) {
    if (!ver_row_on(p, r)) continue;
    const unsigned long long k = atomicExch(p.scratch + r, 0ull);
    const int tok = (int)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
    const float mx = f32_from_order_key((uint32_t)(k >> 32));
    bool in = false;
    if (p.spec_ptr)
      for (int i = p.spec_ptr[r]; i < p.spec_ptr[r + 1]; ++i) in |= (p.spec_ids[i] == tok);
    p.token_out[r] = tok;
    if (p.maxlogit_out) p.maxlogit_out[r] = mx;
    if (p.verified_out) p.verified_out[r] = in ? 1 : 0;
    if (p.full_heads) p.full_heads[r] += 1;
    if (in && p.done_out) {
      p.done_out[r] = 1;
      if (p.exit_layer_out) p.exit_layer_out[r] = p.layer;
    }
  }
  if (threadIdx.x == 0) *p.counter = 0u;
}

// FAST K4 for ONE row (B == 1: the decode step's gated verify and final
// argmax).  Same arithmetic as verify_kernel's FAST path (canonical CDOT,
// folded LayerNorm), so the logits are bit-identical.  Differences are in the
// schedule only: the gate is read first (a non-firing launch reads nothing
// from the head); every warp then issues its first vocab row's loads BEFORE
// the head-side LayerNorm, so the first HBM round trip overlaps the prologue;
// and the loop keeps the next row's loads in flight behind the current row's
// butterflies and argmax.  Two CTAs per SM.
template <typename TW, int CPL>
__global__ void __launch_bounds__(VER_THREADS, 2)
verify1_kernel(VerParams p) {
  const TW *head = reinterpret_cast<const TW *>(p.head);
  extern __shared__ float hn[];           // d
  __shared__ float s_r;
  __shared__ int s_on;
  __shared__ unsigned long long s_best[VER_THREADS / 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = VER_THREADS / 32;
  if (threadIdx.x == 0) s_on = ver_row_on(p, 0) ? 1 : 0;
  __syncthreads();
  const bool on = s_on != 0;
  const int nchunk = p.d / CHUNK;
  const int gw = blockIdx.x * nwarps + warp, tw = gridDim.x * nwarps;
  unsigned long long best = 0ull;
  if (on) {
    Chunk<TW> w[4][CPL];
    float bwn = 0.f;
    if (gw < p.V) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int s = 0; s < CPL; ++s) {
          const int c = 32 * g + lane + NPART * s;
          if (c < nchunk) w[g][s].load(head + (size_t)gw * p.d + CHUNK * c);
          else w[g][s].zero();
        }
      if (p.head_bw) bwn = __ldg(p.head_bw + gw);
    }
    if (warp == 0) {
      int bad = 0;
      float rr = 1.f;
      warp_head_prep<CPL>(p.hidden, p.g, p.b, p.d, hn, lane, false, &rr, &bad);
      if (lane == 0) s_r = rr;
      if (bad && lane == 0) atomicOr(p.err, ERR_HIDDEN_NONFINITE);
    }
    __syncthreads();
    const float rr = s_r;
    for (int v = gw; v < p.V;) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};       // canonical partial groups
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int s = 0; s < CPL; ++s) {
          const int c = 32 * g + lane + NPART * s;
          if (c < nchunk) {
            float wf[4];
            w[g][s].to_f32(wf);
            const float4 h = *reinterpret_cast<const float4 *>(hn + CHUNK * c);
            acc[g] = __fmaf_rn(h.x, wf[0], acc[g]);
            acc[g] = __fmaf_rn(h.y, wf[1], acc[g]);
            acc[g] = __fmaf_rn(h.z, wf[2], acc[g]);
            acc[g] = __fmaf_rn(h.w, wf[3], acc[g]);
          }
        }
      const float bw = bwn;
      const int vn = v + tw;
      if (vn < p.V) {                              // next row in flight during the reductions
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int s = 0; s < CPL; ++s) {
            const int c = 32 * g + lane + NPART * s;
            if (c < nchunk) w[g][s].load(head + (size_t)vn * p.d + CHUNK * c);
          }
        if (p.head_bw) bwn = __ldg(p.head_bw + vn);
      }
      float gs[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) gs[g] = warp_butterfly_sum(acc[g]);
      const float lg = __fadd_rn(__fmul_rn(rr, canon_combine(gs[0], gs[1], gs[2], gs[3])), bw);
      const unsigned long long k = argmax_key(lg, (uint32_t)v);
      best = k > best ? k : best;
      if (p.logits_out && lane == 0) p.logits_out[v] = lg;
      v = vn;
    }
    if (lane == 0) s_best[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long b = 0ull;
      for (int q = 0; q < nwarps; ++q) b = s_best[q] > b ? s_best[q] : b;
      atomicMax(p.scratch, b);
    }
  }
  // ---- last CTA resolves the argmax token, membership and the exit flag
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  if (on) {
    const unsigned long long k = atomicExch(p.scratch, 0ull);
    const int tok = (int)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
    bool in = false;
    if (p.spec_ptr)
      for (int i = p.spec_ptr[0]; i < p.spec_ptr[1]; ++i) in |= (p.spec_ids[i] == tok);
    p.token_out[0] = tok;
    if (p.maxlogit_out) p.maxlogit_out[0] = f32_from_order_key((uint32_t)(k >> 32));
    if (p.verified_out) p.verified_out[0] = in ? 1 : 0;
    if (p.full_heads) p.full_heads[0] += 1;
    if (in && p.done_out) {
      p.done_out[0] = 1;
      if (p.exit_layer_out) p.exit_layer_out[0] = p.layer;
    }
  }
  *p.counter = 0u;
}

// Final LayerNorm of N rows into hn (FAST: canonical, STRICT: sequential).
template <int CPL>
__global__ void final_norm_kernel(const float *x, int64_t stride, const float *g, const float *b,
                                  float *hn, float *r_out, int N, int d, int mode,
                                  int layer_norm_out, int *err) {
  // one warp per CTA and row; the row is normalised in shared memory (the
  // element loops of warp_head_prep are dependent global round trips when
  // run on a global buffer) and written out with coalesced 16-byte stores
  extern __shared__ float fn_row[];
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x;
  if (row >= N) return;
  int bad = 0;
  float r = 1.f;
  warp_head_prep<CPL>(x + (size_t)row * stride, g, b, d, fn_row, lane, mode == SPX_MODE_STRICT,
                      &r, &bad, layer_norm_out != 0);
  float4 *dst = reinterpret_cast<float4 *>(hn + (size_t)row * d);
  for (int j = lane; j < d / 4; j += 32) dst[j] = reinterpret_cast<const float4 *>(fn_row)[j];
  if (lane == 0 && r_out) r_out[row] = r;
  if (bad && lane == 0) atomicOr(err, ERR_HIDDEN_NONFINITE);
}

// bw[v] = CDOT(b, head_v), one warp per vocab row.
template <typename TW, int CPL>
__global__ void head_bias_kernel(const TW *head, const float *b, int V, int d, float *bw) {
  extern __shared__ float bs[];
  for (int j = threadIdx.x; j < d; j += blockDim.x) bs[j] = b[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x / 32;
  for (int v = blockIdx.x * nw + (threadIdx.x >> 5); v < V; v += gridDim.x * nw) {
    float out[1];
    warp_cdot<TW, 1, CPL>(head + (size_t)v * d, bs, d, 1, lane, out);
    if (lane == 0) bw[v] = out[0];
  }
}

}  // namespace spx
#include "spx_verify_tc.cuh"
namespace spx {

struct VerifyTcLaunch {
  const VerParams *p; const float *wmax; uint8_t *scratch; cudaStream_t stream; bool *ok;
  template <int CPL> void operator()() const {
    *ok = launch_verify_tc<CPL>(*p, wmax, scratch, stream);
  }
};

struct NormLaunch {
  const float *x; int64_t st; const float *g, *b; float *hn, *r; int N, d, mode, lno; int *err;
  unsigned grid; int threads; cudaStream_t stream;
  template <int CPL> void operator()() const {
    const size_t sm = (size_t)d * sizeof(float);
    if (sm > 48 * 1024)
      cudaFuncSetAttribute(final_norm_kernel<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    final_norm_kernel<CPL><<<(unsigned)N, 32, sm, stream>>>(x, st, g, b, hn, r, N, d, mode, lno, err);
  }
};

template <typename TW>
struct BiasLaunch {
  const TW *head; const float *b; int V, d; float *bw; cudaStream_t stream;
  template <int CPL> void operator()() const {
    head_bias_kernel<TW, CPL><<<592, 256, (size_t)d * 4, stream>>>(head, b, V, d, bw);
  }
};

}  // namespace spx

using namespace spx;

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename TW, int CPL>
static void launch_verify1(const VerParams &p, cudaStream_t stream) {
  if constexpr (std::is_same<TW, __nv_bfloat16>::value && CPL <= 8) {
    const size_t sm1 = (size_t)p.d * sizeof(float);
    if (sm1 > 48 * 1024)
      cudaFuncSetAttribute(verify1_kernel<TW, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sm1);
    // SPX_VERIFY1_PER_SM: CTAs per SM (1 leaves room for the next layer
    // kernel's CTA -- ~200 KB of shared memory -- to become resident and
    // prefetch its weights while a no-op gated verify drains)
    static const int per_sm = getenv("SPX_VERIFY1_PER_SM") ? atoi(getenv("SPX_VERIFY1_PER_SM")) : 2;
    verify1_kernel<TW, CPL><<<per_sm * num_sms(), VER_THREADS, sm1, stream>>>(p);
  }
}

template <typename TW, int CPL>
static void launch_verify_wide(const VerParams &p, cudaStream_t stream) {
  if constexpr (std::is_same<TW, __nv_bfloat16>::value && CPL <= 8) {
    const size_t sm8 = (size_t)8 * p.d * sizeof(float);
    cudaFuncSetAttribute(verify_kernel<TW, CPL, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm8);
    verify_kernel<TW, CPL, 8><<<num_sms(), VER_THREADS, sm8, stream>>>(p);
  }
}

template <typename TW>
static int launch_verify(const VerParams &p, int nchunk, int grid, size_t smem,
                         cudaStream_t stream) {
  const bool one = p.B == 1 && p.mode != SPX_MODE_STRICT &&
                   std::is_same<TW, __nv_bfloat16>::value && nchunk <= 8 * NPART;
  // SPX_VERIFY_WIDE=1 (A/B, off): 8 rows per pass over the head for more than
  // VER_ROWS rows.  Measured slower (tree draft level, 5-10 rows: 505 vs 283 us
  // per launch): one CTA per SM and 8 shared-memory row reads per weight
  // element make it shared-memory bound.
  static const int env_wide = getenv("SPX_VERIFY_WIDE") ? atoi(getenv("SPX_VERIFY_WIDE")) : 0;
  const bool wide = env_wide && !one && p.B > VER_ROWS && p.mode != SPX_MODE_STRICT &&
                    std::is_same<TW, __nv_bfloat16>::value && nchunk <= 8 * NPART &&
                    (size_t)8 * p.d * sizeof(float) <= 200 * 1024;
#define SPX_LAUNCH_VER(CPL)                                                                    \
  do {                                                                                         \
    if (one) {                                                                                 \
      launch_verify1<TW, CPL>(p, stream);                                                      \
      break;                                                                                   \
    }                                                                                          \
    if (wide) {                                                                                \
      launch_verify_wide<TW, CPL>(p, stream);                                                  \
      break;                                                                                   \
    }                                                                                          \
    if (smem > 48 * 1024)                                                                      \
      cudaFuncSetAttribute(verify_kernel<TW, CPL, VER_ROWS>,                                   \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    verify_kernel<TW, CPL, VER_ROWS><<<grid, VER_THREADS, smem, stream>>>(p);                  \
  } while (0)
  if (nchunk <= NPART) SPX_LAUNCH_VER(1);
  else if (nchunk <= 2 * NPART) SPX_LAUNCH_VER(2);
  else if (nchunk <= 4 * NPART) SPX_LAUNCH_VER(4);
  else if (nchunk <= 8 * NPART) SPX_LAUNCH_VER(8);
  else if (nchunk <= 16 * NPART) SPX_LAUNCH_VER(16);     // d <= 8192 (e.g. Llama2-13B 5120)
  else return SPX_EINVAL;
#undef SPX_LAUNCH_VER
  return spx_launch_status("spx_verify");
}

extern "C" int spx_verify(const spx_verify_args *a, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!a || a->B < 0 || a->d <= 0 || a->d % CHUNK || a->V <= 0 || a->V > 0x7fffffff) return SPX_EINVAL;
  if (!a->hidden || !a->norm_g || !a->norm_b || !a->head || !a->token_out || !a->scratch ||
      !a->counter || !a->err)
    return SPX_EINVAL;
  if (a->B == 0) return 0;
  VerParams p;
  p.hidden = a->hidden; p.hidden_stride = a->hidden_stride ? a->hidden_stride : a->d;
  p.g = a->norm_g; p.b = a->norm_b;
  p.head = a->head; p.head_bw = a->head_bw;
  p.gate = a->gate; p.row_done = a->row_done; p.spec_ptr = a->spec_ptr; p.spec_ids = a->spec_ids;
  p.token_out = a->token_out; p.verified_out = a->verified_out; p.maxlogit_out = a->maxlogit_out;
  p.logits_out = a->logits_out; p.done_out = a->done_out; p.exit_layer_out = a->exit_layer_out;
  p.full_heads = a->full_heads; p.layer = a->layer; p.scratch = a->scratch; p.counter = a->counter;
  p.mode = a->mode; p.err = a->err; p.B = (int)a->B; p.d = (int)a->d; p.V = (int)a->V;
  p.topk_out = nullptr; p.topk_k = 0;
  // many gated rows, FAST, bf16 head: the tensor-core form (spx_verify_tc.cuh)
  static const int env_tc = getenv("SPX_VERIFY_TC") ? atoi(getenv("SPX_VERIFY_TC")) : 1;
  if (env_tc && a->tc_scratch && a->head_wmax && a->mode != SPX_MODE_STRICT &&
      a->head_dtype == SPX_DTYPE_BF16 && !a->logits_out && a->d % TV_BK == 0 &&
      (a->B >= SPX_VERIFY_TC_MIN_ROWS || a->topk_out) && a->B <= 0x7fff) {
    if (a->topk_out && (a->topk_k < 1 || a->topk_k > 64 || a->topk_k > a->V)) return SPX_EINVAL;
    p.topk_out = a->topk_out; p.topk_k = a->topk_out ? a->topk_k : 0;
    bool ok = false;
    if (dispatch_cpl((int)a->d, VerifyTcLaunch{&p, a->head_wmax,
                                               reinterpret_cast<uint8_t *>(a->tc_scratch), stream,
                                               &ok}) && ok)
      return spx_launch_status("spx_verify(tc)");
  }
  if (a->topk_out) return SPX_EINVAL;               // top-K only in the tensor-core form
  const size_t smem = (size_t)VER_ROWS * a->d * sizeof(float);
  const int nchunk = (int)(a->d / CHUNK);
  const int warps_per_cta = VER_THREADS / 32;
  int grid = (int)((a->V + warps_per_cta - 1) / warps_per_cta);
  const int cap = num_sms() * 2;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (a->head_dtype == SPX_DTYPE_BF16)
    return launch_verify<__nv_bfloat16>(p, nchunk, grid, smem, stream);
  if (a->head_dtype == SPX_DTYPE_F32) return launch_verify<float>(p, nchunk, grid, smem, stream);
  return SPX_EINVAL;
}

extern "C" int64_t spx_verify_tc_logits_offset(int64_t B, int64_t d, int64_t V) {
  if (B <= 0 || d <= 0 || V <= 0) return -1;
  return (int64_t)tv_layout((int)B, (int)d, (int)V).tl;
}

extern "C" int64_t spx_verify_tc_scratch_bytes(int64_t B, int64_t d, int64_t V) {
  if (B <= 0 || d <= 0 || V <= 0) return 0;
  return (int64_t)tv_layout((int)B, (int)d, (int)V).total;
}

extern "C" int spx_final_norm(const float *hidden, int64_t hidden_stride, const float *g,
                              const float *b, float *hn, int64_t N, int64_t d, int32_t mode,
                              int32_t *err, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!hidden || !g || !b || !hn || !err || N < 0 || d <= 0 || d % CHUNK) return SPX_EINVAL;
  if (N == 0) return 0;
  const int wpc = 4;
  const unsigned grid = (unsigned)((N + wpc - 1) / wpc);
  const int64_t st = hidden_stride ? hidden_stride : d;
  if (!dispatch_cpl((int)d, NormLaunch{hidden, st, g, b, hn, nullptr, (int)N, (int)d, mode, 1,
                                       err, grid, wpc * 32, stream}))
    return SPX_EINVAL;
  return spx_launch_status("spx_final_norm");
}

extern "C" int spx_head_prep(const float *hidden, int64_t hidden_stride, const float *g,
                             const float *b, float *xg, float *r, int64_t N, int64_t d,
                             int32_t mode, int32_t *err, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!hidden || !g || !b || !xg || !r || !err || N < 0 || d <= 0 || d % CHUNK) return SPX_EINVAL;
  if (N == 0) return 0;
  const int wpc = 4;
  const unsigned grid = (unsigned)((N + wpc - 1) / wpc);
  const int64_t st = hidden_stride ? hidden_stride : d;
  if (!dispatch_cpl((int)d, NormLaunch{hidden, st, g, b, xg, r, (int)N, (int)d, mode, 0, err,
                                       grid, wpc * 32, stream}))
    return SPX_EINVAL;
  return spx_launch_status("spx_head_prep");
}

extern "C" int spx_head_bias(const void *head, int32_t head_dtype, const float *b, int64_t V,
                             int64_t d, float *bw, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!head || !b || !bw || V <= 0 || d <= 0 || d % CHUNK) return SPX_EINVAL;
  if ((size_t)d * 4 > 48 * 1024) return SPX_EINVAL;
  bool ok;
  if (head_dtype == SPX_DTYPE_BF16)
    ok = dispatch_cpl((int)d, BiasLaunch<__nv_bfloat16>{(const __nv_bfloat16 *)head, b, (int)V,
                                                        (int)d, bw, stream});
  else if (head_dtype == SPX_DTYPE_F32)
    ok = dispatch_cpl((int)d, BiasLaunch<float>{(const float *)head, b, (int)V, (int)d, bw, stream});
  else
    return SPX_EINVAL;
  if (!ok) return SPX_EINVAL;
  return spx_launch_status("spx_head_bias");
}
