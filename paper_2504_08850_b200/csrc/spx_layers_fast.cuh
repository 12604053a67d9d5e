// FAST decoder-layer kernels for decode (a handful of rows per layer) at LLM
// shapes -- the flag consumers of the early-exit path (model.py:220-270,
// SURVEY.md §8a-16 / §8f-1).  Included by spx_layers.cu.
//
// A decode step touches every weight byte once and each row of the layer's
// input a few times, so each GEMV is HBM-bound: the design streams the weight
// matrix through shared memory with 1-D TMA bulk copies and keeps the input
// rows in registers.
//
//   * persistent CTAs (<= 1 per SM, 512 threads); CTA c owns a contiguous
//     range of output rows, streamed as stages of `rs` whole weight rows
//     (one cp.async.bulk per stage, ring of `stages` slots, mbarrier
//     complete_tx);
//   * column ownership: thread t owns 8-element chunks t, t+512, ... of the
//     contraction; its slice of every input row (LayerNorm'd in the prologue
//     where the layer has one) sits in registers for the whole kernel;
//   * per stage each thread forms its partial dot for every (weight row,
//     input row) pair (packed FFMA2), a 31-shuffle warp reduce-scatter leaves
//     one finished partial per lane, and 16 warp partials are summed in a
//     fixed order by the epilogue thread (deterministic);
//   * programmatic dependent launch: every kernel calls griddepcontrol.wait
//     before touching data the previous kernel wrote, and triggers its
//     dependents right after, so launch latency and (for Wo/FFN1/FFN2, whose
//     weights do not depend on anything) the first weight stages overlap the
//     previous kernel;
//   * the device exit flag `done` is checked first: an exited stream costs
//     one empty kernel per launch.
//
// One layer = 5 launches: LN1+QKV, attention, Wo+residual, LN2+FFN1+ReLU,
// FFN2+residual (+ frontier update and newest-row copy by the last CTA).
#pragma once
#include <type_traits>

namespace spx {

constexpr int GT = 512;                 // threads per GEMV CTA
constexpr int GW = GT / 32;
constexpr int GEMV_SMEM = 200 * 1024;   // dynamic shared memory budget
constexpr int STAGE_TARGET = 64 * 1024; // bytes per weight stage (target)

enum { EPI_QKV = 0, EPI_WO = 1, EPI_FFN1 = 2, EPI_FFN2 = 3 };

struct GemvGeom {
  int nout, kin;        // weight (nout, kin), out-row major
  int rs;               // weight rows per stage
  int stages;           // ring depth
  int pitch;            // bytes per ring slot (128-aligned)
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ bool flag_set(const uint8_t *f) {
  return f && *reinterpret_cast<const volatile uint8_t *>(f);
}

// Unfrozen rows with frontier == layer (model.py:230), ascending, into smem.
__device__ int cta_row_set(const LayerParams &p, int *rows) {
  __shared__ int s_wc[32];
  __shared__ int s_cnt;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int n = *reinterpret_cast<const volatile int32_t *>(p.n_ctx);
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool take = i < n && __ldcg(p.frontier + i) == p.layer && !(p.frozen && p.frozen[i]);
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (lane == 0) s_wc[w] = __popc(m);
    __syncthreads();
    int off = s_cnt;
    for (int j = 0; j < w; ++j) off += s_wc[j];
    if (take) rows[off + __popc(m & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) for (int j = 0; j < nw; ++j) s_cnt += s_wc[j];
    __syncthreads();
  }
  return s_cnt;
}

// Sum of RP values over the CTA (fixed order -> identical in every CTA).
template <int RP>
__device__ __forceinline__ void cta_sum(float (&v)[RP], float *scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], m);
    if (lane == 0) scr[r * GW + w] = v[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < GW; ++j) t += scr[r * GW + j];
    v[r] = t;
  }
  __syncthreads();
}

// Warp reduce-scatter of 32 values: afterwards lane L holds the warp-wide sum
// of v[L] (16+8+4+2+1 = 31 shuffles instead of 5 per value).
__device__ __forceinline__ float warp_reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int m = 16 >> s, half = 16 >> s;
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  return v[0];
}

// 8 weights from shared memory as floats
template <typename TW> struct SW8;
template <> struct SW8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float *f) {
    const uint4 u = *reinterpret_cast<const uint4 *>(p);
    bf16x4_to_f32(u.x, u.y, f);
    bf16x4_to_f32(u.z, u.w, f + 4);
  }
};
template <> struct SW8<float> {
  static __device__ __forceinline__ void load(const float *p, float *f) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    const float4 b = *reinterpret_cast<const float4 *>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

template <int EPI>
__device__ __forceinline__ const void *gemv_weights(const LayerParams &p) {
  return EPI == EPI_QKV ? p.wqkv : EPI == EPI_WO ? p.wo : EPI == EPI_FFN1 ? p.w1 : p.w2;
}

template <int EPI>
__device__ __forceinline__ void gemv_epilogue(const LayerParams &p, int row, int o, float v) {
  const int d = p.d;
  if (EPI == EPI_QKV) {
    if (o < d) p.s_q[(size_t)row * d + o] = v;
    else if (o < 2 * d) p.kc[(size_t)row * d + (o - d)] = v;
    else p.vc[(size_t)row * d + (o - 2 * d)] = v;
  } else if (EPI == EPI_WO) {
    float *x = p.pending + (size_t)row * d + o;
    *x = __fadd_rn(__ldcg(x), v);
  } else if (EPI == EPI_FFN1) {
    const float z = __fadd_rn(v, p.b1[o]);
    p.s_f[(size_t)row * p.ffn + o] = z > 0.f ? z : 0.f;
  } else {
    float *x = p.pending + (size_t)row * d + o;
    *x = __fadd_rn(__fadd_rn(__ldcg(x), v), p.b2[o]);
  }
}

// Input rows r0 .. r0+nr of this kernel, this thread's chunks, into registers
// (LayerNorm applied for QKV / FFN1, model.py:140-146; FAST statistics).
template <int CPT, int RP, int EPI>
__device__ __forceinline__ void gemv_load_x(const LayerParams &p, const int *rows, int r0, int nr,
                                            int kin, float (&x)[RP][CPT * 8], float *scr) {
  const int nch = kin >> 3;
  const bool ln = EPI == EPI_QKV || EPI == EPI_FFN1;
  const float *src = ln ? p.pending : EPI == EPI_WO ? p.s_att : p.s_f;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci) {
      const int c = threadIdx.x + ci * GT;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (r < nr && c < nch) {
        const float *q = src + (size_t)rows[r0 + r] * kin + c * 8;
        a = __ldcg(reinterpret_cast<const float4 *>(q));
        b = __ldcg(reinterpret_cast<const float4 *>(q + 4));
      }
      x[r][ci * 8 + 0] = a.x; x[r][ci * 8 + 1] = a.y; x[r][ci * 8 + 2] = a.z;
      x[r][ci * 8 + 3] = a.w; x[r][ci * 8 + 4] = b.x; x[r][ci * 8 + 5] = b.y;
      x[r][ci * 8 + 6] = b.z; x[r][ci * 8 + 7] = b.w;
    }
  }
  if (!ln) return;
  const float *g = EPI == EPI_QKV ? p.ln1_g : p.ln2_g;
  const float *bb = EPI == EPI_QKV ? p.ln1_b : p.ln2_b;
  const float df = (float)kin;
  float s[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    s[r] = 0.f;
#pragma unroll
    for (int e = 0; e < CPT * 8; ++e) s[r] += x[r][e];
  }
  cta_sum<RP>(s, scr);
  float mean[RP], v[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    mean[r] = s[r] / df;
    v[r] = 0.f;
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci) {
      if (threadIdx.x + ci * GT < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float c = x[r][ci * 8 + e] - mean[r];
          v[r] = fmaf(c, c, v[r]);
        }
      }
    }
  }
  cta_sum<RP>(v, scr);
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    const float den = sqrtf(v[r] / df + 1e-5f);
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci) {
      const int c = threadIdx.x + ci * GT;
      if (c < nch) {
        const float4 g0 = __ldg(reinterpret_cast<const float4 *>(g + c * 8));
        const float4 g1 = __ldg(reinterpret_cast<const float4 *>(g + c * 8 + 4));
        const float4 b0 = __ldg(reinterpret_cast<const float4 *>(bb + c * 8));
        const float4 b1 = __ldg(reinterpret_cast<const float4 *>(bb + c * 8 + 4));
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          x[r][ci * 8 + e] = (r < nr) ? ln_elem(x[r][ci * 8 + e] - mean[r], den, gg[e], bv[e]) : 0.f;
      }
    }
  }
}

template <typename TW, int CPT, int EPI>
__global__ void __launch_bounds__(GT, 1) gemv_layer_kernel(LayerParams p, GemvGeom g) {
  constexpr int RP = CPT >= 3 ? 2 : 4;     // input rows per pass
  constexpr int RSM = 32 / RP;             // max weight rows per stage
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char *wbuf = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)g.stages * g.pitch);
  float *red = reinterpret_cast<float *>(full + g.stages);   // [2][GW][32]
  float *scr = red + 2 * GW * 32;                             // [RP][GW]
  int *rows = reinterpret_cast<int *>(scr + RP * GW);         // [max_ctx]
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int o_begin = (int)((long long)blockIdx.x * g.nout / G);
  const int o_end = (int)((long long)(blockIdx.x + 1) * g.nout / G);
  const int nst = (o_end - o_begin + g.rs - 1) / g.rs;
  const size_t row_bytes = (size_t)g.kin * sizeof(TW);
  const unsigned char *W = reinterpret_cast<const unsigned char *>(gemv_weights<EPI>(p));

  auto issue = [&](int job) {               // thread 0 only
    const int st = job % nst, slot = job % g.stages;
    const int o = o_begin + st * g.rs;
    const int n = (o_end - o) < g.rs ? (o_end - o) : g.rs;
    const uint32_t bytes = (uint32_t)(n * row_bytes);
    mbar_arrive_expect_tx(&full[slot], bytes);
    bulk_g2s(wbuf + (size_t)slot * g.pitch, W + (size_t)o * row_bytes, bytes, &full[slot]);
  };

  if (tid == 0) {
    for (int s = 0; s < g.stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int issued = 0;
  if (EPI != EPI_QKV && nst > 0 && !flag_set(p.done) && tid == 0) {
    // weights are constant: start streaming before the previous kernel ends
    for (; issued < (nst < g.stages ? nst : g.stages); ++issued) issue(issued);
  }
  pdl_wait();
  const bool skip = flag_set(p.done);
  pdl_trigger();
  if (EPI == EPI_QKV && blockIdx.x == 0 && tid == 0 && !skip) *p.nrows = 0;   // FFN2 counter
  int nrows = 0;
  if (!skip) nrows = cta_row_set(p, rows);
  const int npass = (nrows + RP - 1) / RP;
  const int njobs = npass * nst;
  if (tid == 0 && !skip)
    for (; issued < (njobs < g.stages ? njobs : g.stages); ++issued) issue(issued);
  // drain stages issued before we learnt there is nothing to do
  if (skip || njobs == 0) {
    if (tid == 0)
      for (int j = 0; j < issued; ++j) mbar_wait(&full[j % g.stages], (j / g.stages) & 1);
    __syncthreads();
    if (skip) return;
  }

  const int nch = g.kin >> 3;
  for (int pass = 0; pass < npass; ++pass) {
    const int r0 = pass * RP;
    const int nr = nrows - r0 < RP ? nrows - r0 : RP;
    float x[RP][CPT * 8];
    gemv_load_x<CPT, RP, EPI>(p, rows, r0, nr, g.kin, x, scr);
    for (int st = 0; st < nst; ++st) {
      const int job = pass * nst + st, slot = job % g.stages;
      mbar_wait(&full[slot], (job / g.stages) & 1);
      const int o = o_begin + st * g.rs;
      const int n = (o_end - o) < g.rs ? (o_end - o) : g.rs;
      const TW *ws = reinterpret_cast<const TW *>(wbuf + (size_t)slot * g.pitch);
      float acc[32];
#pragma unroll
      for (int i = 0; i < RSM; ++i) {
        float2 s2[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) s2[r] = make_float2(0.f, 0.f);
        if (i < n) {
#pragma unroll
          for (int ci = 0; ci < CPT; ++ci) {
            const int c = tid + ci * GT;
            if (c < nch) {
              float w[8];
              SW8<TW>::load(ws + (size_t)i * g.kin + c * 8, w);
#pragma unroll
              for (int r = 0; r < RP; ++r) {
                if (r < nr) {
                  const float *xr = &x[r][ci * 8];
                  s2[r] = ffma2(make_float2(xr[0], xr[1]), make_float2(w[0], w[1]), s2[r]);
                  s2[r] = ffma2(make_float2(xr[2], xr[3]), make_float2(w[2], w[3]), s2[r]);
                  s2[r] = ffma2(make_float2(xr[4], xr[5]), make_float2(w[4], w[5]), s2[r]);
                  s2[r] = ffma2(make_float2(xr[6], xr[7]), make_float2(w[6], w[7]), s2[r]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int r = 0; r < RP; ++r) acc[i * RP + r] = s2[r].x + s2[r].y;
      }
      const float part = warp_reduce_scatter32(acc, lane);
      float *rb = red + (job & 1) * GW * 32;
      rb[warp * 32 + lane] = part;           // lane L holds value index L = i*RP + r
      __syncthreads();                        // slot consumed, partials visible
      if (tid == 0 && issued < njobs) issue(issued++);
      for (int idx = tid; idx < n * RP; idx += GT) {
        const int i = idx / RP, r = idx % RP;
        if (r < nr) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < GW; ++w) v += rb[w * 32 + idx];
          gemv_epilogue<EPI>(p, rows[r0 + r], o + i, v);
        }
      }
    }
  }

  if (EPI == EPI_FFN2) {
    // the last CTA advances the frontier and copies the newest row
    // (model.py:269-270 and run_layer's return value)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(p.nrows, 1) == G - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int i = tid; i < nrows; i += GT) p.frontier[rows[i]] = p.layer + 1;
      if (p.cur_hidden && p.new_row) {
        const int nr = *reinterpret_cast<const volatile int32_t *>(p.new_row);
        if (nr >= 0)
          for (int j = tid; j < p.d; j += GT) p.cur_hidden[j] = __ldcg(p.pending + (size_t)nr * p.d + j);
      }
      if (tid == 0) *p.nrows = 0;
    }
  }
}

// Attention for the layer's rows: one CTA per (row, head) item, keys split
// over 4 warps (model.py:247-262); FAST sums, numpy-exp softmax.
constexpr int AT = 128;
__global__ void __launch_bounds__(AT) attn_fast_kernel(LayerParams p) {
  extern __shared__ __align__(16) float asmem[];
  float *scores = asmem;                            // max_ctx
  float *qs = scores + p.max_ctx;                   // dh
  int *rows = reinterpret_cast<int *>(qs + (p.d / p.nh));   // max_ctx
  __shared__ float s_red[AT / 32];
  __shared__ float s_bc;
  pdl_wait();
  if (flag_set(p.done)) return;
  pdl_trigger();
  const int nrows = cta_row_set(p, rows);
  const int d = p.d, nh = p.nh, dh = d / nh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = AT / 32;
  const float scale = (float)(1.0 / sqrt((double)dh));
  for (int item = blockIdx.x; item < nrows * nh; item += gridDim.x) {
    const int row = rows[item / nh], h = item % nh;
    for (int e = tid; e < dh; e += AT) qs[e] = __ldcg(p.s_q + (size_t)row * d + h * dh + e);
    const int *ctx = nullptr;
    int nctx = row + 1;
    if (p.attn_ptr && p.attn_ptr[row + 1] > p.attn_ptr[row]) {
      ctx = p.attn_idx + p.attn_ptr[row];
      nctx = p.attn_ptr[row + 1] - p.attn_ptr[row];
    }
    __syncthreads();
    float mloc = -INFINITY;
    for (int jj = w; jj < nctx; jj += nw) {
      const int pos = ctx ? ctx[jj] : jj;
      const float *k = p.kc + (size_t)pos * d + h * dh;
      float acc = 0.f;
      for (int e = lane * 4; e < dh; e += 128) {
        const float4 kv = __ldcg(reinterpret_cast<const float4 *>(k + e));
        acc = fmaf(kv.x, qs[e], fmaf(kv.y, qs[e + 1], fmaf(kv.z, qs[e + 2], fmaf(kv.w, qs[e + 3], acc))));
      }
#pragma unroll
      for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
      const float sc = acc * scale;
      if (lane == 0) scores[jj] = sc;
      mloc = fmaxf(mloc, sc);
    }
    if (lane == 0) s_red[w] = mloc;
    __syncthreads();
    if (tid == 0) {
      float m = s_red[0];
      for (int j = 1; j < nw; ++j) m = fmaxf(m, s_red[j]);
      s_bc = m;
    }
    __syncthreads();
    const float m = s_bc;
    float sl = 0.f;
    for (int jj = tid; jj < nctx; jj += AT) {
      const float e = np_expf(scores[jj] - m);
      scores[jj] = e;
      sl += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
    __syncthreads();
    if (lane == 0) s_red[w] = sl;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int j = 0; j < nw; ++j) t += s_red[j];
      s_bc = 1.0f / t;
    }
    __syncthreads();
    const float inv = s_bc;
    for (int e = tid; e < dh; e += AT) {
      float acc = 0.f;
      for (int jj = 0; jj < nctx; ++jj) {
        const int pos = ctx ? ctx[jj] : jj;
        acc = fmaf(scores[jj], __ldcg(p.vc + (size_t)pos * d + h * dh + e), acc);
      }
      p.s_att[(size_t)row * d + h * dh + e] = acc * inv;
    }
    __syncthreads();
  }
}

template <typename K, typename... Args>
static void launch_pdl(K kern, int grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// ------------------------------------------------- tensor-core GEMV (bf16 weights)
//
// The CUDA-core kernel above is issue-bound (≈1.4K warp-instructions per 8 KB
// weight row: conversions, FFMA2, reductions).  For bf16 weights the product is
// instead formed on the tensor cores with mma.sync m16n8k16 (bf16 in, f32
// accumulate): D[a][n] = sum_k A[a][k] W[n][k] where the A rows are the input
// rows split into a bf16 head and a bf16 tail (x = hi + lo + O(2^-17 |x|)),
// so the result keeps fp32-level accuracy while the weights stay exact bf16.
// One m16n8k16 covers 8 weight rows x 16 columns for up to 4 input rows: ~3
// instructions per 256 bytes of weights, so the kernel is HBM-bound.
//
// Work: weight rows in groups of 32 (four n8 blocks) x contraction chunks of
// 512 columns ("items", 32 KB of weights each); CTA c takes a contiguous item
// range, so a group's chunks may straddle CTAs (split-K).  Straddling groups
// write their partial sums to s_part; the last arriving CTA (s_flag counter)
// adds the parts in part order -- deterministic.  Within a CTA the 8 warps
// split each chunk's k-steps and are summed in warp order through smem.
// Input rows: QKV/FFN1 LayerNorm'd and WO's attention rows are resident in
// smem as hi/lo bf16; FFN2's input (FFN1's ReLU output, written by FFN1 as
// hi/lo bf16 in the s_f row) is streamed chunk by chunk with the weights.
constexpr int MT = 256, MW = MT / 32;  // threads / warps per CTA
constexpr int MRG = 32;                // weight rows per group
constexpr int MKC = 512;               // contraction columns per chunk
constexpr int MRP = 4;                 // input rows per pass (A rows: 4 hi + 4 lo)
constexpr int MPITCH = MKC * 2 + 16;   // smem bytes per weight / x row segment
constexpr int MMA_SMEM = 225 * 1024;   // dynamic shared memory budget

struct MmaGeom {
  int nout, kin, ngroups, nkc, items, stages, slot_bytes;
};

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1,
                                               uint32_t a2, uint32_t a3, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void split_hilo(float x, __nv_bfloat16 &hi, __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

template <int EPI>
__device__ __forceinline__ void mma_epilogue(const LayerParams &p, int row, int o, float v) {
  if (EPI == EPI_FFN1) {
    // ReLU output stored as hi/lo bf16 in the row's s_f slot (FFN2's A operand)
    const float z = __fadd_rn(v, p.b1[o]);
    __nv_bfloat16 hi, lo;
    split_hilo(z > 0.f ? z : 0.f, hi, lo);
    __nv_bfloat16 *sf = reinterpret_cast<__nv_bfloat16 *>(p.s_f) + (size_t)row * 2 * p.ffn;
    sf[o] = hi;
    sf[p.ffn + o] = lo;
  } else {
    gemv_epilogue<EPI>(p, row, o, v);
  }
}

// CTA that owns item i (inverse of i0(c) = floor(c * items / G)).
__device__ __forceinline__ int mma_cta_of(long long i, int G, int items) {
  return (int)(((i + 1) * G - 1) / items);
}

template <int EPI>
__global__ void __launch_bounds__(MT, 1) gemv_mma_kernel(LayerParams p, MmaGeom g) {
  constexpr bool XS = EPI == EPI_FFN2;      // streamed input rows
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char *ring = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)g.stages * g.slot_bytes);
  const int xres_pitch = (g.kin + 8) * 2;   // bytes per resident hi/lo row
  unsigned char *xres = reinterpret_cast<unsigned char *>(full + g.stages);
  float *red = reinterpret_cast<float *>(xres + (XS ? 0 : (size_t)MRP * 2 * xres_pitch));
  float *scr = red + MW * 4 * 32;           // [MRP][MW]
  int *rows = reinterpret_cast<int *>(scr + MRP * MW);
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const unsigned char *W = reinterpret_cast<const unsigned char *>(gemv_weights<EPI>(p));
  const size_t wrow = (size_t)g.kin * 2;

  // item range: even split (single pass, split-K allowed) or whole groups
  int i0 = (int)((long long)c * g.items / G), i1 = (int)((long long)(c + 1) * g.items / G);
  int q_issue = 0, q_cons = 0, job_base = 0;    // ring sequence counters
  int nr_cur = 0;

  auto issue = [&](int job, int nj) {       // warp 0
    const int it = i0 + job % nj;
    const int grp = it / g.nkc, kc = it % g.nkc;
    const int rw0 = grp * MRG;
    const int nrw = g.nout - rw0 < MRG ? g.nout - rw0 : MRG;
    const int len = g.kin - kc * MKC < MKC ? g.kin - kc * MKC : MKC;
    const uint32_t bytes = (uint32_t)len * 2;
    const int slot = q_issue % g.stages;
    unsigned char *dst = ring + (size_t)slot * g.slot_bytes;
    if (lane == 0) mbar_arrive_expect_tx(&full[slot], bytes * nrw);
    __syncwarp();
    if (lane < nrw)
      bulk_g2s(dst + lane * MPITCH, W + (size_t)(rw0 + lane) * wrow + (size_t)kc * MKC * 2, bytes,
               &full[slot]);
    ++q_issue;
  };
  auto issue_x = [&](int job, int nj, int slot, int r0, int nr) {   // warp 0, XS only
    const int it = i0 + job % nj, kc = it % g.nkc;
    const int len = g.kin - kc * MKC < MKC ? g.kin - kc * MKC : MKC;
    const uint32_t bytes = (uint32_t)len * 2;
    unsigned char *dst = ring + (size_t)slot * g.slot_bytes + MRG * MPITCH;
    if (lane == 0) mbar_arrive_expect_tx(&full[slot], bytes * 2 * nr);
    __syncwarp();
    if (lane < 2 * nr) {
      const int r = lane >> 1, h = lane & 1;
      const __nv_bfloat16 *src = reinterpret_cast<const __nv_bfloat16 *>(p.s_f) +
                                 (size_t)rows[r0 + r] * 2 * g.kin + (size_t)h * g.kin +
                                 (size_t)kc * MKC;
      bulk_g2s(dst + lane * MPITCH, src, bytes, &full[slot]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < g.stages; ++s) mbar_init(&full[s], XS ? 2 : 1);
    fence_mbar_init();
  }
  __syncthreads();
  int nj = i1 - i0;
  int pre = 0;
  if (EPI != EPI_QKV && nj > 0 && !flag_set(p.done) && warp == 0)
    for (; pre < (nj < g.stages ? nj : g.stages); ++pre) issue(pre, nj);
  pdl_wait();
  const bool skip = flag_set(p.done);
  pdl_trigger();
  int nrows = skip ? 0 : cta_row_set(p, rows);
  const int npass = (nrows + MRP - 1) / MRP;
  if (npass > 1) {
    // several passes: whole groups per CTA so passes never share partials
    const int g0 = (int)((long long)c * g.ngroups / G), g1 = (int)((long long)(c + 1) * g.ngroups / G);
    i0 = g0 * g.nkc;
    i1 = g1 * g.nkc;
  }
  const int njn = i1 - i0;
  const int total = npass * njn;
  // drain prefetched stages that turned out useless (exit, no rows, or the
  // item split changed); completes their phases so the ring stays in sync
  if (warp == 0) {
    if (pre > 0 && (skip || total == 0 || npass > 1)) {
      for (int j = 0; j < pre; ++j) {
        const int slot = j % g.stages;
        if (XS && lane == 0) mbar_arrive(&full[slot]);
        mbar_wait(&full[slot], (j / g.stages) & 1);
      }
      q_cons = pre;                          // warp 0's view; broadcast below
    } else if (pre > 0 && XS) {
      nr_cur = nrows < MRP ? nrows : MRP;
      for (int j = 0; j < pre; ++j) issue_x(j, nj, j % g.stages, 0, nr_cur);
    }
  }
  // every thread learns the drained count
  __shared__ int s_drained;
  if (tid == 0) s_drained = (pre > 0 && (skip || total == 0 || npass > 1)) ? pre : 0;
  __syncthreads();
  q_cons = s_drained;
  job_base = q_cons;
  if (warp == 0 && s_drained) q_issue = s_drained;
  if (skip) return;
  nj = njn;
  if (warp == 0) {
    // top the ring up (jobs counted from job_base)
    const int have = s_drained ? 0 : pre;
    for (int job = have; job < (total < g.stages ? total : g.stages); ++job) {
      const int slot = q_issue % g.stages;
      issue(job, nj);
      if (XS) {
        const int pass = job / nj, r0 = pass * MRP;
        issue_x(job, nj, slot, r0, nrows - r0 < MRP ? nrows - r0 : MRP);
      }
    }
  }

  const int g8 = lane >> 2, cq = lane & 3;
  for (int pass = 0; pass < npass; ++pass) {
    const int r0 = pass * MRP;
    const int nr = nrows - r0 < MRP ? nrows - r0 : MRP;
    if (!XS) {
      // resident input rows as hi/lo bf16 (LayerNorm first for QKV / FFN1)
      const bool ln = EPI == EPI_QKV || EPI == EPI_FFN1;
      const float *src = ln ? p.pending : p.s_att;
      const float *gg = EPI == EPI_QKV ? p.ln1_g : p.ln2_g;
      const float *bb = EPI == EPI_QKV ? p.ln1_b : p.ln2_b;
      float mean[MRP], den[MRP];
      if (ln) {
        float s[MRP];
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
          s[r] = 0.f;
          if (r < nr)
            for (int j = tid; j < g.kin; j += MT) s[r] += __ldcg(src + (size_t)rows[r0 + r] * g.kin + j);
        }
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
#pragma unroll
          for (int m = 16; m; m >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], m);
          if (lane == 0) scr[r * MW + warp] = s[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
          float t = 0.f;
#pragma unroll
          for (int w = 0; w < MW; ++w) t += scr[r * MW + w];
          mean[r] = t / (float)g.kin;
          s[r] = 0.f;
          if (r < nr)
            for (int j = tid; j < g.kin; j += MT) {
              const float cc = __ldcg(src + (size_t)rows[r0 + r] * g.kin + j) - mean[r];
              s[r] = fmaf(cc, cc, s[r]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
#pragma unroll
          for (int m = 16; m; m >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], m);
          if (lane == 0) scr[r * MW + warp] = s[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < MRP; ++r) {
          float t = 0.f;
#pragma unroll
          for (int w = 0; w < MW; ++w) t += scr[r * MW + w];
          den[r] = sqrtf(t / (float)g.kin + 1e-5f);
        }
      }
#pragma unroll
      for (int r = 0; r < MRP; ++r) {
        __nv_bfloat16 *hrow = reinterpret_cast<__nv_bfloat16 *>(xres + (size_t)(r * 2) * xres_pitch);
        __nv_bfloat16 *lrow = reinterpret_cast<__nv_bfloat16 *>(xres + (size_t)(r * 2 + 1) * xres_pitch);
        for (int j = tid; j < g.kin; j += MT) {
          float v = 0.f;
          if (r < nr) {
            v = __ldcg(src + (size_t)rows[r0 + r] * g.kin + j);
            if (ln) v = ln_elem(v - mean[r], den[r], gg[j], bb[j]);
          }
          __nv_bfloat16 hi, lo;
          split_hilo(v, hi, lo);
          hrow[j] = hi;
          lrow[j] = lo;
        }
      }
      __syncthreads();
    }
    float D[4][4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) D[b][e] = 0.f;
    for (int j = 0; j < nj; ++j) {
      const int job = pass * nj + j;
      const int seq = job_base + job, slot = seq % g.stages;
      const int it = i0 + j, grp = it / g.nkc, kc = it % g.nkc;
      const int len = g.kin - kc * MKC < MKC ? g.kin - kc * MKC : MKC;
      const int nrw = g.nout - grp * MRG < MRG ? g.nout - grp * MRG : MRG;
      const int nblk = (nrw + 7) >> 3;
      mbar_wait(&full[slot], (seq / g.stages) & 1);
      const unsigned char *wb = ring + (size_t)slot * g.slot_bytes;
      const unsigned char *xb;
      int xp, xc0;
      if (XS) { xb = wb + MRG * MPITCH; xp = MPITCH; xc0 = 0; }
      else { xb = xres; xp = xres_pitch; xc0 = kc * MKC; }
      const int ks = len >> 4;
      const int s0 = warp * ks / MW, s1 = (warp + 1) * ks / MW;
      // A-row g8: input row (g8 & 3), head (g8 < 4) or tail (g8 >= 4)
      const bool arow = (g8 & 3) < nr;
      const unsigned char *xa = xb + (size_t)((g8 & 3) * 2 + (g8 >> 2)) * xp + (size_t)(xc0 + 2 * cq) * 2;
      const unsigned char *wa = wb + (size_t)g8 * MPITCH + 4 * cq;
      for (int s = s0; s < s1; ++s) {
        const int k = s * 16;
        uint32_t a0 = 0u, a2 = 0u;
        if (arow) {
          a0 = *reinterpret_cast<const uint32_t *>(xa + k * 2);
          a2 = *reinterpret_cast<const uint32_t *>(xa + k * 2 + 16);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b < nblk) {
            const unsigned char *wr = wa + (size_t)b * 8 * MPITCH + k * 2;
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(wr);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(wr + 16);
            mma_bf16_16816(D[b], a0, 0u, a2, 0u, b0, b1);
          }
        }
      }
      __syncthreads();                         // slot consumed by every warp
      if (warp == 0 && q_issue - job_base < total) {
        const int nxt = q_issue - job_base;
        const int nslot = q_issue % g.stages;
        issue(nxt, nj);
        if (XS) {
          const int npas = nxt / nj, nr0 = npas * MRP;
          issue_x(nxt, nj, nslot, nr0, nrows - nr0 < MRP ? nrows - nr0 : MRP);
        }
      }
      if (kc == g.nkc - 1 || j == nj - 1) {
        // group finished in this CTA: combine head + tail, then the warps
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const float v0 = D[b][0] + __shfl_xor_sync(0xffffffffu, D[b][0], 16);
          const float v1 = D[b][1] + __shfl_xor_sync(0xffffffffu, D[b][1], 16);
          if (lane < 16) {
            red[(warp * 4 + b) * 32 + lane * 2] = v0;
            red[(warp * 4 + b) * 32 + lane * 2 + 1] = v1;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) D[b][e] = 0.f;
        }
        __syncthreads();
        const long long gi0 = (long long)grp * g.nkc;
        const int first = npass > 1 ? c : mma_cta_of(gi0, G, g.items);
        const int last = npass > 1 ? c : mma_cta_of(gi0 + g.nkc - 1, G, g.items);
        const int nparts = last - first + 1;
        float v = 0.f;
        int idx = tid, row = -1, o = -1;
        if (idx < 128) {
          const int b = idx >> 5, l = (idx & 31) >> 1, e = idx & 1;
#pragma unroll
          for (int w = 0; w < MW; ++w) v += red[(w * 4 + b) * 32 + l * 2 + e];
          const int r = l >> 2, n = b * 8 + (l & 3) * 2 + e;
          if (r < nr && n < nrw) { row = rows[r0 + r]; o = grp * MRG + n; }
        }
        if (nparts == 1) {
          if (row >= 0) mma_epilogue<EPI>(p, row, o, v);
        } else {
          float *part = p.s_part + (size_t)gi0 * 128;
          if (idx < 128) part[(c - first) * 128 + idx] = v;
          __threadfence();
          __syncthreads();
          if (tid == 0) s_last = atomicAdd(p.s_flag + grp, 1) == nparts - 1;
          __syncthreads();
          if (s_last) {
            __threadfence();
            if (idx < 128) {
              float t = 0.f;
              for (int q = 0; q < nparts; ++q) t += __ldcg(part + q * 128 + idx);
              if (row >= 0) mma_epilogue<EPI>(p, row, o, t);
            }
            if (tid == 0) p.s_flag[grp] = 0;
          }
        }
      }
    }
  }

  if (EPI == EPI_FFN2) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(p.nrows, 1) == G - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int i = tid; i < nrows; i += MT) p.frontier[rows[i]] = p.layer + 1;
      if (p.cur_hidden && p.new_row) {
        const int nw = *reinterpret_cast<const volatile int32_t *>(p.new_row);
        if (nw >= 0)
          for (int j = tid; j < p.d; j += MT) p.cur_hidden[j] = __ldcg(p.pending + (size_t)nw * p.d + j);
      }
      if (tid == 0) *p.nrows = 0;
    }
  }
}

// ------------------------------------------------------------------ host side

static MmaGeom mma_geom(int nout, int kin, int sms, int max_ctx, bool xs, int &grid,
                        size_t &smem) {
  MmaGeom g;
  g.nout = nout;
  g.kin = kin;
  g.ngroups = (nout + MRG - 1) / MRG;
  g.nkc = (kin + MKC - 1) / MKC;
  g.items = g.ngroups * g.nkc;
  g.slot_bytes = (MRG * MPITCH + (xs ? 2 * MRP * MPITCH : 0) + 127) / 128 * 128;
  const size_t fixed = (xs ? 0 : (size_t)MRP * 2 * (kin + 8) * 2) + MW * 4 * 32 * 4 +
                       MRP * MW * 4 + (size_t)max_ctx * 4 + 16 * 8 + 1024;
  int st = (int)((MMA_SMEM - fixed) / g.slot_bytes);
  g.stages = st > 8 ? 8 : st;
  grid = g.items < sms ? g.items : sms;
  smem = (size_t)g.stages * g.slot_bytes + g.stages * 8 + fixed - 1024;
  return g;
}

static bool mma_layer_supported(const LayerParams &p) {
  if (p.d % 16 || p.ffn % 16 || !p.s_part || !p.s_flag) return false;
  int grid;
  size_t smem;
  const MmaGeom g = mma_geom(3 * p.d, p.d, 148, p.max_ctx, false, grid, smem);
  return g.stages >= 2;
}

template <int EPI>
static void launch_mma(const LayerParams &p, int nout, int kin, int sms, cudaStream_t s) {
  int grid;
  size_t smem;
  const MmaGeom g = mma_geom(nout, kin, sms, p.max_ctx, EPI == EPI_FFN2, grid, smem);
  cudaFuncSetAttribute(gemv_mma_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  launch_pdl(gemv_mma_kernel<EPI>, grid, MT, smem, s, p, g);
}

template <typename TW>
static GemvGeom gemv_geom(int nout, int kin, int sms, int max_ctx, int &grid, size_t &smem) {
  const int cpt = ((kin >> 3) + GT - 1) / GT;
  const int rp = cpt >= 3 ? 2 : 4;
  const int rsm = 32 / rp;
  GemvGeom g;
  g.nout = nout;
  g.kin = kin;
  const size_t row_bytes = (size_t)kin * sizeof(TW);
  int rs = (int)(STAGE_TARGET / row_bytes);
  rs = rs < 1 ? 1 : rs > rsm ? rsm : rs;
  g.rs = rs;
  g.pitch = (int)((rs * row_bytes + 127) / 128 * 128);
  const size_t fixed = 2 * GW * 32 * 4 + rp * GW * 4 + (size_t)max_ctx * 4 + 64 * 8;
  int st = (int)((GEMV_SMEM - fixed) / g.pitch);
  g.stages = st > 8 ? 8 : st;
  int gr = (nout + rs - 1) / rs;
  grid = gr < sms ? gr : sms;
  smem = (size_t)g.stages * g.pitch + g.stages * 8 + fixed;
  return g;
}

static bool fast_layer_supported(const LayerParams &p, size_t tw_size) {
  const int ks[2] = {p.d, p.ffn};
  for (int k : ks) {
    if (k % 8) return false;
    const int cpt = ((k >> 3) + GT - 1) / GT;
    if (cpt > 4) return false;
    if ((size_t)k * tw_size > (size_t)GEMV_SMEM / 2) return false;   // >= 2 stages of one row
  }
  return (size_t)p.max_ctx * 8 + 64 * 1024 < (size_t)GEMV_SMEM;
}


template <typename TW, int EPI>
static void launch_gemv(const LayerParams &p, int nout, int kin, int sms, cudaStream_t s) {
  int grid;
  size_t smem;
  const GemvGeom g = gemv_geom<TW>(nout, kin, sms, p.max_ctx, grid, smem);
  const int cpt = ((kin >> 3) + GT - 1) / GT;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, grid, GT, smem, s, p, g);
  };
  switch (cpt) {
    case 1: go(gemv_layer_kernel<TW, 1, EPI>); break;
    case 2: go(gemv_layer_kernel<TW, 2, EPI>); break;
    case 3: go(gemv_layer_kernel<TW, 3, EPI>); break;
    default: go(gemv_layer_kernel<TW, 4, EPI>); break;
  }
}

template <typename TW>
static void launch_layer_fast(const LayerParams &p, int sms, cudaStream_t s) {
  if (std::is_same<TW, __nv_bfloat16>::value && mma_layer_supported(p)) {
    launch_mma<EPI_QKV>(p, 3 * p.d, p.d, sms, s);
    const size_t ab = (size_t)p.max_ctx * 8 + (size_t)(p.d / p.nh) * 4;
    cudaFuncSetAttribute(attn_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ab);
    launch_pdl(attn_fast_kernel, 2 * sms, AT, ab, s, p);
    launch_mma<EPI_WO>(p, p.d, p.d, sms, s);
    launch_mma<EPI_FFN1>(p, p.ffn, p.d, sms, s);
    launch_mma<EPI_FFN2>(p, p.d, p.ffn, sms, s);
    return;
  }
  launch_gemv<TW, EPI_QKV>(p, 3 * p.d, p.d, sms, s);
  const size_t asm_bytes = (size_t)p.max_ctx * 8 + (size_t)(p.d / p.nh) * 4;
  cudaFuncSetAttribute(attn_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)asm_bytes);
  launch_pdl(attn_fast_kernel, 2 * sms, AT, asm_bytes, s, p);
  launch_gemv<TW, EPI_WO>(p, p.d, p.d, sms, s);
  launch_gemv<TW, EPI_FFN1>(p, p.ffn, p.d, sms, s);
  launch_gemv<TW, EPI_FFN2>(p, p.d, p.ffn, sms, s);
}

}  // namespace spx
