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
#include <cstdlib>

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
  // the first block of frontier / frozen entries is read together with n_ctx
  // (independent loads: one memory round trip instead of two)
  const int t0 = threadIdx.x;
  const int f0 = t0 < p.max_ctx ? __ldcg(p.frontier + t0) : -1;
  const bool z0 = p.frozen && t0 < p.max_ctx && p.frozen[t0];
  __syncthreads();
  const int n = *reinterpret_cast<const volatile int32_t *>(p.n_ctx);
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool take = i < n && (base == 0 ? (f0 == p.layer && !z0)
                                          : (__ldcg(p.frontier + i) == p.layer &&
                                             !(p.frozen && p.frozen[i])));
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (lane == 0) s_wc[w] = __popc(m);
    __syncthreads();
    int off = s_cnt;
    for (int j = 0; j < w; ++j) off += s_wc[j];
    if (take) {
      const int slot = off + __popc(m & ((1u << lane) - 1u));
      if (slot < p.row_cap) rows[slot] = i;
      else atomicOr(p.err, ERR_ROW_CAP);
    }
    __syncthreads();
    if (threadIdx.x == 0) for (int j = 0; j < nw; ++j) s_cnt += s_wc[j];
    __syncthreads();
  }
  return s_cnt < p.row_cap ? s_cnt : p.row_cap;
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
inline const void *gemv_weights_host(const LayerParams &p) {
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
  float *scores = asmem;                            // att_cap
  float *qs = scores + p.att_cap;                   // dh
  int *rows = reinterpret_cast<int *>(qs + (p.d / p.nh));   // row_cap
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

// Head dim 128 (Llama2-7B / 13B): the same attention, one WARP per
// (row, head) item (no CTA barrier per item; 4 items in flight per CTA), the
// key loops latency-hidden -- 4 keys per iteration (4 independent 512-byte
// K/V row loads in flight), lane = 4 consecutive head dims.  GROWS: the row
// set comes from tcl_rows_kernel (p.rows / *p.nrows) instead of a per-CTA
// frontier scan.
template <bool GROWS>
__global__ void __launch_bounds__(AT) attn_fast128_kernel(LayerParams p) {
  constexpr int DH = 128, NW = AT / 32;
  extern __shared__ __align__(16) float asmem[];
  const int sstride = (p.att_cap + 3) / 4 * 4;
  int *rows = reinterpret_cast<int *>(asmem + NW * sstride);   // row_cap (!GROWS)
  pdl_wait();
  if (flag_set(p.done)) return;
  pdl_trigger();
  int nrows;
  const int *rowp;
  if (GROWS) {
    nrows = *reinterpret_cast<const volatile int32_t *>(p.nrows);
    rowp = p.rows;
  } else {
    nrows = cta_row_set(p, rows);
    rowp = rows;
  }
  const int d = p.d, nh = p.nh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float *scores = asmem + w * sstride;
  const float scale = (float)(1.0 / sqrt((double)DH));
  for (int item = blockIdx.x * NW + w; item < nrows * nh; item += gridDim.x * NW) {
    const int row = rowp[item / nh], h = item % nh;
    const float4 q = __ldcg(reinterpret_cast<const float4 *>(p.s_q + (size_t)row * d + h * DH) + lane);
    const int *ctx = nullptr;
    int nctx = row + 1;
    if (p.attn_ptr && p.attn_ptr[row + 1] > p.attn_ptr[row]) {
      ctx = p.attn_idx + p.attn_ptr[row];
      nctx = p.attn_ptr[row + 1] - p.attn_ptr[row];
    }
    float m = -INFINITY;
    for (int j0 = 0; j0 < nctx; j0 += 4) {
      float4 kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jj = j0 + u < nctx ? j0 + u : j0;
        const int pos = ctx ? ctx[jj] : jj;
        kv[u] = __ldcg(reinterpret_cast<const float4 *>(p.kc + (size_t)pos * d + h * DH) + lane);
      }
      float acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        acc[u] = fmaf(kv[u].x, q.x, fmaf(kv[u].y, q.y, fmaf(kv[u].z, q.z, kv[u].w * q.w)));
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < nctx) {
          const float sc = acc[u] * scale;
          if (lane == 0) scores[j0 + u] = sc;
          m = fmaxf(m, sc);
        }
    }
    __syncwarp();
    float sl = 0.f;
    for (int jj = lane; jj < nctx; jj += 32) {
      const float e = np_expf(scores[jj] - m);
      scores[jj] = e;
      sl += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
    __syncwarp();
    float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j0 = 0; j0 < nctx; j0 += 4) {
      float4 vv[4];
      float sc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jj = j0 + u;
        const int js = jj < nctx ? jj : j0;
        const int pos = ctx ? ctx[js] : js;
        vv[u] = __ldcg(reinterpret_cast<const float4 *>(p.vc + (size_t)pos * d + h * DH) + lane);
        sc[u] = jj < nctx ? scores[jj] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        o4.x = fmaf(sc[u], vv[u].x, o4.x);
        o4.y = fmaf(sc[u], vv[u].y, o4.y);
        o4.z = fmaf(sc[u], vv[u].z, o4.z);
        o4.w = fmaf(sc[u], vv[u].w, o4.w);
      }
    }
    const float inv = 1.0f / sl;
    o4.x *= inv; o4.y *= inv; o4.z *= inv; o4.w *= inv;
    reinterpret_cast<float4 *>(p.s_att + (size_t)row * d + h * DH)[lane] = o4;
    if (GROWS) {
      // the tcgen05 path: Wo's input row parts (hi / lo bf16, row-set order)
      // straight from here instead of a prep pass over s_att
      __nv_bfloat16 *pa = reinterpret_cast<__nv_bfloat16 *>(p.tc_scratch);
      const size_t plane = (size_t)((p.row_cap + 15) / 16 * 16) * d;
      const size_t base = (size_t)(item / nh) * d + h * DH + 4 * lane;
      const float ov[4] = {o4.x, o4.y, o4.z, o4.w};
      __nv_bfloat16 hv[4], lv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hv[e] = __float2bfloat16_rn(ov[e]);
        lv[e] = __float2bfloat16_rn(ov[e] - __bfloat162float(hv[e]));
      }
      *reinterpret_cast<uint2 *>(pa + base) = *reinterpret_cast<uint2 *>(hv);
      *reinterpret_cast<uint2 *>(pa + plane + base) = *reinterpret_cast<uint2 *>(lv);
    }
    __syncwarp();
  }
}

// attention launch for the fast layer paths (dh == 128: attn_fast128_kernel)
static bool launch_attn_fast(const LayerParams &p, int sms, cudaStream_t s, bool grows);

template <typename K, typename... Args>
static void launch_pdl(K kern, dim3 grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // SPX_PDL_LAYERS=0 (A/B): plain stream order for the multi-row layer kernels
  static const int env_pdl = getenv("SPX_PDL_LAYERS") ? atoi(getenv("SPX_PDL_LAYERS")) : 1;
  cfg.numAttrs = env_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

#include "spx_gemv_tc.cuh"
#include "spx_layer_mega.cuh"

// ------------------------------------------------------------------ host side

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
  return (size_t)p.att_cap * 4 + (size_t)p.row_cap * 4 + 64 * 1024 < (size_t)GEMV_SMEM;
}


template <typename TW, int EPI>
static void launch_gemv(const LayerParams &p, int nout, int kin, int sms, cudaStream_t s) {
  int grid;
  size_t smem;
  const GemvGeom g = gemv_geom<TW>(nout, kin, sms, p.row_cap, grid, smem);
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
  // SPX_LAYER_MEGA=0 selects the per-matrix kernel chain (sweeps / A-B runs)
  static const int env_mega = getenv("SPX_LAYER_MEGA") ? atoi(getenv("SPX_LAYER_MEGA")) : 1;
  if (std::is_same<TW, __nv_bfloat16>::value && env_mega && p.rows_hint <= MG_NRP &&
      mega_layer_supported(p, sms) && launch_layer_mega(p, sms, s))
    return;
  static const int env_tc = getenv("SPX_LAYER_TC") ? atoi(getenv("SPX_LAYER_TC")) : 1;
  if (std::is_same<TW, __nv_bfloat16>::value && env_tc && tc_layer_supported(p)) {
    launch_tc<EPI_QKV>(p, 3 * p.d, p.d, sms, s);
    launch_attn_fast(p, sms, s, false);
    launch_tc<EPI_WO>(p, p.d, p.d, sms, s);
    launch_tc<EPI_FFN1>(p, p.ffn, p.d, sms, s);
    launch_tc<EPI_FFN2>(p, p.d, p.ffn, sms, s);
    return;
  }
  launch_gemv<TW, EPI_QKV>(p, 3 * p.d, p.d, sms, s);
  launch_attn_fast(p, sms, s, false);
  launch_gemv<TW, EPI_WO>(p, p.d, p.d, sms, s);
  launch_gemv<TW, EPI_FFN1>(p, p.ffn, p.d, sms, s);
  launch_gemv<TW, EPI_FFN2>(p, p.d, p.ffn, sms, s);
}

// returns true when the launched kernel also wrote Wo's input parts (grows)
static bool launch_attn_fast(const LayerParams &p, int sms, cudaStream_t s, bool grows) {
  static const int env = getenv("SPX_ATTN128") ? atoi(getenv("SPX_ATTN128")) : 1;
  if (env && p.d / p.nh == 128 && p.d % p.nh == 0) {
    const size_t ab = (size_t)(AT / 32) * ((p.att_cap + 3) / 4 * 4) * 4 +
                      (grows ? 0 : (size_t)p.row_cap * 4);
    static size_t set_t = 0, set_f = 0;
    if (grows) {
      if (ab > set_t && ab > 48 * 1024) {
        cudaFuncSetAttribute(attn_fast128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ab);
        set_t = ab;
      }
      launch_pdl(attn_fast128_kernel<true>, 8 * sms, AT, ab, s, p);
    } else {
      if (ab > set_f && ab > 48 * 1024) {
        cudaFuncSetAttribute(attn_fast128_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ab);
        set_f = ab;
      }
      launch_pdl(attn_fast128_kernel<false>, 2 * sms, AT, ab, s, p);
    }
    return grows;
  }
  const size_t ab = (size_t)(p.att_cap + p.row_cap) * 4 + (size_t)(p.d / p.nh) * 4;
  cudaFuncSetAttribute(attn_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ab);
  launch_pdl(attn_fast_kernel, 2 * sms, AT, ab, s, p);
  return false;
}

}  // namespace spx
