// Flag-guarded decoder-layer kernels with lazy KV completion (sm_100a).
//
// Reference: DecodeState (model.py:155-286): begin (:181-212) appends rows at
// frontier 0; run_layer(l) (:220-233) advances every unfrozen row whose
// frontier is l -- the new row plus rows an earlier early exit left behind --
// through _advance (:235-270): pre-LN MHA (causal or explicit ancestor lists)
// + ReLU FFN with biases, residual stream f32.  Every kernel here first reads
// the device exit flag and returns if the stream already exited this token
// (engine.py:205-207 `break`), so the host never synchronises per layer.
//
// One layer = 6 launches: row-set build, LN1+QKV, attention, Wo+residual,
// LN2+FFN1+ReLU, FFN2+residual (+frontier update).  FAST: bf16 weights, fp32
// accumulation with 16-byte vector loads and packed FFMA2 (HBM-bound GEMVs).
// STRICT: the reference's own operation order (sequential chains, no FMA,
// numpy exp), used for bit-exact parity with the reference trace.
#include <cstdio>
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"

namespace spx {

constexpr int LT = 256;            // threads per CTA
constexpr int RMAX = 4;            // rows per pass

struct LayerParams {
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b, *b1, *b2;
  const void *wqkv, *wo, *w1, *w2;
  int wdt;
  float *pending, *kc, *vc;
  int32_t *frontier;
  const int32_t *n_ctx;
  const int32_t *new_row;
  const uint8_t *frozen;
  const int32_t *attn_ptr, *attn_idx;
  const uint8_t *done;
  float *cur_hidden;
  int32_t *rows, *nrows;
  float *s_q, *s_att, *s_f;
  float *s_part;
  int32_t *s_flag;
  int layer, strict;
  int *err;
  int max_ctx, d, nh, ffn;
  int rows_hint;
  int row_cap, att_cap;            // shared-memory row set / attention keys (<= max_ctx)
  void *tc_scratch;                // tensor-core layer path: input parts (spx_layer_tc.cuh)
};

__device__ __forceinline__ bool exited(const LayerParams &p) { return p.done && *p.done; }

// ---- row set: unfrozen rows with frontier == layer (model.py:230), ascending
__global__ void rows_kernel(LayerParams p) {
  if (exited(p)) return;
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int n = *p.n_ctx;
  // ordered compaction: one pass per 256-block, prefix by ballot
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool take = i < n && p.frontier[i] == p.layer && !(p.frozen && p.frozen[i]);
    const unsigned m = __ballot_sync(0xffffffffu, take);
    __shared__ int wcnt[LT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    int off = cnt;
    for (int j = 0; j < w; ++j) off += wcnt[j];
    if (take) p.rows[off + __popc(m & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) for (int j = 0; j < LT / 32; ++j) cnt += wcnt[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) *p.nrows = cnt;
}

// ---- LayerNorm of up to RMAX rows into shared memory (model.py:140-146)
// FAST: CTA-wide tree sums; STRICT: sequential (thread 0) -- bit-exact.
__device__ void ln_rows(const float *src, const int32_t *rows, int nr, int d, const float *g,
                        const float *b, float *dst, bool strict) {
  __shared__ float s_stat[RMAX][2];
  __shared__ float red[LT / 32];
  for (int r = 0; r < nr; ++r) {
    const float *x = src + (size_t)rows[r] * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) dst[(size_t)r * d + j] = x[j];
  }
  __syncthreads();
  const float df = (float)d;
  for (int r = 0; r < nr; ++r) {
    float *xr = dst + (size_t)r * d;
    if (strict) {
      if (threadIdx.x == 0) {
        float m = 0.f;
        for (int j = 0; j < d; ++j) m = __fadd_rn(m, xr[j]);
        m = __fdiv_rn(m, df);
        float v = 0.f;
        for (int j = 0; j < d; ++j) { const float c = __fsub_rn(xr[j], m); v = __fadd_rn(v, __fmul_rn(c, c)); }
        s_stat[r][0] = m;
        s_stat[r][1] = __fsqrt_rn(__fadd_rn(__fdiv_rn(v, df), 1e-5f));
      }
    } else {
      float s = 0.f;
      for (int j = threadIdx.x; j < d; j += blockDim.x) s += xr[j];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        float t = 0.f;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += red[j];
        s_stat[r][0] = t / df;
      }
      __syncthreads();
      const float m = s_stat[r][0];
      float v = 0.f;
      for (int j = threadIdx.x; j < d; j += blockDim.x) { const float c = xr[j] - m; v = fmaf(c, c, v); }
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        float t = 0.f;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += red[j];
        s_stat[r][1] = sqrtf(t / df + 1e-5f);
      }
    }
    __syncthreads();
  }
  for (int r = 0; r < nr; ++r) {
    const float m = s_stat[r][0], den = s_stat[r][1];
    float *xr = dst + (size_t)r * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x)
      xr[j] = ln_elem(__fsub_rn(xr[j], m), den, g[j], b[j]);
  }
  __syncthreads();
}

// 8 weights (16 bytes bf16 / 32 bytes f32) as floats
template <typename TW> struct W8;
template <> struct W8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float *f) {
    const uint4 u = ldg_nc_v4(p);
    bf16x4_to_f32(u.x, u.y, f);
    bf16x4_to_f32(u.z, u.w, f + 4);
  }
};
template <> struct W8<float> {
  static __device__ __forceinline__ void load(const float *p, float *f) {
    const uint4 a = ldg_nc_v4(p), b = ldg_nc_v4(p + 4);
    f[0] = __uint_as_float(a.x); f[1] = __uint_as_float(a.y); f[2] = __uint_as_float(a.z);
    f[3] = __uint_as_float(a.w); f[4] = __uint_as_float(b.x); f[5] = __uint_as_float(b.y);
    f[6] = __uint_as_float(b.z); f[7] = __uint_as_float(b.w);
  }
};

// out[r][o] = sum_j in[r][j] * W[o][j] for o in [0, nout), r < nr; W (nout, kin)
// out-major.  FAST: one warp per output row, 16-byte loads, lane-strided
// partials + butterfly.  STRICT: one thread per (row, output), sequential
// ascending chain without FMA (kernels/_ckern.pyx:16-31).  `fn(r, o, acc)`
// consumes each result.
template <typename TW, typename F>
__device__ void gemv_rows(const TW *W, int nout, int kin, const float *in, int nr, bool strict,
                          F &&fn) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int tw = gridDim.x * (blockDim.x >> 5);
  if (strict) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, tt = gridDim.x * blockDim.x;
    for (int idx = gt; idx < nout * nr; idx += tt) {
      const int o = idx % nout, r = idx / nout;
      const TW *wr = W + (size_t)o * kin;
      const float *x = in + (size_t)r * kin;
      float acc = 0.f;
      for (int j = 0; j < kin; j += 4) {
        float w4[4];
        load4_f32<TW>(wr + j, w4);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc = __fadd_rn(acc, __fmul_rn(x[j + e], w4[e]));
      }
      fn(r, o, acc);
    }
    return;
  }
  for (int o = gw; o < nout; o += tw) {
    const TW *wr = W + (size_t)o * kin;
    float acc[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) acc[r] = 0.f;
    int j = lane * 8;
    for (; j + 8 <= kin; j += 256) {
      float wf[8];
      W8<TW>::load(wr + j, wf);
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        if (r < nr) {
          const float4 a = *reinterpret_cast<const float4 *>(in + (size_t)r * kin + j);
          const float4 b = *reinterpret_cast<const float4 *>(in + (size_t)r * kin + j + 4);
          float2 s2 = make_float2(acc[r], 0.f);
          s2 = ffma2(make_float2(a.x, a.y), make_float2(wf[0], wf[1]), s2);
          s2 = ffma2(make_float2(a.z, a.w), make_float2(wf[2], wf[3]), s2);
          s2 = ffma2(make_float2(b.x, b.y), make_float2(wf[4], wf[5]), s2);
          s2 = ffma2(make_float2(b.z, b.w), make_float2(wf[6], wf[7]), s2);
          acc[r] = s2.x + s2.y;
        }
      }
    }
    for (int jj = j; jj < kin && jj < j + 8; jj += 4) {    // kin % 8 == 4 tail
      float w4[4];
      load4_f32<TW>(wr + jj, w4);
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < nr)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[r] = fmaf(in[(size_t)r * kin + jj + e], w4[e], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      float v = acc[r];
      for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
      if (lane == 0 && r < nr) fn(r, o, v);
    }
  }
}

// ---- LN1 + QKV: q -> s_q, k/v -> cache[row] (model.py:240-245)
template <typename TW>
__global__ void __launch_bounds__(LT) qkv_kernel(LayerParams p) {
  if (exited(p)) return;
  extern __shared__ float hs[];
  const int nrows = *p.nrows, d = p.d;
  for (int c0 = 0; c0 < nrows; c0 += RMAX) {
    const int nr = nrows - c0 < RMAX ? nrows - c0 : RMAX;
    const int32_t *rows = p.rows + c0;
    ln_rows(p.pending, rows, nr, d, p.ln1_g, p.ln1_b, hs, p.strict);
    gemv_rows<TW>(reinterpret_cast<const TW *>(p.wqkv), 3 * d, d, hs, nr, p.strict,
                  [&](int r, int o, float v) {
                    const int row = rows[r];
                    if (o < d) p.s_q[(size_t)row * d + o] = v;
                    else if (o < 2 * d) p.kc[(size_t)row * d + (o - d)] = v;
                    else p.vc[(size_t)row * d + (o - 2 * d)] = v;
                  });
    __syncthreads();
  }
}

// ---- attention: one warp per (row, head) (model.py:247-262)
__global__ void __launch_bounds__(LT) attn_kernel(LayerParams p) {
  if (exited(p)) return;
  const int nrows = *p.nrows, d = p.d, nh = p.nh, dh = d / nh;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int tw = gridDim.x * (blockDim.x >> 5);
  extern __shared__ float sc[];                     // scores: (warps, max_ctx)
  float *scores = sc + (size_t)(threadIdx.x >> 5) * p.att_cap;
  const float scale = __fdiv_rn(1.0f, __fsqrt_rn((float)dh)) ;
  // reference: np.float32(1.0 / math.sqrt(dh)) -- f64 then rounded
  const float scale_ref = (float)(1.0 / sqrt((double)dh));
  (void)scale;
  for (int item = gw; item < nrows * nh; item += tw) {
    const int row = p.rows[item / nh], h = item % nh;
    const float *q = p.s_q + (size_t)row * d + h * dh;
    // context: explicit ancestor list (tree rows) or causal 0..row
    const int *ctx = nullptr;
    int nctx = row + 1;
    if (p.attn_ptr && p.attn_ptr[row + 1] > p.attn_ptr[row]) {
      ctx = p.attn_idx + p.attn_ptr[row];
      nctx = p.attn_ptr[row + 1] - p.attn_ptr[row];
    }
    // scores[j] = (k_j . q) * scale
    for (int jj = lane; jj < nctx; jj += 32) {
      const int pos = ctx ? ctx[jj] : jj;
      const float *k = p.kc + (size_t)pos * d + h * dh;
      float acc = 0.f;
      if (p.strict) {
        for (int e = 0; e < dh; ++e) acc = __fadd_rn(acc, __fmul_rn(k[e], q[e]));
      } else {
        for (int e = 0; e < dh; e += 4) {
          const float4 kv = *reinterpret_cast<const float4 *>(k + e);
          const float4 qv = *reinterpret_cast<const float4 *>(q + e);
          acc = fmaf(kv.x, qv.x, fmaf(kv.y, qv.y, fmaf(kv.z, qv.z, fmaf(kv.w, qv.w, acc))));
        }
      }
      scores[jj] = __fmul_rn(acc, scale_ref);
    }
    __syncwarp();
    // softmax_1d (model.py:149-152): max, np exp, strict sum, divide
    float m = -INFINITY;
    for (int jj = lane; jj < nctx; jj += 32) m = fmaxf(m, scores[jj]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int jj = lane; jj < nctx; jj += 32) scores[jj] = np_expf(__fsub_rn(scores[jj], m));
    __syncwarp();
    float ssum = 0.f;
    if (p.strict) {
      if (lane == 0) for (int jj = 0; jj < nctx; ++jj) ssum = __fadd_rn(ssum, scores[jj]);
      ssum = __shfl_sync(0xffffffffu, ssum, 0);
    } else {
      for (int jj = lane; jj < nctx; jj += 32) ssum += scores[jj];
      for (int o = 16; o; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    }
    for (int jj = lane; jj < nctx; jj += 32) scores[jj] = __fdiv_rn(scores[jj], ssum);
    __syncwarp();
    // out[e] = sum_j probs[j] * v_j[e]  (strict: ascending j, no FMA)
    for (int e = lane; e < dh; e += 32) {
      float acc = 0.f;
      for (int jj = 0; jj < nctx; ++jj) {
        const int pos = ctx ? ctx[jj] : jj;
        const float vv = p.vc[(size_t)pos * d + h * dh + e];
        acc = p.strict ? __fadd_rn(acc, __fmul_rn(scores[jj], vv)) : fmaf(scores[jj], vv, acc);
      }
      p.s_att[(size_t)row * d + h * dh + e] = acc;
    }
    __syncwarp();
  }
}

// ---- Wo + residual: pending[row] += attn @ Wo (model.py:262-263)
template <typename TW>
__global__ void __launch_bounds__(LT) wo_kernel(LayerParams p) {
  if (exited(p)) return;
  extern __shared__ float hs[];
  const int nrows = *p.nrows, d = p.d;
  for (int c0 = 0; c0 < nrows; c0 += RMAX) {
    const int nr = nrows - c0 < RMAX ? nrows - c0 : RMAX;
    const int32_t *rows = p.rows + c0;
    for (int r = 0; r < nr; ++r)
      for (int j = threadIdx.x; j < d; j += blockDim.x) hs[(size_t)r * d + j] = p.s_att[(size_t)rows[r] * d + j];
    __syncthreads();
    gemv_rows<TW>(reinterpret_cast<const TW *>(p.wo), d, d, hs, nr, p.strict,
                  [&](int r, int o, float v) {
                    float *x = p.pending + (size_t)rows[r] * d + o;
                    *x = __fadd_rn(*x, v);
                  });
    __syncthreads();
  }
}

// ---- LN2 + FFN1 + bias + ReLU -> s_f (model.py:265-266)
template <typename TW>
__global__ void __launch_bounds__(LT) ffn1_kernel(LayerParams p) {
  if (exited(p)) return;
  extern __shared__ float hs[];
  const int nrows = *p.nrows, d = p.d, f = p.ffn;
  for (int c0 = 0; c0 < nrows; c0 += RMAX) {
    const int nr = nrows - c0 < RMAX ? nrows - c0 : RMAX;
    const int32_t *rows = p.rows + c0;
    ln_rows(p.pending, rows, nr, d, p.ln2_g, p.ln2_b, hs, p.strict);
    gemv_rows<TW>(reinterpret_cast<const TW *>(p.w1), f, d, hs, nr, p.strict,
                  [&](int r, int o, float v) {
                    const float z = __fadd_rn(v, p.b1[o]);
                    p.s_f[(size_t)rows[r] * f + o] = z > 0.f ? z : 0.f;
                  });
    __syncthreads();
  }
}

// ---- FFN2 + bias + residual (model.py:267): x = (x + f@W2) + b2
template <typename TW>
__global__ void __launch_bounds__(LT) ffn2_kernel(LayerParams p) {
  if (exited(p)) return;
  extern __shared__ float hs[];
  const int nrows = *p.nrows, d = p.d, f = p.ffn;
  for (int c0 = 0; c0 < nrows; c0 += RMAX) {
    const int nr = nrows - c0 < RMAX ? nrows - c0 : RMAX;
    const int32_t *rows = p.rows + c0;
    for (int r = 0; r < nr; ++r)
      for (int j = threadIdx.x; j < f; j += blockDim.x) hs[(size_t)r * f + j] = p.s_f[(size_t)rows[r] * f + j];
    __syncthreads();
    gemv_rows<TW>(reinterpret_cast<const TW *>(p.w2), d, f, hs, nr, p.strict,
                  [&](int r, int o, float v) {
                    float *x = p.pending + (size_t)rows[r] * d + o;
                    *x = __fadd_rn(__fadd_rn(*x, v), p.b2[o]);
                  });
    __syncthreads();
  }
}

// ---- frontier update + newest-row copy (model.py:269-270, run_layer return)
__global__ void finish_kernel(LayerParams p) {
  if (exited(p)) return;
  const int nrows = *p.nrows, d = p.d;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) p.frontier[p.rows[i]] = p.layer + 1;
  if (p.cur_hidden && p.new_row) {
    const int nr = *p.new_row;
    if (nr >= 0)
      for (int j = threadIdx.x; j < d; j += blockDim.x) p.cur_hidden[j] = p.pending[(size_t)nr * d + j];
  }
}

}  // namespace spx

#include "spx_layers_fast.cuh"
#include "spx_layer_tc.cuh"

using namespace spx;

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename TW>
static void launch_layer(const LayerParams &p, cudaStream_t s) {
  const int sms = sm_count();
  if constexpr (std::is_same<TW, __nv_bfloat16>::value) {
    if (!p.strict && tcl_supported(p) && fast_layer_supported(p, sizeof(TW))) {
      launch_layer_tcgen05(p, sms, s);               // >= 16 rows: tcgen05 GEMMs
      return;
    }
  }
  if (!p.strict && fast_layer_supported(p, sizeof(TW))) {
    launch_layer_fast<TW>(p, sms, s);
    return;
  }
  const size_t ln_smem = (size_t)RMAX * p.d * sizeof(float);
  const size_t f_smem = (size_t)RMAX * (p.ffn > p.d ? p.ffn : p.d) * sizeof(float);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(qkv_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(wo_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(ffn1_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(ffn2_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    configured = true;
  }
  const int wpc = LT / 32;
  auto grid_for = [&](int nout) {
    int g = (nout + wpc - 1) / wpc;
    return g < sms ? g : sms;
  };
  spx_debug_capture(s, "strict layer: entry");
  rows_kernel<<<1, LT, 0, s>>>(p);
  spx_debug_capture(s, "strict layer: rows");
  qkv_kernel<TW><<<grid_for(3 * p.d), LT, ln_smem, s>>>(p);
  spx_debug_capture(s, "strict layer: qkv");
  const size_t a_smem = (size_t)wpc * p.att_cap * sizeof(float);
  attn_kernel<<<sms, LT, a_smem, s>>>(p);
  spx_debug_capture(s, "strict layer: attn");
  wo_kernel<TW><<<grid_for(p.d), LT, ln_smem, s>>>(p);
  ffn1_kernel<TW><<<grid_for(p.ffn), LT, ln_smem, s>>>(p);
  ffn2_kernel<TW><<<grid_for(p.d), LT, f_smem, s>>>(p);
  finish_kernel<<<1, LT, 0, s>>>(p);
  spx_debug_capture(s, "strict layer: exit");
}

extern "C" int spx_layer_forward(const spx_layer_args *a, void *stream) {
  if (!a || !a->pending || !a->kcache || !a->vcache || !a->frontier || !a->n_ctx || !a->rows ||
      !a->nrows || !a->s_q || !a->s_att || !a->s_f || !a->err)
    return SPX_EINVAL;
  if (a->d <= 0 || a->d % 8 || a->n_heads <= 0 || a->d % a->n_heads || (a->d / a->n_heads) % 4 ||
      a->ffn <= 0 || a->ffn % 4 || a->max_ctx <= 0)
    return SPX_EINVAL;
  if ((size_t)RMAX * (a->ffn > a->d ? a->ffn : a->d) * 4 > 225 * 1024 ||
      (size_t)(LT / 32) * (a->att_cap > 0 && a->att_cap < a->max_ctx ? a->att_cap : a->max_ctx) * 4 >
          225 * 1024)
    return SPX_EINVAL;
  LayerParams p;
  p.ln1_g = a->ln1_g; p.ln1_b = a->ln1_b; p.ln2_g = a->ln2_g; p.ln2_b = a->ln2_b;
  p.b1 = a->b1; p.b2 = a->b2;
  p.wqkv = a->wqkv; p.wo = a->wo; p.w1 = a->w1; p.w2 = a->w2; p.wdt = a->w_dtype;
  p.pending = a->pending; p.kc = a->kcache; p.vc = a->vcache; p.frontier = a->frontier;
  p.n_ctx = a->n_ctx; p.new_row = a->new_row; p.frozen = a->frozen;
  p.attn_ptr = a->attn_ptr; p.attn_idx = a->attn_idx; p.done = a->done;
  p.cur_hidden = a->cur_hidden; p.rows = a->rows; p.nrows = a->nrows;
  p.s_q = a->s_q; p.s_att = a->s_att; p.s_f = a->s_f;
  p.s_part = a->s_part; p.s_flag = a->s_flag;
  p.layer = a->layer; p.strict = a->mode == SPX_MODE_STRICT; p.err = a->err;
  p.max_ctx = (int)a->max_ctx; p.d = (int)a->d; p.nh = (int)a->n_heads; p.ffn = (int)a->ffn;
  p.rows_hint = a->rows_hint;
  p.row_cap = a->row_cap > 0 && a->row_cap < p.max_ctx ? a->row_cap : p.max_ctx;
  p.att_cap = a->att_cap > 0 && a->att_cap < p.max_ctx ? a->att_cap : p.max_ctx;
  p.tc_scratch = a->tc_scratch;
  cudaStream_t s = (cudaStream_t)stream;
  if (a->w_dtype == SPX_DTYPE_BF16) launch_layer<__nv_bfloat16>(p, s);
  else if (a->w_dtype == SPX_DTYPE_F32) launch_layer<float>(p, s);
  else return SPX_EINVAL;
  return spx_launch_status("spx_layer_forward");
}

static int64_t tc_units(int64_t nout, int64_t kin) {
  return ((nout + 7) / 8) * ((kin + TUC - 1) / TUC);
}
extern "C" int64_t spx_layer_part_floats(int64_t d, int64_t ffn) {
  int64_t m = tc_units(3 * d, d);
  m = tc_units(ffn, d) > m ? tc_units(ffn, d) : m;
  m = tc_units(d, ffn) > m ? tc_units(d, ffn) : m;
  return m * 64;
}
extern "C" int64_t spx_layer_tc_scratch_bytes(int64_t d, int64_t ffn, int64_t row_cap) {
  if (d <= 0 || ffn <= 0 || row_cap <= 0) return -1;
  return (int64_t)tcl_scratch_bytes((int)d, (int)ffn, (int)row_cap);
}

extern "C" int64_t spx_layer_flag_ints(int64_t d, int64_t ffn) {
  const int64_t n = 3 * d > ffn ? 3 * d : ffn;
  return (n + 7) / 8;
}

// ---- begin(): append T rows (model.py:181-212): pending = emb[tok] + pe[pos]
template <typename TW>
__global__ void embed_kernel(const TW *emb, const float *pe, const int32_t *tokens,
                             const int32_t *pos_ids, int T, int d, int V, int max_ctx,
                             float *pending, int32_t *frontier, int32_t *n_ctx, int32_t *new_row,
                             const uint8_t *frozen_reset, int *err) {
  // grid (rows, d / (4 * blockDim)): every thread owns 4 consecutive
  // elements of one row (d % 4 == 0), so a single decode row is spread over
  // d / 512 CTAs instead of one CTA's strided loop
  const int n0 = *n_ctx;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int row = n0 + t;
    int tok = tokens[t];
    if (tok < 0 || tok >= V || row >= max_ctx) {
      if (threadIdx.x == 0 && blockIdx.y == 0) atomicOr(err, ERR_ID_RANGE);
      continue;
    }
    const int pos = pos_ids ? pos_ids[t] : row;
    const TW *e = emb + (size_t)tok * d;
    for (int j = 4 * (blockIdx.y * blockDim.x + threadIdx.x); j < d; j += 4 * blockDim.x * gridDim.y) {
      float w[4];
      load4_f32<TW>(e + j, w);
      const float4 pv = *reinterpret_cast<const float4 *>(pe + (size_t)pos * d + j);
      float4 o;
      o.x = __fadd_rn(w[0], pv.x); o.y = __fadd_rn(w[1], pv.y);
      o.z = __fadd_rn(w[2], pv.z); o.w = __fadd_rn(w[3], pv.w);
      *reinterpret_cast<float4 *>(pending + (size_t)row * d + j) = o;
    }
    if (threadIdx.x == 0 && blockIdx.y == 0) frontier[row] = 0;
  }
  (void)frozen_reset;
}

__global__ void embed_commit_kernel(int T, int32_t *n_ctx, int32_t *new_row, int max_ctx) {
  const int n0 = *n_ctx;
  *new_row = n0 + T - 1 < max_ctx ? n0 + T - 1 : -1;
  *n_ctx = n0 + T < max_ctx ? n0 + T : max_ctx;
}

extern "C" int spx_embed(const void *embedding, int32_t w_dtype, const float *pos_encoding,
                         const int32_t *tokens, const int32_t *pos_ids, int64_t T, int64_t d,
                         int64_t V, int64_t max_ctx, float *pending, int32_t *frontier,
                         int32_t *n_ctx, int32_t *new_row, int32_t *err, void *stream) {
  if (!embedding || !pos_encoding || !tokens || !pending || !frontier || !n_ctx || !new_row ||
      !err || T <= 0 || d <= 0 || d % 4)
    return SPX_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  spx_debug_capture(s, "embed: entry");
  const dim3 grid((unsigned)(T < 1024 ? T : 1024), (unsigned)((d + 511) / 512 < 16 ? (d + 511) / 512 : 16));
  if (w_dtype == SPX_DTYPE_BF16)
    embed_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>((const __nv_bfloat16 *)embedding, pos_encoding,
                                                      tokens, pos_ids, (int)T, (int)d, (int)V,
                                                      (int)max_ctx, pending, frontier, n_ctx,
                                                      new_row, nullptr, err);
  else if (w_dtype == SPX_DTYPE_F32)
    embed_kernel<float><<<grid, 128, 0, s>>>((const float *)embedding, pos_encoding, tokens,
                                              pos_ids, (int)T, (int)d, (int)V, (int)max_ctx,
                                              pending, frontier, n_ctx, new_row, nullptr, err);
  else
    return SPX_EINVAL;
  embed_commit_kernel<<<1, 1, 0, s>>>((int)T, n_ctx, new_row, (int)max_ctx);
  return spx_launch_status("spx_embed");
}
