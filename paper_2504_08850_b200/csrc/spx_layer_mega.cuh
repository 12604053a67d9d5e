// Persistent whole-layer decode kernel (FAST mode, bf16 weights) -- included
// by spx_layers_fast.cuh.  One launch runs a decoder layer (model.py:235-270)
// for the layer's row set: LN1 + QKV -> attention -> Wo + residual -> LN2 +
// FFN1 + ReLU -> FFN2 + residual, with grid-wide barriers between phases.
//
// Why one launch: a decode step is HBM-bound on the weights (314.6 MB per
// layer at 7B) and the weights do not depend on the activations.  A producer
// warp per CTA streams the CTA's share of ALL four weight matrices of the
// layer in phase order through one shared-memory ring (cp.async.bulk of whole
// contiguous weight-row blocks, mbarrier complete_tx), so the weight stream
// never stops at a phase boundary: while the consumer warps wait at a grid
// barrier for the previous phase's activations, the next phase's weights are
// already landing.  The separate-kernel chain drained the pipe at every
// kernel boundary (launch, prologue, ramp) five times per layer.
//
//   CTA c (one per SM, grid = #SMs, all co-resident) owns the contiguous
//   output rows [c*n/G, (c+1)*n/G) of every matrix.
//   16 consumer warps: thread t holds chunks t, t+512, ... (8 elements) of
//   the phase's input rows in registers (LayerNorm applied for QKV / FFN1);
//   per stage each thread forms its partial dots for every (weight row,
//   input row) pair with packed FFMA2, a warp reduce-scatter + a fixed-order
//   sum over the 16 warps gives each output (deterministic).
//   Attention: one warp per (row, head) item over the grid, online softmax
//   with numpy's f32 exp.
//   Rows: up to NRP input rows per pass; more rows (long lazy-completion
//   chains) take several passes over the weights.
//
// The early-exit flag `done` is read before griddepcontrol.wait (an exit
// decided by an earlier kernel) and after it (decided by the kernel just
// before): an exited stream streams nothing or drains its prefetch and
// returns.  launch_dependents fires after grid barrier 1, i.e. once every CTA
// of this grid is resident and running, so a dependent kernel can never take
// an SM this grid still needs.
// Co-residency of the whole grid (one CTA per SM, spun on by the grid
// barriers) is guaranteed by the launch: the occupancy API must report one
// CTA per SM for every SM, and the kernel is launched with the cooperative
// attribute, so the driver rejects a grid that cannot be co-resident (MPS SM
// limits, green contexts) instead of letting it spin; the caller then takes
// the per-matrix kernel chain.
#pragma once

constexpr int MG_CW = 16;                       // consumer warps
constexpr int MG_T = 32 * (MG_CW + 1);          // + producer warp
constexpr int MG_CT = 32 * MG_CW;               // consumer threads
constexpr int MG_NRP = 2;                       // input rows per pass
constexpr int MG_CPT = 4;                       // max 8-element chunks per thread (kin <= 16384: Llama2-13B ffn 13824)
constexpr int MG_STAGE = 48 * 1024;             // max bytes per ring slot
constexpr int MG_RMAX = 8;                      // max weight rows per stage
constexpr int MG_SLOTS = 4;

struct MegaGeom {
  int nout[4], kin[4], R[4];                    // per matrix: QKV, Wo, FFN1, FFN2
  int red_stride;                               // floats per warp row of `red`
  int dbg;                                      // tuning: 1 = no math, 2 = one copy per row
  size_t smem;
};

__device__ unsigned long long g_mega_trace[4][16];   // debug: phase stamps of CTAs 0, G/2

__device__ __forceinline__ void mg_stamp(int k) {
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2))
    g_mega_trace[blockIdx.x == 0 ? 0 : 1][k] = gtimer();
}

__device__ __forceinline__ void mg_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mg_cbar() {
  asm volatile("bar.sync 1, %0;" ::"r"(MG_CT) : "memory");
}

// grid-wide barrier number b (0-based) on a monotonic counter, among the
// consumer warps only (the producer keeps streaming weights meanwhile)
__device__ __forceinline__ void mg_grid_barrier(int32_t *ctr, int b) {
  mg_cbar();
  if (threadIdx.x == 0) {
    const int target = (b + 1) * (int)gridDim.x;
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  mg_cbar();
}

template <int EPI>
__device__ __forceinline__ const __nv_bfloat16 *mg_weights(const LayerParams &p) {
  return reinterpret_cast<const __nv_bfloat16 *>(gemv_weights<EPI>(p));
}

// reduce-scatter of 16 values over a warp: lane L ends with the warp sum of
// value L >> 1 (pairs of lanes hold the same value)
__device__ __forceinline__ float mg_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int m = 16 >> s, half = 8 >> s;
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <int EPI, int CPT>
__device__ __forceinline__ void mg_load_x(const LayerParams &p, const int *rows, int r0, int nr,
                                          int kin, float (&x)[MG_NRP][CPT * 8], float *scr) {
  const int nch = kin >> 3, tid = threadIdx.x;
  const bool ln = EPI == EPI_QKV || EPI == EPI_FFN1;
  const float *src = ln ? p.pending : EPI == EPI_WO ? p.s_att : p.s_f;
#pragma unroll
  for (int r = 0; r < MG_NRP; ++r)
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci) {
      const int c = tid + ci * MG_CT;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (r < nr && c < nch) {
        const float *q = src + (size_t)rows[r0 + r] * kin + c * 8;
        a = __ldcg(reinterpret_cast<const float4 *>(q));
        b = __ldcg(reinterpret_cast<const float4 *>(q + 4));
      }
      x[r][ci * 8 + 0] = a.x; x[r][ci * 8 + 1] = a.y; x[r][ci * 8 + 2] = a.z; x[r][ci * 8 + 3] = a.w;
      x[r][ci * 8 + 4] = b.x; x[r][ci * 8 + 5] = b.y; x[r][ci * 8 + 6] = b.z; x[r][ci * 8 + 7] = b.w;
    }
  if (!ln) return;
  const float *gg = EPI == EPI_QKV ? p.ln1_g : p.ln2_g;
  const float *bb = EPI == EPI_QKV ? p.ln1_b : p.ln2_b;
  const int lane = tid & 31, w = tid >> 5;
  const float df = (float)kin;
  float s[MG_NRP];
#pragma unroll
  for (int r = 0; r < MG_NRP; ++r) {
    s[r] = 0.f;
#pragma unroll
    for (int e = 0; e < CPT * 8; ++e) s[r] += x[r][e];
#pragma unroll
    for (int m = 16; m; m >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], m);
    if (lane == 0) scr[r * MG_CW + w] = s[r];
  }
  mg_cbar();
  float mean[MG_NRP], v[MG_NRP];
#pragma unroll
  for (int r = 0; r < MG_NRP; ++r) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < MG_CW; ++j) t += scr[r * MG_CW + j];
    mean[r] = t / df;
    v[r] = 0.f;
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci)
      if (tid + ci * MG_CT < nch)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float c = x[r][ci * 8 + e] - mean[r];
          v[r] = fmaf(c, c, v[r]);
        }
  }
  mg_cbar();
#pragma unroll
  for (int r = 0; r < MG_NRP; ++r) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], m);
    if (lane == 0) scr[r * MG_CW + w] = v[r];
  }
  mg_cbar();
#pragma unroll
  for (int r = 0; r < MG_NRP; ++r) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < MG_CW; ++j) t += scr[r * MG_CW + j];
    const float den = sqrtf(t / df + 1e-5f);
#pragma unroll
    for (int ci = 0; ci < CPT; ++ci) {
      const int c = tid + ci * MG_CT;
      if (c < nch) {
        const float4 g0 = __ldg(reinterpret_cast<const float4 *>(gg + c * 8));
        const float4 g1 = __ldg(reinterpret_cast<const float4 *>(gg + c * 8 + 4));
        const float4 b0 = __ldg(reinterpret_cast<const float4 *>(bb + c * 8));
        const float4 b1 = __ldg(reinterpret_cast<const float4 *>(bb + c * 8 + 4));
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          x[r][ci * 8 + e] = (r < nr) ? ln_elem(x[r][ci * 8 + e] - mean[r], den, gv[e], bv[e]) : 0.f;
      }
    }
  }
  mg_cbar();                                      // scr reused by the next pass
}

// One matrix phase for the consumers: passes over the row set, stages of R
// weight rows.  No CTA-wide barrier per stage: each warp reduces its partial
// dots (reduce-scatter) into its own row of `red` and releases the slot on its
// own (the slot's empty barrier counts the 16 consumer warps); the fixed-order
// sum over warps and the epilogue run once per pass.
template <int EPI, int CPT>
__device__ __forceinline__ void mg_phase(const LayerParams &p, const MegaGeom &g, const int *rows,
                                         int nrows, unsigned char *ring, uint64_t *full,
                                         uint64_t *empty, float *red, float *scr, int &job) {
  constexpr int M = EPI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, kin = g.kin[M], R = g.R[M], nch = kin >> 3;
  const int o_begin = (int)((long long)blockIdx.x * g.nout[M] / G);
  const int o_end = (int)((long long)(blockIdx.x + 1) * g.nout[M] / G);
  const int nloc = o_end - o_begin;
  const int nst = (nloc + R - 1) / R;
  float *myred = red + (size_t)warp * g.red_stride;
  for (int r0 = 0; r0 < nrows; r0 += MG_NRP) {
    const int nr = nrows - r0 < MG_NRP ? nrows - r0 : MG_NRP;
    float x[MG_NRP][CPT * 8];
    mg_load_x<EPI, CPT>(p, rows, r0, nr, kin, x, scr);
    // the epilogue's operands (residual row entries, biases) of this thread's
    // first output are fetched now, so their latency hides behind the stages
    float pre_a = 0.f, pre_b = 0.f;
    const int idx0 = tid;
    const bool has0 = idx0 < nloc * MG_NRP && (idx0 % MG_NRP) < nr;
    if (has0) {
      const int o = o_begin + idx0 / MG_NRP, row = rows[r0 + idx0 % MG_NRP];
      if (EPI == EPI_WO || EPI == EPI_FFN2) pre_a = __ldcg(p.pending + (size_t)row * p.d + o);
      if (EPI == EPI_FFN1) pre_b = __ldg(p.b1 + o);
      if (EPI == EPI_FFN2) pre_b = __ldg(p.b2 + o);
    }
    for (int st = 0; st < nst; ++st, ++job) {
      const int slot = job % MG_SLOTS;
      mbar_wait(&full[slot], (job / MG_SLOTS) & 1);
      const int n = (nloc - st * R) < R ? (nloc - st * R) : R;
      const __nv_bfloat16 *ws =
          reinterpret_cast<const __nv_bfloat16 *>(ring + (size_t)slot * MG_STAGE);
      float acc[16];
#pragma unroll
      for (int i = 0; i < MG_RMAX; ++i) {
        float2 s2[MG_NRP];
#pragma unroll
        for (int r = 0; r < MG_NRP; ++r) s2[r] = make_float2(0.f, 0.f);
        if (i < n && !(g.dbg & 1)) {
#pragma unroll
          for (int ci = 0; ci < CPT; ++ci) {
            const int c = tid + ci * MG_CT;
            if (c < nch) {
              float w[8];
              const uint4 u = *reinterpret_cast<const uint4 *>(ws + (size_t)i * kin + c * 8);
              bf16x4_to_f32(u.x, u.y, w);
              bf16x4_to_f32(u.z, u.w, w + 4);
#pragma unroll
              for (int r = 0; r < MG_NRP; ++r) {
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
        for (int r = 0; r < MG_NRP; ++r) acc[i * MG_NRP + r] = s2[r].x + s2[r].y;
      }
      __syncwarp();
      if (lane == 0) mg_arrive(&empty[slot]);     // this warp is done with the slot
      const float part = mg_reduce16(acc, lane);  // value index lane >> 1 = i * NRP + r
      const int vi = lane >> 1;
      if ((lane & 1) == 0 && vi < n * MG_NRP) myred[st * R * MG_NRP + vi] = part;
    }
    mg_cbar();                                    // all warps' partials of the pass
    for (int idx = tid; idx < nloc * MG_NRP; idx += MG_CT) {
      const int i = idx / MG_NRP, r = idx % MG_NRP;
      if (r < nr) {
        float v = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < MG_CW; ++w2) v += red[(size_t)w2 * g.red_stride + idx];
        const int row = rows[r0 + r], o = o_begin + i;
        if (idx != idx0 || EPI == EPI_QKV) {
          gemv_epilogue<EPI>(p, row, o, v);
        } else if (EPI == EPI_WO) {
          p.pending[(size_t)row * p.d + o] = __fadd_rn(pre_a, v);
        } else if (EPI == EPI_FFN1) {
          const float z = __fadd_rn(v, pre_b);
          p.s_f[(size_t)row * p.ffn + o] = z > 0.f ? z : 0.f;
        } else {
          p.pending[(size_t)row * p.d + o] = __fadd_rn(__fadd_rn(pre_a, v), pre_b);
        }
      }
    }
    mg_cbar();                                    // red reused by the next pass
  }
}

// Attention of the row set (model.py:247-262), one warp per (row, head) over
// the grid.  The weight stream keeps HBM saturated during this phase, so every
// dependent global load costs ~1 us: keys are processed in batches of 16 whose
// K and V loads (lane = 4 dims of the head) are all issued before any is used,
// i.e. one memory round trip per 16 keys; online softmax across batches with
// numpy's f32 exp.
constexpr int MG_ATT_KEYS = 512;                // max context per item
constexpr int MG_ATT_W = 8;                     // attention warps per CTA
constexpr int MG_AB = 8;                        // keys per batch
// Items (row, head) are few at decode (32 at 7B) and the HBM is saturated by
// the weight stream, so latency dominates: each item takes one CTA and its 8
// attention warps split the keys (contiguous ranges); every warp runs the
// batched online softmax over its range, then the 8 partial (max, sum, acc)
// triples are merged in shared memory in warp order.
template <int NP>
__device__ void mg_attention_split(const LayerParams &p, const int *rows, int nrows, float *sc_all) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = p.d, nh = p.nh, dh = d / nh;
  const float scale = (float)(1.0 / sqrt((double)dh));
  float *part = sc_all;                        // [MG_ATT_W][4 + 128 * NP]: m, l, pad, acc
  const int pstride = 4 + 128 * NP;
  for (int item = blockIdx.x; item < nrows * nh; item += gridDim.x) {
    const int row = rows[item / nh], h = item % nh;
    const int *ctx = nullptr;
    int nctx = row + 1;
    if (p.attn_ptr && p.attn_ptr[row + 1] > p.attn_ptr[row]) {
      ctx = p.attn_idx + p.attn_ptr[row];
      nctx = p.attn_ptr[row + 1] - p.attn_ptr[row];
    }
    const size_t hoff = (size_t)h * dh;
    if (warp < MG_ATT_W) {
      const int per = (nctx + MG_ATT_W - 1) / MG_ATT_W;
      const int ja = warp * per, jb = ja + per < nctx ? ja + per : nctx;
      float4 qv[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int e = lane * 4 + 128 * k;
        qv[k] = e < dh ? __ldcg(reinterpret_cast<const float4 *>(p.s_q + (size_t)row * d + hoff + e))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float m = -INFINITY, l = 0.f;
      float4 acc[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j0 = ja; j0 < jb; j0 += MG_AB) {
        float4 kb[MG_AB][NP], vb[MG_AB][NP];
#pragma unroll
        for (int t = 0; t < MG_AB; ++t) {
          const int jj = j0 + t;
          const int pos = jj < jb ? (ctx ? ctx[jj] : jj) : 0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const int e = lane * 4 + 128 * k;
            const bool ok = jj < jb && e < dh;
            kb[t][k] = ok ? __ldcg(reinterpret_cast<const float4 *>(p.kc + (size_t)pos * d + hoff + e))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            vb[t][k] = ok ? __ldcg(reinterpret_cast<const float4 *>(p.vc + (size_t)pos * d + hoff + e))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        float sc[MG_AB];
#pragma unroll
        for (int t = 0; t < MG_AB; ++t) {
          float a = 0.f;
#pragma unroll
          for (int k = 0; k < NP; ++k)
            a = fmaf(kb[t][k].x, qv[k].x, fmaf(kb[t][k].y, qv[k].y,
                fmaf(kb[t][k].z, qv[k].z, fmaf(kb[t][k].w, qv[k].w, a))));
          sc[t] = a;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
          for (int t = 0; t < MG_AB; ++t) sc[t] += __shfl_xor_sync(0xffffffffu, sc[t], o);
        float bm = m;
#pragma unroll
        for (int t = 0; t < MG_AB; ++t) {
          sc[t] = (j0 + t < jb) ? sc[t] * scale : -INFINITY;
          bm = fmaxf(bm, sc[t]);
        }
        const float corr = np_expf(m - bm);
        l *= corr;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          acc[k].x *= corr; acc[k].y *= corr; acc[k].z *= corr; acc[k].w *= corr;
        }
#pragma unroll
        for (int t = 0; t < MG_AB; ++t) {
          const float pe = np_expf(sc[t] - bm);
          l += pe;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            acc[k].x = fmaf(pe, vb[t][k].x, acc[k].x); acc[k].y = fmaf(pe, vb[t][k].y, acc[k].y);
            acc[k].z = fmaf(pe, vb[t][k].z, acc[k].z); acc[k].w = fmaf(pe, vb[t][k].w, acc[k].w);
          }
        }
        m = bm;
      }
      float *pw = part + (size_t)warp * pstride;
      if (lane == 0) { pw[0] = m; pw[1] = l; }
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int e = lane * 4 + 128 * k;
        if (e < dh) *reinterpret_cast<float4 *>(pw + 4 + e) = acc[k];
      }
    }
    mg_cbar();
    // merge the warps' partials in warp order (threads own dims)
    for (int e = threadIdx.x; e < dh; e += MG_CT) {
      float M = -INFINITY;
      for (int w = 0; w < MG_ATT_W; ++w) M = fmaxf(M, part[(size_t)w * pstride]);
      float L = 0.f, A = 0.f;
      for (int w = 0; w < MG_ATT_W; ++w) {
        const float mw = part[(size_t)w * pstride];
        const float f = mw == -INFINITY ? 0.f : np_expf(mw - M);
        L = fmaf(part[(size_t)w * pstride + 1], f, L);
        A = fmaf(part[(size_t)w * pstride + 4 + e], f, A);
      }
      p.s_att[(size_t)row * d + hoff + e] = A / L;
    }
    mg_cbar();
  }
}

__device__ __forceinline__ void mg_attention(const LayerParams &p, const int *rows, int nrows,
                                             float *sc) {
  if (p.d / p.nh <= 128) mg_attention_split<1>(p, rows, nrows, sc);
  else mg_attention_split<2>(p, rows, nrows, sc);
}

template <int CD, int CF>                       // chunks per thread for d / ffn inputs
__global__ void __launch_bounds__(MG_T, 1) layer_mega_kernel(LayerParams p, MegaGeom g) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char *ring = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)MG_SLOTS * MG_STAGE);
  uint64_t *empty = full + MG_SLOTS;
  float *red = reinterpret_cast<float *>(empty + MG_SLOTS);          // [16][red_stride]
  float *scr = red + (size_t)MG_CW * g.red_stride;                    // [NRP][16]
  int *rows = reinterpret_cast<int *>(scr + MG_NRP * MG_CW);          // [max_ctx]
  float *att_sc = red;        // attention scores [8][512] alias the idle partial buffer
  __shared__ int s_last, s_skip, s_skip2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  int32_t *bar_ctr = p.s_flag, *end_ctr = p.s_flag + 1;

  mg_stamp(0);
  if (tid == 0) {
    for (int s = 0; s < MG_SLOTS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MG_CW); }
    fence_mbar_init();
    s_skip = flag_set(p.done) ? 1 : 0;            // exit decided by an earlier kernel
  }
  __syncthreads();
  if (s_skip) return;

  // producer: weight stages of the four matrices, in phase order, across passes
  auto stages_of = [&](int M) {
    const int o0 = (int)((long long)blockIdx.x * g.nout[M] / G);
    const int o1 = (int)((long long)(blockIdx.x + 1) * g.nout[M] / G);
    return (o1 - o0 + g.R[M] - 1) / g.R[M];
  };
  auto issue = [&](int job, int M, int st) {
    const int o0 = (int)((long long)blockIdx.x * g.nout[M] / G);
    const int o1 = (int)((long long)(blockIdx.x + 1) * g.nout[M] / G);
    const int o = o0 + st * g.R[M];
    const int n = (o1 - o) < g.R[M] ? (o1 - o) : g.R[M];
    const size_t rb = (size_t)g.kin[M] * 2;
    const unsigned char *W = reinterpret_cast<const unsigned char *>(
        M == 0 ? p.wqkv : M == 1 ? p.wo : M == 2 ? p.w1 : p.w2);
    const int slot = job % MG_SLOTS;
    if (job >= MG_SLOTS) mbar_wait(&empty[slot], ((job / MG_SLOTS) - 1) & 1);
    mbar_arrive_expect_tx(&full[slot], (uint32_t)(n * rb));
    if (g.dbg & 2) {
      for (int i = 0; i < n; ++i)
        bulk_g2s(ring + (size_t)slot * MG_STAGE + i * rb, W + (size_t)(o + i) * rb, (uint32_t)rb,
                 &full[slot]);
    } else {
      bulk_g2s(ring + (size_t)slot * MG_STAGE, W + (size_t)o * rb, (uint32_t)(n * rb), &full[slot]);
    }
  };
  int pre = 0;                                    // stages issued before the wait
  if (warp == MG_CW && lane == 0) {
    const int n0 = stages_of(0);
    for (; pre < MG_SLOTS && pre < n0; ++pre) issue(pre, 0, pre);
  }
  pdl_wait();
  if (tid == 0) s_skip2 = flag_set(p.done) ? 1 : 0;
  __syncthreads();
  if (s_skip2) {                                  // exit decided just before: drain
    if (warp == MG_CW && lane == 0)
      for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0);
    __syncthreads();
    return;
  }
  mg_stamp(1);
  const int nrows = cta_row_set(p, rows);        // every CTA: the same ascending set
  const int npass = (nrows + MG_NRP - 1) / MG_NRP;
  mg_stamp(2);

  if (warp == MG_CW) {
    if (lane == 0) {
      int job = 0;
      for (int M = 0; M < 4; ++M) {
        const int ns = stages_of(M);
        for (int ps = 0; ps < npass; ++ps)
          for (int st = 0; st < ns; ++st, ++job)
            if (job >= pre) issue(job, M, st);
      }
      // drain prefetched stages nobody consumes (no rows at this layer)
      if (npass == 0)
        for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0);
    }
  } else {
    int job = 0;
    mg_phase<EPI_QKV, CD>(p, g, rows, nrows, ring, full, empty, red, scr, job);
    mg_stamp(3);
    mg_grid_barrier(bar_ctr, 0);
    mg_stamp(4);
    mg_attention(p, rows, nrows, att_sc);
    mg_stamp(5);
    mg_grid_barrier(bar_ctr, 1);
    mg_stamp(6);
    pdl_trigger();
    mg_phase<EPI_WO, CD>(p, g, rows, nrows, ring, full, empty, red, scr, job);
    mg_stamp(7);
    mg_grid_barrier(bar_ctr, 2);
    mg_stamp(8);
    mg_phase<EPI_FFN1, CD>(p, g, rows, nrows, ring, full, empty, red, scr, job);
    mg_stamp(9);
    mg_grid_barrier(bar_ctr, 3);
    mg_stamp(10);
    mg_phase<EPI_FFN2, CF>(p, g, rows, nrows, ring, full, empty, red, scr, job);
    mg_stamp(11);
  }
  // the last CTA advances the frontier, copies the newest row and resets the
  // barrier counters (model.py:269-270, run_layer's return value)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(end_ctr, 1) == G - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int i = tid; i < nrows; i += MG_T) p.frontier[rows[i]] = p.layer + 1;
    if (p.cur_hidden && p.new_row) {
      const int nw = *reinterpret_cast<const volatile int32_t *>(p.new_row);
      if (nw >= 0)
        for (int j = tid; j < p.d; j += MG_T) p.cur_hidden[j] = __ldcg(p.pending + (size_t)nw * p.d + j);
    }
    __syncthreads();
    if (tid == 0) { *bar_ctr = 0; *end_ctr = 0; }
  }
  mg_stamp(12);
}

static size_t mega_smem(const LayerParams &p, int sms) {
  const int no[4] = {3 * p.d, p.d, p.ffn, p.d}, ki[4] = {p.d, p.d, p.d, p.ffn};
  int mx = 0;
  for (int m = 0; m < 4; ++m) {
    int R = (int)(MG_STAGE / ((size_t)ki[m] * 2));
    R = R < 1 ? 1 : R > MG_RMAX ? MG_RMAX : R;
    const int per = (no[m] + sms - 1) / sms;
    const int padded = ((per + R - 1) / R) * R;
    mx = padded > mx ? padded : mx;
  }
  const size_t redf = (size_t)mx * MG_NRP * MG_CW > (size_t)MG_ATT_KEYS * MG_ATT_W
                          ? (size_t)mx * MG_NRP * MG_CW : (size_t)MG_ATT_KEYS * MG_ATT_W;
  return (size_t)MG_SLOTS * MG_STAGE + 2 * MG_SLOTS * 8 + redf * 4 +
         MG_NRP * MG_CW * 4 + (size_t)p.row_cap * 4 + 64;
}

static bool mega_layer_supported(const LayerParams &p, int sms) {
  if (p.d % 8 || p.ffn % 8) return false;
  if (p.d > MG_CT * 8 * 2 || p.ffn > MG_CT * 8 * MG_CPT || p.ffn < p.d) return false;
  if ((size_t)p.ffn * 2 > MG_STAGE || (size_t)p.d * 2 > MG_STAGE) return false;   // >= 1 row/stage
  if ((p.d / p.nh) > 256 || (p.d / p.nh) % 4 || p.att_cap > MG_ATT_KEYS) return false;
  if (!p.s_flag) return false;
  return sms > 0 && mega_smem(p, sms) <= 220 * 1024;
}

static bool launch_layer_mega(const LayerParams &p, int sms, cudaStream_t s) {
  MegaGeom g;
  const int no[4] = {3 * p.d, p.d, p.ffn, p.d}, ki[4] = {p.d, p.d, p.d, p.ffn};
  for (int m = 0; m < 4; ++m) {
    g.nout[m] = no[m];
    g.kin[m] = ki[m];
    int R = (int)(MG_STAGE / ((size_t)ki[m] * 2));
    g.R[m] = R < 1 ? 1 : R > MG_RMAX ? MG_RMAX : R;
  }
  int mx = 0;
  for (int m = 0; m < 4; ++m) {
    const int per = (no[m] + sms - 1) / sms;
    const int padded = ((per + g.R[m] - 1) / g.R[m]) * g.R[m];
    mx = padded > mx ? padded : mx;
  }
  g.red_stride = mx * MG_NRP > MG_ATT_KEYS * MG_ATT_W / MG_CW ? mx * MG_NRP
                                                              : MG_ATT_KEYS * MG_ATT_W / MG_CW;
  static const int env_dbg = getenv("SPX_MEGA_DBG") ? atoi(getenv("SPX_MEGA_DBG")) : 0;
  g.dbg = env_dbg;
  g.smem = mega_smem(p, sms);
  const int cd = (p.d / 8 + MG_CT - 1) / MG_CT, cf = (p.ffn / 8 + MG_CT - 1) / MG_CT;
  static const int env_coop = getenv("SPX_MEGA_COOP") ? atoi(getenv("SPX_MEGA_COOP")) : 1;
  auto go = [&](auto kern) -> bool {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)g.smem);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MG_T, g.smem);
    if (e != cudaSuccess || per_sm < 1) { cudaGetLastError(); return false; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(MG_T);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = env_coop ? 2 : 1;
    e = cudaLaunchKernelEx(&cfg, kern, p, g);
    if (e != cudaSuccess) {
      fprintf(stderr, "spx mega: launch: %s\n", cudaGetErrorString(e));
      cudaGetLastError();
      return false;
    }
    return true;
  };
  if (cd == 1 && cf == 1) return go(layer_mega_kernel<1, 1>);
  if (cd == 1 && cf == 2) return go(layer_mega_kernel<1, 2>);
  if (cd == 1 && cf == 3) return go(layer_mega_kernel<1, 3>);
  if (cd == 2 && cf == 2) return go(layer_mega_kernel<2, 2>);
  if (cd == 2 && cf == 3) return go(layer_mega_kernel<2, 3>);
  return go(layer_mega_kernel<2, 4>);                // Llama2-13B: d = 5120, ffn = 13824
}

extern "C" void spx_debug_mega_trace(void *host_out) {
  cudaMemcpyFromSymbol(host_out, g_mega_trace, sizeof(unsigned long long) * 64);
}
