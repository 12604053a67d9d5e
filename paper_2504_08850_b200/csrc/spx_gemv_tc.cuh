// Tensor-core decode GEMV for bf16 decoder weights (included by
// spx_layers_fast.cuh).
//
//   out[r][n] = sum_k x[r][k] * W[n][k]      W: (nout, kin) bf16, x: nr <= 8 rows f32
//
// Formed with mma.sync m16n8k16 (bf16 x bf16 -> f32): the 16 A rows are the
// input rows split into a bf16 head (rows 0-7) and a bf16 tail (rows 8-15),
// x = hi + lo + O(2^-17 |x|), so D[g] + D[g+8] is the fp32-accurate dot with
// the exact bf16 weights.  The 8 B columns are 8 weight rows.
//
// Weights go HBM -> registers with 16-byte non-allocating loads: lane (g, c)
// loads columns 8c..8c+7 of weight row g of a 32-column slab; the MMA's k
// order is permuted per lane (virtual k 2c+j <-> column 8c+j, 2c+8+j <->
// 8c+2+j, and the next k-step takes 8c+4..7), which is legal because A and B
// use the same permutation -- so one 16-byte load feeds two k-steps with no
// shuffles and no shared-memory staging of weights.  x (hi/lo) is resident in
// shared memory, read with one 16-byte load per k-step pair.
//
// Work: "units" of 8 weight rows x 512 columns (8 KB), numbered block-major,
// split evenly over all warps of the grid (split-K at warp granularity, so
// every SM streams the same byte count).  Each warp double-buffers its loads
// in half-units (8 x 16 B per lane in flight).  A block whose units span
// several warps is combined through global scratch: every segment writes its
// partial, the last arrival (atomic counter) adds the segments in segment
// order and runs the epilogue -- deterministic.  With more than `maxr` rows
// (prefill, or many lazily completed rows) the kernel switches to whole
// blocks per warp and passes over the rows (no cross-warp combine).
#pragma once
// (included inside namespace spx)

constexpr int TT = 512, TWARPS = TT / 32;
constexpr int TUC = 512;                 // columns per unit
constexpr int TLD = TUC / 32;            // 16-byte loads per lane per unit
constexpr int THALF = TLD / 2;
constexpr int TC_SMEM = 210 * 1024;

struct TcGeom {
  int nout, kin, nblk, P, units, maxr, xpitch;
  int r_begin, last;       // row slice of this launch (multi-row calls: one launch per slice)
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
__device__ __forceinline__ void split_hilo(float x, __nv_bfloat16 &hi, __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}
__device__ __forceinline__ uint4 ldg_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int EPI>
__device__ __forceinline__ void tc_epilogue(const LayerParams &p, int row, int o, float v) {
  if (EPI == EPI_FFN1) {
    // ReLU output kept as hi/lo bf16 in the row's s_f slot: FFN2's A operand
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

// warp (global index) owning unit u under the even split
__device__ __forceinline__ int tc_warp_of(long long u, int Wt, int units) {
  return (int)(((u + 1) * Wt - 1) / units);
}

struct TcUnit {
  const __nv_bfloat16 *wp;   // this lane's first 16-byte load
  int col0;                  // this lane's first column
  int nld;                   // 16-byte loads in the unit (<= TLD)
};

__device__ __forceinline__ TcUnit tc_unit(const TcGeom &g, const __nv_bfloat16 *W, int u, int g8,
                                          int cq) {
  const int b = u / g.P, q = u - (u / g.P) * g.P;
  const int n = b * 8 + g8;
  const int k0 = q * TUC;
  const int len = g.kin - k0 < TUC ? g.kin - k0 : TUC;
  TcUnit t;
  t.nld = n < g.nout ? (len >> 5) : 0;
  t.col0 = k0 + 8 * cq;
  t.wp = W + (size_t)(n < g.nout ? n : 0) * g.kin + t.col0;
  return t;
}

__device__ __forceinline__ void tc_load_half(const TcUnit &t, int h, uint4 (&w)[THALF]) {
#pragma unroll
  for (int i = 0; i < THALF; ++i) {
    const int li = h * THALF + i;
    w[i] = li < t.nld ? ldg_stream(t.wp + 32 * li) : make_uint4(0u, 0u, 0u, 0u);
  }
}

__device__ __forceinline__ void tc_mma_half(const TcUnit &t, int h, const uint4 (&w)[THALF],
                                            const unsigned char *xhi, const unsigned char *xlo,
                                            bool arow, float (&D)[4]) {
#pragma unroll
  for (int i = 0; i < THALF; ++i) {
    const int li = h * THALF + i;
    if (li < t.nld) {
      uint4 hi = make_uint4(0u, 0u, 0u, 0u), lo = hi;
      if (arow) {
        const int off = (t.col0 + 32 * li) * 2;
        hi = *reinterpret_cast<const uint4 *>(xhi + off);
        lo = *reinterpret_cast<const uint4 *>(xlo + off);
      }
      mma_bf16_16816(D, hi.x, lo.x, hi.y, lo.y, w[i].x, w[i].y);
      mma_bf16_16816(D, hi.z, lo.z, hi.w, lo.w, w[i].z, w[i].w);
    }
  }
}

// Resident A operand: hi/lo bf16 rows of the pass's input rows.
template <int EPI>
__device__ void tc_load_x(const LayerParams &p, const TcGeom &g, const int *rows, int r0, int nr,
                          unsigned char *xa, float *scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kin = g.kin;
  if (EPI == EPI_FFN2) {
    // FFN1 already wrote hi/lo bf16: copy 16-byte pieces
    const int n16 = kin / 8;
    for (int r = 0; r < nr; ++r) {
      const uint4 *src = reinterpret_cast<const uint4 *>(
          reinterpret_cast<const __nv_bfloat16 *>(p.s_f) + (size_t)rows[r0 + r] * 2 * kin);
      uint4 *dh = reinterpret_cast<uint4 *>(xa + (size_t)r * g.xpitch);
      uint4 *dl = reinterpret_cast<uint4 *>(xa + (size_t)(g.maxr + r) * g.xpitch);
      for (int j = tid; j < n16; j += TT) {
        dh[j] = __ldcg(src + j);
        dl[j] = __ldcg(src + n16 + j);
      }
    }
    __syncthreads();
    return;
  }
  const bool ln = EPI == EPI_QKV || EPI == EPI_FFN1;
  const float *src = ln ? p.pending : p.s_att;
  const float *gg = EPI == EPI_QKV ? p.ln1_g : p.ln2_g;
  const float *bb = EPI == EPI_QKV ? p.ln1_b : p.ln2_b;
  for (int r = 0; r < nr; ++r) {
    const float *x = src + (size_t)rows[r0 + r] * kin;
    float mean = 0.f, den = 1.f;
    if (ln) {
      float s = 0.f;
      for (int j = tid; j < kin; j += TT) s += __ldcg(x + j);
#pragma unroll
      for (int m = 16; m; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
      if (lane == 0) scr[warp] = s;
      __syncthreads();
      s = 0.f;
#pragma unroll
      for (int w = 0; w < TWARPS; ++w) s += scr[w];
      mean = s / (float)kin;
      __syncthreads();
      float v = 0.f;
      for (int j = tid; j < kin; j += TT) {
        const float c = __ldcg(x + j) - mean;
        v = fmaf(c, c, v);
      }
#pragma unroll
      for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
      if (lane == 0) scr[warp] = v;
      __syncthreads();
      v = 0.f;
#pragma unroll
      for (int w = 0; w < TWARPS; ++w) v += scr[w];
      den = sqrtf(v / (float)kin + 1e-5f);
      __syncthreads();
    }
    __nv_bfloat16 *dh = reinterpret_cast<__nv_bfloat16 *>(xa + (size_t)r * g.xpitch);
    __nv_bfloat16 *dl = reinterpret_cast<__nv_bfloat16 *>(xa + (size_t)(g.maxr + r) * g.xpitch);
    for (int j = tid; j < kin; j += TT) {
      float v = __ldcg(x + j);
      if (ln) v = ln_elem(v - mean, den, gg[j], bb[j]);
      __nv_bfloat16 hi, lo;
      split_hilo(v, hi, lo);
      dh[j] = hi;
      dl[j] = lo;
    }
  }
  __syncthreads();
}

template <int EPI>
__global__ void __launch_bounds__(TT, 1) gemv_tc_kernel(LayerParams p, TcGeom g) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *xa = smem;
  float *scr = reinterpret_cast<float *>(smem + (size_t)2 * g.maxr * g.xpitch);
  int *rows_all = reinterpret_cast<int *>(scr + TWARPS);
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, cq = lane & 3;
  const int G = gridDim.x, gw = blockIdx.x * TWARPS + warp;
  // active warps: never more than units, so every active warp owns >= 1 unit
  const int Wt = G * TWARPS < g.units ? G * TWARPS : g.units;
  const __nv_bfloat16 *W = reinterpret_cast<const __nv_bfloat16 *>(gemv_weights<EPI>(p));

  // even split of the units over all warps (assumed before the row count is known)
  const int u0 = gw < Wt ? (int)((long long)gw * g.units / Wt) : 0;
  const int u1 = gw < Wt ? (int)((long long)(gw + 1) * g.units / Wt) : 0;
  uint4 wa[THALF], wb[THALF];
  bool pre = false;
  if (EPI != EPI_QKV && u0 < u1 && !flag_set(p.done)) {
    // weights are constant: start streaming before the previous kernel ends
    const TcUnit t = tc_unit(g, W, u0, g8, cq);
    tc_load_half(t, 0, wa);
    tc_load_half(t, 1, wb);
    pre = true;
  }
  pdl_wait();
  if (flag_set(p.done)) return;
  pdl_trigger();
  const int nall = cta_row_set(p, rows_all);
  // this launch's slice of the row set: maxr rows, or everything left (last)
  const int rb = g.r_begin < nall ? g.r_begin : nall;
  const int nrows = g.last ? nall - rb : (nall - rb < g.maxr ? nall - rb : g.maxr);
  const int *rows = rows_all + rb;

  if (nrows <= g.maxr) {
    const int nr = nrows;
    if (nr > 0) tc_load_x<EPI>(p, g, rows, 0, nr, xa, scr);
    const bool arow = g8 < nr;
    const unsigned char *xhi = xa + (size_t)g8 * g.xpitch;
    const unsigned char *xlo = xa + (size_t)(g.maxr + g8) * g.xpitch;
    float D[4] = {0.f, 0.f, 0.f, 0.f};
    if (nr > 0 && u0 < u1) {
      TcUnit t = tc_unit(g, W, u0, g8, cq);
      if (!pre) {
        tc_load_half(t, 0, wa);
        tc_load_half(t, 1, wb);
      }
      for (int u = u0; u < u1; ++u) {
        const bool more = u + 1 < u1;
        const TcUnit tn = more ? tc_unit(g, W, u + 1, g8, cq) : t;
        tc_mma_half(t, 0, wa, xhi, xlo, arow, D);
        if (more) tc_load_half(tn, 0, wa);
        tc_mma_half(t, 1, wb, xhi, xlo, arow, D);
        if (more) tc_load_half(tn, 1, wb);
        const int b = u / g.P, q = u - b * g.P;
        if (q == g.P - 1 || !more) {
          // block b done in this warp: D[0..1] hi + D[2..3] lo -> rows g8, cols 2cq+e
          const float v0 = D[0] + D[2], v1 = D[1] + D[3];
          D[0] = D[1] = D[2] = D[3] = 0.f;
          const long long bu0 = (long long)b * g.P;
          const int first = tc_warp_of(bu0, Wt, g.units);
          const int last = tc_warp_of(bu0 + g.P - 1, Wt, g.units);
          const int nseg = last - first + 1;
          const int n0 = b * 8 + 2 * cq;
          if (nseg == 1) {
            if (arow) {
              if (n0 < g.nout) tc_epilogue<EPI>(p, rows[g8], n0, v0);
              if (n0 + 1 < g.nout) tc_epilogue<EPI>(p, rows[g8], n0 + 1, v1);
            }
          } else {
            float *part = p.s_part + (size_t)bu0 * 64;
            part[(gw - first) * 64 + lane * 2] = v0;
            part[(gw - first) * 64 + lane * 2 + 1] = v1;
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(p.s_flag + b, 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == nseg - 1) {
              __threadfence();
              float s0 = 0.f, s1 = 0.f;
              for (int s = 0; s < nseg; ++s) {
                s0 += __ldcg(part + s * 64 + lane * 2);
                s1 += __ldcg(part + s * 64 + lane * 2 + 1);
              }
              if (arow) {
                if (n0 < g.nout) tc_epilogue<EPI>(p, rows[g8], n0, s0);
                if (n0 + 1 < g.nout) tc_epilogue<EPI>(p, rows[g8], n0 + 1, s1);
              }
              if (lane == 0) p.s_flag[b] = 0;
            }
          }
        }
        t = tn;
      }
    }
  } else {
    // many rows: whole blocks per warp, passes of maxr rows (no split-K)
    for (int r0 = 0; r0 < nrows; r0 += g.maxr) {
      const int nr = nrows - r0 < g.maxr ? nrows - r0 : g.maxr;
      tc_load_x<EPI>(p, g, rows, r0, nr, xa, scr);
      const bool arow = g8 < nr;
      const unsigned char *xhi = xa + (size_t)g8 * g.xpitch;
      const unsigned char *xlo = xa + (size_t)(g.maxr + g8) * g.xpitch;
      for (int b = gw; b < g.nblk; b += Wt) {
        float D[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < g.P; ++q) {
          const TcUnit t = tc_unit(g, W, b * g.P + q, g8, cq);
          tc_load_half(t, 0, wa);
          tc_load_half(t, 1, wb);
          tc_mma_half(t, 0, wa, xhi, xlo, arow, D);
          tc_mma_half(t, 1, wb, xhi, xlo, arow, D);
        }
        const int n0 = b * 8 + 2 * cq;
        if (arow) {
          if (n0 < g.nout) tc_epilogue<EPI>(p, rows[r0 + g8], n0, D[0] + D[2]);
          if (n0 + 1 < g.nout) tc_epilogue<EPI>(p, rows[r0 + g8], n0 + 1, D[1] + D[3]);
        }
      }
      __syncthreads();
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
      if (g.last)
        for (int i = tid; i < nall; i += TT) p.frontier[rows_all[i]] = p.layer + 1;
      if (g.last && p.cur_hidden && p.new_row) {
        const int nw = *reinterpret_cast<const volatile int32_t *>(p.new_row);
        if (nw >= 0)
          for (int j = tid; j < p.d; j += TT) p.cur_hidden[j] = __ldcg(p.pending + (size_t)nw * p.d + j);
      }
      if (tid == 0) *p.nrows = 0;
    }
  }
}

static TcGeom tc_geom(int nout, int kin, int max_ctx, size_t &smem) {
  TcGeom g;
  g.nout = nout;
  g.kin = kin;
  g.nblk = (nout + 7) / 8;
  g.P = (kin + TUC - 1) / TUC;
  g.units = g.nblk * g.P;
  // row pitch = 64 (mod 128) bytes: the 8 lanes of a 16-byte LDS phase
  // (2 rows x 4 column groups) hit distinct bank groups
  int pitch = kin * 2;
  pitch += (64 - (pitch % 128) + 128) % 128;
  g.xpitch = pitch;
  const size_t fixed = TWARPS * 4 + (size_t)max_ctx * 4 + 256;
  int mr = (int)((TC_SMEM - fixed) / (2 * (size_t)pitch));
  g.maxr = mr > 8 ? 8 : mr;
  g.r_begin = 0;
  g.last = 1;
  smem = 2 * (size_t)g.maxr * pitch + fixed;
  return g;
}

static bool tc_layer_supported(const LayerParams &p) {
  if (p.d % 32 || p.ffn % 32 || !p.s_part || !p.s_flag) return false;
  size_t smem;
  return tc_geom(p.d, p.ffn, p.row_cap, smem).maxr >= 1 &&
         tc_geom(p.ffn, p.d, p.row_cap, smem).maxr >= 1;
}

// Multi-row calls (rows_hint > maxr: prefill, token trees) run one launch per
// slice of maxr rows so every slice takes the split-K path; the frontier and
// newest-row copy happen in the last slice only, so all slices see the same
// row set.
template <int EPI>
static void launch_tc(const LayerParams &p, int nout, int kin, int sms, cudaStream_t s) {
  size_t smem;
  TcGeom g = tc_geom(nout, kin, p.row_cap, smem);
  cudaFuncSetAttribute(gemv_tc_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  int grid = g.units / TWARPS;
  grid = grid < 1 ? 1 : grid > sms ? sms : grid;
  const int slices = p.rows_hint > g.maxr ? (p.rows_hint + g.maxr - 1) / g.maxr : 1;
  for (int sl = 0; sl < slices; ++sl) {
    g.r_begin = sl * g.maxr;
    g.last = sl == slices - 1;
    launch_pdl(gemv_tc_kernel<EPI>, grid, TT, smem, s, p, g);
  }
}
