// Multi-row decoder layers on the 5th-generation tensor cores (sm_100a):
// batched streams (BatchedExitEngine), token trees, prefill -- every call
// that advances >= 16 rows.  Included by spx_layers.cu after
// spx_layers_fast.cuh.
//
// The 8-row mma.sync path (spx_gemv_tc.cuh) re-streams each weight matrix
// once per 8-row slice; here every matrix is ONE weight-streaming GEMM per
// call:
//
//   D[o][n] (TMEM f32, 128 lanes = 128 output features x <= 128 rows)
//     += W[o0 .. o0+127][k-block] . X_part[n0 .. n0+127][k-block]^T
//
// for the two bf16 parts of the f32 input rows (hi + lo: 16 mantissa bits,
// relative representation error <= 2^-17, as the 8-row mma.sync path), with
// exact bf16 x bf16 products and f32 accumulation -- FAST-mode tolerance.
// Per call:
//
//   tcl_rows      the row set (frontier == layer, not frozen), once
//   per matrix:   tcl_prep  input rows -> LayerNorm (QKV, FFN1) -> 2 bf16 parts
//                 tcl_gemm  grid (128-feature tiles, 128-row tiles); 16-byte
//                           cp.async into 128B-swizzled K-major stages, one
//                           thread issues tcgen05.mma kind::f16, tcgen05.commit
//                           releases stages; epilogue tcgen05.ld -> the layer's
//                           epilogue (Q/K/V scatter, residual adds, bias + ReLU)
//   attention     attn_fast_kernel (unchanged)
//   tcl_finish    frontier + newest-row copy
//
// The weights are read once per 128-row tile (once for <= 128 rows).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <unordered_map>
#include "spx_umma.cuh"

namespace spx {

constexpr int TL_M = 128;             // output features per tile (UMMA M)
constexpr int TL_NT = 128;            // rows per tile (UMMA N)
constexpr int TL_BK = 64;             // K elements per stage (one 128-byte swizzle atom)
constexpr int TL_STAGES = 4;
constexpr int TL_AHEAD = 2;           // K-blocks loaded ahead; a slot is refilled TL_AHEAD
                                      // iterations after its MMAs were issued
constexpr int TL_THREADS = 128;
constexpr int TL_PARTS = 2;           // hi + lo bf16: 16 mantissa bits of the f32 rows
constexpr size_t TL_TILE_A = (size_t)TL_M * TL_BK * 2;
constexpr size_t TL_TILE_B = (size_t)TL_NT * TL_BK * 2;
constexpr size_t TL_STAGE = TL_TILE_A + TL_PARTS * TL_TILE_B;          // 48 KB

inline int tl_npad(const LayerParams &p) { return (p.row_cap + 15) / 16 * 16; }
__device__ __forceinline__ int tl_npad_dev(const LayerParams &p) { return (p.row_cap + 15) / 16 * 16; }

// bytes of one row-part region (two bf16 planes of Npad x max(d, ffn)); the
// scratch holds two regions (A: the QKV / Wo / FFN1 inputs, B: the FFN2
// input, written by FFN1's epilogue while FFN1 still reads A) + the K-split
// partials
__host__ __device__ inline size_t tcl_parts_bytes(int d, int ffn, int row_cap) {
  const size_t npad = (size_t)(row_cap + 15) / 16 * 16;
  return ((size_t)TL_PARTS * npad * (size_t)(ffn > d ? ffn : d) * 2 + 255) / 256 * 256;
}

constexpr size_t TL_PARTIAL_BYTES = 96ull << 20;      // K-split partial sums
constexpr int TL_FIX_SLOTS = 65536;                   // K-split tile counters (int32)

// the two bf16 parts of x (hi = RNE(x), lo = RNE(x - hi): tcl_prep_kernel's split)
__device__ __forceinline__ void tl_put_parts(__nv_bfloat16 *parts, size_t plane, size_t idx,
                                             float x) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  parts[idx] = h;
  parts[plane + idx] = __float2bfloat16_rn(x - __bfloat162float(h));
}

// the layer epilogue of output o of row-set entry n; FFN1 also emits FFN2's
// input parts (relu(v + b1), no LayerNorm) into region B -- no FFN2 prep pass
template <int EPI>
__device__ __forceinline__ void tcl_epilogue(const LayerParams &p, int n, int o, float v) {
  gemv_epilogue<EPI>(p, p.rows[n], o, v);
  if (EPI == EPI_FFN1) {
    const float z = __fadd_rn(v, p.b1[o]);
    __nv_bfloat16 *pb = reinterpret_cast<__nv_bfloat16 *>(
        reinterpret_cast<uint8_t *>(p.tc_scratch) + tcl_parts_bytes(p.d, p.ffn, p.row_cap));
    tl_put_parts(pb, (size_t)tl_npad_dev(p) * p.ffn, (size_t)n * p.ffn + o, z > 0.f ? z : 0.f);
  }
}

// the row set once per call, into p.rows / *p.nrows (global)
__global__ void __launch_bounds__(512) tcl_rows_kernel(LayerParams p) {
  pdl_wait();
  pdl_trigger();
  if (flag_set(p.done)) return;
  extern __shared__ int trows[];
  const int n = cta_row_set(p, trows);
  for (int i = threadIdx.x; i < n; i += blockDim.x) p.rows[i] = trows[i];
  if (threadIdx.x == 0) *p.nrows = n;
}

// input rows (row-set order) -> [LayerNorm] -> two bf16 parts (2, Npad, kin);
// one CTA per row, 4 elements per thread per step
template <int EPI>
__global__ void __launch_bounds__(256) tcl_prep_kernel(LayerParams p, int kin, int Npad,
                                                     __nv_bfloat16 *parts) {
  pdl_wait();
  pdl_trigger();
  if (flag_set(p.done)) return;
  const int n = *reinterpret_cast<const volatile int32_t *>(p.nrows);
  const bool ln = EPI == EPI_QKV || EPI == EPI_FFN1;
  const float *src = ln ? p.pending : EPI == EPI_WO ? p.s_att : p.s_f;
  const float *gg = EPI == EPI_QKV ? p.ln1_g : p.ln2_g;
  const float *bb = EPI == EPI_QKV ? p.ln1_b : p.ln2_b;
  __shared__ float s_red[8];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const size_t plane = (size_t)Npad * kin;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const float4 *x4 = reinterpret_cast<const float4 *>(src + (size_t)p.rows[i] * kin);
    const int k4 = kin / 4;
    float mean = 0.f, den = 1.f;
    if (ln) {
      float sm = 0.f;
#pragma unroll 4
      for (int j = tid; j < k4; j += 256) {
        const float4 v = __ldcg(x4 + j);
        sm += (v.x + v.y) + (v.z + v.w);
      }
      sm = warp_butterfly_sum(sm);
      if (lane == 0) s_red[w] = sm;
      __syncthreads();
      sm = 0.f;
      for (int q = 0; q < 8; ++q) sm += s_red[q];
      mean = sm / (float)kin;
      __syncthreads();
      float v2 = 0.f;
#pragma unroll 4
      for (int j = tid; j < k4; j += 256) {
        const float4 v = __ldcg(x4 + j);
        const float a0 = v.x - mean, a1 = v.y - mean, a2 = v.z - mean, a3 = v.w - mean;
        v2 = fmaf(a0, a0, fmaf(a1, a1, fmaf(a2, a2, fmaf(a3, a3, v2))));
      }
      v2 = warp_butterfly_sum(v2);
      if (lane == 0) s_red[w] = v2;
      __syncthreads();
      v2 = 0.f;
      for (int q = 0; q < 8; ++q) v2 += s_red[q];
      den = sqrtf(v2 / (float)kin + 1e-5f);
      __syncthreads();
    }
    __nv_bfloat16 *o = parts + (size_t)i * kin;
#pragma unroll 4
    for (int j = tid; j < k4; j += 256) {
      const float4 v4 = __ldcg(x4 + j);
      float v[4] = {v4.x, v4.y, v4.z, v4.w};
      __nv_bfloat16 h[4], m[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = v[e];
        if (ln) x = ln_elem(x - mean, den, gg[4 * j + e], bb[4 * j + e]);
        h[e] = __float2bfloat16_rn(x);
        m[e] = __float2bfloat16_rn(x - __bfloat162float(h[e]));
      }
      *reinterpret_cast<uint2 *>(o + 4 * j) = *reinterpret_cast<uint2 *>(h);
      *reinterpret_cast<uint2 *>(o + plane + 4 * j) = *reinterpret_cast<uint2 *>(m);
    }
  }
}

template <int EPI, int AHEAD>
__global__ void __launch_bounds__(TL_THREADS, 1) tcl_gemm_kernel(LayerParams p, int nout, int kin,
                                                                 int Npad,
                                                                 const __nv_bfloat16 *parts,
                                                                 float *partial) {
  extern __shared__ __align__(1024) uint8_t tlsm[];
  uint8_t *ring = reinterpret_cast<uint8_t *>(((uintptr_t)tlsm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mma_done[TL_STAGES];
  __shared__ uint64_t all_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (flag_set(p.done)) return;
  const int nrows = *reinterpret_cast<const volatile int32_t *>(p.nrows);
  const int o0 = blockIdx.x * TL_M, n0 = blockIdx.y * TL_NT;
  if (n0 >= nrows) return;
  const int ntile = (nrows - n0 < TL_NT ? (nrows - n0 + 15) / 16 * 16 : TL_NT);
  // K split over blockIdx.z (partials reduced by tcl_reduce_kernel)
  const int kbt = kin / TL_BK, ks = blockIdx.z, nks = gridDim.z;
  const int kb0 = (int)((long long)ks * kbt / nks), kb1 = (int)((long long)(ks + 1) * kbt / nks);
  const int nkb = kb1 - kb0;
  const __nv_bfloat16 *W = reinterpret_cast<const __nv_bfloat16 *>(gemv_weights<EPI>(p));
  if (tid == 0) {
    for (int s = 0; s < TL_STAGES; ++s) mbar_init(&mma_done[s], 1);
    mbar_init(&all_done, 1);
  }
  fence_mbar_init();
  // two accumulators (even / odd k-steps): two independent MMA chains
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&tmem_base)), "n"(2 * TL_NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int my_o = o0 + tid;
  const size_t plane = (size_t)Npad * kin;
  auto load_stage = [&](int i) {
    uint8_t *st = ring + (size_t)(i % TL_STAGES) * TL_STAGE;
    const int k0 = (kb0 + i) * TL_BK;
    {
      const __nv_bfloat16 *src = W + (size_t)(my_o < nout ? my_o : 0) * kin + k0;
      uint8_t *dst = st + (size_t)tid * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) cp_async16(dst + ((c ^ (tid & 7)) << 4), src + c * 8, my_o < nout);
    }
    for (int pp = 0; pp < TL_PARTS; ++pp) {
      uint8_t *bt = st + TL_TILE_A + (size_t)pp * TL_TILE_B;
      const __nv_bfloat16 *pb = parts + (size_t)pp * plane;
      for (int q = tid; q < ntile * 8; q += TL_THREADS) {
        const int n = q >> 3, c = q & 7;
        cp_async16(bt + (size_t)n * 128 + ((c ^ (n & 7)) << 4),
                   pb + (size_t)(n0 + n) * kin + k0 + c * 8, n0 + n < nrows);
      }
    }
    cp_async_commit();
  };
  const uint32_t idesc = umma_idesc_bf16(TL_M, ntile);
  for (int i = 0; i < AHEAD; ++i) {
    if (i < nkb) load_stage(i); else cp_async_commit();
  }
  for (int i = 0; i < nkb; ++i) {
    // block i + AHEAD goes into the slot block i + AHEAD - STAGES used, whose
    // MMAs were issued STAGES - AHEAD iterations ago
    const int nxt = i + AHEAD;
    if (nxt < nkb) {
      const int old = nxt - TL_STAGES;
      if (old >= 0) mbar_wait(&mma_done[old % TL_STAGES], (old / TL_STAGES) & 1);
      load_stage(nxt);
    } else {
      cp_async_commit();
    }
    cp_async_wait<AHEAD>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(ring + (size_t)(i % TL_STAGES) * TL_STAGE);
#pragma unroll
      for (int k = 0; k < TL_BK / 16; ++k) {
        const uint64_t ad = umma_desc_sw128(sa + k * 32);
        const uint32_t dt = tmem + (uint32_t)((k & 1) * TL_NT);
#pragma unroll
        for (int pp = 0; pp < TL_PARTS; ++pp) {
          const uint64_t bd = umma_desc_sw128(sa + (uint32_t)(TL_TILE_A + pp * TL_TILE_B) + k * 32);
          umma_bf16(dt, ad, bd, idesc, (i > 0 || k > 1 || pp > 0) ? 1u : 0u);
        }
      }
      umma_commit(&mma_done[i % TL_STAGES]);
      if (i == nkb - 1) umma_commit(&all_done);
    }
  }
  mbar_wait(&all_done, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < ntile; c0 += 32) {
    uint32_t v[32], v1[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(TL_NT + c0), v1);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v1[j]));
    if (my_o < nout) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + c0 + j;
        if (c0 + j < ntile && n < nrows) {
          if (nks == 1) tcl_epilogue<EPI>(p, n, my_o, __uint_as_float(v[j]));
          else partial[((size_t)ks * Npad + n) * nout + my_o] = __uint_as_float(v[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TL_NT));
}

// ---------------------------------------------------------------------------
// TMA-fed, warp-specialised form of the same GEMM (default).  Warps 0-3 are
// the epilogue (thread = output feature = TMEM lane), warp 4 is the TMA
// producer (one elected lane: a 2-D cp.async.bulk.tensor of the 128 x 64
// weight block and of the two 64-wide row-part blocks per stage, 128-byte
// swizzle done by the copy engine, completion on full[s]), warp 5 issues the
// UMMAs (one lane) and releases stages with tcgen05.commit on empty[s].  No
// CTA-wide barrier inside the K loop, and no per-thread copy instructions:
// the ring is as deep as shared memory allows (4 stages at 128 rows, 7 at 64).
// Same MMA sequence as tcl_gemm_kernel (even/odd k-step accumulators), so the
// results are bit-identical to it.
constexpr int TT_THREADS = 192;
constexpr int TT_MAX_STAGES = 8;

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y),
        "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tl_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Row tiles: the grid's z extent covers the rows this call expects
// (rows_hint); a CTA then walks row tiles z, z + gridDim.z, ... while they
// hold rows (lazily completed rows can exceed the expectation), with the
// stage ring and the barrier phases running on across tiles and TMEM handed
// back by the epilogue (tmem_free) before the next tile's first MMA.
template <int EPI>
__global__ void __launch_bounds__(TT_THREADS, 2) tcl_tma_kernel(
    const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
    LayerParams p, int nout, int kin, int Npad, int nbox, int stages, float *partial,
    int *fix) {
  extern __shared__ __align__(1024) uint8_t tlsm[];
  uint8_t *ring = reinterpret_cast<uint8_t *>(((uintptr_t)tlsm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[TT_MAX_STAGES], empty[TT_MAX_STAGES];
  __shared__ uint64_t all_done, tmem_free;
  __shared__ int s_last;
  __shared__ uint32_t tmem_base;
  __shared__ int s_go;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // grid (output tiles, K splits, row tiles)
  const int o0 = blockIdx.x * TL_M;
  const int kbt = kin / TL_BK, ks = blockIdx.y, nks = gridDim.y;
  const int kb0 = (int)((long long)ks * kbt / nks), kb1 = (int)((long long)(ks + 1) * kbt / nks);
  const int nkb = kb1 - kb0;
  const uint32_t tile_b = (uint32_t)nbox * 128u;
  const uint32_t stage_bytes = (uint32_t)TL_TILE_A + TL_PARTS * tile_b;
  // the weights do not depend on the previous kernels: the first tile's
  // first weight stages are requested before griddepcontrol.wait
  // (programmatic dependent launch), its row parts after it
  const int first_n0 = blockIdx.z * nbox;
  const int pre = nkb < stages ? nkb : stages;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&all_done, 1);
    mbar_init(&tmem_free, 128);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    for (int i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full[i], stage_bytes);
      tma_load_2d(ring + (size_t)i * stage_bytes, &tmW, (kb0 + i) * TL_BK, o0, &full[i]);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (tid == 0) {
    const int nrows0 = *reinterpret_cast<const volatile int32_t *>(p.nrows);
    s_go = !flag_set(p.done) && first_n0 < nrows0;
    // complete the prefetched stages (their row parts) either way; drain
    // them if this CTA has nothing to do
    for (int i = 0; i < pre; ++i)
#pragma unroll
      for (int pp = 0; pp < TL_PARTS; ++pp)
        tma_load_2d(ring + (size_t)i * stage_bytes + TL_TILE_A + pp * tile_b, &tmX,
                    (kb0 + i) * TL_BK, pp * Npad + first_n0, &full[i]);
    if (!s_go)
      for (int i = 0; i < pre; ++i) mbar_wait(&full[i], 0);
  }
  __syncthreads();
  if (!s_go) return;
  const int nrows = *reinterpret_cast<const volatile int32_t *>(p.nrows);
  if (warp == 5) {
    // two accumulators (even / odd k-steps) of acc = max(nbox, 128) columns:
    // 256 columns, or all 512 for 256-row tiles (one CTA per SM then)
    if (nbox > TL_NT)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(&tmem_base)), "n"(4 * TL_NT));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(&tmem_base)), "n"(2 * TL_NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t acc = nbox > TL_NT ? 2 * TL_NT : TL_NT;    // accumulator column stride
  const int zstep = gridDim.z * nbox;
  if (warp == 4) {
    if (lane == 0) {
      int it = 0;
      for (int n0 = first_n0; n0 < nrows; n0 += zstep, ++it)
        for (int i = 0; i < nkb; ++i) {
          const int gi = it * nkb + i;
          if (gi < pre) continue;                   // issued before the wait
          const int s = gi % stages;
          if (gi >= stages) mbar_wait(&empty[s], ((gi / stages) - 1) & 1);
          uint8_t *st = ring + (size_t)s * stage_bytes;
          const int k0 = (kb0 + i) * TL_BK;
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          tma_load_2d(st, &tmW, k0, o0, &full[s]);
#pragma unroll
          for (int pp = 0; pp < TL_PARTS; ++pp)
            tma_load_2d(st + TL_TILE_A + pp * tile_b, &tmX, k0, pp * Npad + n0, &full[s]);
        }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(TL_M, nbox);
      int it = 0;
      for (int n0 = first_n0; n0 < nrows; n0 += zstep, ++it) {
        if (it > 0) {                               // the epilogue has read the last tile
          mbar_wait(&tmem_free, (it - 1) & 1);
          tc_fence_after();
        }
        for (int i = 0; i < nkb; ++i) {
          const int gi = it * nkb + i;
          const int s = gi % stages;
          mbar_wait(&full[s], (gi / stages) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + (size_t)s * stage_bytes);
#pragma unroll
          for (int k = 0; k < TL_BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(sa + k * 32);
            const uint32_t dt = tmem + (uint32_t)(k & 1) * acc;
#pragma unroll
            for (int pp = 0; pp < TL_PARTS; ++pp) {
              const uint64_t bd = umma_desc_sw128(sa + (uint32_t)TL_TILE_A + pp * tile_b + k * 32);
              umma_bf16(dt, ad, bd, idesc, (i > 0 || k > 1 || pp > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
          if (i == nkb - 1) umma_commit(&all_done);
        }
      }
    }
  } else {
    const int my_o = o0 + tid;
    int it = 0;
    for (int n0 = first_n0; n0 < nrows; n0 += zstep, ++it) {
      mbar_wait(&all_done, it & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < nbox; c0 += 32) {
        uint32_t v[32], v1[32];
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + acc + (uint32_t)c0, v1);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v1[j]));
        if (my_o < nout) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + c0 + j;
            if (c0 + j < nbox && n < nrows) {
              if (nks == 1) tcl_epilogue<EPI>(p, n, my_o, __uint_as_float(v[j]));
              else partial[((size_t)ks * Npad + n) * nout + my_o] = __uint_as_float(v[j]);
            }
          }
        }
      }
      tc_fence_before();
      tl_mbar_arrive(&tmem_free);
      if (nks > 1 && fix) {
        // K-split fixup: the last split CTA of this (output tile, row tile)
        // sums the nks partials in split order (tcl_reduce_kernel's order)
        // and runs the epilogue -- no separate reduce launch
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        int *ctr = fix + (size_t)blockIdx.x * (Npad / 16) + n0 / 16;
        if (tid == 0) s_last = atomicAdd(ctr, 1) == nks - 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (s_last) {
          __threadfence();
          if (my_o < nout)
            for (int c = 0; c < nbox && n0 + c < nrows; ++c) {
              const int n = n0 + c;
              float sum = 0.f;
              for (int k = 0; k < nks; ++k) sum += __ldcg(partial + ((size_t)k * Npad + n) * nout + my_o);
              tcl_epilogue<EPI>(p, n, my_o, sum);
            }
          if (tid == 0) *ctr = 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    if (nbox > TL_NT)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(4 * TL_NT));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TL_NT));
  }
}

// 2-D bf16 tensor map, 64-element (128-byte) inner box, 128-byte swizzle
static bool tl_tensor_map_encode(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols,
                                 uint32_t box_rows);
// encoded maps cached per (pointer, shape, box): the host cost of a layer call
// matters where it is not graph-captured (the tree step)
struct TlMapKey {
  const void *ptr; uint64_t rows, cols; uint32_t box;
  bool operator==(const TlMapKey &o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && box == o.box;
  }
};
struct TlMapHash {
  size_t operator()(const TlMapKey &k) const {
    return std::hash<const void *>()(k.ptr) ^ (k.rows * 0x9E3779B97F4A7C15ull) ^ (k.cols << 7) ^ k.box;
  }
};
static bool tl_tensor_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols,
                          uint32_t box_rows) {
  static std::unordered_map<TlMapKey, CUtensorMap, TlMapHash> cache;
  const TlMapKey key{ptr, rows, cols, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) { *m = it->second; return true; }
  if (!tl_tensor_map_encode(m, ptr, rows, cols, box_rows)) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}
static bool tl_tensor_map_encode(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols,
                                 uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      encode = nullptr;
    if (!encode) return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)TL_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the K-split partials of every (row, output) in split order -> the epilogue
template <int EPI>
__global__ void __launch_bounds__(256) tcl_reduce_kernel(LayerParams p, int nout, int Npad,
                                                       int nks, const float *partial) {
  pdl_wait();
  pdl_trigger();
  if (flag_set(p.done)) return;
  const int n = *reinterpret_cast<const volatile int32_t *>(p.nrows);
  // grid (output quads, rows): 4 consecutive outputs per thread (16-byte
  // partial loads, all splits in flight), rows strided by gridDim.y; the
  // split order of the sum is unchanged (k = 0, 1, ...)
  const int o = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (o >= nout) return;
  for (int r = blockIdx.y; r < n; r += gridDim.y) {
    float4 a = __ldcg(reinterpret_cast<const float4 *>(partial + (size_t)r * nout + o));
    float sv[4] = {a.x, a.y, a.z, a.w};
    sv[0] = 0.f + sv[0]; sv[1] = 0.f + sv[1]; sv[2] = 0.f + sv[2]; sv[3] = 0.f + sv[3];
    for (int k = 1; k < nks; ++k) {
      const float4 b = __ldcg(reinterpret_cast<const float4 *>(partial + ((size_t)k * Npad + r) * nout + o));
      sv[0] += b.x; sv[1] += b.y; sv[2] += b.z; sv[3] += b.w;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) tcl_epilogue<EPI>(p, r, o + e, sv[e]);
  }
}

// frontier of the advanced rows, newest-row copy (model.py:269-270), reset
__global__ void tcl_finish_kernel(LayerParams p) {
  pdl_wait();
  pdl_trigger();
  if (flag_set(p.done)) return;
  const int n = *reinterpret_cast<const volatile int32_t *>(p.nrows);
  for (int i = threadIdx.x; i < n; i += blockDim.x) p.frontier[p.rows[i]] = p.layer + 1;
  if (p.cur_hidden && p.new_row) {
    const int nw = *p.new_row;
    if (nw >= 0) {                                // 16-byte copies, all in flight at once
      const float4 *src = reinterpret_cast<const float4 *>(p.pending + (size_t)nw * p.d);
      float4 *dst = reinterpret_cast<float4 *>(p.cur_hidden);
#pragma unroll 4
      for (int j = threadIdx.x; j < p.d / 4; j += blockDim.x) dst[j] = __ldcg(src + j);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *p.nrows = 0;
}


inline size_t tcl_scratch_bytes(int d, int ffn, int row_cap) {
  // parts A, parts B, partials, the K-split tile counters (zero-initialised
  // by the caller, self-resetting)
  return 2 * tcl_parts_bytes(d, ffn, row_cap) + TL_PARTIAL_BYTES + (size_t)TL_FIX_SLOTS * 4;
}

inline bool tcl_supported(const LayerParams &p) {
  static const int env = getenv("SPX_LAYER_TCGEN05") ? atoi(getenv("SPX_LAYER_TCGEN05")) : 1;
  // SPX_TCL_MIN_ROWS: smallest row count routed here (the 8-row mma.sync
  // slices below it re-stream nothing for <= 8 rows but run ~2x slower per
  // byte than the TMA-fed UMMA GEMM)
  static const int min_rows = getenv("SPX_TCL_MIN_ROWS") ? atoi(getenv("SPX_TCL_MIN_ROWS")) : 3;
  return env && p.tc_scratch && p.rows_hint >= min_rows && p.d % TL_BK == 0 && p.ffn % TL_BK == 0;
}

template <int EPI>
static void tcl_matrix(const LayerParams &p, int nout, int kin, int Npad, int sms,
                       cudaStream_t s, bool prep = true) {
  const size_t pbytes = tcl_parts_bytes(p.d, p.ffn, p.row_cap);
  __nv_bfloat16 *parts = reinterpret_cast<__nv_bfloat16 *>(
      reinterpret_cast<uint8_t *>(p.tc_scratch) + (EPI == EPI_FFN2 ? pbytes : 0));
  float *partial = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(p.tc_scratch) + 2 * pbytes);
  int *fix = reinterpret_cast<int *>(reinterpret_cast<uint8_t *>(p.tc_scratch) + 2 * pbytes +
                                     TL_PARTIAL_BYTES);
  // SPX_TCL_FIXUP=1 (A/B, off): the last split CTA of a tile reduces the
  // partials itself instead of a reduce launch.  Measured slower (tree step
  // 13.2 vs 10.4 ms, 13B B=64 21.2 vs 10.5 ms): one thread per output walks
  // the tile's rows x splits as a dependent load chain, where the reduce
  // kernel spreads the same sums over the whole GPU.
  static const int env_fix = getenv("SPX_TCL_FIXUP") ? atoi(getenv("SPX_TCL_FIXUP")) : 0;
  bool fixed = false;                               // K split reduced inside the GEMM
  if (prep)
    launch_pdl(tcl_prep_kernel<EPI>, p.row_cap < 2 * sms ? p.row_cap : 2 * sms, 256, 0, s, p, kin,
               Npad, parts);
  // K split so that the live CTAs (expected row tiles) fill one wave
  // (rows_hint), bounded by the partial buffer and >= 8 K-blocks per split
  const int otiles = (nout + TL_M - 1) / TL_M;
  const int nt_exp = (p.rows_hint + TL_NT - 1) / TL_NT;
  int nks = sms / (otiles * (nt_exp > 0 ? nt_exp : 1));    // one wave (1 CTA per SM; cp.async form)
  nks = nks < 1 ? 1 : nks > 8 ? 8 : nks;
  while (nks > 1 && ((size_t)nks * Npad * nout * 4 > TL_PARTIAL_BYTES || kin / TL_BK / nks < 8))
    --nks;
  const size_t smem = (size_t)TL_STAGES * TL_STAGE + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tcl_gemm_kernel<EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(tcl_gemm_kernel<EPI, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = true;
  }
  // SPX_TCL_TMA=0 (A/B): the cp.async form below
  static const int env_tma = getenv("SPX_TCL_TMA") ? atoi(getenv("SPX_TCL_TMA")) : 1;
  // row tile sized by the rows this call expects (rows_hint), not the state's
  // capacity: the B operand (two parts) is loaded box-sized per stage
  const int rows_exp = p.rows_hint > 16 ? (p.rows_hint + 15) / 16 * 16 : 16;
  // SPX_TCL_N256=1 (A/B, off): 256-row tiles (UMMA N = 256, weights read
  // once for up to 256 rows, all 512 TMEM columns, 2 stages, one CTA per SM)
  // when the call expects >= 256 rows.  Measured slower: 13B B=256 step 22.3
  // vs 19.3 ms (two 80 KB stages per SM keep too few weight bytes in flight)
  static const int env_n256 = getenv("SPX_TCL_N256") ? atoi(getenv("SPX_TCL_N256")) : 0;
  const int nmax = (env_n256 && rows_exp >= 2 * TL_NT) ? 2 * TL_NT : TL_NT;
  int nbox = Npad < nmax ? Npad : nmax;
  nbox = rows_exp < nbox ? rows_exp : nbox;
  CUtensorMap tmW, tmX;
  if (env_tma && tl_tensor_map(&tmW, gemv_weights_host<EPI>(p), (uint64_t)nout, (uint64_t)kin, TL_M) &&
      tl_tensor_map(&tmX, parts, (uint64_t)TL_PARTS * Npad, (uint64_t)kin, (uint32_t)nbox)) {
    const size_t stage = TL_TILE_A + (size_t)TL_PARTS * nbox * 128;
    // two CTAs per SM (two independent TMA -> UMMA pipelines per SM, and a
    // K split that fills one wave of 2 x 148 CTAs) when at least 2 stages fit
    // in half the shared memory (measured: 2 x 2 stages beat 1 x 4 stages at
    // 128-row tiles, 78 vs 113 us for the 13B QKV at 256 rows), else one
    // CTA per SM with a deep ring
    const int nt0 = (rows_exp + nbox - 1) / nbox;
    int per_sm = 2;
    int stages = (int)((113 * 1024 - 1024) / stage);
    static const int env_min2 = getenv("SPX_TCL_MIN2") ? atoi(getenv("SPX_TCL_MIN2")) : 2;
    (void)nt0;
    const int min_stages = env_min2;
    if (stages < min_stages) {
      per_sm = 1;
      stages = (int)((227 * 1024 - 1024) / stage);
    }
    stages = stages > TT_MAX_STAGES ? TT_MAX_STAGES : stages;
    // K split: the expected live CTAs fill one wave of per_sm CTAs per SM
    const int nt = (rows_exp + nbox - 1) / nbox;
    nks = per_sm * sms / (otiles * nt);
    // SPX_TCL_MIN_OTILES_SPLIT (A/B): matrices with at least this many output
    // tiles run without a K split (no partials, no reduce pass)
    static const int env_nosplit = getenv("SPX_TCL_MIN_OTILES_SPLIT") ? atoi(getenv("SPX_TCL_MIN_OTILES_SPLIT")) : 0;
    if (env_nosplit > 0 && otiles * nt >= env_nosplit) nks = 1;
    nks = nks < 1 ? 1 : nks > 8 ? 8 : nks;
    while (nks > 1 && ((size_t)nks * Npad * nout * 4 > TL_PARTIAL_BYTES || kin / TL_BK / nks < 8))
      --nks;
    const size_t tsm = (size_t)stages * stage + 1024;
    static size_t tsm_set = 0;
    if (tsm > tsm_set) {
      cudaFuncSetAttribute(tcl_tma_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      tsm_set = tsm;
    }
    // row tiles for the rows this call expects; more rows (lazy completion)
    // are walked by the same CTAs
    const int zt = (rows_exp + nbox - 1) / nbox;
    dim3 tgrid((unsigned)otiles, (unsigned)nks, (unsigned)(zt < 1 ? 1 : zt));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = tgrid;
    cfg.blockDim = dim3(TT_THREADS);
    cfg.dynamicSmemBytes = tsm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const int env_pdl = getenv("SPX_PDL_LAYERS") ? atoi(getenv("SPX_PDL_LAYERS")) : 1;
    cfg.numAttrs = env_pdl ? 1 : 0;
    const int otiles_l = (nout + TL_M - 1) / TL_M;
    fixed = env_fix && nks > 1 && (size_t)otiles_l * (Npad / 16) <= (size_t)TL_FIX_SLOTS;
    cudaLaunchKernelEx(&cfg, tcl_tma_kernel<EPI>, tmW, tmX, p, nout, kin, Npad, nbox, stages,
                       partial, fixed ? fix : static_cast<int *>(nullptr));
  } else {
  dim3 grid((unsigned)otiles, (unsigned)((Npad + TL_NT - 1) / TL_NT), (unsigned)nks);
  // SPX_TCL_AHEAD (A/B): K-blocks in flight ahead of the MMA (3 leaves one
  // iteration of MMA slack per slot, 2 leaves two)
  static const int env_ahead = getenv("SPX_TCL_AHEAD") ? atoi(getenv("SPX_TCL_AHEAD")) : 2;
  if (env_ahead == 3)
    tcl_gemm_kernel<EPI, 3><<<grid, TL_THREADS, smem, s>>>(p, nout, kin, Npad, parts, partial);
  else
    tcl_gemm_kernel<EPI, 2><<<grid, TL_THREADS, smem, s>>>(p, nout, kin, Npad, parts, partial);
  }
  if (nks > 1 && !fixed) {
    const long long work = (long long)(p.rows_hint > 0 ? p.rows_hint : 1) * nout;
    const int rg = (int)((work + 255) / 256 < 8 * sms ? (work + 255) / 256 : 8 * sms);
    (void)rg;
    const int rows_y = p.rows_hint > 0 ? (p.rows_hint < 256 ? p.rows_hint : 256) : 1;
    launch_pdl(tcl_reduce_kernel<EPI>, dim3((unsigned)((nout / 4 + 255) / 256), (unsigned)rows_y),
               256, 0, s, p, nout, Npad, nks, static_cast<const float *>(partial));
  }
}

static void launch_layer_tcgen05(const LayerParams &p, int sms, cudaStream_t s) {
  const int Npad = tl_npad(p);
  const size_t rsm = (size_t)p.row_cap * 4;
  if (rsm > 48 * 1024)
    cudaFuncSetAttribute(tcl_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
  launch_pdl(tcl_rows_kernel, 1, 512, rsm, s, p);
  tcl_matrix<EPI_QKV>(p, 3 * p.d, p.d, Npad, sms, s);
  // head dim 128: the attention kernel emits Wo's input parts itself;
  // FFN1's epilogue emits FFN2's
  const bool att_parts = launch_attn_fast(p, sms, s, true);
  tcl_matrix<EPI_WO>(p, p.d, p.d, Npad, sms, s, !att_parts);
  tcl_matrix<EPI_FFN1>(p, p.ffn, p.d, Npad, sms, s);
  tcl_matrix<EPI_FFN2>(p, p.d, p.ffn, Npad, sms, s, false);
  launch_pdl(tcl_finish_kernel, 1, 1024, 0, s, p);
}

}  // namespace spx
