// K4 for MANY gated rows on the 5th-generation tensor cores (FAST mode, bf16
// head): the batched engine's per-layer gated verify and its final argmax,
// token-tree path verification.  Included by spx_verify.cu.
//
// Reference: verify_exit (engine.py:59-64) = argmax(full_head_logits) in the
// speculative set; full_head_logits (model.py:289-295).
//
// The CUDA-core verify_kernel re-reads the (V, d) head once per 4 gated rows
// (911 us per launch for ~64 rows of the Llama2-13B head).  Here the whole
// head is read once per 128 rows:
//
//   tcv_prep    the gated rows, compacted; per row the FAST head
//               normalisation (warp_head_prep: xg, r -- the same bits as
//               verify_kernel) split EXACTLY into three bf16 parts
//               (hi + mid + lo = the f32 mantissa), and S = sum |xg|
//   tcv_gemm    D[v][n] (TMEM f32) = W_v . (hi + mid + lo)_n  -- TMA-fed,
//               warp-specialised UMMA (kind::f16, exact bf16 x bf16 products);
//               epilogue tl[n][v] = r_n * D + bw_v
//   tcv_select  per row: M = max_v tl; every v whose tensor-core logit is
//               within the stated bound of M is re-evaluated in the canonical
//               CDOT order (warp_cdot, exactly verify_kernel's arithmetic) and
//               the argmax is taken over those exact logits -> token, max
//               logit, membership, the exit flag: bit-identical to
//               verify_kernel.
//
// Candidate bound: the tensor-core and CDOT logits are two f32 sums of the
// same d exact products |xg_j W_vj| <= wmax_v |xg_j|, so each differs from
// the exact dot by <= 2 d u wmax_v S (u = 2^-24, a factor 2 over the
// textbook (d-1)u for the tensor pipe's accumulation), plus the rounding of
// r * dot + bw.  With e_v = r (4 d u wmax_v S) + 4 u (|tl_v| + |bw_v|):
// the CDOT argmax v* satisfies tl_v* >= M - e_v* - e_vhat (vhat = the
// tensor-core argmax), so it is always a candidate.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "spx_umma.cuh"

namespace spx {

constexpr int TV_M = 128;            // vocab rows per tile (UMMA M)
constexpr int TV_NT = 128;           // gated rows per tile (UMMA N)
constexpr int TV_BK = 64;            // K elements per stage (128-byte swizzle atom)
constexpr int TV_PARTS = 3;
constexpr int TV_THREADS = 192;      // warps 0-3 epilogue, 4 TMA, 5 MMA
constexpr int TV_MAX_STAGES = 8;
constexpr size_t TV_TILE_A = (size_t)TV_M * TV_BK * 2;

struct TvLayout {
  size_t rows, r, s, parts, xg, tl, total;
};
__host__ __device__ inline int tv_npad(int B) { return (B + 15) / 16 * 16; }
__host__ __device__ inline TvLayout tv_layout(int B, int d, int V) {
  TvLayout L;
  const size_t np = (size_t)tv_npad(B);
  L.rows = 256;                                   // [0] = row count
  L.r = L.rows + (np * 4 + 255) / 256 * 256;
  L.s = L.r + (np * 4 + 255) / 256 * 256;
  L.parts = L.s + (np * 4 + 255) / 256 * 256;
  L.xg = L.parts + ((size_t)TV_PARTS * np * d * 2 + 255) / 256 * 256;
  L.tl = L.xg + (np * (size_t)d * 4 + 255) / 256 * 256;
  L.total = L.tl + np * (size_t)V * 4;
  return L;
}

// one CTA (one warp) per potential row: the i-th gated row (ballot scan of
// the flags), its FAST normalisation, the three parts, S and r
template <int CPL>
__global__ void __launch_bounds__(32) tcv_prep_kernel(VerParams p, uint8_t *scratch, int Npad) {
  extern __shared__ float hn[];
  const TvLayout L = tv_layout(p.B, p.d, p.V);
  int32_t *rows = reinterpret_cast<int32_t *>(scratch + L.rows);
  const int lane = threadIdx.x, want = blockIdx.x;
  int seen = 0, row = -1;
  for (int base = 0; base < p.B; base += 32) {
    const int r = base + lane;
    const bool on = r < p.B && ver_row_on(p, r);
    const unsigned m = __ballot_sync(0xffffffffu, on);
    const int c = __popc(m);
    if (row < 0 && want >= seen && want < seen + c) {
      // the (want - seen)-th set bit of m
      unsigned mm = m;
      for (int k = 0; k < want - seen; ++k) mm &= mm - 1;
      row = base + __ffs(mm) - 1;
    }
    seen += c;
  }
  if (want == 0 && lane == 0) reinterpret_cast<int32_t *>(scratch)[0] = seen;
  if (row < 0) return;
  int bad = 0;
  float rr = 1.f;
  warp_head_prep<CPL>(p.hidden + (size_t)row * p.hidden_stride, p.g, p.b, p.d, hn, lane, false,
                      &rr, &bad);
  if (bad && lane == 0) atomicOr(p.err, ERR_HIDDEN_NONFINITE);
  __nv_bfloat16 *parts = reinterpret_cast<__nv_bfloat16 *>(scratch + L.parts);
  float *xg_out = reinterpret_cast<float *>(scratch + L.xg) + (size_t)want * p.d;
  const size_t plane = (size_t)Npad * p.d;
  float sa = 0.f;
  for (int j = lane; j < p.d; j += 32) {
    const float x = hn[j];
    xg_out[j] = x;                                  // for tcv_select's exact dots
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float x1 = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(x1);
    const __nv_bfloat16 l = __float2bfloat16_rn(x1 - __bfloat162float(m));
    parts[(size_t)want * p.d + j] = h;
    parts[plane + (size_t)want * p.d + j] = m;
    parts[2 * plane + (size_t)want * p.d + j] = l;
    sa += fabsf(x);
  }
  sa = warp_butterfly_sum(sa);
  if (lane == 0) {
    rows[want] = row;
    reinterpret_cast<float *>(scratch + L.r)[want] = rr;
    reinterpret_cast<float *>(scratch + L.s)[want] = sa * (1.f + 1e-3f);   // sum rounding
  }
}

__device__ __forceinline__ void tv_tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                               uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y),
        "r"(smem_u32(bar))
      : "memory");
}

// D[v][n] for a 128-vocab-row x nbox-row tile; epilogue tl[n][v] = r_n D + bw_v
__global__ void __launch_bounds__(TV_THREADS, 1) tcv_gemm_kernel(
    const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
    VerParams p, uint8_t *scratch, int Npad, int nbox, int stages) {
  extern __shared__ __align__(1024) uint8_t tvsm[];
  uint8_t *ring = reinterpret_cast<uint8_t *>(((uintptr_t)tvsm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[TV_MAX_STAGES], empty[TV_MAX_STAGES];
  __shared__ uint64_t all_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const TvLayout L = tv_layout(p.B, p.d, p.V);
  const int nrows = *reinterpret_cast<const volatile int32_t *>(scratch);
  const int v0 = blockIdx.x * TV_M, n0 = blockIdx.y * nbox;
  if (n0 >= nrows) return;
  const int nkb = p.d / TV_BK;
  const uint32_t tile_b = (uint32_t)nbox * 128u;
  const uint32_t stage_bytes = (uint32_t)TV_TILE_A + TV_PARTS * tile_b;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&all_done, 1);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  fence_mbar_init();
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&tmem_base)), "n"(2 * TV_NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        if (i >= stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
        uint8_t *st = ring + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tv_tma_load_2d(st, &tmW, i * TV_BK, v0, &full[s]);
#pragma unroll
        for (int pp = 0; pp < TV_PARTS; ++pp)
          tv_tma_load_2d(st + TV_TILE_A + pp * tile_b, &tmX, i * TV_BK, pp * Npad + n0, &full[s]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(TV_M, nbox);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        mbar_wait(&full[s], (i / stages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(ring + (size_t)s * stage_bytes);
#pragma unroll
        for (int k = 0; k < TV_BK / 16; ++k) {
          const uint64_t ad = umma_desc_sw128(sa + k * 32);
          const uint32_t dt = tmem + (uint32_t)((k & 1) * TV_NT);
#pragma unroll
          for (int pp = 0; pp < TV_PARTS; ++pp) {
            const uint64_t bd = umma_desc_sw128(sa + (uint32_t)TV_TILE_A + pp * tile_b + k * 32);
            umma_bf16(dt, ad, bd, idesc, (i > 0 || k > 1 || pp > 0) ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
        if (i == nkb - 1) umma_commit(&all_done);
      }
    }
  } else {
    const int v = v0 + tid;
    const float bw = (v < p.V && p.head_bw) ? p.head_bw[v] : 0.f;
    const float *rr = reinterpret_cast<const float *>(scratch + L.r);
    float *tl = reinterpret_cast<float *>(scratch + L.tl);
    mbar_wait(&all_done, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < nbox; c0 += 32) {
      uint32_t a[32], b[32];
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, a);
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(TV_NT + c0), b);
      if (v < p.V) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = n0 + c0 + j;
          if (c0 + j < nbox && n < nrows) {
            const float dot = __uint_as_float(a[j]) + __uint_as_float(b[j]);
            tl[(size_t)n * p.V + v] = __fadd_rn(__fmul_rn(rr[n], dot), bw);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TV_NT));
}

// one CTA per compacted row: the tensor-core top keys, the candidates, their
// exact CDOT logits, the argmax (and the stable top-K when topk_k > 0) and
// verify_kernel's row finalisation.  With Kt = max(topk_k, 1) tensor-core
// winners, T = the Kt-th largest tensor-core logit and E = the largest bound
// e_v among the winners, every member of the exact top-Kt has tl_v + e_v >=
// T - E (Kt elements have exact logits >= T - E), so it is a candidate.
constexpr int TV_CAND = 1024;
template <typename TW, int CPL>
__global__ void __launch_bounds__(VER_THREADS) tcv_select_kernel(VerParams p,
                                                                 const float *head_wmax,
                                                                 const uint8_t *scratch) {
  extern __shared__ float hn[];
  __shared__ unsigned long long s_key[VER_THREADS / 32];
  __shared__ unsigned long long s_cand[TV_CAND];
  __shared__ int s_nc;
  __shared__ float s_thr;
  const TvLayout L = tv_layout(p.B, p.d, p.V);
  const int nrows = *reinterpret_cast<const volatile int32_t *>(scratch);
  const int i = blockIdx.x;
  if (i >= nrows) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = VER_THREADS / 32;
  const int row = reinterpret_cast<const int32_t *>(scratch + L.rows)[i];
  const float S = reinterpret_cast<const float *>(scratch + L.s)[i];
  const float *tl = reinterpret_cast<const float *>(scratch + L.tl) + (size_t)i * p.V;
  const TW *head = reinterpret_cast<const TW *>(p.head);
  const int Kt = p.topk_k > 0 ? p.topk_k : 1;
  {
    // the row's FAST normalisation as tcv_prep computed it (warp_head_prep:
    // the very bits verify_kernel uses), staged with 16-byte loads
    const float4 *src = reinterpret_cast<const float4 *>(scratch + L.xg) + (size_t)i * (p.d / 4);
    for (int j = tid; j < p.d / 4; j += VER_THREADS) reinterpret_cast<float4 *>(hn)[j] = __ldcg(src + j);
    if (tid == 0) hn[p.d] = reinterpret_cast<const float *>(scratch + L.r)[i];
  }
  if (tid == 0) s_nc = 0;
  __syncthreads();
  const float r = hn[p.d];
  const float du = 4.f * (float)p.d * 5.9604645e-8f;          // 4 d u
  const float u4 = 4.f * 5.9604645e-8f;
  auto bound = [&](int v, float t) {
    const float bwv = p.head_bw ? p.head_bw[v] : 0.f;
    return r * du * head_wmax[v] * S + u4 * (fabsf(t) + fabsf(bwv));
  };
  auto block_max = [&](unsigned long long k) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, m);
      k = o > k ? o : k;
    }
    if (lane == 0) s_key[warp] = k;
    __syncthreads();
    unsigned long long b = 0ull;
    for (int w = 0; w < nw; ++w) b = s_key[w] > b ? s_key[w] : b;
    __syncthreads();
    return b;
  };
  // the Kt largest tensor-core keys
  unsigned long long below = ~0ull, last = 0ull;
  float E = 0.f;
  if (Kt <= 8) {
    // one scan: every thread keeps its 8 best keys in registers; Kt rounds
    // of a block max pop the winner from its owner's list (a thread is asked
    // for at most Kt <= 8 keys, so its list never runs dry)
    unsigned long long l[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) l[q] = 0ull;
    for (int v = tid; v < p.V; v += VER_THREADS) {
      unsigned long long k = argmax_key(tl[v], (uint32_t)v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool sw = k > l[q];
        const unsigned long long t = l[q];
        l[q] = sw ? k : t;
        k = sw ? t : k;
      }
    }
    for (int q = 0; q < Kt; ++q) {
      last = block_max(l[0]);
      if (l[0] == last && last != 0ull) {
#pragma unroll
        for (int r = 0; r < 7; ++r) l[r] = l[r + 1];
        l[7] = 0ull;
      }
      const int vw = (int)(0xffffffffu - (uint32_t)(last & 0xffffffffull));
      E = fmaxf(E, bound(vw, f32_from_order_key((uint32_t)(last >> 32))));
    }
  } else {
    for (int q = 0; q < Kt; ++q) {                // one block max per round
      unsigned long long best = 0ull;
      for (int v = tid; v < p.V; v += VER_THREADS) {
        const unsigned long long k = argmax_key(tl[v], (uint32_t)v);
        if (k < below && k > best) best = k;
      }
      last = block_max(best);
      below = last;
      const int vw = (int)(0xffffffffu - (uint32_t)(last & 0xffffffffull));
      E = fmaxf(E, bound(vw, f32_from_order_key((uint32_t)(last >> 32))));
    }
  }
  const float thr = f32_from_order_key((uint32_t)(last >> 32)) - E;
  // candidates, re-evaluated exactly (warp per candidate), keys into s_cand
  for (int base = warp * 32; base < p.V; base += nw * 32) {
    const int v = base + lane;
    bool cand = false;
    if (v < p.V) {
      const float t = tl[v];
      cand = t + bound(v, t) >= thr || !(t == t);
    }
    unsigned m = __ballot_sync(0xffffffffu, cand);
    while (m) {
      const int vc = base + __ffs(m) - 1;
      m &= m - 1;
      float lg;
      warp_cdot<TW, 1, CPL>(head + (size_t)vc * p.d, hn, p.d, 1, lane, &lg);
      const float bw = p.head_bw ? p.head_bw[vc] : 0.f;
      lg = __fadd_rn(__fmul_rn(r, lg), bw);
      if (lane == 0) {
        const int slot = atomicAdd(&s_nc, 1);
        if (slot < TV_CAND) s_cand[slot] = argmax_key(lg, (uint32_t)vc);
      }
    }
  }
  __syncthreads();
  const int nc = s_nc < TV_CAND ? s_nc : TV_CAND;
  if (s_nc > TV_CAND && tid == 0) atomicOr(p.err, ERR_CAND_OVERFLOW);
  // exact top-Kt of the candidates (stable: value desc, index asc)
  below = ~0ull;
  unsigned long long top = 0ull;
  for (int q = 0; q < Kt; ++q) {
    unsigned long long best = 0ull;
    for (int c = tid; c < nc; c += VER_THREADS)
      if (s_cand[c] < below && s_cand[c] > best) best = s_cand[c];
    const unsigned long long k = block_max(best);
    if (q == 0) top = k;
    below = k;
    if (p.topk_out && tid == 0)
      p.topk_out[(size_t)row * p.topk_k + q] = (int32_t)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
  }
  if (tid == 0) {
    const int tok = (int)(0xffffffffu - (uint32_t)(top & 0xffffffffull));
    const float mx = f32_from_order_key((uint32_t)(top >> 32));
    bool in = false;
    if (p.spec_ptr)
      for (int j = p.spec_ptr[row]; j < p.spec_ptr[row + 1]; ++j) in |= (p.spec_ids[j] == tok);
    p.token_out[row] = tok;
    if (p.maxlogit_out) p.maxlogit_out[row] = mx;
    if (p.verified_out) p.verified_out[row] = in ? 1 : 0;
    if (p.full_heads) p.full_heads[row] += 1;
    if (in && p.done_out) {
      p.done_out[row] = 1;
      if (p.exit_layer_out) p.exit_layer_out[row] = p.layer;
    }
  }
}

// 2-D bf16 tensor map, 64-element (128-byte) inner box, 128-byte swizzle
static bool tv_tensor_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols,
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
  cuuint32_t box[2] = {(cuuint32_t)TV_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CPL>
static bool launch_verify_tc(const VerParams &p, const float *head_wmax, uint8_t *scratch,
                             cudaStream_t stream) {
  const int Npad = tv_npad(p.B);
  const TvLayout L = tv_layout(p.B, p.d, p.V);
  const int nbox = Npad < TV_NT ? Npad : TV_NT;
  CUtensorMap tmW, tmX;
  if (!tv_tensor_map(&tmW, p.head, (uint64_t)p.V, (uint64_t)p.d, TV_M) ||
      !tv_tensor_map(&tmX, scratch + L.parts, (uint64_t)TV_PARTS * Npad, (uint64_t)p.d,
                     (uint32_t)nbox))
    return false;
  const size_t hsm = (size_t)(p.d + 1) * sizeof(float);
  if (hsm > 48 * 1024) {
    cudaFuncSetAttribute(tcv_prep_kernel<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    cudaFuncSetAttribute(tcv_select_kernel<__nv_bfloat16, CPL>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
  }
  tcv_prep_kernel<CPL><<<p.B, 32, hsm, stream>>>(p, scratch, Npad);
  const size_t stage = TV_TILE_A + (size_t)TV_PARTS * nbox * 128;
  int stages = (int)((227 * 1024 - 1024) / stage);
  stages = stages > TV_MAX_STAGES ? TV_MAX_STAGES : stages;
  const size_t tsm = (size_t)stages * stage + 1024;
  cudaFuncSetAttribute(tcv_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
  dim3 grid((unsigned)((p.V + TV_M - 1) / TV_M), (unsigned)((Npad + nbox - 1) / nbox));
  tcv_gemm_kernel<<<grid, TV_THREADS, tsm, stream>>>(tmW, tmX, p, scratch, Npad, nbox, stages);
  tcv_select_kernel<__nv_bfloat16, CPL><<<p.B, VER_THREADS, hsm, stream>>>(p, head_wmax, scratch);
  return true;
}

}  // namespace spx
