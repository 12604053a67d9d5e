// K6 on the 5th-generation tensor cores: the merged-mapping contraction for
// DENSE node x unique-id tiles (batched token trees, SURVEY.md §8a-14,
// north-star (e)).
//
// Reference: grouped_speculative_logits (tree.py:92-113): per live node j,
// LN(h_j) . lm_head[:, ids_j].  After the merged mapping (spx_tree.cu) the
// work is D[u][n] = W_u . xg_n for the U unique LM-head rows u and the N live
// nodes n, needed only at the (n, u) pairs the nodes asked for.  When the
// node x id tile is large and dense, the whole tile is one GEMM:
//
//   A (M = 128 unique ids, K-major) = gathered bf16 LM-head rows
//   B (N <= 128 nodes,     K-major) = xg split EXACTLY into three bf16 parts
//       xg = hi + mid + lo (8 + 8 + 8 mantissa bits = the whole f32 mantissa)
//   D (TMEM, f32, 128 lanes x N columns) += A . B_hi^T + A . B_mid^T + A . B_lo^T
//
// bf16 x bf16 products are exact in f32, so the only difference from the
// CUDA-core CDOT order is the tensor core's accumulation order / rounding
// (FAST-mode tolerance; STRICT never takes this path).  Data movement:
// 16-byte cp.async into the 128-byte-swizzled K-major canonical layout
// (chunk ^ (row & 7)), a 3-stage ring released by tcgen05.commit; one thread
// issues tcgen05.mma (kind::f16, cta_group::1); the epilogue reads TMEM with
// tcgen05.ld 32x32b, stages D in shared memory and writes logit =
// r_n * D[u][n] + bw_u for the requested pairs.  K is split over CTAs so the
// grid covers the SMs; each split writes its dense partial tile and a gather
// kernel sums the partials of every requested pair in split order
// (deterministic).
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"
#include "spx_umma.cuh"

namespace spx {

constexpr int TC_M = 128;            // unique ids per tile (UMMA M)
constexpr int TC_NT = 128;           // nodes per tile (UMMA N, multiple of 16)
constexpr int TC_BK = 64;            // K elements per stage (128 bytes of bf16: one swizzle atom)
constexpr int TC_STAGES = 3;
constexpr int TC_THREADS = 128;
constexpr int TC_PARTS = 3;          // hi / mid / lo
constexpr size_t TC_TILE_A = (size_t)TC_M * TC_BK * 2;            // 16 KB
constexpr size_t TC_TILE_B = (size_t)TC_NT * TC_BK * 2;           // 16 KB per part
constexpr size_t TC_STAGE = TC_TILE_A + TC_PARTS * TC_TILE_B;     // 64 KB

// ---- prep: xg (N, d) f32 -> three exact bf16 parts (3, Npad, d) -------------
__global__ void tree_tc_split_kernel(const float *xg, int N, int Npad, int d,
                                     __nv_bfloat16 *parts) {
  const size_t total = (size_t)Npad * d;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / d);
    const float x = n < N ? xg[i] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(hi);                  // exact
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mid);                // exact
    parts[i] = hi;
    parts[total + i] = mid;
    parts[2 * total + i] = __float2bfloat16_rn(r2);             // exact for normal x
  }
}

struct TreeTcArgs {
  const __nv_bfloat16 *parts; int Npad;   // (3, Npad, d)
  const float *r; int N;
  const __nv_bfloat16 *head; const float *head_bw; int V, d;
  const int32_t *uniq; int U;
  const int32_t *uniq_ptr, *pair_node, *pair_out, *pair_uid;
  float *logits;
  float *partial; int P;                  // (ksplit, Upad, Npad) dense partial tiles; P pairs
  int Upad;
  int ksplit, kblocks;
  int *err;
};

__global__ void __launch_bounds__(TC_THREADS, 1) tree_tc_kernel(TreeTcArgs a) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  uint8_t *ring = reinterpret_cast<uint8_t *>(((uintptr_t)tsm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mma_done[TC_STAGES];
  __shared__ uint64_t all_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int ut = blockIdx.x, nt = blockIdx.y, ks = blockIdx.z;
  const int u0 = ut * TC_M, n0 = nt * TC_NT;
  const int ntile = min(TC_NT, a.Npad - n0);                  // multiple of 16
  const int kb0 = (int)((long long)ks * a.kblocks / a.ksplit);
  const int kb1 = (int)((long long)(ks + 1) * a.kblocks / a.ksplit);
  const int nkb = kb1 - kb0;

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) mbar_init(&mma_done[s], 1);
    mbar_init(&all_done, 1);
  }
  fence_mbar_init();
  if (warp == 0) {                                            // TMEM: 128 lanes x 128 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&tmem_base)), "n"(TC_NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  // this thread's unique id row for the A loads (row u of the tile), validated
  const int my_u = u0 + tid;
  int my_id = -1;
  if (my_u < a.U) {
    my_id = a.uniq[my_u];
    if (my_id < 0 || my_id >= a.V) { atomicOr(a.err, ERR_ID_RANGE); my_id = -1; }
  }
  auto load_stage = [&](int i) {                              // K-block kb0 + i -> slot i % S
    uint8_t *st = ring + (size_t)(i % TC_STAGES) * TC_STAGE;
    const int k0 = (kb0 + i) * TC_BK;
    // A: thread t copies row t (8 chunks of 16 B), swizzled
    {
      const __nv_bfloat16 *src = a.head + (size_t)(my_id < 0 ? 0 : my_id) * a.d + k0;
      uint8_t *dst = st + (size_t)tid * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        cp_async16(dst + ((c ^ (tid & 7)) << 4), src + c * 8, my_id >= 0);
    }
    // B: the three parts, rows n0 .. n0 + ntile
    for (int p = 0; p < TC_PARTS; ++p) {
      uint8_t *bt = st + TC_TILE_A + (size_t)p * TC_TILE_B;
      const __nv_bfloat16 *pb = a.parts + (size_t)p * a.Npad * a.d;
      for (int q = tid; q < ntile * 8; q += TC_THREADS) {
        const int n = q >> 3, c = q & 7;
        cp_async16(bt + (size_t)n * 128 + ((c ^ (n & 7)) << 4),
                   pb + (size_t)(n0 + n) * a.d + k0 + c * 8, true);
      }
    }
    cp_async_commit();
  };

  const uint32_t idesc = umma_idesc_bf16(TC_M, ntile);
  // prologue: fill the ring
  for (int i = 0; i < TC_STAGES - 1; ++i) {
    if (i < nkb) load_stage(i); else cp_async_commit();
  }
  for (int i = 0; i < nkb; ++i) {
    // refill: K-block i + S - 1 into the slot K-block i - 1 used (its MMAs done)
    const int nxt = i + TC_STAGES - 1;
    if (nxt < nkb) {
      if (i >= 1) mbar_wait(&mma_done[(i - 1) % TC_STAGES], ((i - 1) / TC_STAGES) & 1);
      load_stage(nxt);
    } else {
      cp_async_commit();
    }
    cp_async_wait<TC_STAGES - 1>();                           // K-block i has landed (this thread)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
    __syncthreads();                                          // ... for every thread
    if (tid == 0) {
      tc_fence_after();
      uint8_t *st = ring + (size_t)(i % TC_STAGES) * TC_STAGE;
      const uint32_t sa = smem_u32(st);
#pragma unroll
      for (int k = 0; k < TC_BK / 16; ++k) {
        const uint64_t ad = umma_desc_sw128(sa + k * 32);
#pragma unroll
        for (int p = 0; p < TC_PARTS; ++p) {
          const uint64_t bd = umma_desc_sw128(sa + (uint32_t)(TC_TILE_A + p * TC_TILE_B) + k * 32);
          umma_bf16(tmem, ad, bd, idesc, (i > 0 || k > 0 || p > 0) ? 1u : 0u);
        }
      }
      umma_commit(&mma_done[i % TC_STAGES]);                  // frees the slot when done
      if (i == nkb - 1) umma_commit(&all_done);
    }
  }
  // ---- epilogue: TMEM -> registers -> this split's dense partial tile
  // partial[ks][u][n] (thread = TMEM lane = unique id row u, 32 columns per
  // tcgen05.ld); the requested pairs are gathered by tree_tc_gather_kernel
  float *dst = a.partial + ((size_t)ks * a.Upad + u0 + tid) * a.Npad + n0;
  if (nkb > 0) {
    mbar_wait(&all_done, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < ntile; c0 += 32) {
      uint32_t v[32];
      const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (c0 + 32 <= ntile) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          __stcg(reinterpret_cast<float4 *>(dst + c0 + j),
                 make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                             __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < ntile) dst[c0 + j] = __uint_as_float(v[j]);
      }
    }
  } else {
    for (int j = 0; j < ntile; ++j) dst[j] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_NT));
}

// The requested pairs from the dense partial tiles: logit = r_n * (sum of the
// K-split partials in split order) + bw_u.  One thread per pair, all SMs.
__global__ void tree_tc_gather_kernel(TreeTcArgs a) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.P; q += gridDim.x * blockDim.x) {
    const int u = a.pair_uid[q], n = a.pair_node[q];
    const int id = a.uniq[u];
    if (id < 0 || id >= a.V) continue;                      // flagged by the GEMM kernel
    const float *pp = a.partial + (size_t)u * a.Npad + n;
    float s = 0.f;
    for (int k = 0; k < a.ksplit; ++k) s = __fadd_rn(s, __ldcg(pp + (size_t)k * a.Upad * a.Npad));
    a.logits[a.pair_out[q]] = __fadd_rn(__fmul_rn(a.r[n], s), a.head_bw ? a.head_bw[id] : 0.f);
  }
}

}  // namespace spx

using namespace spx;

static int tc_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int tc_ksplit(int64_t U, int64_t N, int64_t d) {
  const int tiles = (int)(((U + TC_M - 1) / TC_M) * ((N + TC_NT - 1) / TC_NT));
  const int kblocks = (int)(d / TC_BK);
  // split K over CTAs to cover the SMs, but keep >= 8 K-blocks per CTA and
  // <= 8 splits (the last CTA of a tile sums the partials)
  int ks = tc_sms() / (tiles > 0 ? tiles : 1);
  ks = ks < 1 ? 1 : ks > 8 ? 8 : ks;
  while (ks > 1 && kblocks / ks < 8) --ks;
  return ks;
}

extern "C" int64_t spx_tree_tc_scratch_bytes(int64_t N, int64_t d, int64_t U, int64_t P) {
  if (N < 0 || d <= 0 || U < 0 || P < 0) return -1;
  const int64_t Npad = (N + 15) / 16 * 16, Upad = (U + TC_M - 1) / TC_M * TC_M;
  const int64_t ks = tc_ksplit(U, Npad, d);
  return ((int64_t)TC_PARTS * Npad * d * 2 + 255) / 256 * 256 + ks * Upad * Npad * 4;
}

extern "C" int spx_tree_merged_logits_tc(const float *xg, const float *r, int64_t N,
                                         const void *head, int32_t head_dtype,
                                         const float *head_bw, int64_t V, int64_t d,
                                         const int32_t *uniq, int64_t U, const int32_t *uniq_ptr,
                                         const int32_t *pair_node, const int32_t *pair_out,
                                         const int32_t *pair_uid, int64_t P, float *logits,
                                         void *scratch, int32_t *err, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!xg || !r || !head || !uniq || !uniq_ptr || !pair_node || !pair_out || !pair_uid ||
      !logits || !err || !scratch || N < 0 || U < 0 || P < 0 || V <= 0 || head_dtype != SPX_DTYPE_BF16 ||
      d <= 0 || d % TC_BK)
    return SPX_EINVAL;
  if (U == 0 || N == 0 || P == 0) return 0;
  const int64_t Npad = (N + 15) / 16 * 16;
  const int ks = tc_ksplit(U, Npad, d);
  TreeTcArgs a{};
  uint8_t *sp = reinterpret_cast<uint8_t *>(scratch);
  a.parts = reinterpret_cast<const __nv_bfloat16 *>(sp);
  sp += ((int64_t)TC_PARTS * Npad * d * 2 + 255) / 256 * 256;
  a.partial = reinterpret_cast<float *>(sp);
  a.Upad = (int)((U + TC_M - 1) / TC_M * TC_M);
  a.Npad = (int)Npad; a.r = r; a.N = (int)N;
  a.head = reinterpret_cast<const __nv_bfloat16 *>(head); a.head_bw = head_bw;
  a.V = (int)V; a.d = (int)d; a.uniq = uniq; a.U = (int)U;
  a.uniq_ptr = uniq_ptr; a.pair_node = pair_node; a.pair_out = pair_out; a.pair_uid = pair_uid;
  a.logits = logits; a.P = (int)P; a.ksplit = ks; a.kblocks = (int)(d / TC_BK); a.err = err;
  const int sgrid = (int)((Npad * d + 255) / 256 < 4096 ? (Npad * d + 255) / 256 : 4096);
  tree_tc_split_kernel<<<sgrid, 256, 0, stream>>>(xg, (int)N, (int)Npad, (int)d,
                                                  const_cast<__nv_bfloat16 *>(a.parts));
  const size_t smem = (size_t)TC_STAGES * TC_STAGE + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tree_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  dim3 grid((unsigned)((U + TC_M - 1) / TC_M), (unsigned)((Npad + TC_NT - 1) / TC_NT),
            (unsigned)ks);
  tree_tc_kernel<<<grid, TC_THREADS, smem, stream>>>(a);
  const int gg = (int)((P + 255) / 256 < 4 * tc_sms() ? (P + 255) / 256 : 4 * tc_sms());
  tree_tc_gather_kernel<<<gg, 256, 0, stream>>>(a);
  return spx_launch_status("spx_tree_merged_logits_tc");
}
