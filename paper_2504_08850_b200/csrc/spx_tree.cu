// K6: context-aware merged mapping for token trees (sm_100a).
//
// Reference: grouped_speculative_logits (tree.py:92-113) -- per live tree
// node j, LN(h_j) . lm_head[:, ids_j].  The reference computes the FULL
// vocabulary per node and gathers (tree.py:111-113).  Here the feature ids of
// all live nodes are de-duplicated into U unique LM-head rows (the merged
// mapping of the paper, §6.2); one warp owns one unique row, holds it in
// registers (read from HBM exactly once), and dots it with every node that
// asked for it (normed node rows come from L2).  FAST: the canonical CDOT
// order, so every logit is bit-identical to the predictor kernel's sliced
// logit for the same (row, id) -- the reference's "grouped == sliced"
// contract (tests/test_tree.py:32-42).  STRICT: each (node, id) dot is the
// reference's sequential chain (kernels/_ckern.pyx:16-31), one lane per pair.
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"

namespace spx {

constexpr int TREE_THREADS = 128;

template <typename TW, int CPL>
__global__ void __launch_bounds__(TREE_THREADS)
tree_merged_kernel(const float *hn, const float *rr, int N, const TW *head, const float *bwv,
                   int V, int d, const int32_t *uniq, int U, const int32_t *uniq_ptr,
                   const int32_t *pair_node, const int32_t *pair_out, float *logits, int strict,
                   int *err) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * (TREE_THREADS / 32) + (threadIdx.x >> 5);
  if (u >= U) return;
  const int id = uniq[u];
  if (id < 0 || id >= V) {
    if (lane == 0) atomicOr(err, ERR_ID_RANGE);
    return;
  }
  const TW *wrow = head + (size_t)id * d;
  if (strict) {
    for (int q = uniq_ptr[u] + lane; q < uniq_ptr[u + 1]; q += 32) {
      const float *h = hn + (size_t)pair_node[q] * d;
      float acc = 0.f;
      for (int j = 0; j < d; j += CHUNK) {
        float w[4];
        load4_f32<TW>(wrow + j, w);
#pragma unroll
        for (int e = 0; e < CHUNK; ++e) acc = __fadd_rn(acc, __fmul_rn(h[j + e], w[e]));
      }
      logits[pair_out[q]] = acc;
    }
    return;
  }
  const int nchunk = d / CHUNK;
  Chunk<TW> w[4][CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s)
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int c = 32 * g + lane + NPART * s;
      if (c < nchunk) w[g][s].load(wrow + CHUNK * c);
      else w[g][s].zero();
    }
  const float bw = bwv ? bwv[id] : 0.f;
  for (int q = uniq_ptr[u]; q < uniq_ptr[u + 1]; ++q) {
    const float *h = hn + (size_t)pair_node[q] * d;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < CPL; ++s)
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int c = 32 * g + lane + NPART * s;
        if (c < nchunk) {
          const float4 h0 = __ldg(reinterpret_cast<const float4 *>(h + CHUNK * c));
          float wf[4];
          w[g][s].to_f32(wf);
          acc[g] = __fmaf_rn(h0.x, wf[0], acc[g]);
          acc[g] = __fmaf_rn(h0.y, wf[1], acc[g]);
          acc[g] = __fmaf_rn(h0.z, wf[2], acc[g]);
          acc[g] = __fmaf_rn(h0.w, wf[3], acc[g]);
        }
      }
    float gs[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) gs[g] = warp_butterfly_sum(acc[g]);
    const float lg = canon_combine(gs[0], gs[1], gs[2], gs[3]);
    if (lane == 0) logits[pair_out[q]] = __fadd_rn(__fmul_rn(rr[pair_node[q]], lg), bw);
  }
}

template <typename TW>
struct TreeLaunch {
  const float *hn, *rr; int N; const TW *head; const float *bw; int V, d;
  const int32_t *uniq; int U; const int32_t *uniq_ptr, *pair_node, *pair_out;
  float *logits; int strict; int *err; unsigned grid; cudaStream_t stream;
  template <int CPL> void operator()() const {
    tree_merged_kernel<TW, CPL><<<grid, TREE_THREADS, 0, stream>>>(
        hn, rr, N, head, bw, V, d, uniq, U, uniq_ptr, pair_node, pair_out, logits, strict, err);
  }
};

}  // namespace spx

using namespace spx;

extern "C" int spx_tree_merged_logits(const float *xg, const float *r, int64_t N, const void *head,
                                      int32_t head_dtype, const float *head_bw, int64_t V,
                                      int64_t d, const int32_t *uniq, int64_t U,
                                      const int32_t *uniq_ptr, const int32_t *pair_node,
                                      const int32_t *pair_out, float *logits, int32_t mode,
                                      int32_t *err, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!xg || !r || !head || !uniq || !uniq_ptr || !pair_node || !pair_out || !logits || !err ||
      N < 0 || U < 0 || d <= 0 || d % CHUNK || V <= 0)
    return SPX_EINVAL;
  if (U == 0) return 0;
  const int wpc = TREE_THREADS / 32;
  const unsigned grid = (unsigned)((U + wpc - 1) / wpc);
  const int strict = mode == SPX_MODE_STRICT;
  bool ok;
  if (head_dtype == SPX_DTYPE_F32)
    ok = dispatch_cpl((int)d, TreeLaunch<float>{xg, r, (int)N, (const float *)head, head_bw,
                                                (int)V, (int)d, uniq, (int)U, uniq_ptr, pair_node,
                                                pair_out, logits, strict, err, grid, stream});
  else if (head_dtype == SPX_DTYPE_BF16)
    ok = dispatch_cpl((int)d, TreeLaunch<__nv_bfloat16>{
                                  xg, r, (int)N, (const __nv_bfloat16 *)head, head_bw, (int)V,
                                  (int)d, uniq, (int)U, uniq_ptr, pair_node, pair_out, logits,
                                  strict, err, grid, stream});
  else
    return SPX_EINVAL;
  if (!ok) return SPX_EINVAL;
  return spx_launch_status("spx_tree_merged_logits");
}
