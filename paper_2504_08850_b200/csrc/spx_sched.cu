// K5: two-level predictor scheduler on device, and K7: hyper-token
// conjunction.  Integer-only -- exact by construction.
//
// Reference: scheduler.py:49-102 (OnlineState, _neighborhood, update_online,
// online_hot_layers, active_layers), engine.py:170-174 ("all" mode) and
// tree.py:116-122 / :389-390 (per-path AND of node decisions).
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"

namespace spx {

// scheduler.py:61-62  range(max(e-r,0), min(e+r, L-1)+1)
__device__ __forceinline__ void neighborhood_add(int32_t *counts, int e, int L, int r, int delta) {
  const int lo = e - r > 0 ? e - r : 0;
  const int hi = e + r < L - 1 ? e + r : L - 1;
  for (int i = lo; i <= hi; ++i) counts[i] += delta;
}

__global__ void sched_update_kernel(spx_online_state st, const int32_t *exit_layer,
                                    const uint8_t *gate, int B, int L, int qlen, int radius,
                                    int *err) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B || (gate && !gate[r])) return;
  const int e = exit_layer[r];
  if (e < 0 || e >= L) { atomicOr(err, ERR_BAD_LAYER); return; }   // scheduler.py:69-70
  int32_t *q = st.queue + (size_t)r * qlen;
  int32_t *counts = st.counts + (size_t)r * L;
  int head = st.head[r], len = st.len[r];
  if (len == qlen) {                              // evict the oldest (:72-75)
    neighborhood_add(counts, q[head], L, radius, -1);
    head = (head + 1) % qlen;
    --len;
  }
  q[(head + len) % qlen] = e;                     // push (:76-78)
  ++len;
  neighborhood_add(counts, e, L, radius, +1);
  st.head[r] = head;
  st.len[r] = len;
}

__global__ void sched_active_kernel(spx_online_state st, uint64_t offline_mask, int B, int L,
                                    int mode, uint64_t *out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const uint64_t capable = (L - 1 >= 64) ? ~0ull : ((1ull << (L - 1)) - 1ull);   // 0..L-2
  if (mode == 0) { out[r] = capable; return; }
  uint64_t m = offline_mask;
  const int32_t *counts = st.counts + (size_t)r * L;
  for (int i = 0; i < L - 1; ++i)
    if (counts[i] > 0) m |= (1ull << i);
  out[r] = m & capable;
}

__global__ void path_and_kernel(const uint8_t *node_fired, const int32_t *path_ptr,
                                const int32_t *path_nodes, const uint8_t *live, int P,
                                uint8_t *path_fire) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  if (live && !live[p]) { path_fire[p] = 0; return; }
  bool all = path_ptr[p + 1] > path_ptr[p];
  for (int i = path_ptr[p]; i < path_ptr[p + 1]; ++i) all &= node_fired[path_nodes[i]] != 0;
  path_fire[p] = all ? 1 : 0;
}

}  // namespace spx

using namespace spx;

extern "C" int spx_sched_update(spx_online_state st, const int32_t *exit_layer,
                                const uint8_t *gate, int64_t B, int32_t L, int32_t queue_len,
                                int32_t radius, int32_t *err, void *stream) {
  if (B < 0 || L < 1 || L > 64 || queue_len < 1 || radius < 0 || !exit_layer || !err ||
      !st.queue || !st.head || !st.len || !st.counts)
    return SPX_EINVAL;
  if (B == 0) return 0;
  sched_update_kernel<<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      st, exit_layer, gate, (int)B, L, queue_len, radius, err);
  return spx_launch_status("spx_sched_update");
}

extern "C" int spx_sched_active(spx_online_state st, uint64_t offline_mask, int64_t B, int32_t L,
                                int32_t mode, uint64_t *active_out, void *stream) {
  if (B < 0 || L < 1 || L > 64 || !active_out || (mode != 0 && !st.counts)) return SPX_EINVAL;
  if (B == 0) return 0;
  sched_active_kernel<<<(unsigned)((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      st, offline_mask, (int)B, L, mode, active_out);
  return spx_launch_status("spx_sched_active");
}

extern "C" int spx_path_and(const uint8_t *node_fired, const int32_t *path_ptr,
                            const int32_t *path_nodes, const uint8_t *live, int64_t P,
                            uint8_t *path_fire, void *stream) {
  if (P < 0 || !node_fired || !path_ptr || !path_nodes || !path_fire) return SPX_EINVAL;
  if (P == 0) return 0;
  path_and_kernel<<<(unsigned)((P + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      node_fired, path_ptr, path_nodes, live, (int)P, path_fire);
  return spx_launch_status("spx_path_and");
}

// K7b: which rows need the full-head check after the path AND
// (tree.py:221-227): every node on a firing live path, plus the root (its
// argmax opens every path's chain) when any path fires.  One CTA; the
// all-or-nothing writes of 1 race benignly.
namespace spx {
__global__ void tree_gate_kernel(const uint8_t *path_fire, const int32_t *path_ptr,
                                 const int32_t *path_nodes, int P, int n_nodes,
                                 uint8_t *node_gate) {
  for (int j = threadIdx.x; j < n_nodes; j += blockDim.x) node_gate[j] = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    if (!path_fire[p]) continue;
    node_gate[0] = 1;
    for (int q = path_ptr[p]; q < path_ptr[p + 1]; ++q) node_gate[path_nodes[q]] = 1;
  }
}
}  // namespace spx

extern "C" int spx_tree_gate(const uint8_t *path_fire, const int32_t *path_ptr,
                             const int32_t *path_nodes, int64_t P, int64_t n_nodes,
                             uint8_t *node_gate, void *stream) {
  if (!path_fire || !path_ptr || !path_nodes || !node_gate || P < 0 || n_nodes < 1)
    return SPX_EINVAL;
  spx::tree_gate_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(path_fire, path_ptr, path_nodes,
                                                             (int)P, (int)n_nodes, node_gate);
  return spx_launch_status("spx_tree_gate");
}

// Elementwise numpy-float32 exp (the softmax's exp, model.py:151), exposed so
// the tests can compare the device restatement with the host's np.exp over
// large input sweeps.
namespace spx {
__global__ void np_expf_kernel(const float *x, float *y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = np_expf(x[i]);
}
}  // namespace spx

extern "C" int spx_np_expf(const float *x, float *y, int64_t n, void *stream) {
  if (!x || !y || n < 0) return SPX_EINVAL;
  if (n == 0) return 0;
  spx::np_expf_kernel<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(x, y, n);
  return spx_launch_status("spx_np_expf");
}
