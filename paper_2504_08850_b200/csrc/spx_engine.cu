// Per-token control kernels of the device-resident early-exit engine.
//
// Reference: ExitEngine.step (engine.py:176-217) and speculative_set_from_logits
// / topk_from_logits (speculation.py:57-84).  The whole token step (draft,
// schedule, L flag-guarded layers, predictor + verify per scheduled layer,
// final argmax, online update, trace record) is enqueued on one stream with
// device-resident state, so it is captured once into a CUDA graph and
// replayed per token with no host synchronisation.
#include "spx_common.cuh"
#include "../../include/specexit_b200.h"

namespace spx {

// Stable top-K (value desc, index asc) of n logits; one CTA.
__global__ void topk_kernel(const float *logits, int n, int K, int32_t *ids_out) {
  extern __shared__ unsigned long long keys[];      // blockDim.x * K
  const int tid = threadIdx.x;
  unsigned long long best[64];
  for (int q = 0; q < 64; ++q) best[q] = 0ull;
  for (int i = tid; i < n; i += blockDim.x) {
    unsigned long long k = argmax_key(logits[i], (uint32_t)i);
    // insert into the descending list
    for (int q = 0; q < K; ++q) {
      if (k > best[q]) { const unsigned long long t = best[q]; best[q] = k; k = t; }
    }
  }
  for (int q = 0; q < K; ++q) keys[(size_t)tid * K + q] = best[q];
  __syncthreads();
  // tree merge of sorted lists
  for (int stride = 1; stride < (int)blockDim.x; stride <<= 1) {
    if ((tid % (2 * stride)) == 0 && tid + stride < (int)blockDim.x) {
      unsigned long long *a = keys + (size_t)tid * K, *b = keys + (size_t)(tid + stride) * K;
      unsigned long long m[64];
      int i = 0, j = 0;
      for (int q = 0; q < K; ++q) m[q] = (a[i] >= b[j]) ? a[i++] : b[j++];
      for (int q = 0; q < K; ++q) a[q] = m[q];
    }
    __syncthreads();
  }
  if (tid < K) ids_out[tid] = (int32_t)(0xffffffffu - (uint32_t)(keys[tid] & 0xffffffffull));
}

// Per-token reset (engine.py:183-191): prev = uniform(K) as f32, flags clear.
__global__ void token_begin_kernel(spx_token_state st, int K, int L, float inv_k) {
  const int t = threadIdx.x;
  if (t < K) st.prev[t] = inv_k;                       // np.float32(1.0 / k), host-rounded
  if (t == 0) {
    *st.done = 0; *st.fired = 0; *st.fired_any = 0;
    *st.exit_layer = L - 1; *st.evals = 0; *st.full_heads = 0;
  }
}

// Token end (engine.py:208-217): choose the token, record, push the exit
// layer into the online window (scheduler.py:65-79), set next_in.
__global__ void token_end_kernel(spx_token_state st, spx_online_state os, int L, int qlen,
                                 int radius, int max_steps) {
  if (threadIdx.x != 0) return;
  const bool verified = *st.done != 0;
  const int token = verified ? *st.exit_token : *st.final_token;
  const int el = verified ? *st.exit_layer : L - 1;
  const int step = *st.step;
  if (step < max_steps) {
    st.rec_token[step] = token;
    st.rec_exit_layer[step] = el;
    st.rec_fired[step] = *st.fired_any;
    st.rec_verified[step] = verified ? 1 : 0;
    st.rec_evals[step] = *st.evals;
    st.rec_full_heads[step] = *st.full_heads;
    st.rec_active[step] = *st.active;
  }
  *st.next_in = token;
  *st.step = step + 1;
  // update_online for this stream (row 0)
  int head = os.head[0], len = os.len[0];
  int32_t *counts = os.counts;
  if (len == qlen) {
    const int ev = os.queue[head];
    for (int i = (ev - radius > 0 ? ev - radius : 0); i <= (ev + radius < L - 1 ? ev + radius : L - 1); ++i)
      counts[i] -= 1;
    head = (head + 1) % qlen;
    --len;
  }
  os.queue[(head + len) % qlen] = el;
  ++len;
  for (int i = (el - radius > 0 ? el - radius : 0); i <= (el + radius < L - 1 ? el + radius : L - 1); ++i)
    counts[i] += 1;
  os.head[0] = head;
  os.len[0] = len;
}

// fired_any |= fired (per scheduled layer, after the predictor launch)
__global__ void or_flag_kernel(const uint8_t *src, uint8_t *dst) {
  if (threadIdx.x == 0 && *src) *dst = 1;
}

// generate_forced (engine.py:227-246): next_in = forced[step - 1]
__global__ void force_next_kernel(const int32_t *forced, const int32_t *step, int32_t *next_in,
                                  int n_forced) {
  if (threadIdx.x != 0) return;
  const int s = *step - 1;
  if (s >= 0 && s < n_forced) *next_in = forced[s];
}

}  // namespace spx

using namespace spx;

extern "C" int spx_topk(const float *logits, int64_t n, int32_t K, int32_t *ids_out,
                        void *stream) {
  if (!logits || !ids_out || n <= 0 || K < 1 || K > 64 || K > n) return SPX_EINVAL;
  const int threads = 256;
  topk_kernel<<<1, threads, (size_t)threads * K * 8, (cudaStream_t)stream>>>(logits, (int)n, K,
                                                                              ids_out);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}

extern "C" int spx_token_begin(spx_token_state st, int32_t K, int32_t L, float inv_k,
                               void *stream) {
  if (!st.prev || !st.done || K < 1 || K > 64) return SPX_EINVAL;
  token_begin_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(st, K, L, inv_k);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}

extern "C" int spx_token_end(spx_token_state st, spx_online_state os, int32_t L,
                             int32_t queue_len, int32_t radius, int64_t max_steps,
                             void *stream) {
  if (!st.step || !st.next_in || L < 1 || L > 64 || queue_len < 1 || radius < 0)
    return SPX_EINVAL;
  token_end_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(st, os, L, queue_len, radius,
                                                       (int)max_steps);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}

extern "C" int spx_force_next(const int32_t *forced, const int32_t *step, int32_t *next_in,
                              int64_t n_forced, void *stream) {
  if (!forced || !step || !next_in || n_forced < 0) return SPX_EINVAL;
  force_next_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(forced, step, next_in, (int)n_forced);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}

extern "C" int spx_or_flag(const uint8_t *src, uint8_t *dst, void *stream) {
  if (!src || !dst) return SPX_EINVAL;
  or_flag_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(src, dst);
  return cudaGetLastError() == cudaSuccess ? 0 : SPX_ECUDA;
}
