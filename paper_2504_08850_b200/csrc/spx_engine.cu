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

// Stable top-K (value desc, index asc) of n logits (speculation.py:57-60
// topk_from_logits: np.argsort(-x, kind="stable")[:K]).  One CTA of 1024
// threads: each thread keeps the best TK keys of its strided share in
// registers (fully unrolled insertion, no local memory); K rounds of a block
// argmax pop the winner from its owner's list.  An owner whose list runs dry
// rescans its share for the best keys below the last one it gave up (keys are
// unique, so "below" is exact).  Keys: order-preserving value bits << 32 |
// ~index, i.e. ties go to the lower index (np.argmax / stable argsort).
constexpr int TOPK_THREADS = 1024;
constexpr int TK = 4;

__device__ __forceinline__ void topk_insert(unsigned long long (&l)[TK], unsigned long long k) {
#pragma unroll
  for (int q = 0; q < TK; ++q) {
    const bool sw = k > l[q];
    const unsigned long long t = l[q];
    l[q] = sw ? k : t;
    k = sw ? t : k;
  }
}

__global__ void __launch_bounds__(TOPK_THREADS) topk_kernel(const float *logits, int n, int K,
                                                           int32_t *ids_out) {
  // one CTA per row (gridDim.x rows of n logits, K ids each)
  logits += (size_t)blockIdx.x * n;
  ids_out += (size_t)blockIdx.x * K;
  __shared__ unsigned long long s_red[TOPK_THREADS / 32];
  __shared__ unsigned long long s_win;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned long long l[TK];
  auto scan = [&](unsigned long long below) {
#pragma unroll
    for (int q = 0; q < TK; ++q) l[q] = 0ull;
    for (int i = tid; i < n; i += TOPK_THREADS) {
      const unsigned long long k = argmax_key(logits[i], (uint32_t)i);
      if (k < below) topk_insert(l, k);
    }
  };
  scan(~0ull);
  int taken = 0;
  for (int r = 0; r < K; ++r) {
    unsigned long long m = l[0];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    if (lane == 0) s_red[wid] = m;
    __syncthreads();
    if (wid == 0) {
      m = s_red[lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
        m = v > m ? v : m;
      }
      if (lane == 0) {
        s_win = m;
        ids_out[r] = (int32_t)(0xffffffffu - (uint32_t)(m & 0xffffffffull));
      }
    }
    __syncthreads();
    const unsigned long long win = s_win;
    if (l[0] == win && win != 0ull) {              // the owner pops its head
#pragma unroll
      for (int q = 0; q + 1 < TK; ++q) l[q] = l[q + 1];
      l[TK - 1] = 0ull;
      if (++taken % TK == 0) scan(win);            // list dry: next keys below
    }
  }
}

// Per-token reset (engine.py:183-191): prev = uniform(K) as f32, flags clear.
__global__ void token_begin_kernel(spx_token_state st, int K, int L, float inv_k) {
  const int t = threadIdx.x;
  if (t < K) st.prev[t] = inv_k;                       // np.float32(1.0 / k), host-rounded
  if (t == 0) {
    if (st.prev_err) *st.prev_err = 0.f;                // the uniform prior is exact
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

// Injected-spec hook (on the reference's _speculative_set,
// engine.py:162-168): at a flagged step the target's final argmax -- the
// forced token of generate_forced -- replaces the last draft id unless it is
// already among the K ids.  One thread.
__global__ void inject_spec_kernel(int32_t *spec, int K, const int32_t *forced,
                                   const int32_t *step, const uint8_t *flags, int n) {
  if (threadIdx.x != 0) return;
  const int s = *step;
  if (s < 0 || s >= n || !flags[s]) return;
  const int tok = forced[s];
  for (int k = 0; k < K; ++k)
    if (spec[k] == tok) return;
  spec[K - 1] = tok;
}

}  // namespace spx

using namespace spx;

extern "C" int spx_inject_spec(int32_t *spec_ids, int32_t K, const int32_t *forced,
                               const int32_t *step, const uint8_t *flags, int64_t n,
                               void *stream) {
  if (!spec_ids || !forced || !step || !flags || K < 1 || K > 64 || n < 0) return SPX_EINVAL;
  inject_spec_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(spec_ids, K, forced, step, flags, (int)n);
  return spx_launch_status("spx_inject_spec");
}

extern "C" int spx_topk(const float *logits, int64_t n, int32_t K, int32_t *ids_out,
                        void *stream) {
  if (!logits || !ids_out || n <= 0 || K < 1 || K > 64 || K > n) return SPX_EINVAL;
  topk_kernel<<<1, TOPK_THREADS, 0, (cudaStream_t)stream>>>(logits, (int)n, K, ids_out);
  return spx_launch_status("spx_topk");
}

extern "C" int spx_topk_rows(const float *logits, int64_t rows, int64_t n, int32_t K,
                             int32_t *ids_out, void *stream) {
  if (!logits || !ids_out || rows < 0 || n <= 0 || K < 1 || K > 64 || K > n) return SPX_EINVAL;
  if (rows == 0) return 0;
  topk_kernel<<<(unsigned)rows, TOPK_THREADS, 0, (cudaStream_t)stream>>>(logits, (int)n, K,
                                                                         ids_out);
  return spx_launch_status("spx_topk_rows");
}

extern "C" int spx_token_begin(spx_token_state st, int32_t K, int32_t L, float inv_k,
                               void *stream) {
  if (!st.prev || !st.done || K < 1 || K > 64) return SPX_EINVAL;
  token_begin_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(st, K, L, inv_k);
  return spx_launch_status("spx_token_begin");
}

extern "C" int spx_token_end(spx_token_state st, spx_online_state os, int32_t L,
                             int32_t queue_len, int32_t radius, int64_t max_steps,
                             void *stream) {
  if (!st.step || !st.next_in || L < 1 || L > 64 || queue_len < 1 || radius < 0)
    return SPX_EINVAL;
  token_end_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(st, os, L, queue_len, radius,
                                                       (int)max_steps);
  return spx_launch_status("spx_token_end");
}

extern "C" int spx_force_next(const int32_t *forced, const int32_t *step, int32_t *next_in,
                              int64_t n_forced, void *stream) {
  if (!forced || !step || !next_in || n_forced < 0) return SPX_EINVAL;
  force_next_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(forced, step, next_in, (int)n_forced);
  return spx_launch_status("spx_force_next");
}

extern "C" int spx_or_flag(const uint8_t *src, uint8_t *dst, void *stream) {
  if (!src || !dst) return SPX_EINVAL;
  or_flag_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(src, dst);
  return spx_launch_status("spx_or_flag");
}
