// Bandwidth probe for the predictor's access pattern (not product code):
// per eval one contiguous f32 hidden row (16 KB) + K random bf16 LM-head rows
// (8 KB each).  One producer thread per CTA streams whole evals into a ring of
// S slots with cp.async.bulk; 16 consumer warps reduce each slot (all warps on
// one slot) and release it.  Prints us/launch and GB/s for several S, B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(n), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n"
               ::"r"(smem_u32(b)), "r"(ph) : "memory");
}

constexpr int D = 4096, K = 4, NW = 16;
constexpr int SLOT = D * 4 + K * D * 2;   // 48 KB

template <int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
probe(const float *hidden, const __nv_bfloat16 *head, const int *ids, int B, float *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + S * SLOT);
  uint64_t *empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, NW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrows = B > (int)blockIdx.x ? (B - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == NW) {
    if (lane == 0) {
      for (int i = 0; i < nrows; ++i) {
        const int s = i % S, r = blockIdx.x + i * gridDim.x;
        if (i >= S) wait(empty + s, ((i / S) - 1) & 1);
        unsigned char *dst = sm + s * SLOT;
        expect_tx(full + s, SLOT);
        bulk(dst, hidden + (size_t)r * D, D * 4, full + s);
        for (int c = 0; c < K; ++c)
          bulk(dst + D * 4 + c * D * 2, head + (size_t)ids[r * K + c] * D, D * 2, full + s);
      }
    }
    return;
  }
  for (int i = 0; i < nrows; ++i) {
    const int s = i % S, r = blockIdx.x + i * gridDim.x;
    wait(full + s, (i / S) & 1);
    const float4 *h = reinterpret_cast<const float4 *>(sm + s * SLOT);
    const uint4 *w = reinterpret_cast<const uint4 *>(sm + s * SLOT + D * 4);
    float acc = 0.f;
    for (int j = threadIdx.x; j < D / 4; j += 32 * NW) { float4 v = h[j]; acc += v.x + v.y + v.z + v.w; }
    for (int j = threadIdx.x; j < K * D / 8; j += 32 * NW) {
      uint4 v = w[j];
      acc += __uint_as_float(v.x << 16) + __uint_as_float(v.y << 16) + __uint_as_float(v.z << 16) + __uint_as_float(v.w << 16);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __syncwarp();
    if (lane == 0) { arrive(empty + s); if (acc == 12345.f) out[r] = acc; }
  }
}

template <int S>
void run(const float *h, const __nv_bfloat16 *w, const int *ids, float *out, int B, int grid) {
  const size_t smem = S * SLOT + 2 * S * 8;
  cudaFuncSetAttribute(probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int L = 31;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 20; ++it)
    probe<S><<<grid, 32 * (NW + 1), smem>>>(h + (size_t)(it % L) * B * D, w, ids + (size_t)(it % L) * B * K, B, out);
  cudaEventRecord(a);
  const int N = 200;
  for (int it = 0; it < N; ++it)
    probe<S><<<grid, 32 * (NW + 1), smem>>>(h + (size_t)(it % L) * B * D, w, ids + (size_t)(it % L) * B * K, B, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1e3 / N, bytes = (double)B * SLOT;
  printf("S=%d B=%5d grid=%d: %7.2f us/launch  %7.1f GB/s  (err=%s)\n", S, B, grid, us, bytes / us / 1e3,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int V = 32000, L = 31, BMAX = 4096;
  float *h; __nv_bfloat16 *w; int *ids; float *out;
  cudaMalloc(&h, (size_t)L * BMAX * D * 4);
  cudaMalloc(&w, (size_t)V * D * 2);
  cudaMalloc(&ids, (size_t)L * BMAX * K * 4);
  cudaMalloc(&out, BMAX * 4);
  cudaMemset(h, 0, (size_t)L * BMAX * D * 4);
  cudaMemset(w, 0, (size_t)V * D * 2);
  std::vector<int> hid((size_t)L * BMAX * K);
  std::mt19937 g(1);
  for (auto &x : hid) x = g() % V;
  cudaMemcpy(ids, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice);
  for (int B : {148, 1024, 4096}) {
    run<2>(h, w, ids, out, B, 148);
    run<3>(h, w, ids, out, B, 148);
    run<4>(h, w, ids, out, B, 148);
  }
  return 0;
}
