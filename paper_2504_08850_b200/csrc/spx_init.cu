// Synthetic-weight generation on device: the reference's seeded init
// (rng.py:14-32, model.py:121-137) evaluated element-parallel in HBM, so the
// Llama2-7B-shaped random-init model (6.7 B params) is produced in seconds
// instead of minutes of numpy, with bit-identical values.
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/specexit_b200.h"
#include "spx_common.cuh"

namespace spx {

// splitmix64 output i (1-based) of stream `seed` (rng.py:14-21).
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// rng.py:24-27: f32( low + (high-low) * (f64(z>>11) * 2^-53) ), no contraction.
__device__ __forceinline__ float uniform_at(uint64_t seed, uint64_t i, double low, double span) {
  const double u = __dmul_rn((double)(splitmix64_at(seed, i) >> 11), 0x1p-53);
  return __double2float_rn(__dadd_rn(low, __dmul_rn(span, u)));
}

__global__ void init_uniform_kernel(void *out, int f32, int64_t rows, int64_t cols, int transpose,
                                    uint64_t seed, double low, double span) {
  const int64_t n = rows * cols;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    // o indexes the OUTPUT layout; i is the element's index in the
    // reference's row-major (rows, cols) order.
    int64_t i = o;
    if (transpose) {
      const int64_t c = o / rows, r = o - c * rows;
      i = r * cols + c;
    }
    const float v = uniform_at(seed, (uint64_t)i + 1ull, low, span);
    if (f32) reinterpret_cast<float *>(out)[o] = v;
    else reinterpret_cast<__nv_bfloat16 *>(out)[o] = __float2bfloat16_rn(v);
  }
}

}  // namespace spx

extern "C" int spx_init_uniform(void *out, int32_t out_f32, int64_t rows, int64_t cols,
                                int32_t transpose, uint64_t seed, double low, double high,
                                void *stream) {
  if (!out || rows < 0 || cols < 0) return SPX_EINVAL;
  if (rows * cols == 0) return 0;
  const double span = high - low;   // Python float arithmetic in the reference
  spx::init_uniform_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      out, out_f32, rows, cols, transpose, seed, low, span);
  return spx_launch_status("spx_init_uniform");
}

extern "C" const char *spx_version(void) {
  return "libspecexit_b200 0.1 (sm_100a; K1-K7 predictor path)";
}
