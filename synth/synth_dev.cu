// synth/synth_dev.cu — device twin of synth/synth.c (same counter-based generator), so
// multi-GiB benchmark inputs are generated in HBM instead of over PCIe.  Test/bench
// infrastructure only; holds none of the Kron-Matmul arithmetic.  The sub-block variant
// (`synth_fill_block_dev_*`) generates X[r0:r0+rows, c0:c0+cols] of a matrix with `ld`
// columns, which is how each distributed rank builds its own block of X.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double value(uint64_t key, uint64_t idx, int mode) {
  uint64_t h = splitmix64(key ^ idx);
  switch (mode) {
    case 0: return (double)(h >> 40) * (1.0 / 16777216.0);
    case 1: return 2.0 * ((double)(h >> 40) * (1.0 / 16777216.0)) - 1.0;
    case 2: return (double)(int)(h % 5u) - 2.0;
    case 3: return (double)(int)(h % 3u) - 1.0;
    default: return 0.0;
  }
}
uint64_t host_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
template <typename T>
__global__ void fill_block(T *out, int64_t rows, int64_t cols, int64_t r0, int64_t c0, int64_t ld,
                           uint64_t key, int mode) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i % cols;
    out[i] = (T)value(key, (uint64_t)((r0 + r) * ld + (c0 + c)), mode);
  }
}
template <typename T>
int launch(T *out, int64_t rows, int64_t cols, int64_t r0, int64_t c0, int64_t ld, uint64_t seed,
           uint64_t tensor_id, int mode, cudaStream_t s) {
  if (!out || rows < 0 || cols < 0 || mode < 0 || mode > 3) return 1;
  if (rows * cols == 0) return 0;
  uint64_t key = host_splitmix64(seed) ^ (tensor_id << 56);
  int64_t blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  fill_block<T><<<(unsigned)blocks, 256, 0, s>>>(out, rows, cols, r0, c0, ld, key, mode);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
}  // namespace

extern "C" {
int synth_fill_block_dev_f32(float *out, int64_t rows, int64_t cols, int64_t r0, int64_t c0, int64_t ld,
                             uint64_t seed, uint64_t tensor_id, int mode, void *stream) {
  return launch<float>(out, rows, cols, r0, c0, ld, seed, tensor_id, mode, (cudaStream_t)stream);
}
int synth_fill_block_dev_f64(double *out, int64_t rows, int64_t cols, int64_t r0, int64_t c0, int64_t ld,
                             uint64_t seed, uint64_t tensor_id, int mode, void *stream) {
  return launch<double>(out, rows, cols, r0, c0, ld, seed, tensor_id, mode, (cudaStream_t)stream);
}
}
