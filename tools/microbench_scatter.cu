// Write-pattern microbenchmark for the fused chunk kernels' direct-index store: each CTA stages a
// contiguous tile of R chunks x C values of one row in shared memory (coalesced loads), then writes
// value (g, u) to Y[row][u*WC + g0 + g] (runs of R*4 bytes at stride WC*4 bytes, WC = W/C), lanes
// along g.  Compared with a plain contiguous copy.  Prints GB/s (read + write).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_scatter tools/microbench_scatter.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void scatter(const float *__restrict__ X, float *__restrict__ Y, long M, long W, int C, int R) {
  extern __shared__ float tile[];
  const long WC = W / C, tpr = W / ((long)R * C), tiles = M * tpr;
  for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long row = t / tpr, cb = t - row * tpr;
    const float4 *src = reinterpret_cast<const float4 *>(X + row * W + cb * (long)R * C);
    __syncthreads();
    for (int i = threadIdx.x; i < R * C / 4; i += blockDim.x) reinterpret_cast<float4 *>(tile)[i] = src[i];
    __syncthreads();
    float *dst = Y + row * W + cb * R;
    for (int i = threadIdx.x; i < R * C; i += blockDim.x) {
      const int g = i % R, u = i / R;
      dst[(long)u * WC + g] = tile[g * C + (u ^ (g & 31))];  // xor: spread banks (values irrelevant)
    }
  }
}

// same pattern with 16-byte stores: lane = 4 consecutive chunks of one u
__global__ void scatter4(const float *__restrict__ X, float *__restrict__ Y, long M, long W, int C, int R) {
  extern __shared__ float tile[];
  const long WC = W / C, tpr = W / ((long)R * C), tiles = M * tpr;
  for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long row = t / tpr, cb = t - row * tpr;
    const float4 *src = reinterpret_cast<const float4 *>(X + row * W + cb * (long)R * C);
    __syncthreads();
    for (int i = threadIdx.x; i < R * C / 4; i += blockDim.x) reinterpret_cast<float4 *>(tile)[i] = src[i];
    __syncthreads();
    float *dst = Y + row * W + cb * R;
    for (int i = threadIdx.x; i < R * C / 4; i += blockDim.x) {
      const int g4 = i % (R / 4), u = i / (R / 4);
      float4 v;
      v.x = tile[(4 * g4) * C + u];
      v.y = tile[(4 * g4 + 1) * C + u];
      v.z = tile[(4 * g4 + 2) * C + u];
      v.w = tile[(4 * g4 + 3) * C + u];
      *reinterpret_cast<float4 *>(dst + (long)u * WC + 4 * g4) = v;
    }
  }
}

__global__ void copy(const float4 *__restrict__ X, float4 *__restrict__ Y, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) Y[i] = X[i];
}

int main() {
  const long W = 1L << 20, M = 1024;  // 4 GB per matrix
  const long n = W * M;
  float *X, *Y;
  cudaMalloc(&X, n * 4);
  cudaMalloc(&Y, n * 4);
  cudaMemset(X, 0, n * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    copy<<<148 * 8, 256>>>((const float4 *)X, (float4 *)Y, n / 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("{\"kind\": \"copy\", \"GBps\": %.1f}\n", 2.0 * n * 4 / ms / 1e6);
  struct Cfg { int C, R; } cfgs[] = {{1024, 8}, {1024, 16}, {256, 8}, {256, 16}, {256, 32}, {256, 64}, {64, 128}, {64, 256}};
  for (auto c : cfgs) {
    const int smem = c.R * c.C * 4;
    cudaFuncSetAttribute(scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int per_sm = smem <= 32 * 1024 ? 4 : (smem <= 64 * 1024 ? 2 : 1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      scatter<<<148 * per_sm, 512, smem>>>(X, Y, M, W, c.C, c.R);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("{\"kind\": \"scatter\", \"C\": %d, \"R\": %d, \"run_bytes\": %d, \"stride_bytes\": %ld, \"GBps\": %.1f}\n",
           c.C, c.R, c.R * 4, W / c.C * 4, 2.0 * n * 4 / ms / 1e6);
    cudaFuncSetAttribute(scatter4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      scatter4<<<148 * per_sm, 512, smem>>>(X, Y, M, W, c.C, c.R);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("{\"kind\": \"scatter_st128\", \"C\": %d, \"R\": %d, \"run_bytes\": %d, \"stride_bytes\": %ld, \"GBps\": %.1f}\n",
           c.C, c.R, c.R * 4, W / c.C * 4, 2.0 * n * 4 / ms / 1e6);
  }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
