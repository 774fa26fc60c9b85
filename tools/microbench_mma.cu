// Legacy warp-level tensor-core throughput on sm_100a (mma.sync -> SASS HMMA / DMMA): TF32 m16n8k8,
// BF16 m16n8k16 and FP64 m16n8k4, 8 independent accumulators per warp, 16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_mma tools/microbench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tf32(float *out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[0] = s;
}

__global__ void bf16(float *out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  float *out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 4, threads = 128;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    tf32<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  double flops = 2.0 * 16 * 8 * 8 * 8 * (double)iters * blocks * (threads / 32);
  printf("{\"kind\": \"mma.sync tf32 m16n8k8\", \"TFLOPS\": %.1f}\n", flops / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    bf16<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  flops = 2.0 * 16 * 8 * 16 * 8 * (double)iters * blocks * (threads / 32);
  printf("{\"kind\": \"mma.sync bf16 m16n8k16\", \"TFLOPS\": %.1f}\n", flops / ms / 1e9);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
