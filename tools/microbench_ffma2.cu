// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) issue/throughput probe for the fused kernel's inner loop shape:
// acc[q] += x[p] * F[p][q] with F in registers (8x8), 1-2 slices per thread.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{.reg .b64 ra, rb, rc, rd;\n\t"
               "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
               "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
               : "=f"(d.x), "=f"(d.y)
               : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

__global__ void k_ffma(float *out, const float *in, int iters) {
  float F[8][8], x[2][8];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = 0; q < 8; ++q) F[p][q] = in[p * 8 + q];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int p = 0; p < 8; ++p) x[r][p] = in[64 + r * 8 + p] + threadIdx.x;
  float s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = x[r][0] * F[0][q];
#pragma unroll
      for (int p = 1; p < 8; ++p)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fmaf(x[r][p], F[p][q], acc[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) x[r][q] = acc[q];
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[0][q] + x[1][q];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float *out, const float *in, int iters) {
  float2 F[8][4];
  float x[2][8];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) F[p][q] = make_float2(in[p * 8 + 2 * q], in[p * 8 + 2 * q + 1]);
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int p = 0; p < 8; ++p) x[r][p] = in[64 + r * 8 + p] + threadIdx.x;
  float s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float2 acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const float2 xx = make_float2(x[r][p], x[r][p]);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = ffma2(xx, F[p][q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) { x[r][2 * q] = acc[q].x; x[r][2 * q + 1] = acc[q].y; }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[0][q] + x[1][q];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float *d;
  cudaMalloc(&d, 4096);
  cudaMemset(d, 0, 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int occ = 1; occ <= 4; occ *= 2) {
    int iters = 2000, blocks = 148 * occ, threads = 256;
    k_ffma<<<blocks, threads>>>(d, d, 10);
    cudaEventRecord(a);
    k_ffma<<<blocks, threads>>>(d, d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 2 * 64 * iters * (double)blocks * threads;
    printf("{\"test\":\"ffma_8x8_regs\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", occ * 8, fl / ms / 1e9);
    k_ffma2<<<blocks, threads>>>(d, d, 10);
    cudaEventRecord(a);
    k_ffma2<<<blocks, threads>>>(d, d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"test\":\"ffma2_8x8_regs\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", occ * 8, fl / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
