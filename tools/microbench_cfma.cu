// Constant-bank factor operands: FFMA with the factor entry read straight from the kernel-parameter
// constant bank (c[0x0][...], uniform across the warp) vs FFMA / FFMA2 with the factor in registers.
// Inner-loop shape of a sliced multiply: acc[q] = sum_p x[p] * F[p][q], then x <- acc (the next factor).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbc tools/microbench_cfma.cu && /tmp/mbc
#include <cstdio>
#include <cuda_runtime.h>

template <int P, int NF>
struct Fac {
  float f[NF][P][P];
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// scalar FFMA, factor from the constant bank; R slices per thread (independent chains)
template <int P, int NF, int R>
__global__ void __launch_bounds__(256) k_cfma(float *out, const __grid_constant__ Fac<P, NF> F, int iters) {
  float x[R][P];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int p = 0; p < P; ++p) x[r][p] = (float)(threadIdx.x + p + r) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float acc[P];
#pragma unroll
        for (int q = 0; q < P; ++q) acc[q] = x[r][0] * F.f[j][0][q];
#pragma unroll
        for (int p = 1; p < P; ++p)
#pragma unroll
          for (int q = 0; q < P; ++q) acc[q] = fmaf(x[r][p], F.f[j][p][q], acc[q]);
#pragma unroll
        for (int q = 0; q < P; ++q) x[r][q] = acc[q];
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q < P; ++q) s += x[r][q];
  if (s == 1234.5f) out[0] = s;
}

// FFMA2 over two slices at once: acc2[q] = (x0[p], x1[p]) * (F[p][q], F[p][q]) + acc2[q]; the factor
// pair is a broadcast of one constant
template <int P, int NF>
__global__ void __launch_bounds__(256) k_cfma2(float *out, const __grid_constant__ Fac<P, NF> F, int iters) {
  float2 x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = make_float2((threadIdx.x + p) * 1e-3f, (threadIdx.x + 2 * p) * 1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      float2 acc[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const float f = F.f[j][0][q];
        acc[q] = make_float2(x[0].x * f, x[0].y * f);
      }
#pragma unroll
      for (int p = 1; p < P; ++p)
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const float f = F.f[j][p][q];
          acc[q] = ffma2(x[p], make_float2(f, f), acc[q]);
        }
#pragma unroll
      for (int q = 0; q < P; ++q) x[q] = acc[q];
    }
  }
  float s = 0;
#pragma unroll
  for (int q = 0; q < P; ++q) s += x[q].x + x[q].y;
  if (s == 1234.5f) out[0] = s;
}

template <typename K, typename A>
double run(K kern, const A &arg, double flop_per_thread_iter, int blocks, int threads, int iters, float *d) {
  kern<<<blocks, threads>>>(d, arg, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(d, arg, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return flop_per_thread_iter * iters * (double)blocks * threads / ms / 1e9;
}

template <int P, int NF, int R>
void one(float *d, int occ) {
  Fac<P, NF> F;
  for (int j = 0; j < NF; ++j)
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < P; ++q) F.f[j][p][q] = (p == q ? 0.5f : 0.01f) + 0.001f * j;
  const int blocks = 148 * occ, threads = 256, iters = 4096 / (P * NF) * 16;
  double t1 = run(k_cfma<P, NF, R>, F, 2.0 * NF * P * P * R, blocks, threads, iters, d);
  printf("{\"test\":\"cfma\",\"P\":%d,\"NF\":%d,\"R\":%d,\"param_bytes\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", P, NF,
         R, (int)sizeof(F), occ * 8, t1);
  double t2 = run(k_cfma2<P, NF>, F, 2.0 * NF * P * P * 2, blocks, threads, iters, d);
  printf("{\"test\":\"cfma2\",\"P\":%d,\"NF\":%d,\"param_bytes\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", P, NF,
         (int)sizeof(F), occ * 8, t2);
}

int main() {
  float *d;
  cudaMalloc(&d, 4096);
  for (int occ = 1; occ <= 4; occ *= 2) {
    one<8, 1, 2>(d, occ);
    one<16, 1, 1>(d, occ);
    one<16, 1, 2>(d, occ);
    one<16, 3, 1>(d, occ);
    one<16, 3, 2>(d, occ);
    one<32, 1, 1>(d, occ);
    one<32, 2, 1>(d, occ);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
