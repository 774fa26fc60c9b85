// Do FP64 tensor-core MMAs (DMMA) and FP64 FMAs (DFMA) share one pipe on sm_100a?  Each warp runs either
// independent DMMA m16n8k4 chains or independent DFMA chains; mode 0 = all DMMA, 1 = all DFMA, 2 = half the
// warps of every SM sub-partition each.  If the mix beats both pure modes, fp64 kernels could split work
// between the two.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbf tools/microbench_f64mix.cu && /tmp/mbf
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

template <int DFMA_REPS>
__global__ void mix(double *out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool use_dmma = mode == 0 ? true : mode == 1 ? false : ((w >> 2) & 1) == 0;
  double s = 0;
  if (use_dmma) {
    double c[8][4] = {};
    const double a0 = threadIdx.x * 1e-3, a1 = a0 * 3, b = a0 * 5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(c[j], a0, a1, b);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  } else {
    double c[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = threadIdx.x * 1e-3 + j;
    const double x = 1.0000001, y = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int r = 0; r < DFMA_REPS; ++r)
#pragma unroll
        for (int j = 0; j < 32; ++j) c[j] = fma(c[j], x, y);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) s += c[j];
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048, threads = 512;  // 16 warps per CTA, one CTA per SM
  for (int mode = 0; mode < 3; ++mode) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      mix<4><<<sms, threads>>>(out, iters, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    // each warp-iteration is 8 DMMA (16x8x4 FMAs = 512 each) = 4096 FMAs, or 32 lanes x 128 FMAs = 4096 FMAs
    const double fl = 4096.0 * 2 * iters * (threads / 32) * sms;
    printf("{\"test\":\"f64mix\",\"mode\":\"%s\",\"ms\":%.3f,\"tflops\":%.2f}\n",
           mode == 0 ? "dmma" : mode == 1 ? "dfma" : "half_dmma_half_dfma", ms, fl / ms / 1e9);
  }
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
