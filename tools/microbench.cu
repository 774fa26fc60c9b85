// Day-1 B200 micro-benchmarks: the roofline denominators this build
// reports against besides MEASURED_PEAKS.json.  Not part of the product path.
//   FFMA / DFMA pipe peak, DMMA (mma.sync f64) peak, HBM copy, and the HBM rate of the
//   Kron-Matmul store pattern (runs of R contiguous elements at stride W/C) vs R.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void ffma_kernel(float *out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

// register-register-register FFMA as in a GEMM micro-tile (no immediate operands)
__global__ void ffma_rrr_kernel(float *out, const float *in, int iters) {
  float x[8], f[8], acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = in[i]; f[i] = in[8 + i]; }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(x[i], f[j], acc[i][j]);
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] += 1e-7f; }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[i][j];
  if (s == 12345.f) out[0] = s;
}

__global__ void dfma_rrr_kernel(double *out, const double *in, int iters) {
  double x[4], f[8], acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = in[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = in[4 + i];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fma(x[i], f[j], acc[i][j]);
#pragma unroll
    for (int i = 0; i < 4; ++i) { x[i] += 1e-15; }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[i][j];
  if (s == 12345.0) out[0] = s;
}

// DMMA: mma.sync.aligned.m16n8k4.row.col.f64 (sm_90+)  -> 2*16*8*4 = 1024 flop / warp-instr
__global__ void dmma_kernel(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 1.0, b0 = 0.5;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_kernel(const float4 *__restrict__ in, float4 *__restrict__ out, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

// Store pattern of one sliced-multiply pass with chunk C and run R (fp32):
// input element (m, g*C + r) -> output (m, u*(W/C) + g) for a "tile" of R chunks.
// Here: each thread copies one 16B vector; the tile of R*C contiguous input elements is
// written as C runs of R elements (u = r), i.e. exactly the permuted store of a fused pass.
__global__ void runstore_kernel(const float *__restrict__ in, float *__restrict__ out, size_t W,
                                size_t M, int C, int R) {
  // tile = (m, tile index j) covering input [j*R*C, (j+1)*R*C)
  size_t tiles_per_row = W / ((size_t)R * C);
  size_t ntiles = tiles_per_row * M;
  size_t vec_per_tile = (size_t)R * C / 4;
  size_t total = ntiles * vec_per_tile;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += stride) {
    size_t tile = v / vec_per_tile, e = (v % vec_per_tile) * 4;
    size_t m = tile / tiles_per_row, j = tile % tiles_per_row;
    float4 x = *reinterpret_cast<const float4 *>(in + m * W + j * R * C + e);
    // local output layout u*R + t  ->  global u*(W/C) + j*R + t
    size_t u = e / R, t = e % R;
    *reinterpret_cast<float4 *>(out + m * W + u * (W / C) + j * R + t) = x;
  }
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int smem_optin = 0, l2 = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  size_t fr, tot;
  cudaMemGetInfo(&fr, &tot);
  printf("{\"name\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"smem_optin\":%d,\"l2\":%d,\"mem_total\":%zu,\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, smem_optin, l2, tot, p.clockRate);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  float *dout;
  CK(cudaMalloc(&dout, 1 << 20));
  CK(cudaMemset(dout, 0, 1 << 20));

  {  // FFMA imm-free (a,b are kernel args -> uniform regs)
    int iters = 20000, blocks = sms * 8, threads = 256;
    ffma_kernel<16><<<blocks, threads>>>(dout, 100, 1.0001f, 1e-6f);
    cudaEventRecord(e0);
    ffma_kernel<16><<<blocks, threads>>>(dout, iters, 1.0001f, 1e-6f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf("{\"test\":\"ffma_uniform\",\"tflops\":%.2f}\n", fl / ms / 1e9);
  }
  {
    int iters = 5000, blocks = sms * 4, threads = 256;
    ffma_rrr_kernel<<<blocks, threads>>>(dout, dout, 10);
    cudaEventRecord(e0);
    ffma_rrr_kernel<<<blocks, threads>>>(dout, dout, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"test\":\"ffma_rrr_8x8\",\"tflops\":%.2f}\n", fl / ms / 1e9);
  }
  {
    int iters = 5000, blocks = sms * 4, threads = 256;
    double *dd = (double *)dout;
    dfma_rrr_kernel<<<blocks, threads>>>(dd, dd, 10);
    cudaEventRecord(e0);
    dfma_rrr_kernel<<<blocks, threads>>>(dd, dd, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 32 * iters * (double)blocks * threads;
    printf("{\"test\":\"dfma_rrr_4x8\",\"tflops\":%.2f}\n", fl / ms / 1e9);
  }
  {
    int iters = 4000, blocks = sms * 4, threads = 256;
    double *dd = (double *)dout;
    dmma_kernel<<<blocks, threads>>>(dd, 10);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(dd, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 1024.0 * 4 * iters * (double)blocks * (threads / 32);
    printf("{\"test\":\"dmma_m16n8k4\",\"tflops\":%.2f}\n", fl / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 1 GiB fp32
  float *a, *b;
  CK(cudaMalloc(&a, n * 4));
  CK(cudaMalloc(&b, n * 4));
  CK(cudaMemset(a, 0, n * 4));
  {
    for (int rep = 0; rep < 2; ++rep) {
      copy_kernel<<<sms * 16, 256>>>((float4 *)a, (float4 *)b, n / 4);
    }
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 16, 256>>>((float4 *)a, (float4 *)b, n / 4);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"test\":\"hbm_copy\",\"gbs\":%.1f}\n", 2.0 * n * 4 / best / 1e6);
  }
  size_t W = (size_t)1 << 18, M = n / W;
  int Cs[] = {64, 512, 4096};
  int Rs[] = {4, 8, 16, 32, 64};
  for (int ci = 0; ci < 3; ++ci)
    for (int ri = 0; ri < 5; ++ri) {
      int C = Cs[ci], R = Rs[ri];
      runstore_kernel<<<sms * 16, 256>>>(a, b, W, M, C, R);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        runstore_kernel<<<sms * 16, 256>>>(a, b, W, M, C, R);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("{\"test\":\"run_store\",\"C\":%d,\"R\":%d,\"gbs\":%.1f}\n", C, R, 2.0 * n * 4 / best / 1e6);
    }
  CK(cudaGetLastError());
  return 0;
}
