// Probe of the tcgen05 building blocks used by csrc/tc.cu: one CTA, D[128 x N] = A[128 x K] . B[K x N] in
// kind::tf32 with A K-major (128B swizzle) or MN-major (128B swizzle) and B K-major, TMEM accumulator read
// back with tcgen05.ld 32x32b.  Checks against a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2401_10187_b200/csrc -o /tmp/tcp tools/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda.h>
#include "ptx.cuh"

using namespace kron;
constexpr int M = 128, N = 32, K = 32;

// A: [M][K] values a[m][k]; B: [K][N] values b[k][n]; layout mode 0: A K-major SW128, 1: A MN-major SW128
__global__ void probe(const float *A, const float *B, float *D, int amode, int lbo, int sbo) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char *base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  unsigned char *sa = base, *sb = base + 16384;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base + 32768);
  uint32_t *slot = reinterpret_cast<uint32_t *>(base + 32768 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    uint32_t off;
    if (amode == 0) off = swz128((uint32_t)m * 128u + (uint32_t)k * 4u);  // row m, 128 B
    else {
      // MN-major: [k group (8 rows)][m block (32)][8 rows][128 B]
      const uint32_t row = (uint32_t)(k / 8) * 4096u + (uint32_t)(m / 32) * 1024u + (uint32_t)(k % 8) * 128u;
      off = row + ((((uint32_t)(m % 32)) * 4u) ^ ((uint32_t)(k % 8) << 4));
    }
    *reinterpret_cast<float *>(sa + off) = A[i];
  }
  // B^T K-major: [n][k], 128 B rows
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    *reinterpret_cast<float *>(sb + swz128((uint32_t)n * 128u + (uint32_t)k * 4u)) = B[i];
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(slot, 32);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t id = umma_idesc_tf32(M, N, amode, 0);
    for (int k = 0; k < K / 8; ++k) {
      uint64_t ad;
      if (amode == 0) ad = umma_desc(smem_u32(sa) + k * 32u, 16, 1024, 2);
      else ad = umma_desc(smem_u32(sa) + k * 4096u, (uint32_t)lbo, (uint32_t)sbo, 2);
      const uint64_t bd = umma_desc(smem_u32(sb) + k * 32u, 16, 1024, 2);
      umma_tf32(tmem, ad, bd, id, k > 0 ? 1u : 0u);
    }
    umma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), r);
    tmem_ld_wait();
    for (int n = 0; n < N; ++n) D[(32 * warp + lane) * N + n] = __uint_as_float(r[n]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 32);
  }
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, M * K * 4);
  cudaMallocManaged(&B, K * N * 4);
  cudaMallocManaged(&D, M * N * 4);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7) % 11 - 5);
  for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5) % 7 - 3);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int cfg[][3] = {{0, 16, 1024}, {1, 1024, 4096}, {1, 4096, 1024}, {1, 1024, 1024}, {1, 4096, 4096},
                        {1, 16, 1024}, {1, 1024, 16}, {1, 8192, 1024}, {1, 1024, 8192}};
  for (auto &cf : cfg) {
    const int amode = cf[0];
    cudaMemset(D, 0, M * N * 4);
    probe<<<1, 256, 40000>>>(A, B, D, amode, cf[1], cf[2]);
    cudaError_t e = cudaDeviceSynchronize();
    int bad = 0;
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
        const double err = fabs(ref - D[m * N + n]);
        if (err > 1e-3) ++bad;
        if (err > maxerr) maxerr = err;
      }
    printf("lbo %d sbo %d ", cf[1], cf[2]);
    printf("amode %d: %s, mismatches %d of %d, max err %g, D[0..3] = %g %g %g %g\n", amode, cudaGetErrorString(e), bad,
           M * N, maxerr, D[0], D[1], D[2], D[3]);
  }
  return 0;
}
