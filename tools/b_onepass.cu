// Prototype: config B (M = 1024, six 8 x 8 fp32 factors, W = 8^6) in ONE pass on an 8-CTA cluster
// (fusion bounded by what one CTA holds -> let a cluster hold the row).
//
// Each cluster owns whole rows.  CTA r of the cluster holds x[row][r*32768 .. (r+1)*32768) = the p1 = r slab
// (128 KB of shared memory), then
//   1. local steps: F6 .. F2 applied in place to its 32768-vector (in-register slices, __syncthreads between
//      the read and the write half of each step: out[q*4096 + s] = sum_p in[s*8 + p] F[p][q]) -> Z_r[v];
//   2. cluster barrier; exchange + F1: CTA r takes u in [r*4096, (r+1)*4096), reads Z_p1[u] for p1 = 0..7
//      from the 8 CTAs' shared memory (DSMEM, 7/8 remote) and writes Y[row][q1*32768 + u] = sum_p1 F1[p1][q1]
//      Z_p1[u] straight from registers (float4 runs);
//   3. cluster barrier (nobody refills its slab while a peer may still read it).
// No double buffering (the slab is 128 KB of the 227 KB).  Timed with CUDA events over `reps` launches;
// mode 1 skips the local steps, mode 2 skips the exchange (component times).  Checks two rows against a
// host fp64 reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2401_10187_b200/csrc -o /tmp/b1 tools/b_onepass.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace kron;
constexpr int P = 8, NF = 6, W = 262144, SEG = W / 8, S = SEG / P;  // S: slices of the local vector
__constant__ float cF[NF][P * P];

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int F>
__device__ __forceinline__ void local_step(float *seg, int tid) {
  const int lane = tid & 31, h = (lane >> 2) & 1;
  const float4 *s4 = reinterpret_cast<const float4 *>(seg);
  float v[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int s = tid + 512 * i;
    // halves in the order that puts lanes 0-3 / 4-7 of a phase on different 16-byte granules (no conflict)
    const float4 a = s4[2 * s + h], b = s4[2 * s + 1 - h];
    const float4 lo = h ? b : a, hi = h ? a : b;
    v[i][0] = lo.x; v[i][1] = lo.y; v[i][2] = lo.z; v[i][3] = lo.w;
    v[i][4] = hi.x; v[i][5] = hi.y; v[i][6] = hi.z; v[i][7] = hi.w;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int s = tid + 512 * i;
    float2 o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = __ffma2_rn(make_float2(v[i][p], v[i][p]), make_float2(cF[F][p * 8 + 2 * j], cF[F][p * 8 + 2 * j + 1]), o[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      seg[(2 * j) * S + s] = o[j].x;
      seg[(2 * j + 1) * S + s] = o[j].y;
    }
  }
  __syncthreads();
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1)
    onepass(const float *__restrict__ X, float *__restrict__ Y, int M, int mode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *seg = reinterpret_cast<float *>(smem_raw);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + SEG * 4);
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x / 8, ncl = gridDim.x / 8;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  int it = 0;
  for (int row = cid; row < M; row += ncl, ++it) {
    if (tid == 0) {
      mbar_arrive_expect_tx(bar, SEG * 4);
      for (int c = 0; c < 4; ++c)
        bulk_g2s(seg + c * (SEG / 4), X + (size_t)row * W + (size_t)rank * SEG + c * (SEG / 4), SEG, bar);
    }
    mbar_wait(bar, (uint32_t)(it & 1));
    if (mode != 1) {
      local_step<5>(seg, tid);
      local_step<4>(seg, tid);
      local_step<3>(seg, tid);
      local_step<2>(seg, tid);
      local_step<1>(seg, tid);
    }
    cluster_sync_all();
    if (mode != 2) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int u = (int)rank * (SEG / 8) + 4 * (tid + 512 * k);
        float4 z[8];
        const uint32_t la = smem_u32(seg + u);
#pragma unroll
        for (int p1 = 0; p1 < 8; ++p1) z[p1] = ld_dsmem_f32x4(mapa_shared(la, (uint32_t)p1));
#pragma unroll
        for (int q1 = 0; q1 < 8; ++q1) {
          float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int p1 = 0; p1 < 8; ++p1) {
            const float f = cF[0][p1 * 8 + q1];
            y.x = fmaf(z[p1].x, f, y.x);
            y.y = fmaf(z[p1].y, f, y.y);
            y.z = fmaf(z[p1].z, f, y.z);
            y.w = fmaf(z[p1].w, f, y.w);
          }
          *reinterpret_cast<float4 *>(Y + (size_t)row * W + (size_t)q1 * SEG + u) = y;
        }
      }
    }
    cluster_sync_all();
  }
}

int main(int argc, char **argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 1024, reps = argc > 2 ? atoi(argv[2]) : 20;
  std::vector<float> hX((size_t)2 * W), hF(NF * P * P);
  uint32_t st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (float)((st >> 8) & 0xFFFF) / 65536.f; };
  for (auto &x : hF) x = rnd();
  for (auto &x : hX) x = rnd();
  float *X, *Y;
  cudaMalloc(&X, (size_t)M * W * 4);
  cudaMalloc(&Y, (size_t)M * W * 4);
  cudaMemset(X, 0, (size_t)M * W * 4);
  cudaMemcpy(X, hX.data(), (size_t)2 * W * 4, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(cF, hF.data(), hF.size() * 4);
  const size_t smem = SEG * 4 + 16;
  cudaFuncSetAttribute(onepass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 8;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(8);
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, onepass, &cfg);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    const int grid = 8 * ncl;
    onepass<<<grid, 512, smem>>>(X, Y, M, mode);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(err));
      return 1;
    }
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) onepass<<<grid, 512, smem>>>(X, Y, M, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    double maxrel = -1;
    if (mode == 0) {
      // host fp64 reference for rows 0, 1: Algorithm 1, F6 first
      std::vector<float> hY((size_t)2 * W);
      cudaMemcpy(hY.data(), Y, hY.size() * 4, cudaMemcpyDeviceToHost);
      maxrel = 0;
      for (int r = 0; r < 2; ++r) {
        std::vector<double> t(hX.begin() + (size_t)r * W, hX.begin() + (size_t)(r + 1) * W), o(W);
        for (int f = NF - 1; f >= 0; --f) {
          const int Sl = W / P;
          for (int s = 0; s < Sl; ++s)
            for (int q = 0; q < P; ++q) {
              double acc = 0;
              for (int p = 0; p < P; ++p) acc += t[(size_t)s * P + p] * hF[f * 64 + p * 8 + q];
              o[(size_t)q * Sl + s] = acc;
            }
          t.swap(o);
        }
        for (int i = 0; i < W; ++i) maxrel = fmax(maxrel, fabs(hY[(size_t)r * W + i] - t[i]) / fabs(t[i]));
      }
    }
    const double bytes = 2.0 * M * W * 4, flops = 2.0 * M * W * P * NF;
    printf("{\"mode\": %d, \"M\": %d, \"clusters\": %d, \"ms\": %.4f, \"GBs_alg\": %.1f, \"TFLOPs\": %.2f, \"max_rel_err\": %.3g}\n",
           mode, M, ncl, ms, bytes / ms * 1e-6, flops / ms * 1e-9, maxrel);
  }
  return 0;
}
