// Compute-only microbenchmark of config E's fused 16x16 triple (v10): the cb_pair16 / cb_top16 chunk steps of
// fused.cu on a shared-memory tile that never changes (no TMA, no stream-out, no mbarriers), to separate
// the arithmetic's own FMA-pipe rate from the pipeline around it in kron_fused_gemm3c_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I paper_2401_10187_b200/csrc -lcuda \
//        -o /tmp/mbt tools/microbench_tri.cu && /tmp/mbt
// Prints one JSON line per variant: TFLOP/s counted as 48 FMA (2 flops each) per element of every chunk.
#include "../paper_2401_10187_b200/csrc/fused.cu"

#include <cstdio>

namespace kron {  // tc.cu is not linked into the microbenchmark
int launch_tc(const PassPlan &, int64_t, const void *, void *, const void *const *, void *) { return 1; }
}  // namespace kron

namespace kron {
namespace {

// MODE 0: as the kernel (groups of four warps, named barrier between phase 1 and phase 2)
// MODE 1: no named barrier (each warp's phase 2 reads columns other warps may still be writing: timing only)
// MODE 2: phase 1 only (cb_pair16), MODE 3: phase 2 only (cb_top16)
template <int NCW, int MODE>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) mb_tri(float *out, int iters) {
  constexpr uint32_t CE = 1024, TB = 64 * CE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  for (uint32_t i = threadIdx.x; i < 3 * TB / 4; i += blockDim.x)
    reinterpret_cast<float *>(base)[i] = 1e-3f * (float)((i * 2654435761u) >> 20);
  __syncthreads();
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  if (warp < NCW) {
    constexpr int NG = NCW / 4;
    const int grp = warp >> 2, wi = warp & 3;
    const float *F1c = c_fac3, *F2c = c_fac3 + 256, *F3c = c_fac3 + 512;
    for (int ci = grp; ci < iters; ci += NG) {
      const int t = ci & 3, st = (ci >> 2) % 3;
      unsigned char *buf = base + (size_t)st * TB;
      if (MODE != 3) cb_pair16(buf, (uint32_t)(t * 16 + wi * 4), lane, F1c, F2c);
      if (MODE == 0) named_bar_sync(1 + grp, 128);
      if (MODE != 2) cb_top16(buf + (uint32_t)(t * 16) * CE, (uint32_t)(wi * 64 + 2 * lane), F3c);
      __syncwarp();
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = reinterpret_cast<float *>(base)[5];
}

template <int NCW, int MODE>
void run(float *d_out, int sms) {
  auto k = mb_tri<NCW, MODE>;
  const int smem = 3 * 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;  // chunks per CTA
  k<<<sms, (NCW + 4) * 32, smem>>>(d_out, iters);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k<<<sms, (NCW + 4) * 32, smem>>>(d_out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double fma_per_chunk = MODE == 2 ? 32.0 * 4096 : MODE == 3 ? 16.0 * 4096 : 48.0 * 4096;
  const double tf = 2.0 * fma_per_chunk * iters * sms / (ms * 1e-3) / 1e12;
  printf("{\"test\":\"tri\",\"ncw\":%d,\"mode\":%d,\"ms\":%.3f,\"tflops\":%.2f,\"err\":\"%s\"}\n", NCW, MODE, ms, tf,
         cudaGetErrorString(cudaGetLastError()));
}

}  // namespace
}  // namespace kron

int main() {
  float h[768];
  for (int i = 0; i < 768; ++i) h[i] = 0.0625f * (float)((i * 37) % 17) / 16.0f;
  cudaMemcpyToSymbol(kron::c_fac3, h, sizeof(h));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *d_out;
  cudaMalloc(&d_out, 4096 * sizeof(float));
  kron::run<12, 0>(d_out, sms);
  kron::run<12, 1>(d_out, sms);
  kron::run<12, 2>(d_out, sms);
  kron::run<12, 3>(d_out, sms);
  kron::run<16, 0>(d_out, sms);
  kron::run<8, 0>(d_out, sms);
  return 0;
}
