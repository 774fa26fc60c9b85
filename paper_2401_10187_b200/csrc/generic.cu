// generic.cu — the fallback sliced multiply for any factor shape (odd P/Q, mixed shapes, widths the
// TMA kernels cannot tile).  One pass = one factor, Algorithm 1:
//     out[m, q*S + s] = sum_p in[m, s*P + p] * F[p, q],   S = W/P.
// Consecutive threads own consecutive s for a fixed (m, q): the store is fully coalesced and the
// loads of neighbouring slices share cache lines (consecutive outputs are consecutive
// slices times the same factor column, so no transpose is needed).
#include <cuda_runtime.h>

#include "kron_internal.h"

namespace kron {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) sliced_generic_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                             const T *__restrict__ F, int64_t M, int64_t W, int P,
                                                             int Q, int f_in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *Fs = reinterpret_cast<T *>(smem_raw);
  if (f_in_smem) {
    for (int i = threadIdx.x; i < P * Q; i += blockDim.x) Fs[i] = F[i];
    __syncthreads();
  }
  const T *Fr = f_in_smem ? Fs : F;
  const int64_t S = W / P, Wout = S * Q, total = M * Wout;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx / Wout, j = idx - m * Wout;
    const int64_t q = j / S, s = j - q * S;
    const T *x = in + m * W + s * P;
    T acc = 0;
    for (int p = 0; p < P; ++p) acc = fma(x[p], Fr[(int64_t)p * Q + q], acc);
    out[idx] = acc;
  }
}

}  // namespace

int launch_generic(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F,
                   void *stream) {
  const int64_t total = M * pp.W_out;
  if (total == 0) return 0;
  const size_t es = dtype == KRON_F32 ? 4 : 8;
  const size_t fbytes = (size_t)pp.P * pp.Q * es;
  const int f_in_smem = fbytes <= 48 * 1024;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KRON_F32)
    sliced_generic_kernel<float><<<(unsigned)blocks, 256, f_in_smem ? fbytes : 0, s>>>(
        (const float *)in, (float *)out, (const float *)F, M, pp.W_in, pp.P, pp.Q, f_in_smem);
  else
    sliced_generic_kernel<double><<<(unsigned)blocks, 256, f_in_smem ? fbytes : 0, s>>>(
        (const double *)in, (double *)out, (const double *)F, M, pp.W_in, pp.P, pp.Q, f_in_smem);
  return (int)cudaGetLastError();
}

}  // namespace kron
