// generic.cu — the sliced multiply for any factor shape (odd P/Q, mixed shapes, widths the TMA
// kernels cannot tile).  One pass = one factor, Algorithm 1:
//     out[m, q*S + s] = sum_p in[m, s*P + p] * F[p, q],   S = W/P.
// This is the paper's SlicedMultiplyKernel shape (Fig 3) with TileP = P: a CTA stages a
// contiguous tile of TS slices (TS*P elements) of one row in shared memory with coalesced loads,
// each thread multiplies its slice by every column of F (F in shared memory), and for every column q
// the CTA stores TS consecutive outputs at q*S + s0 (the direct-index store).  Small odd
// P (3..7) get compile-time slice registers; other P loop over shared memory.
#include <cuda_runtime.h>

#include "kron_internal.h"

namespace kron {
namespace {

constexpr int TS = 256;  // slices per tile = threads per CTA

template <typename T, int PC>
__global__ void __launch_bounds__(TS) sliced_generic_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                            const T *__restrict__ F, int64_t M, int64_t W, int Pr,
                                                            int Q) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = PC > 0 ? PC : Pr;
  T *Fs = reinterpret_cast<T *>(smem_raw);  // [P][Q]
  T *Xs = Fs + ((P * Q + 3) & ~3);          // [TS * P]
  for (int i = threadIdx.x; i < P * Q; i += TS) Fs[i] = F[i];
  const int64_t S = W / P, Wout = S * Q;
  const int64_t tiles_row = (S + TS - 1) / TS, ntiles = M * tiles_row;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t m = tile / tiles_row, s0 = (tile - m * tiles_row) * TS;
    const int ns = (int)(S - s0 < TS ? S - s0 : TS);
    __syncthreads();  // previous tile's reads done (and F staged on the first pass)
    const T *src = in + m * W + s0 * P;
    for (int i = threadIdx.x; i < ns * P; i += TS) Xs[i] = src[i];
    __syncthreads();
    const int t = threadIdx.x;
    if (t < ns) {
      T *dst = out + m * Wout + s0 + t;
      if constexpr (PC > 0) {
        T x[PC];
#pragma unroll
        for (int p = 0; p < PC; ++p) x[p] = Xs[t * PC + p];
        for (int q = 0; q < Q; ++q) {
          T acc = x[0] * Fs[q];
#pragma unroll
          for (int p = 1; p < PC; ++p) acc = fma(x[p], Fs[p * Q + q], acc);
          dst[(int64_t)q * S] = acc;
        }
      } else {
        for (int q = 0; q < Q; ++q) {
          T acc = 0;
          for (int p = 0; p < P; ++p) acc = fma(Xs[t * P + p], Fs[p * Q + q], acc);
          dst[(int64_t)q * S] = acc;
        }
      }
    }
  }
}

// Fallback for factors too large for shared memory: one thread per output, F read through L1/L2.
template <typename T>
__global__ void __launch_bounds__(256) sliced_generic_global_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                                    const T *__restrict__ F, int64_t M, int64_t W,
                                                                    int P, int Q) {
  const int64_t S = W / P, Wout = S * Q, total = M * Wout;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = idx / Wout, j = idx - m * Wout;
    const int64_t q = j / S, s = j - q * S;
    const T *x = in + m * W + s * P;
    T acc = 0;
    for (int p = 0; p < P; ++p) acc = fma(x[p], F[(int64_t)p * Q + q], acc);
    out[idx] = acc;
  }
}

template <typename T>
using GenFn = void (*)(const T *, T *, const T *, int64_t, int64_t, int, int);

template <typename T>
GenFn<T> pick(int P) {
  switch (P) {
    case 1: return sliced_generic_kernel<T, 1>;
    case 2: return sliced_generic_kernel<T, 2>;
    case 3: return sliced_generic_kernel<T, 3>;
    case 4: return sliced_generic_kernel<T, 4>;
    case 5: return sliced_generic_kernel<T, 5>;
    case 6: return sliced_generic_kernel<T, 6>;
    case 7: return sliced_generic_kernel<T, 7>;
    case 8: return sliced_generic_kernel<T, 8>;
  }
  return sliced_generic_kernel<T, 0>;
}

template <typename T>
int launch_t(const PassPlan &pp, int64_t M, const void *in, void *out, const void *F, void *stream) {
  const size_t smem = ((size_t)((pp.P * pp.Q + 3) & ~3) + (size_t)TS * pp.P) * sizeof(T);
  if (smem > 200 * 1024) {
    const int64_t total = M * pp.W_out;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    sliced_generic_global_kernel<T><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        (const T *)in, (T *)out, (const T *)F, M, pp.W_in, pp.P, pp.Q);
    return (int)cudaGetLastError();
  }
  GenFn<T> k = pick<T>(pp.P);
  if (smem > 48 * 1024) {
    const int e = set_smem_attr((const void *)k, smem);
    if (e != 0) return e;
  }
  const int64_t S = pp.W_in / pp.P, ntiles = M * ((S + TS - 1) / TS);
  int64_t grid = ntiles < 148 * 8 ? ntiles : 148 * 8;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, TS, smem, (cudaStream_t)stream>>>((const T *)in, (T *)out, (const T *)F, M, pp.W_in, pp.P,
                                                        pp.Q);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_generic(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F,
                   void *stream) {
  if (M * pp.W_out == 0) return 0;
  return dtype == KRON_F32 ? launch_t<float>(pp, M, in, out, F, stream)
                           : launch_t<double>(pp, M, in, out, F, stream);
}

}  // namespace kron
