// chain.cu — fused multi-factor passes for square factors of ANY size P (NEXT-3).
//
// The TMA-staged fused kernels (fused.cu) need 16-byte-aligned row strides and 128-byte lines, so odd P
// (3, 5, 6, 7 ... — the paper's Table 4 shapes 3^7, 6^7) used to run one unfused generic pass per
// factor.  This kernel fuses a group of k consecutive P x P factors (chunk C = P^k, Fused <= floor(log_P TileK),
// P:524) with plain coalesced loads:
//   a2  a CTA copies a tile of R consecutive chunks (R*C contiguous elements of one row) into shared memory
//       (coalesced 4 / 8-byte loads, any alignment);
//   a4/a5  the k sliced multiplies run in place: step j contracts digit j of the chunk index
//       (stride P^j): each thread owns whole slices, reads its P values and writes its P outputs to the same
//       positions (one barrier per step) — odd strides keep consecutive slices on distinct banks; an even chunk
//       is padded by one element so the chunk-to-chunk stride stays odd;
//   a6  direct-index store Y[row][u*(W/C) + g0 + t]: threads walk (u, t) with t fastest, so each
//       warp writes runs of R consecutive outputs.
// Several small CTAs per SM (no warp specialisation): the loads of one CTA overlap the arithmetic of others.
#include <cuda_runtime.h>

#include "kron_internal.h"

namespace kron {
namespace {

constexpr int kChainThreads = 256;

__device__ __forceinline__ uint32_t sptr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int BYTES>
__device__ __forceinline__ void cp_async(void *dst, const void *src) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sptr(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sptr(dst)), "l"(src), "n"(BYTES) : "memory");
}
// n / d for n < 2^31 by multiply-high and shift (divisor fixed per launch; Granlund-Montgomery): 2-3
// instructions instead of a ~20-instruction integer division in the slice-index math
struct FastDiv {
  uint32_t d = 1, m = 0;
  int shift = 0;
  __host__ void set(uint32_t div) {
    d = div;
    int l = 0;
    while ((1ull << l) < div) ++l;  // ceil(log2 d)
    const int p = 31 + l;
    m = (uint32_t)(((1ull << p) + div - 1) / div);
    shift = p - 32;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return d == 1 ? n : (__umulhi(n, m) >> shift); }
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct ChainArgs {
  const void *F[kMaxFused];  // factors in processing order (step 0 first)
  int k;                     // fused factors
  int64_t C;                 // chunk = P^k
  int64_t CS;                // chunk stride in shared memory: C + 1 (even C) / C (odd C); 16-byte copies: C + pad
  int vec;                   // 1: 16-byte asynchronous copies (aligned rows and chunks)
  FastDiv dCP, dR;           // division by C/P (slices per chunk) and by R
  FastDiv dst[kMaxFused];    // division by P^j (step j's digit stride)
  FastDiv dCP2;              // slice-pair path (even P, 16-byte layout): division by C/(2P)
  FastDiv dsth[kMaxFused];   // ... and by P^j / 2
  int R;                     // chunks per tile
  int64_t W, WC;             // row width (in = out for square factors), W / C
  int64_t M, tiles_k, ntiles;
};

template <typename T, int P>
__global__ void __launch_bounds__(kChainThreads) kron_chain_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                                   const ChainArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *Fs = reinterpret_cast<T *>(smem_raw);            // [k][P][P]
  const int tid = threadIdx.x;
  for (int i = tid; i < a.k * P * P; i += kChainThreads) Fs[i] = reinterpret_cast<const T *>(a.F[i / (P * P)])[i % (P * P)];
  // tile-local index math in 32 bits (a tile is < 2^25 elements): 64-bit divisions cost ~100 instructions each
  const uint32_t C = (uint32_t)a.C, CS = (uint32_t)a.CS, R = (uint32_t)a.R, CP = C / P;
  const uint32_t nsl = R * CP;  // slices per tile
  // two tile buffers: the next tile's rows stream in with cp.async (LDGSTS, many copies in flight, no register
  // round trip) while this tile is multiplied and stored
  // (buffer = base + cur * tile: a runtime-indexed pointer array would demote every tile access to a generic
  // LD / ST — ncu counted them on Table 4 #19)
  T *const buf0 = Fs + ((a.k * P * P + 3) & ~3);
  const uint32_t tileE = R * CS;
  auto fetch = [&](int64_t tile, T *dst) {
    if (tile < a.ntiles) {
      const int64_t row = tile / a.tiles_k, tk = tile - row * a.tiles_k;
      const T *src = in + row * a.W + tk * R * C;
      if (a.vec) {
        constexpr int V = 16 / sizeof(T);
        for (uint32_t t = 0; t < R; ++t)
          for (uint32_t e = tid * V; e < C; e += kChainThreads * V) cp_async<16>(dst + t * CS + e, src + (int64_t)t * C + e);
      } else {
        for (uint32_t t = 0; t < R; ++t)
          for (uint32_t e = tid; e < C; e += kChainThreads) cp_async<sizeof(T)>(dst + t * CS + e, src + (int64_t)t * C + e);
      }
    }
    cp_async_commit();
  };
  fetch(blockIdx.x, buf0);
  int cur = 0;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, cur ^= 1) {
    const int64_t row = tile / a.tiles_k, tk = tile - row * a.tiles_k;
    const int64_t g0 = tk * R;                         // first chunk of the tile
    T *buf = buf0 + cur * tileE;
    fetch(tile + gridDim.x, buf0 + (cur ^ 1) * tileE);  // the other buffer was released at the last barrier
    cp_async_wait<1>();                                // this tile's copies (all but the newest group) landed
    __syncthreads();
    uint32_t st = 1;  // stride of the digit contracted in this step (P^j)
    for (int j = 0; j < a.k; ++j, st *= P) {
      // the step's factor in registers for P <= 8 (<= 64 values; a shared-memory operand per FMA doubled the
      // instruction count), else read from shared memory as warp-uniform broadcasts
      constexpr bool kFReg = P <= 8;
      T Fr[kFReg ? P * P : 1];
      const T *F = Fs + j * P * P;
      if constexpr (kFReg) {
#pragma unroll
        for (int i = 0; i < P * P; ++i) Fr[i] = F[i];
      }
      // slices of this step: (chunk t, hi, lo) with element base t*CS + hi*st*P + lo, elements at + p*st; a
      // thread writes its outputs over exactly the positions it read (P = Q), so a step needs no barrier
      // between its reads and writes, only one before the next step
      if constexpr (kFReg && sizeof(T) == 4 && P % 2 == 0) {
        if (a.vec) {
          // even P on the 16-byte layout (CS, P, st even: every slice pair below is 8-byte aligned).
          // Step 0 (st = 1): a slice is P contiguous values -> P/2 LDS.64 in, P/2 STS.64 out (lanes 2P words
          // apart: the 16 lanes of a phase cover 32 distinct banks).  Steps j >= 1: a thread takes the slice
          // PAIR (lo, lo + 1) — its elements p are adjacent — as one float2 per p and runs
          // FFMA2(x pair, F[p][q] broadcast): half the loads, stores and index math per FMA of the scalar path
          // (Table 4 #19, 6^7: 40% of the wavefronts were conflicts, FMA pipe at 29-40%)
          if (j == 0) {
            for (uint32_t sl = tid; sl < nsl; sl += kChainThreads) {
              const uint32_t t = a.dCP.div(sl), w = sl - t * CP;
              T *bp = buf + t * CS + w * P;
              float x[P];
#pragma unroll
              for (int p = 0; p < P; p += 2) {
                const float2 v = *reinterpret_cast<const float2 *>(bp + p);
                x[p] = v.x;
                x[p + 1] = v.y;
              }
#pragma unroll
              for (int q = 0; q < P; q += 2) {
                float2 acc = __fmul2_rn(make_float2(x[0], x[0]), make_float2(Fr[q], Fr[q + 1]));
#pragma unroll
                for (int p = 1; p < P; ++p)
                  acc = __ffma2_rn(make_float2(x[p], x[p]), make_float2(Fr[p * P + q], Fr[p * P + q + 1]), acc);
                *reinterpret_cast<float2 *>(bp + q) = acc;
              }
            }
          } else {
            const uint32_t half = st / 2, CP2 = CP / 2;
            for (uint32_t pr = tid; pr < nsl / 2; pr += kChainThreads) {
              const uint32_t t = a.dCP2.div(pr), w = pr - t * CP2, hi = a.dsth[j].div(w), lo = 2 * (w - hi * half);
              T *bp = buf + t * CS + hi * st * P + lo;
              float2 x2[P];
#pragma unroll
              for (int p = 0; p < P; ++p) x2[p] = *reinterpret_cast<const float2 *>(bp + p * st);
#pragma unroll
              for (int q = 0; q < P; ++q) {
                float2 acc = __fmul2_rn(x2[0], make_float2(Fr[q], Fr[q]));
#pragma unroll
                for (int p = 1; p < P; ++p) acc = __ffma2_rn(x2[p], make_float2(Fr[p * P + q], Fr[p * P + q]), acc);
                *reinterpret_cast<float2 *>(bp + q * st) = acc;
              }
            }
          }
          __syncthreads();
          continue;
        }
      }
      for (uint32_t sl = tid; sl < nsl; sl += kChainThreads) {
        const uint32_t t = a.dCP.div(sl), w = sl - t * CP, hi = a.dst[j].div(w), lo = w - hi * st;
        const uint32_t b = t * CS + hi * st * P + lo;
        T x[P];
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = buf[b + p * st];
        if constexpr (kFReg && sizeof(T) == 4 && P % 2 == 0) {
          // FFMA2: outputs (q, q+1) as a pair, x[p] broadcast, factor pair from registers
#pragma unroll
          for (int q = 0; q < P; q += 2) {
            float2 acc = make_float2(x[0] * Fr[q], x[0] * Fr[q + 1]);
#pragma unroll
            for (int p = 1; p < P; ++p)
              acc = __ffma2_rn(make_float2(x[p], x[p]), make_float2(Fr[p * P + q], Fr[p * P + q + 1]), acc);
            buf[b + q * st] = acc.x;
            buf[b + (q + 1) * st] = acc.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < P; ++q) {
            T acc = x[0] * (kFReg ? Fr[q] : F[q]);
#pragma unroll
            for (int p = 1; p < P; ++p) acc = fma(x[p], kFReg ? Fr[p * P + q] : F[p * P + q], acc);
            buf[b + q * st] = acc;
          }
        }
      }
      __syncthreads();
    }
    // a6: composite column u of chunk t -> out[row][u*WC + g0 + t]; t fastest = runs of R
    T *dst = out + row * a.W + g0;
    for (uint32_t i = tid; i < R * C; i += kChainThreads) {
      const uint32_t u = a.dR.div(i), t = i - u * R;
      dst[(int64_t)u * a.WC + t] = buf[t * CS + u];
    }
    __syncthreads();  // every read of this buffer is done before the next iteration's prefetch overwrites it
  }
  cp_async_wait<0>();
}

template <typename T>
using ChainFn = void (*)(const T *, T *, const ChainArgs);

template <typename T>
ChainFn<T> chain_pick(int P) {
  switch (P) {
    case 2: return kron_chain_kernel<T, 2>;
    case 3: return kron_chain_kernel<T, 3>;
    case 4: return kron_chain_kernel<T, 4>;
    case 5: return kron_chain_kernel<T, 5>;
    case 6: return kron_chain_kernel<T, 6>;
    case 7: return kron_chain_kernel<T, 7>;
    case 8: return kron_chain_kernel<T, 8>;
    case 9: return kron_chain_kernel<T, 9>;
    case 10: return kron_chain_kernel<T, 10>;
    case 11: return kron_chain_kernel<T, 11>;
    case 12: return kron_chain_kernel<T, 12>;
    case 13: return kron_chain_kernel<T, 13>;
    case 14: return kron_chain_kernel<T, 14>;
    case 15: return kron_chain_kernel<T, 15>;
    case 16: return kron_chain_kernel<T, 16>;
  }
  return nullptr;
}

// chunk stride in shared memory: odd (conflict-free strided slices) unless the 16-byte copy path needs it
// to be a multiple of 16 bytes (then C + 16 bytes: the chunk-to-chunk bank offset still varies)
int64_t chain_cs(int64_t C, int es, bool vec) {
  if (vec) return C + 16 / es;
  return C % 2 ? C : C + 1;
}
bool chain_vec(int64_t C, int64_t W, int es) { return (C * es) % 16 == 0 && (W * es) % 16 == 0; }
size_t chain_smem(int P, int k, int64_t C, int R, int es, bool vec) {
  return (size_t)(((int64_t)k * P * P + 3) & ~3) * es + 2 * (size_t)R * chain_cs(C, es, vec) * es;
}

}  // namespace

// Geometry of a chain pass over factors of size P (square), k of them, on rows of width W: chunk C = P^k must
// divide W; R chunks per tile — the largest divisor of W/C up to 16 whose tile fits `budget` bytes, preferring
// output runs of >= 32 bytes (R*es >= 32) — policy.chain_rdiv halves R (autotuner tile-size candidates).
bool chain_geometry(int P, int k, int dtype, int64_t W, int rdiv, PassPlan *pp) {
  if (P < 2 || P > 16 || k < 1 || k > kMaxFused) return false;
  const int es = dtype == KRON_F64 ? 8 : 4;
  int64_t C = 1;
  for (int i = 0; i < k; ++i) C *= P;
  if (W % C) return false;
  const int64_t WC = W / C;
  const size_t budget = 100 * 1024;
  int best = 0, best8 = 0;
  const bool vec = chain_vec(C, W, es);
  for (int R = 1; R <= 64 && R <= WC; ++R)
    if (WC % R == 0 && chain_smem(P, k, C, R, es, vec) <= budget) {
      if (R <= 16) best = R;
      if (R % 8 == 0) best8 = R;
    }
  // tiles of a multiple of 8 chunks, up to 64 when the chunk is small (Table 4 #19: 6^4 pass 8 chunks, 6^3 pass 48
  // chunks = 192-byte output runs; with the shared-space and FMUL2 fixes below: 2.39 -> 2.07 ms.  Warp-owned chunks
  // (one __syncwarp instead of a CTA barrier per step) measured no faster: 2.10 ms)
  if (best8 > 0) best = best8;
  if (best == 0) return false;
  if (rdiv > 1) {
    int r2 = best / rdiv;
    while (r2 > 1 && WC % r2) --r2;
    if (r2 < 1) r2 = 1;
    best = r2;
  }
  // short runs only when the whole row is the tile (no run to speak of) or nothing longer fits
  if ((int64_t)best * es < 32 && best < WC && k > 1) return false;
  pp->kind = KIND_CHAIN;
  pp->nf = k;
  pp->P = pp->Q = P;
  pp->C = pp->Qc = C;
  pp->R = best;
  pp->tileK = best * C;
  pp->tileM = 1;
  pp->stages = 1;
  return true;
}

int launch_chain(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *const *Fgroup,
                 void *stream) {
  ChainArgs a{};
  for (int i = 0; i < pp.nf; ++i) a.F[i] = Fgroup[i];
  a.k = pp.nf;
  a.C = pp.C;
  const int es = dtype == KRON_F64 ? 8 : 4;
  const bool vec = chain_vec(pp.C, pp.W_in, es);
  a.CS = chain_cs(pp.C, es, vec);
  a.vec = vec ? 1 : 0;
  a.R = pp.R;
  a.W = pp.W_in;
  a.WC = pp.W_in / pp.C;
  a.M = M;
  a.tiles_k = a.WC / pp.R;
  a.dCP.set((uint32_t)(pp.C / pp.P));
  a.dR.set((uint32_t)pp.R);
  for (int j = 0, st = 1; j < pp.nf; ++j, st *= pp.P) {
    a.dst[j].set((uint32_t)st);
    a.dsth[j].set((uint32_t)(st > 1 ? st / 2 : 1));
  }
  a.dCP2.set((uint32_t)(pp.C / pp.P / 2 > 0 ? pp.C / pp.P / 2 : 1));
  a.ntiles = M * a.tiles_k;
  if (a.ntiles == 0) return 0;
  const size_t smem = chain_smem(pp.P, pp.nf, pp.C, pp.R, es, vec);
  const void *fn = dtype == KRON_F64 ? (const void *)chain_pick<double>(pp.P) : (const void *)chain_pick<float>(pp.P);
  if (!fn) return (int)cudaErrorInvalidValue;
  const int slots = kernel_slots(fn, kChainThreads, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > a.ntiles) grid = a.ntiles;
  if (dtype == KRON_F64)
    chain_pick<double>(pp.P)<<<(unsigned)grid, kChainThreads, smem, (cudaStream_t)stream>>>(
        static_cast<const double *>(in), static_cast<double *>(out), a);
  else
    chain_pick<float>(pp.P)<<<(unsigned)grid, kChainThreads, smem, (cudaStream_t)stream>>>(
        static_cast<const float *>(in), static_cast<float *>(out), a);
  return (int)cudaGetLastError();
}

}  // namespace kron
