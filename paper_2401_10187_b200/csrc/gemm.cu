// gemm.cu — the large-P sliced multiply as a register-tiled GEMM.
//
// For large P (64, 128: configs D1/D2) one factor per pass; fusion does not pay.  The pass
//     Y[m, q*S + s] = sum_p T[m, s*P + p] * F[p, q]          (Alg 1, S = W/P)
// is the GEMM  A (M*S x P, row-major: row m*S+s is slice s of row m)  x  F (P x Q), with the
// permuted epilogue of the paper's direct-index store: for a fixed column q
// consecutive slices are consecutive outputs, so the store needs no transpose.
//
//   * A and F tiles stream HBM/L2 -> shared memory with TMA (A: 128B-swizzled [slice][p] rows of
//     BK elements; F: [p][q] rows), through an mbarrier ring of NS stages (the paper's t_P loop,
//     P:351-365);
//   * 256 threads, each a TM x TN register tile (FFMA for fp32, DFMA for fp64 — the DFMA and DMMA
//     pipes measured the same 37 TF on B200, profiles/r01_microbench.jsonl), slices strided by
//     BM/TM and columns interleaved by BN/TN so that A reads (LDS.128 of p-pairs/quads) and F
//     reads (LDS.64/32) are conflict-free;
//   * the epilogue writes Y straight from registers: for each (slice i, column j) a quad of lanes
//     stores 4 consecutive slices (one 32-byte sector for fp64).
#include <cuda.h>
#include <cuda_runtime.h>

#include "kron_internal.h"
#include "ptx.cuh"

namespace kron {

namespace {

struct GemmArgs {
  int64_t rows;   // M * S  (rows of A)
  int64_t S;      // slices per row of T
  int P, Q;
  int64_t Wout;   // S * Q
  int64_t tiles_m;
  int tiles_n;
  int64_t ntiles;
  int nk;         // k-chunks per tile
};

template <typename T, int BM, int BN, int TM, int TN, int NS>
__global__ void __launch_bounds__(256, 1) kron_gemm_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                          const __grid_constant__ CUtensorMap tm_b, T *__restrict__ Y,
                                                          const GemmArgs g) {
  constexpr int ES = sizeof(T);
  constexpr int BK = 128 / ES;            // one 128-byte swizzle line of A per slice
  constexpr int VA = 16 / ES;             // p-values per LDS.128 of A
  constexpr int GM = BM / TM, GN = BN / TN;  // thread grid
  static_assert(GM * GN == 256, "256 threads");
  static_assert(GM % 4 == 0 && GN % 8 == 0, "warp = 4 x 8 threads");
  constexpr uint32_t A_BYTES = BM * BK * ES, B_BYTES = BK * BN * ES, STAGE = A_BYTES + B_BYTES;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + NS * STAGE);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WM = GM / 4;
  const int tm = (warp % WM) * 4 + (lane & 3);  // slice group
  const int tn = (warp / WM) * 8 + (lane >> 2); // column group

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
  }
  __syncthreads();

  const int64_t nsteps = g.ntiles * g.nk;  // this CTA walks tiles blockIdx.x, +gridDim.x, ...
  auto tile_of = [&](int64_t z, int64_t &tile, int &k) {
    const int64_t t = z / g.nk;
    k = (int)(z - t * g.nk);
    tile = blockIdx.x + t * gridDim.x;
  };
  auto issue = [&](int64_t z) {
    int64_t tile;
    int k;
    tile_of(z, tile, k);
    if (tile >= g.ntiles) return;
    const int st = (int)(z % NS);
    const int64_t mt = tile / g.tiles_n;
    const int nt = (int)(tile - mt * g.tiles_n);
    unsigned char *sa = base + st * STAGE;
    mbar_arrive_expect_tx(&bars[st], STAGE);
    tma_load_2d(sa, &tm_a, &bars[st], k * BK, (int)(mt * BM));
    tma_load_2d(sa + A_BYTES, &tm_b, &bars[st], nt * BN, k * BK);
  };
  if (tid == 0)
    for (int z = 0; z < NS; ++z) issue(z);

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int64_t z = 0;; ++z) {
    int64_t tile;
    int k;
    tile_of(z, tile, k);
    if (tile >= g.ntiles) break;
    const int st = (int)(z % NS);
    mbar_wait(&bars[st], (uint32_t)((z / NS) & 1));
    const unsigned char *sa = base + st * STAGE;
    const T *sb = reinterpret_cast<const T *>(sa + A_BYTES);
#pragma unroll
    for (int pp = 0; pp < BK; pp += VA) {
      T a[TM][VA];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int s = tm + GM * i;  // slice row of the A tile
        const uint32_t off = (uint32_t)s * 128u + (uint32_t)pp * ES;
        const unsigned char *src = sa + swz128(off);
        if constexpr (ES == 8) {
          const double2 v = *reinterpret_cast<const double2 *>(src);
          a[i][0] = v.x;
          a[i][1] = v.y;
        } else {
          const float4 v = *reinterpret_cast<const float4 *>(src);
          a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
      }
#pragma unroll
      for (int e = 0; e < VA; ++e) {
        T b[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = sb[(pp + e) * BN + tn + GN * j];
        if constexpr (ES == 4) {
          // FFMA2: two columns per instruction, a[i] broadcast
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float2 aa = make_float2(a[i][e], a[i][e]);
#pragma unroll
            for (int j = 0; j < TN; j += 2) {
              float2 c = __ffma2_rn(aa, make_float2(b[j], b[j + 1]), make_float2(acc[i][j], acc[i][j + 1]));
              acc[i][j] = c.x;
              acc[i][j + 1] = c.y;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i][e], b[j], acc[i][j]);
        }
      }
    }
    __syncthreads();  // stage st fully read
    if (tid == 0) issue(z + NS);
    if (k == g.nk - 1) {
      // epilogue: A row r = m*S + s  ->  Y[m, q*S + s]
      const int64_t mt = tile / g.tiles_n;
      const int nt = (int)(tile - mt * g.tiles_n);
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int64_t r = mt * BM + tm + GM * i;
        if (r < g.rows) {
          const int64_t m = r / g.S, s = r - m * g.S;
          T *yrow = Y + m * g.Wout + s;
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            const int q = nt * BN + tn + GN * j;
            if (q < g.Q) yrow[(int64_t)q * g.S] = acc[i][j];
          }
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
      }
    }
  }
}

struct GemmInst {
  int dtype, BM, BN, TM, TN, NS;
};
// fp64: 128x128 (Q >= 96) and 256x32 (small Q) tiles; fp32 the same shapes with 32-wide k chunks
const GemmInst kGemm[] = {
    {KRON_F64, 128, 128, 8, 8, 4},
    {KRON_F64, 256, 32, 8, 4, 4},
    {KRON_F32, 128, 128, 8, 8, 4},
    {KRON_F32, 256, 32, 8, 4, 4},
};

using GemmFn = void (*)(const CUtensorMap, const CUtensorMap, void *, const GemmArgs);

GemmFn gemm_kernel(int i) {
  switch (i) {
    case 0: return reinterpret_cast<GemmFn>(kron_gemm_kernel<double, 128, 128, 8, 8, 4>);
    case 1: return reinterpret_cast<GemmFn>(kron_gemm_kernel<double, 256, 32, 8, 4, 4>);
    case 2: return reinterpret_cast<GemmFn>(kron_gemm_kernel<float, 128, 128, 8, 8, 4>);
    case 3: return reinterpret_cast<GemmFn>(kron_gemm_kernel<float, 256, 32, 8, 4, 4>);
  }
  return nullptr;
}

int gemm_pick(int dtype, int Q) {
  const int small = Q <= 64 ? 1 : 0;
  return (dtype == KRON_F64 ? 0 : 2) + small;
}

}  // namespace

bool gemm_supported(int dtype, int64_t M, int64_t W, int P, int Q) {
  const int es = dtype == KRON_F32 ? 4 : 8;
  if (P < 48 || Q < 16) return false;                 // small factors: fused / generic kernels
  if ((int64_t)P * es % 16 || (int64_t)Q * es % 16) return false;  // TMA row strides
  const int64_t rows = M * (W / P);
  if (rows >= ((int64_t)1 << 31)) return false;       // TMA coordinates are int32
  return true;
}

int launch_gemm(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F, void *stream) {
  const int es = dtype == KRON_F32 ? 4 : 8;
  const int gi = gemm_pick(dtype, pp.Q);
  const GemmInst &gs = kGemm[gi];
  const int BK = 128 / es;
  GemmArgs g{};
  g.S = pp.W_in / pp.P;
  g.rows = M * g.S;
  g.P = pp.P;
  g.Q = pp.Q;
  g.Wout = g.S * pp.Q;
  g.tiles_m = (g.rows + gs.BM - 1) / gs.BM;
  g.tiles_n = (pp.Q + gs.BN - 1) / gs.BN;
  g.ntiles = g.tiles_m * g.tiles_n;
  g.nk = (pp.P + BK - 1) / BK;
  CUtensorMap ta, tb;
  {
    uint64_t dims[2] = {(uint64_t)pp.P, (uint64_t)g.rows};
    uint64_t strides[1] = {(uint64_t)pp.P * es};
    uint32_t box[2] = {(uint32_t)BK, (uint32_t)gs.BM};
    if (!encode_tmap(&ta, dtype, 2, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
  }
  {
    uint64_t dims[2] = {(uint64_t)pp.Q, (uint64_t)pp.P};
    uint64_t strides[1] = {(uint64_t)pp.Q * es};
    uint32_t box[2] = {(uint32_t)gs.BN, (uint32_t)BK};
    if (!encode_tmap(&tb, dtype, 2, F, dims, strides, box, false)) return (int)cudaErrorInvalidValue;
  }
  const size_t stage = (size_t)gs.BM * BK * es + (size_t)BK * gs.BN * es;
  const size_t smem = 1024 + gs.NS * stage + 8 * gs.NS;
  GemmFn k = gemm_kernel(gi);
  cudaError_t e = cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, 256, smem);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > g.ntiles) grid = g.ntiles;
  k<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(ta, tb, out, g);
  return (int)cudaGetLastError();
}

}  // namespace kron
