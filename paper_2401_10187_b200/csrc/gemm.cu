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

#include <cstdlib>

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

// ------------------------------------------------------------------ fp32 large-P pass, round 2 (sgemm)
//
// The fp32 GEMM above (TN = 4 columns per thread read as scalar LDS with stride GN) issues 24 shared loads per
// 64 FFMA2 and reached 0.34 (P = 64) / 0.54 (P = 128) of the FP32 peak on the Fig 11 workloads.  This kernel
// reorganises the thread tile around FFMA2's broadcast operand form `FFMA2 acc(q,q+1), x.F32, F(q,q+1).F32x2`:
//   * every lane of a warp shares the warp's QT-column range [q0, q0+QT) and owns RS = 8 slices
//     s = sg*256 + lane + 32*i, so a factor row segment F[p][q0..q0+QT) is one broadcast LDS.128 per 4 columns
//     (1 wavefront) and feeds 8 slices;
//   * the slices' elements come from the TMA-staged [slice][32 p] 128-byte lines (128B swizzle: lanes 0-7 of a
//     phase hit 8 distinct 16-byte chunks), one LDS.128 per 4 p per slice;
//   -> per 4 p: 8 + QT/4*4 shared loads for 4*8*QT/2 FFMA2 (QT = 16: 24 loads per 256 FFMA2);
//   * F (padded to whole 32-p chunks, zero rows) stays resident in shared memory for the CTA's life;
//   * the epilogue stores from registers: for a fixed (slice i, column q) the warp's 32 lanes hold 32
//     consecutive slices, i.e. 128 contiguous bytes of Y[m, q*S + s] (the direct-index store).
// CTA = 8 warps = QR column ranges x SG = 8/QR slice groups; a tile is SG*256 slices x QR*QT columns.
struct SgemmArgs {
  int64_t ntiles;
  int rows;   // M * S  (< 2^31: TMA coordinates)
  int S;      // slices per row of T
  int P, Q;
  int64_t Wout;
  int nk;     // 32-p chunks
};

__device__ __forceinline__ void st_global_f32(float *p, float v) { asm("st.global.f32 [%0], %1;" ::"l"(p), "f"(v)); }

template <int QT, int QR, int SG, int RS, int NS>
__global__ void __launch_bounds__(QR *SG * 32, 1) kron_sgemm_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                  const float *__restrict__ F, float *__restrict__ Y,
                                                                  const SgemmArgs g) {
  constexpr int NT = QR * SG * 32, SL = SG * 32 * RS, QTILE = QT * QR, QP = QT / 2;
  static_assert(SL % 256 == 0, "whole 256-row TMA boxes");
  constexpr uint32_t STAGE = SL * 128u;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float *Fs = reinterpret_cast<float *>(base + NS * STAGE);  // [nk*32][QTILE]
  uint64_t *bars = reinterpret_cast<uint64_t *>(Fs + g.nk * 32 * QTILE);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int qr = warp % QR, sg = warp / QR, q0 = qr * QT;

  for (int i = tid; i < g.nk * 32 * QTILE; i += NT) {
    const int p = i / QTILE, q = i - p * QTILE;
    Fs[i] = (p < g.P && q < g.Q) ? F[(int64_t)p * g.Q + q] : 0.f;
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_a);
  }
  __syncthreads();

  auto issue = [&](int64_t z) {
    const int64_t t = z / g.nk;
    const int k = (int)(z - t * g.nk);
    const int64_t tile = blockIdx.x + t * gridDim.x;
    if (tile >= g.ntiles) return;
    const int st = (int)(z % NS);
    unsigned char *sa = base + st * STAGE;
    mbar_arrive_expect_tx(&bars[st], STAGE);
#pragma unroll
    for (int b = 0; b < SL / 256; ++b) tma_load_2d(sa + b * 256 * 128, &tm_a, &bars[st], k * 32, (int)(tile * SL) + b * 256);
  };
  if (tid == 0)
    for (int z = 0; z < NS; ++z) issue(z);

  float2 acc[RS][QP];
#pragma unroll
  for (int i = 0; i < RS; ++i)
#pragma unroll
    for (int j = 0; j < QP; ++j) acc[i][j] = make_float2(0.f, 0.f);

  const bool active = q0 < g.Q;
  const uint32_t xsw = (uint32_t)(lane & 7) << 4;  // 128B swizzle of the lane's slice rows (sg*256 + 32i = 0 mod 8)
  for (int64_t z = 0;; ++z) {
    const int64_t t = z / g.nk;
    const int k = (int)(z - t * g.nk);
    const int64_t tile = blockIdx.x + t * gridDim.x;
    if (tile >= g.ntiles) break;
    const int st = (int)(z % NS);
    mbar_wait(&bars[st], (uint32_t)((z / NS) & 1));
    if (active) {
      const unsigned char *xs = base + st * STAGE + (size_t)(sg * 32 * RS + lane) * 128;
      const float *fk = Fs + (k * 32) * QTILE + q0;
#pragma unroll 2
      for (int pc = 0; pc < 8; ++pc) {
        float4 xv[RS];
#pragma unroll
        for (int i = 0; i < RS; ++i)
          xv[i] = *reinterpret_cast<const float4 *>(xs + i * 32 * 128 + (((uint32_t)pc << 4) ^ xsw));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float4 fv[QT / 4];
#pragma unroll
          for (int j = 0; j < QT / 4; ++j) fv[j] = *reinterpret_cast<const float4 *>(fk + (pc * 4 + e) * QTILE + 4 * j);
          // factor pair outer: consecutive FFMA2s share the F pair operand (W64 47.0 -> 45.7 ms against the
          // slice-outer order)
#pragma unroll
          for (int j = 0; j < QP; ++j) {
            const float2 ff = (j & 1) ? make_float2(fv[j >> 1].z, fv[j >> 1].w) : make_float2(fv[j >> 1].x, fv[j >> 1].y);
#pragma unroll
            for (int i = 0; i < RS; ++i) {
              const float xe = e == 0 ? xv[i].x : e == 1 ? xv[i].y : e == 2 ? xv[i].z : xv[i].w;
              acc[i][j] = __ffma2_rn(make_float2(xe, xe), ff, acc[i][j]);
            }
          }
        }
      }
    }
    __syncthreads();  // stage st fully read
    if (tid == 0) issue(z + NS);
    if (k == g.nk - 1 && active) {
      // one division per tile; slice i+1 is 32 slices on (s += 32, carrying into m); a 64-bit row pointer and
      // 32-bit offsets s + q*S (< Wout < 2^31)
      const int r0 = (int)(tile * SL) + sg * 32 * RS + lane;
      int m = r0 / g.S, sidx = r0 - m * g.S;
      const bool fullq = q0 + QT <= g.Q;
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        if (i > 0) {
          sidx += 32;
          while (sidx >= g.S) {
            sidx -= g.S;
            ++m;
          }
        }
        if (r0 + 32 * i < g.rows) {
          float *yrow = Y + (int64_t)m * g.Wout;
          asm volatile("" : "+l"(yrow));  // keep the row pointer: each store is then one IMAD.WIDE.U32 off, 4, yrow
          uint32_t off = (uint32_t)(sidx + q0 * g.S);
          const uint32_t S = (uint32_t)g.S;
          if (fullq) {
#pragma unroll
            for (int j = 0; j < QP; ++j) {
              st_global_f32(yrow + off, acc[i][j].x);
              off += S;
              st_global_f32(yrow + off, acc[i][j].y);
              off += S;
            }
          } else {
#pragma unroll
            for (int j = 0; j < QP; ++j) {
              if (q0 + 2 * j < g.Q) st_global_f32(yrow + off, acc[i][j].x);
              off += S;
              if (q0 + 2 * j + 1 < g.Q) st_global_f32(yrow + off, acc[i][j].y);
              off += S;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < QP; ++j) acc[i][j] = make_float2(0.f, 0.f);
      }
    }
  }
}

template <int QT, int QR, int SG, int RS, int NS>
int launch_sgemm_t(const PassPlan &pp, int64_t M, const void *in, void *out, const void *F, void *stream) {
  constexpr int SL = SG * 32 * RS, QTILE = QT * QR, NT = QR * SG * 32;
  SgemmArgs g{};
  g.S = (int)(pp.W_in / pp.P);
  g.rows = (int)(M * g.S);
  g.P = pp.P;
  g.Q = pp.Q;
  g.Wout = (int64_t)g.S * pp.Q;
  g.nk = (pp.P + 31) / 32;
  g.ntiles = ((int64_t)g.rows + SL - 1) / SL;
  CUtensorMap ta;
  uint64_t dims[2] = {(uint64_t)pp.P, (uint64_t)g.rows};
  uint64_t strides[1] = {(uint64_t)pp.P * 4};
  uint32_t box[2] = {32, 256};
  if (!encode_tmap(&ta, KRON_F32, 2, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
  const size_t smem = 1024 + (size_t)NS * SL * 128 + (size_t)g.nk * 32 * QTILE * 4 + 8 * NS;
  auto k = kron_sgemm_kernel<QT, QR, SG, RS, NS>;
  const int slots = kernel_slots((const void *)k, NT, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > g.ntiles) grid = g.ntiles;
  k<<<(unsigned)grid, NT, smem, (cudaStream_t)stream>>>(ta, (const float *)F, (float *)out, g);
  return (int)cudaGetLastError();
}

// QT x QR column tile and stage count of the sgemm instance for (P, Q); 0 = not eligible (the old kernel runs)
int sgemm_pick(int64_t M, int64_t W, int P, int Q) {
  if (P % 4 || Q % 16 || Q > 128) return 0;
  if (M * (W / P) >= ((int64_t)1 << 31) - 1024) return 0;
  const int nk = (P + 31) / 32;
  if (Q <= 32) return nk * 32 * 32 * 4 <= 32768 ? 1 : 0;   // QT 8 x QR 4, 512 slices, 3 stages
  if (Q <= 64) return nk * 32 * 64 * 4 <= 32768 ? 2 : 0;   // QT 16 x QR 4, 512 slices, 3 stages
  return nk * 32 * 128 * 4 <= 65536 ? 3 : 0;               // QT 16 x QR 8, 256 slices, 4 stages
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


// ------------------------------------------------------------------ fp64 tensor-core path (DMMA)
//
// fp64 large-P passes on the FP64 tensor cores: mma.sync.m16n8k4 f64 (SASS DMMA; tcgen05 has no f64
// kind).  The day-1 microbenchmark measured 37.1 TF for DMMA — the same peak as DFMA — but one DMMA
// does the work of 16 DFMA instructions, so the issue slots are free for operand loads and the
// epilogue.  CTA: 8 warps along the slice dimension, each a 32 (slices) x 32 (q) warp tile = 2 x 4
// MMA tiles.  A (slices x P) and F (P x Q) stream through a 3-stage TMA ring in 256-byte rows
// (3-D boxes {16, 2, rows} with the 128B swizzle: the two 128-byte lines of a row get different XOR
// patterns, which makes both fragment gathers bank-conflict free); the epilogue writes C fragments
// straight to Y[m, q*S + s] (8 consecutive slices = 64 bytes per column).
//
// NSW > 0: store-warp epilogue.  ncu on config D1 put 16% of the stall samples in the register epilogue
// (32 scattered 8-byte stores per lane while every compute warp of the CTA, finishing the same tile,
// leaves the DMMA pipe idle).  With store warps the compute warps drop the tile's C block into a
// shared-memory staging tile [q][row] (one STS per element, then straight on to the next tile) and NSW
// warps stream it out: for each column q the BM consecutive slices are one contiguous run of Y
// (512 bytes per store instruction, 16 bytes per lane).
template <int NWARP, int NS, int WN, int NSW = 0>
__global__ void __launch_bounds__((NWARP + 1 + NSW) * 32, 1) kron_dmma_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                             const __grid_constant__ CUtensorMap tm_b,
                                                                             double *__restrict__ Y, const GemmArgs g) {
  // WN warps along q (BN = 32*WN columns per CTA tile): with WN = 4 a Q = 128 factor is one column tile,
  // so every A row block is fetched from HBM once instead of once per 32 columns
  constexpr int BK = 32, WTM = 32, BM = (NWARP / WN) * WTM, BN = WN * 32;
  constexpr uint32_t A_BYTES = BM * BK * 8, B_BYTES = BK * BN * 8, STAGE = A_BYTES + B_BYTES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double *stg = reinterpret_cast<double *>(base + NS * STAGE);  // NSW > 0: [BN][BM] staging tile
  uint64_t *full = reinterpret_cast<uint64_t *>(base + NS * STAGE + (NSW > 0 ? (size_t)BM * BN * 8 : 0));
  uint64_t *empty = full + NS;
  uint64_t *sfull = empty + NS, *sempty = sfull + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // fragment coordinates: group (row/col) and thread-in-group (k)

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP * 32);
    }
    if (NSW > 0) {
      mbar_init(sfull, NWARP * 32);
      mbar_init(sempty, NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
  }
  __syncthreads();

  auto tile_of = [&](int64_t z, int64_t &tile, int &k) {
    const int64_t t = z / g.nk;
    k = (int)(z - t * g.nk);
    tile = blockIdx.x + t * gridDim.x;
  };

  if (warp == NWARP) {
    // ---------------- producer warp: the stage ring never waits on a CTA-wide barrier
    if (lane == 0) {
      for (int64_t z = 0;; ++z) {
        int64_t tile;
        int k;
        tile_of(z, tile, k);
        if (tile >= g.ntiles) break;
        const int st = (int)(z % NS);
        if (z >= NS) mbar_wait(&empty[st], (uint32_t)(((z / NS) - 1) & 1));
        const int64_t mt = tile / g.tiles_n;
        const int nt = (int)(tile - mt * g.tiles_n);
        unsigned char *sa = base + st * STAGE;
        mbar_arrive_expect_tx(&full[st], STAGE);
        tma_load_3d(sa, &tm_a, &full[st], 0, k * (BK / 16), (int)(mt * BM));
        for (int j = 0; j < WN; ++j)  // one [BK][32] slab (256-byte rows) per warp column
          tma_load_3d(sa + A_BYTES + j * (BK * 256), &tm_b, &full[st], 0, nt * (BN / 16) + 2 * j, k * BK);
      }
    }
    return;
  }
  if (NSW > 0 && warp > NWARP) {
    // ---------------- store warps: staging column q -> Y[m, q*S + s] for the BM rows of the tile
    const int sw = warp - NWARP - 1;
    for (int64_t t = 0;; ++t) {
      const int64_t tile = blockIdx.x + t * gridDim.x;
      if (tile >= g.ntiles) break;
      mbar_wait_sleep(sfull, (uint32_t)(t & 1));
      const int64_t mt0 = tile / g.tiles_n;
      const int ntile = (int)(tile - mt0 * g.tiles_n);
      for (int rb = 0; rb < BM; rb += 64) {
        const int64_t r0 = mt0 * BM + rb + 2 * lane;  // this lane's two rows
        const int64_t m0 = r0 / g.S, s0 = r0 - m0 * g.S;
        const bool pair = r0 + 1 < g.rows && s0 + 1 < g.S && (s0 & 1) == 0 && (g.S & 1) == 0;
        for (int q = sw; q < BN; q += NSW) {
          const int qg = ntile * BN + q;
          if (qg >= g.Q) break;
          const double2 v = *reinterpret_cast<const double2 *>(stg + (size_t)q * BM + ((rb + 2 * lane) ^ (4 * ((q >> 1) & 3))));
          if (pair) {
            *reinterpret_cast<double2 *>(Y + m0 * g.Wout + (int64_t)qg * g.S + s0) = v;
          } else {
            if (r0 < g.rows) Y[m0 * g.Wout + (int64_t)qg * g.S + s0] = v.x;
            if (r0 + 1 < g.rows) {
              const int64_t m1 = (r0 + 1) / g.S, s1 = (r0 + 1) - m1 * g.S;
              Y[m1 * g.Wout + (int64_t)qg * g.S + s1] = v.y;
            }
          }
        }
      }
      __syncwarp();
      mbar_arrive(sempty);
    }
    return;
  }

  const int wm = warp / WN, wn = warp % WN;
  // A fragment bases: rows r = wm*32 + mt*16 + gq + 8v, two 128-byte lines (k < 16, k >= 16)
  uint32_t abase[2][2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t row = (uint32_t)(wm * WTM + mt * 16 + gq + 8 * v);
        const uint32_t line = 2 * row + h;
        abase[mt][v][h] = line * 128u + (((uint32_t)tq * 8u) ^ ((line & 7u) << 4));
      }
  // B fragment bases: element (k = k0 + tq, n = nt*8 + gq): line = 2k + n/16
  uint32_t bbase[4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const uint32_t n = (uint32_t)(nt * 8 + gq), h = n >> 4, x = (n & 15u) * 8u;
    const uint32_t line0 = 2u * (uint32_t)tq + h;
    bbase[nt] = line0 * 128u + (x ^ ((line0 & 7u) << 4));
  }

  double acc[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0;

  for (int64_t z = 0;; ++z) {
    int64_t tile;
    int k;
    tile_of(z, tile, k);
    if (tile >= g.ntiles) break;
    const int st = (int)(z % NS);
    mbar_wait(&full[st], (uint32_t)((z / NS) & 1));
    const unsigned char *sa = base + st * STAGE;
    const unsigned char *sb = sa + A_BYTES + wn * (BK * 256);
#pragma unroll
    for (int k0 = 0; k0 < BK; k0 += 4) {
      const int h = k0 >> 4;
      const uint32_t kx = (uint32_t)(k0 & 15) * 8u;
      double a[2][2], b[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v = 0; v < 2; ++v) a[mt][v] = *reinterpret_cast<const double *>(sa + (abase[mt][v][h] ^ kx));
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = *reinterpret_cast<const double *>(sb + bbase[nt] + (uint32_t)k0 * 256u);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_m16n8k4(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
    mbar_arrive(&empty[st]);  // this thread is done with stage st
    if (NSW > 0 && k == g.nk - 1) {
      // hand the C block to the store warps through the staging tile [q][row]
      const int64_t t = z / g.nk;
      if (t >= 1) mbar_wait(sempty, (uint32_t)((t - 1) & 1));
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int row = wm * WTM + mt * 16 + gq + 8 * (e >> 1), col = wn * 32 + nt * 8 + 2 * tq + (e & 1);
            // rows XOR 4*((col/2) % 4): the four tq lanes of an accumulator column pair land in four different
            // 8-row bank groups (unswizzled, the 1 KB column stride put them on the same banks: ncu counted
            // 8 wavefronts per STS.64 against 2 ideal, profiles/r02_banks_D1.json); row pairs stay adjacent
            stg[(size_t)col * BM + (row ^ (4 * ((col >> 1) & 3)))] = acc[mt][nt][e];
            acc[mt][nt][e] = 0.0;
          }
      mbar_arrive(sfull);
    } else if (k == g.nk - 1) {
      // epilogue: C[row][col] with row = A row (m*S + s), col = q -> Y[m, q*S + s]
      const int64_t mt0 = tile / g.tiles_n;
      const int ntile = (int)(tile - mt0 * g.tiles_n);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1) {
          const int64_t r = mt0 * BM + wm * WTM + mt * 16 + gq + 8 * v1;
          if (r < g.rows) {
            const int64_t m = r / g.S, s = r - m * g.S;
            double *yrow = Y + m * g.Wout + s;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
              for (int v0 = 0; v0 < 2; ++v0) {
                const int q = ntile * BN + wn * 32 + nt * 8 + 2 * tq + v0;
                if (q < g.Q) yrow[(int64_t)q * g.S] = acc[mt][nt][v1 * 2 + v0];
              }
          }
        }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0;
    }
  }
}

template <int NWARP, int NS, int WN, int NSW = 0>
int launch_dmma_t(const PassPlan &pp, int64_t M, const void *in, void *out, const void *F, void *stream) {
  constexpr int BK = 32, BN = WN * 32, BM = (NWARP / WN) * 32;
  GemmArgs g{};
  g.S = pp.W_in / pp.P;
  g.rows = M * g.S;
  g.P = pp.P;
  g.Q = pp.Q;
  g.Wout = g.S * pp.Q;
  g.tiles_m = (g.rows + BM - 1) / BM;
  g.tiles_n = (pp.Q + BN - 1) / BN;
  g.ntiles = g.tiles_m * g.tiles_n;
  g.nk = (pp.P + BK - 1) / BK;
  CUtensorMap ta, tb;
  {
    uint64_t dims[3] = {16, (uint64_t)pp.P / 16, (uint64_t)g.rows};
    uint64_t strides[2] = {128, (uint64_t)pp.P * 8};
    uint32_t box[3] = {16, 2, (uint32_t)BM};
    if (!encode_tmap(&ta, KRON_F64, 3, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
  }
  {
    uint64_t dims[3] = {16, (uint64_t)(pp.Q + 15) / 16, (uint64_t)pp.P};
    uint64_t strides[2] = {128, (uint64_t)pp.Q * 8};
    uint32_t box[3] = {16, 2, (uint32_t)BK};
    if (!encode_tmap(&tb, KRON_F64, 3, F, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
  }
  const size_t smem = 1024 + NS * ((size_t)BM * BK * 8 + (size_t)BK * BN * 8) + 16 * NS +
                     (NSW > 0 ? (size_t)BM * BN * 8 + 16 : 0);
  auto k = kron_dmma_kernel<NWARP, NS, WN, NSW>;
  const int threads = (NWARP + 1 + NSW) * 32;
  const int slots = kernel_slots((const void *)k, threads, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > g.ntiles) grid = g.ntiles;
  k<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(ta, tb, (double *)out, g);
  return (int)cudaGetLastError();
}

int launch_dmma(const PassPlan &pp, int64_t M, const void *in, void *out, const void *F, void *stream) {
  // store-warp epilogue (NSW = 2): D1 18.53 -> 15.82 ms (0.75 -> 0.88 of the FP64 peak)
  if (pp.Q % 128 == 0) return launch_dmma_t<8, 3, 4, 2>(pp, M, in, out, F, stream);
  // (the Q = 32 tile, BM = 256, has no shared memory left for a staging tile beside a 3-stage ring; a
  //  2-stage ring with store warps measured 0.408 vs 0.399 ms on D2)
  // Q <= 32 (config D2's last factor): two CTAs per SM of 4 warps, BM = 128, 2 stages: 0.0694 -> 0.0676 ms per
  // pass (BM = 128 with 3 stages, one CTA per SM: 0.088 ms)
  if (pp.Q <= 32) return launch_dmma_t<4, 2, 1>(pp, M, in, out, F, stream);
  return launch_dmma_t<8, 3, 1>(pp, M, in, out, F, stream);
}
}  // namespace

bool sgemm_supported(int64_t M, int64_t W, int P, int Q) { return sgemm_pick(M, W, P, Q) != 0; }

bool gemm_supported(int dtype, int64_t M, int64_t W, int P, int Q) {
  const int es = dtype == KRON_F32 ? 4 : 8;
  if (P < 48 || Q < 16) return false;                 // small factors: fused / generic kernels
  if ((int64_t)P * es % 16 || (int64_t)Q * es % 16) return false;  // TMA row strides
  const int64_t rows = M * (W / P);
  if (rows >= ((int64_t)1 << 31)) return false;       // TMA coordinates are int32
  return true;
}

int launch_gemm(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F, void *stream) {
  if (dtype == KRON_F32 && pp.variant == 2) {
    // measured on the Fig 11 workloads (tools/gpu_sgemm_var.sh): 2 CTAs of 4 warps per SM, 16 warps with RS = 4 or
    // QT = 8, unroll 1 / 4 of the p-quad loop were all 1-10% slower than these
    switch (sgemm_pick(M, pp.W_in, pp.P, pp.Q)) {
      case 1: return launch_sgemm_t<8, 4, 2, 8, 3>(pp, M, in, out, F, stream);
      case 2: return launch_sgemm_t<16, 4, 2, 8, 3>(pp, M, in, out, F, stream);
      case 3: return launch_sgemm_t<16, 8, 1, 8, 4>(pp, M, in, out, F, stream);
    }  // not eligible at this M: the register-tiled kernel below
  }
  if (dtype == KRON_F64 && pp.variant == 1 && pp.P % 16 == 0 && pp.Q % 16 == 0 && !getenv("KRON_NO_DMMA"))
    return launch_dmma(pp, M, in, out, F, stream);
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
  const int slots = kernel_slots((const void *)k, 256, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > g.ntiles) grid = g.ntiles;
  k<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(ta, tb, out, g);
  return (int)cudaGetLastError();
}

}  // namespace kron
