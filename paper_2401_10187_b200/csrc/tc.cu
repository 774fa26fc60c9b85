// tc.cu — NEXT-4: the fused fp32 chunk pair on Blackwell's 5th-generation tensor cores.
//
// A pair of P x P factors (P = 16 / 32) applied to a P^2 chunk is the sandwich (reading G23)
//     OUT[q2][q1] = sum_s F2[s][q2] * Z[s][q1],   Z[s][q1] = sum_p X[s][p] * F1[p][q1]
// with X[s][p] the chunk viewed as a P x P matrix (s = slice, p = element, Alg 1).  Here both
// contractions run as tcgen05.mma kind::tf32 with TMEM accumulators, batched over a tile of R chunks:
//   GEMM1  D1[(c,s)][q1] = sum_p X[(c,s)][p] . F1[p][q1]           M = 128 rows (c,s), N = P, K = P
//          A = the TMA-staged tile itself: with the 128B (P = 32) / 64B (P = 16) swizzle it is the canonical
//          K-major UMMA layout; B = F1^T, K-major, staged once per CTA.
//   GEMM2  D2[(c,q1)][q2] = sum_s Z[c][s][q1] . F2[s][q2]          M = 128 rows (c,q1), N = P, K = P
//          A = Z^T per chunk, K-major (the same swizzled layout as X): the transform warps read D1 from TMEM
//          (tcgen05.ld, one TMEM lane = one (c,s) row per thread) and scatter each row into column s of the
//          rows (c,q1) — for a fixed q1 a warp writes one contiguous swizzled row, conflict-free; B = F2^T,
//          K-major.  (An MN-major A operand would take vector stores, but kind::tf32 with an MN-major A
//          produced all-zero accumulators on this B200 — tools/tc_probe.cu — so the transpose is done by the
//          stores.)
//   epilogue: the transform warps read D2 (lane = (c,q1), registers = q2) and write OUT[q2][q1] over the
//          chunk in the chunk-fastest stream-out layout, from which four store warps write the direct-index
//          runs Y[row][u*(W/C) + g0 + c], u = q2*P + q1.
// Modes (reported separately from the fp32 CUDA-core path, north_star): TF32 — one MMA per K step; 3xTF32 —
// every operand split x = hi + lo with hi = x truncated to TF32 (exact in both parts) and the products
// hi.hi + hi.lo + lo.hi (+ lo.lo) accumulated in fp32 (relative error ~2^-21 per product, within the fp32 parity
// bar; small integers are exact, so integer data stays bit-exact).
// Warp roles (768 threads, one CTA per SM): warp 0 TMA producer, warp 1 MMA issuer (one thread) + TMEM owner,
// warps 4-11 and 12-19 two transform groups taking alternate tiles (warp w reads TMEM lanes 32*(w%4) .., the two
// warps of a lane quarter split the columns; each group owns its TMEM columns and lo buffer), so one group's
// split / Z staging / epilogue overlaps the other group's GEMMs; warps 20-23 store; warps 2-3 idle.
// Round 2 (second version): the hi parts are never written — kind::tf32 reads only the top 19 bits of each fp32
// operand word, so the TMA tile itself is X_hi and Z is staged once (as Z_hi) over the consumed tile, Z_lo in the
// group's lo buffer; 3xTF32 multiplies by [F_hi | F_lo] (N = 2P) in two MMAs per K step (A = hi, A = lo).
// C32 per pass: TF32 1.67 -> 1.52 ms (0.88 of HBM); 3xTF32 3.2 -> 2.20 ms (0.61 of HBM; round 1's mma.sync
// kernel 2.78 ms).  What remains: the transform groups wait on the MMAs ~60% of their time (ncu source view);
// with K = 8 per kind::tf32 MMA every A byte feeds only N MACs, so the operand reads, not the MMA rate, set the
// pace (DESIGN §5 B).
#include <cuda.h>
#include <cuda_runtime.h>

#include "kron_internal.h"
#include "ptx.cuh"

namespace kron {
namespace {

struct TcArgs {
  const float *F1, *F2;  // factor applied first (F^{f}) and second (F^{f-1}), P x P row-major, device
  float *Y;              // output T'[M][Wout]
  int64_t WC, Wout, M, ntiles;
  int tiles_k, R, stages;
};

// 16-byte granule XOR of the 1 KB-aligned rows of a K-major operand: 128B swizzle for 128-byte rows (P = 32),
// 64B swizzle (bits 4-5 ^= bits 7-8) for 64-byte rows (P = 16)
template <int P>
__device__ __forceinline__ uint32_t kswz(uint32_t off) {
  if constexpr (P == 32) return off ^ (((off >> 7) & 7u) << 4);
  else return off ^ (((off >> 7) & 3u) << 4);
}
// chunk-dependent granule XOR of the stream-out layout (conflict-free chunk-fastest reads, as the v6 kernels)
__device__ __forceinline__ uint32_t out_gx(uint32_t chunk) {
  const uint32_t g0 = chunk & 1u, g1 = (chunk >> 1) & 1u, g2 = (chunk >> 2) & 1u;
  return (g2 | (g1 << 1) | ((g0 ^ g1) << 2)) << 4;
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int P, bool X3>
__global__ void __launch_bounds__(768, 1) kron_tc_pair_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                              const TcArgs a) {
  constexpr int C = P * P;
  constexpr uint32_t CE = C * 4;                       // chunk bytes
  constexpr uint32_t ROWB = P * 4;                     // bytes per K-major row (one slice)
  constexpr uint32_t SBO_K = 8 * ROWB;                 // 8-row swizzle atom of the K-major operands
  constexpr uint32_t LAY_K = P == 32 ? 2u : 4u;        // UMMA layout type: 128B / 64B swizzle
  constexpr uint32_t A2M = 128 * P * 4;                // one M-tile of the K-major Z^T operand
  constexpr uint32_t FB = (uint32_t)C * 4 < 1024u ? 1024u : (uint32_t)C * 4;  // factor tile slot (1 KB-aligned)
  // 3xTF32: B = [F_hi | F_lo] along N (the two factor tiles are adjacent K-major row blocks), so one MMA with
  // A = X gives hi.hi | hi.lo and one with A = X_lo gives lo.hi | lo.lo; the epilogues add the two halves
  constexpr int NB = X3 ? 2 * P : P;                   // MMA N
  constexpr uint32_t ID1 = umma_idesc_tf32(128, NB, 0, 0);
  constexpr int NG = 2, NTW = 8, HP = P / 2;           // transform groups, warps per group, columns per warp
  const int R = a.R, S = a.stages;
  const uint32_t TILE = (uint32_t)R * CE;              // stage bytes (= the Z^T operand of the tile)
  const int MT = R * P / 128;                          // M-tiles of 128 rows per tile
  const uint32_t NCOL = (uint32_t)MT * 2 * NB;         // TMEM columns per group: D1 and D2 per M-tile

  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *xlo = base + (size_t)S * TILE;                     // per group: X lo, then Z lo (3xTF32)
  unsigned char *fT = xlo + (X3 ? (size_t)NG * TILE : 0);           // F1hi, F1lo, F2hi, F2lo (transposed)
  uint64_t *full = reinterpret_cast<uint64_t *>(fT + 4 * FB);
  uint64_t *empty = full + S, *cdone = empty + S;
  uint64_t *xrdy = cdone + S, *d1full = xrdy + NG, *a2rdy = d1full + NG, *d2full = a2rdy + NG;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(d2full + NG);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;

  // factors, transposed to K-major B operands: FT[q][p] = F[p][q] (hi / lo split in 3xTF32)
  for (int i = tid; i < C; i += 768) {
    const int p = i / P, q = i % P;
    const uint32_t o = kswz<P>((uint32_t)q * ROWB + (uint32_t)p * 4u);
    const float f1 = a.F1[i], f2 = a.F2[i];
    const float h1 = X3 ? tf32_hi(f1) : f1, h2 = X3 ? tf32_hi(f2) : f2;
    *reinterpret_cast<float *>(fT + o) = h1;
    *reinterpret_cast<float *>(fT + FB + o) = f1 - h1;
    *reinterpret_cast<float *>(fT + 2 * FB + o) = h2;
    *reinterpret_cast<float *>(fT + 3 * FB + o) = f2 - h2;
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4 * 32);    // every store lane
      mbar_init(&cdone[s], NTW * 32);  // every transform lane of the tile's group
    }
    for (int g = 0; g < NG; ++g) {
      mbar_init(&xrdy[g], NTW * 32);
      mbar_init(&d1full[g], 1);
      mbar_init(&a2rdy[g], NTW * 32);
      mbar_init(&d2full[g], 1);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  const uint32_t ncol_alloc = NG * NCOL <= 32    ? 32u
                              : NG * NCOL <= 64  ? 64u
                              : NG * NCOL <= 128 ? 128u
                              : NG * NCOL <= 256 ? 256u
                                                 : 512u;
  if (warp == 1) tmem_alloc(tmem_slot, ncol_alloc);
  fence_proxy_async_smem();  // the factor tiles (generic writes) are read by the tensor cores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % S;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    mbar_arrive_expect_tx(&full[st], TILE);
    // one box = R*P rows of P floats (<= 256 rows)
    tma_load_3d(base + (size_t)st * TILE, &tm_in, &full[st], 0, cb * R * P, rb);
  };

  if (warp == 0) {
    if (lane == 0)
      for (int it = 0; it < S; ++it) issue_load(it);
  } else if (warp == 1) {
    // ---------------- MMA issuer.  Tiles alternate between the two transform groups.  GEMM1's A operand is the
    // TMA tile itself: kind::tf32 reads only the top 19 bits of each fp32 word, i.e. the truncated hi part
    // (3xTF32 adds the MMA on the lo parts the group wrote to xlo).  MMAs into one accumulator are issued back to
    // back (k inner): interleaving the two M-tiles' chains measured slower (C32 TF32 3.05 -> 3.34 ms).
    if (lane == 0) {
      const uint32_t fa = smem_u32(fT);
      auto gemm = [&](uint32_t xa, uint32_t xl, uint32_t arow, uint32_t fofs, uint32_t d0) {
        for (int i = 0; i < MT; ++i) {
          const uint32_t d = d0 + (uint32_t)(i * 2 * NB);
#pragma unroll
          for (int k = 0; k < P / 8; ++k) {
            const uint32_t ko = (uint32_t)i * arow + (uint32_t)k * 32u;
            const uint64_t bh = umma_desc(fa + fofs + k * 32u, 16, SBO_K, LAY_K);
            umma_tf32(d, umma_desc(xa + ko, 16, SBO_K, LAY_K), bh, ID1, k > 0 ? 1u : 0u);
            if constexpr (X3) umma_tf32(d, umma_desc(xl + ko, 16, SBO_K, LAY_K), bh, ID1, 1u);
          }
        }
      };
      int64_t nt = 0;  // tiles of this CTA
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) ++nt;
      // GEMM1 of the next tile and GEMM2 of the oldest staged one are issued in whichever order their groups get
      // ready (polled): a fixed order made each group's epilogue wait for the other group's split
      int i1 = 0, i2 = 0;  // next tile for GEMM1 / GEMM2 (i2 <= i1 <= i2 + 2)
      while (i2 < nt) {
        if (i2 < i1 && mbar_try_wait(&a2rdy[i2 & 1], (uint32_t)((i2 >> 1) & 1))) {
          const int g = i2 & 1, st = i2 % S;
          tc_fence_after();
          gemm(smem_u32(base + (size_t)st * TILE), smem_u32(xlo + (size_t)g * TILE), A2M, 2 * FB,
               tmem + (uint32_t)g * NCOL + NB);
          umma_commit(&d2full[g]);
          ++i2;
        } else if (i1 < nt && i1 < i2 + 2 && mbar_try_wait(&xrdy[i1 & 1], (uint32_t)((i1 >> 1) & 1))) {
          const int g = i1 & 1, st = i1 % S;
          tc_fence_after();
          gemm(smem_u32(base + (size_t)st * TILE), smem_u32(xlo + (size_t)g * TILE), 128 * ROWB, 0,
               tmem + (uint32_t)g * NCOL);
          umma_commit(&d1full[g]);
          ++i1;
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + NG * NTW) {
    // ---------------- transform groups: group g takes tiles it = g, g+2, ...: lo split of X, D1 -> Z^T operand
    // (hi = z over the consumed tile, lo = z - hi in xlo), D2 -> stream-out layout over the tile
    const int g = (warp - 4) / NTW, wg = (warp - 4) % NTW;
    const int q = warp & 3, hc = wg >> 2, tt = wg * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t)g * NCOL + ((uint32_t)(32 * q) << 16) + (uint32_t)(hc * HP);
    unsigned char *xl = xlo + (size_t)g * TILE;
    // this warp's HP accumulator columns of D (3xTF32: the sum of the hi-factor and lo-factor halves)
    auto ldacc = [&](uint32_t col, float (&v)[HP]) {
      uint32_t r[HP];
      if constexpr (P == 32) tmem_ld16(lane_base + col, r);
      else tmem_ld8(lane_base + col, r);
      if constexpr (X3) {
        uint32_t r2[HP];
        if constexpr (P == 32) tmem_ld16(lane_base + col + P, r2);
        else tmem_ld8(lane_base + col + P, r2);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < HP; ++j) v[j] = __uint_as_float(r[j]) + __uint_as_float(r2[j]);
      } else {
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < HP; ++j) v[j] = __uint_as_float(r[j]);
      }
    };
    for (int it = g;; it += NG) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t ph = (uint32_t)((it >> 1) & 1);
      unsigned char *xt = base + (size_t)st * TILE;
      mbar_wait(&full[st], (uint32_t)((it / S) & 1));
      if constexpr (X3) {
        for (uint32_t e = (uint32_t)tt; e < TILE / 16u; e += NTW * 32u) {
          const float4 x = *reinterpret_cast<const float4 *>(xt + e * 16u);
          *reinterpret_cast<float4 *>(xl + e * 16u) =
              make_float4(x.x - tf32_hi(x.x), x.y - tf32_hi(x.y), x.z - tf32_hi(x.z), x.w - tf32_hi(x.w));
        }
        fence_proxy_async_smem();
      }
      mbar_arrive(&xrdy[g]);
      // Z rows: TMEM lane 32q + lane of M-tile i is row m = i*128 + 32q + lane = (chunk c, slice s)
      mbar_wait(&d1full[g], ph);
      tc_fence_after();
      for (int i = 0; i < MT; ++i) {
        float v[HP];
        ldacc((uint32_t)(i * 2 * NB), v);
        const int m = 32 * q + lane, cl = m / P, s = m % P;  // chunk within the M-tile, slice
        // K-major Z^T: element (row cl*P + q1, column s) of this M-tile's operand (this warp's half of q1)
        unsigned char *zh = xt + (size_t)i * A2M;
#pragma unroll
        for (int j = 0; j < HP; ++j) {
          const int q1 = hc * HP + j;
          const uint32_t o = kswz<P>((uint32_t)(cl * P + q1) * ROWB + (uint32_t)s * 4u);
          *reinterpret_cast<float *>(zh + o) = v[j];
          if constexpr (X3) *reinterpret_cast<float *>(xl + (size_t)i * A2M + o) = v[j] - tf32_hi(v[j]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&a2rdy[g]);
      // OUT rows: TMEM lane of M-tile i = (chunk c, q1), registers q2 -> composite column u = q2*P + q1 of chunk
      // c, written over the tile in the stream-out layout swz128(u*4) ^ gx(c)
      mbar_wait(&d2full[g], ph);
      tc_fence_after();
      for (int i = 0; i < MT; ++i) {
        float v[HP];
        ldacc((uint32_t)(i * 2 * NB + NB), v);
        const int m = 32 * q + lane, c = i * (128 / P) + m / P, q1 = m % P;
        unsigned char *ch = xt + (uint32_t)c * CE;
        const uint32_t gx = out_gx((uint32_t)c);
#pragma unroll
        for (int j = 0; j < HP; ++j) {
          const uint32_t u = (uint32_t)((hc * HP + j) * P + q1);
          *reinterpret_cast<float *>(ch + (swz128(u * 4u) ^ gx)) = v[j];
        }
      }
      tc_fence_before();
      mbar_arrive(&cdone[st]);
    }
  } else if (warp >= 4 + NG * NTW) {
    // ---------------- store warps: chunk-fastest stream-out, Y[row][u*(W/C) + cb*R + g]: 8 consecutive chunks
    // = one 32-byte run per composite column, four columns per instruction
    const int sw = warp - 4 - NG * NTW;
    const int gl = lane & 7, uq = lane >> 3;
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      mbar_wait_sleep(&cdone[st], par);
      const unsigned char *buf = base + (size_t)st * TILE;
      const int rb = (int)(tile / a.tiles_k), cbk = (int)(tile - (int64_t)rb * a.tiles_k);
      for (int oct = 0; oct < R / 8; ++oct) {
        const uint32_t gg = (uint32_t)(oct * 8 + gl);
        const uint32_t gx = out_gx(gg);
        const unsigned char *ch = buf + gg * CE;
        const int64_t gcol = (int64_t)cbk * R + gg;
        if (rb < a.M && gcol < a.WC) {
          float *yg = a.Y + (int64_t)rb * a.Wout + gcol;
          const int64_t wc = a.WC;
#pragma unroll 2
          for (int u16 = sw; u16 < C / 16; u16 += 4) {
            const uint32_t u = (uint32_t)(u16 * 16 + uq * 4);
            const float4 v = *reinterpret_cast<const float4 *>(ch + (swz128(u * 4u) ^ gx));
            float *p = yg + (int64_t)u * wc;
            p[0] = v.x;
            p[wc] = v.y;
            p[2 * wc] = v.z;
            p[3 * wc] = v.w;
          }
        }
      }
      __syncwarp();
      mbar_arrive(&empty[st]);
      if (sw == 0) {
        if (lane == 0) {
          mbar_wait_sleep(&empty[st], par);
          fence_proxy_async_smem();
          issue_load(it + S);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, ncol_alloc);
  }
}

template <int P, bool X3>
size_t tc_smem(int R, int S) {
  const size_t tile = (size_t)R * P * P * 4;
  const size_t fb = (size_t)P * P * 4 < 1024 ? 1024 : (size_t)P * P * 4;
  return 1024 + (size_t)S * tile + (X3 ? 2 * tile : 0) + 4 * fb + 8 * (3 * S + 8) + 16;
}

}  // namespace

// Tile geometry of the tensor-core pair (host): R chunks per tile (P = 32: 8 -> 32-byte runs, two M-tiles;
// P = 16: 16 -> 64-byte runs, two M-tiles) and as many ring stages as fit 227 KB.
bool tc_geometry(int P, int mode, int64_t W, PassPlan *pp) {
  if (P != 16 && P != 32) return false;
  const int R = P == 32 ? 8 : 16;
  const int64_t C = (int64_t)P * P;
  if (W % (R * C)) return false;
  const bool x3 = mode == 2;
  int S = 0;
  for (int s = 2; s <= 8; ++s) {
    const size_t b = P == 32 ? (x3 ? tc_smem<32, true>(R, s) : tc_smem<32, false>(R, s))
                             : (x3 ? tc_smem<16, true>(R, s) : tc_smem<16, false>(R, s));
    if (b <= 227 * 1024) S = s;
  }
  if (S < 2) return false;
  pp->kind = KIND_FUSED;
  pp->nf = 2;
  pp->P = pp->Q = P;
  pp->C = pp->Qc = C;
  pp->R = R;
  pp->tileK = R * C;
  pp->tileM = 1;
  pp->stages = S;
  pp->nout = 0;
  pp->tc_mode = mode;
  return true;
}

int launch_tc(const PassPlan &pp, int64_t M, const void *in, void *out, const void *const *Fgroup, void *stream) {
  const int P = pp.P, R = pp.R, S = pp.stages;
  const bool x3 = pp.tc_mode == 2;
  const int64_t W = pp.W_in, C = pp.C;
  TcArgs a{};
  a.F1 = static_cast<const float *>(Fgroup[0]);
  a.F2 = static_cast<const float *>(Fgroup[1]);
  a.Y = static_cast<float *>(out);
  a.WC = W / C;
  a.Wout = pp.W_out;
  a.M = M;
  a.R = R;
  a.stages = S;
  a.tiles_k = (int)(a.WC / R);
  a.ntiles = M * a.tiles_k;
  // X viewed as rows of P floats (one slice each): [M][W/P][P], boxes of R*P slices of one row
  CUtensorMap tin;
  const uint64_t dims[3] = {(uint64_t)P, (uint64_t)(W / P), (uint64_t)M};
  const uint64_t strides[2] = {(uint64_t)P * 4, (uint64_t)W * 4};
  const uint32_t box[3] = {(uint32_t)P, (uint32_t)(R * P), 1};
  if (!encode_tmap_sw(&tin, KRON_F32, 3, in, dims, strides, box, P * 4)) return (int)cudaErrorInvalidValue;
  using K = void (*)(const CUtensorMap, const TcArgs);
  K k = P == 32 ? (x3 ? kron_tc_pair_kernel<32, true> : kron_tc_pair_kernel<32, false>)
                : (x3 ? kron_tc_pair_kernel<16, true> : kron_tc_pair_kernel<16, false>);
  const size_t smem = P == 32 ? (x3 ? tc_smem<32, true>(R, S) : tc_smem<32, false>(R, S))
                              : (x3 ? tc_smem<16, true>(R, S) : tc_smem<16, false>(R, S));
  const int slots = kernel_slots((const void *)k, 768, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > a.ntiles) grid = a.ntiles;
  k<<<(unsigned)grid, 768, smem, (cudaStream_t)stream>>>(tin, a);
  return (int)cudaGetLastError();
}

}  // namespace kron
