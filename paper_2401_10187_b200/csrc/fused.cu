// fused.cu — the small-P fused sliced-multiply kernel for sm_100a.
//
// One launch applies a GROUP of consecutive square factors F^f, F^{f-1}, ..., F^{f-nf+1}
// (processing order N -> 1, Algorithm 1) to a row-major intermediate T[M][W]:
//
//   a2  a persistent CTA streams tiles of tileM rows x tileK = R*C contiguous columns (C = P^nf,
//       "the P^k-element chunk") from HBM into shared memory with TMA
//       (cp.async.bulk.tensor, 128B swizzle) through an mbarrier ring of `stages` buffers;
//   a3  the group's factors sit in shared memory and are read as warp-uniform broadcasts;
//   a4  each thread owns RS whole slices (P contiguous elements, Alg 1) in registers and
//       computes out[q*S_t + s] = sum_p x[s][p] * F[p][q] with FFMA / DFMA (lines 311-315);
//   a5  the nf sliced multiplies run IN PLACE on the shared-memory tile ("fusion"): all
//       slices are read into registers, a barrier, then the outputs are written back (swizzled,
//       so the next step's slice reads are bank-conflict free — the B200 replacement for shift
//       caching);
//   a6  after the last step the tile holds, for every composite column u < Q^nf, R contiguous
//       outputs at u*R + t; ONE 4-D TMA tensor store writes each run to its final
//       position u*(W/C) + g0 + t of the next intermediate (StoreFusedShMem generalised, Fig 7
//       P:560-574, reading G7) — the direct-index store that removes the transpose.
//
// Runs must be >= 32 bytes: the day-1 microbenchmark (profiles/r01_microbench.jsonl) measured 1.2-1.5
// TB/s for 16-byte runs against ~5 TB/s for >= 32-byte runs, so the planner keeps R*s >= 32.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "kron_internal.h"
#include "ptx.cuh"

namespace kron {

struct FusedArgs {
  const void *F[kMaxFused];  // factor device pointers in processing order (step 0 applied first)
  int nf;
  int tileM;
  int tileK;      // columns per tile row (R*C)
  int R;          // chunks per tile row = output run length
  int Sl;         // slices per tile row (tileK / P)
  int nslices;    // tileM * Sl
  int C;          // chunk = P^nf
  int nout;       // output buffers (warp-chain kernel): 2 = double-buffered TMA-store source
  int tiles_k;    // tiles along a row
  int64_t ntiles;
  int nbox;       // input TMA boxes per tile (along dim1)
  int box_lines;  // 128-byte lines per input box
  uint32_t tile_bytes;
  uint32_t stage_bytes;
  int stages;
};

namespace {



// Loads RS whole slices (P contiguous elements each) from shared memory; offs are byte offsets of
// the 16-byte (or smaller) vectors, already swizzled.
template <typename T, int P, int RS, int NV, int VB, bool GUARD = true>
__device__ __forceinline__ void load_slices(const unsigned char *buf, const uint32_t (&offs)[RS][NV],
                                            const bool (&act)[RS], T (&x)[RS][P]) {
  constexpr int ES = sizeof(T), EPV = VB / ES;
#pragma unroll
  for (int r = 0; r < RS; ++r) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const unsigned char *src = buf + offs[r][v];
      if (!GUARD || act[r]) {
        if constexpr (VB == 16 && ES == 4) {
          const float4 t4 = *reinterpret_cast<const float4 *>(src);
          x[r][v * EPV + 0] = t4.x; x[r][v * EPV + 1] = t4.y; x[r][v * EPV + 2] = t4.z; x[r][v * EPV + 3] = t4.w;
        } else if constexpr (VB == 16 && ES == 8) {
          const double2 t2 = *reinterpret_cast<const double2 *>(src);
          x[r][v * EPV + 0] = t2.x; x[r][v * EPV + 1] = t2.y;
        } else if constexpr (VB == 8 && ES == 4) {
          const float2 t2 = *reinterpret_cast<const float2 *>(src);
          x[r][v * EPV + 0] = t2.x; x[r][v * EPV + 1] = t2.y;
        } else {
          x[r][v] = *reinterpret_cast<const T *>(src);
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPV; ++e) x[r][v * EPV + e] = T(0);
      }
    }
  }
}

// One sliced multiply of the register-resident slices with the factor Fst (shared, [p][q]) and the
// in-place store of out[row][q*Sl + s].  SWZ: 0 linear layout (last step, TMA-store source),
// 1 swizzled with the q-stride a multiple of 1024 B (swizzle commutes with +q*stride), 2 general.
template <typename T, int P, int RS, int SWZ>
__device__ __forceinline__ void multiply_store(unsigned char *buf, const T *Fst, const T (&x)[RS][P],
                                               const uint32_t (&wb)[RS], const bool (&act)[RS], uint32_t strideQ) {
  constexpr int ES = sizeof(T);
  constexpr int QB = (P * ES >= 32) ? 32 / ES : P;  // factor columns per broadcast group
  constexpr int FVB = (QB * ES) < 16 ? QB * ES : 16;
  constexpr int FNV = QB * ES / FVB;
  constexpr int FEPV = FVB / ES;
#pragma unroll
  for (int q0 = 0; q0 < P; q0 += QB) {
    T acc[RS][QB];
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int j = 0; j < QB; ++j) acc[r][j] = T(0);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      T f[QB];
      const T *fp = Fst + p * P + q0;
#pragma unroll
      for (int v = 0; v < FNV; ++v) {
        if constexpr (FVB == 16 && ES == 4) {
          const float4 t4 = *reinterpret_cast<const float4 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t4.x; f[v * FEPV + 1] = t4.y; f[v * FEPV + 2] = t4.z; f[v * FEPV + 3] = t4.w;
        } else if constexpr (FVB == 16 && ES == 8) {
          const double2 t2 = *reinterpret_cast<const double2 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t2.x; f[v * FEPV + 1] = t2.y;
        } else {
#pragma unroll
          for (int e = 0; e < FEPV; ++e) f[v * FEPV + e] = fp[v * FEPV + e];
        }
      }
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int j = 0; j < QB; ++j) acc[r][j] = fma(x[r][p], f[j], acc[r][j]);
    }
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      if (!act[r]) continue;
#pragma unroll
      for (int j = 0; j < QB; ++j) {
        uint32_t off = wb[r] + (uint32_t)(q0 + j) * strideQ;
        if constexpr (SWZ == 2) off = swz128(off);
        *reinterpret_cast<T *>(buf + off) = acc[r][j];
      }
    }
  }
}

template <typename T, int P, int RS, int NT>
__global__ void __launch_bounds__(NT) kron_fused_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                       const __grid_constant__ CUtensorMap tm_out,
                                                       const FusedArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int SLICE_BYTES = P * ES;
  constexpr int VB = SLICE_BYTES < 16 ? SLICE_BYTES : 16;  // bytes per shared-memory vector access
  constexpr int NV = SLICE_BYTES / VB;                      // vector loads per slice
  constexpr int LINE = 128 / ES;

  // Shared memory: [stages x stage_bytes (1024-aligned, 128B-swizzled tiles)] [factors] [mbarriers].
  // Offsets stay derived from the __shared__ array so every access is LDS/STS.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  T *Fs = reinterpret_cast<T *>(base + (size_t)a.stages * a.stage_bytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(Fs) +
                                                ((a.nf * P * P * ES + 15) & ~15));
  const int tid = threadIdx.x;

  // a3: the group's factors -> shared memory, [step][p][q]
  for (int i = tid; i < a.nf * P * P; i += NT) {
    const int st = i / (P * P), e = i - st * (P * P);
    Fs[i] = reinterpret_cast<const T *>(a.F[st])[e];
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_in);
    prefetch_tmap(&tm_out);
  }

  // Per-thread slice bookkeeping: identical for every tile (same tile geometry).
  bool act[RS];
  uint32_t rd[RS][NV], wlin[RS], wswz[RS];
  const uint32_t strideQ = (uint32_t)a.Sl * ES;
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const int sl = tid + r * NT;
    act[r] = sl < a.nslices;
    const int row = sl / a.Sl, s = sl - row * a.Sl;
#pragma unroll
    for (int v = 0; v < NV; ++v) rd[r][v] = swz128((uint32_t)sl * SLICE_BYTES + v * VB);
    wlin[r] = ((uint32_t)row * a.tileK + (uint32_t)s) * ES;
    wswz[r] = swz128(wlin[r]);
  }
  const bool fast_swz = (strideQ & 1023u) == 0;
  __syncthreads();

  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      tma_load_3d(dst + (size_t)b * a.box_lines * 128, &tm_in, &bars[st], 0, line0 + b * a.box_lines, rb * a.tileM);
  };

  if (tid == 0)
    for (int it = 0; it < a.stages - 1; ++it) issue_load(it);

  for (int it = 0;; ++it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) break;
    const int st = it % a.stages;
    mbar_wait(&bars[st], (uint32_t)((it / a.stages) & 1));
    unsigned char *buf = base + (size_t)st * a.stage_bytes;

    for (int step = 0; step < a.nf; ++step) {
      const T *Fst = Fs + step * P * P;
      T x[RS][P];
      load_slices<T, P, RS, NV, VB>(buf, rd, act, x);  // a4: my slices -> registers
      __syncthreads();  // every slice of this step is in registers: the tile may be overwritten
      if (step == a.nf - 1) {
        multiply_store<T, P, RS, 0>(buf, Fst, x, wlin, act, strideQ);  // a6 source: linear layout
        fence_proxy_async_smem();
      } else if (fast_swz) {
        multiply_store<T, P, RS, 1>(buf, Fst, x, wswz, act, strideQ);  // a5: swizzled for the next step
      } else {
        multiply_store<T, P, RS, 2>(buf, Fst, x, wlin, act, strideQ);
      }
      __syncthreads();
    }
    if (tid == 0) {
      // a6: one tensor store writes the R-long runs of all Q^nf composite columns
      const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
      tma_store_4d(&tm_out, buf, cb * a.R, 0, 0, rb * a.tileM);
      bulk_commit();
      // refill the buffer of the previous tile once its store has finished reading it
      bulk_wait_read<1>();
      issue_load(it + a.stages - 1);
    }
  }
  if (tid == 0) bulk_wait<0>();
}

// ------------------------------------------------------------------ warp-local chain (v2)
//
// When a warp's share of the tile (32*RS slices = GE elements) is a whole number of chunks, every
// intermediate step of the fused chain stays inside the warp: the warp multiplies its
// slices, writes the outputs back in place into its own region (chunk-local order q*C/P + s) and
// only needs __syncwarp.  The LAST step is done CTA-wide in "chunk-fastest" order, so that a
// thread group writes consecutive composite columns of consecutive chunks — the tile's final
// u*R + g layout — with conflict-free consecutive stores into a separate output buffer that one
// TMA tensor store sends to HBM.  Two CTA barriers per tile instead of two per factor.

// chunk-dependent 16-byte-granule XOR on top of the 128B swizzle: keeps the warp-phase stores and
// the chunk-fastest last-step loads free of bank conflicts (checked by a bank model).
// The mask must be constant over each 128-byte line to stay a bijection, so it is used only when a
// chunk spans whole lines (C*s >= 128); smaller chunks use the plain 128B swizzle (gx = 0).
__device__ __forceinline__ uint32_t gmix(uint32_t g) { return (g ^ (g << 1) ^ (g << 2)) & 7u; }
__device__ __forceinline__ uint32_t swz_m(uint32_t off, uint32_t gx) { return off ^ (((off >> 3) ^ gx) & 0x70u); }

// multiply register slices by Fst and store each output (slice r, column q) at its chunk-swizzled
// position: byte offset off = wbase[r] + q*strideCP, then swz_m(off, gx[r]) (gx = gmix(chunk) << 4).
// For small RS*P the swizzled offsets are precomputed (wo), otherwise they are formed per store.
template <typename T, int P, int RS, bool PRE>
__device__ __forceinline__ void multiply_store_swz(unsigned char *buf, const T *Fst, const T (&x)[RS][P],
                                                   const uint32_t (&wo)[PRE ? RS : 1][PRE ? P : 1],
                                                   const uint32_t (&wbase)[RS], const uint32_t (&gx)[RS],
                                                   uint32_t strideCP) {
  constexpr int ES = sizeof(T);
  constexpr int QB = (P * ES >= 32) ? 32 / ES : P;
  constexpr int FVB = (QB * ES) < 16 ? QB * ES : 16;
  constexpr int FNV = QB * ES / FVB;
  constexpr int FEPV = FVB / ES;
#pragma unroll
  for (int q0 = 0; q0 < P; q0 += QB) {
    T acc[RS][QB];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      T f[QB];
      const T *fp = Fst + p * P + q0;
#pragma unroll
      for (int v = 0; v < FNV; ++v) {
        if constexpr (FVB == 16 && ES == 4) {
          const float4 t4 = *reinterpret_cast<const float4 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t4.x; f[v * FEPV + 1] = t4.y; f[v * FEPV + 2] = t4.z; f[v * FEPV + 3] = t4.w;
        } else if constexpr (FVB == 16 && ES == 8) {
          const double2 t2 = *reinterpret_cast<const double2 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t2.x; f[v * FEPV + 1] = t2.y;
        } else {
#pragma unroll
          for (int e = 0; e < FEPV; ++e) f[v * FEPV + e] = fp[v * FEPV + e];
        }
      }
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int j = 0; j < QB; ++j) acc[r][j] = (p == 0) ? x[r][0] * f[j] : fma(x[r][p], f[j], acc[r][j]);
    }
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int j = 0; j < QB; ++j) {
        uint32_t off;
        if constexpr (PRE) {
          off = wo[r][q0 + j];
        } else {
          off = wbase[r] + (uint32_t)(q0 + j) * strideCP;
          off ^= ((off >> 3) ^ gx[r]) & 0x70u;
        }
        *reinterpret_cast<T *>(buf + off) = acc[r][j];
      }
  }
}

// multiply and store to a linear layout: out byte offset wb[r] + q*strideQ
template <typename T, int P, int RS>
__device__ __forceinline__ void multiply_store_lin(unsigned char *buf, const T *Fst, const T (&x)[RS][P],
                                                   const uint32_t (&wb)[RS], uint32_t strideQ) {
  constexpr int ES = sizeof(T);
  constexpr int QB = (P * ES >= 32) ? 32 / ES : P;
  constexpr int FVB = (QB * ES) < 16 ? QB * ES : 16;
  constexpr int FNV = QB * ES / FVB;
  constexpr int FEPV = FVB / ES;
#pragma unroll
  for (int q0 = 0; q0 < P; q0 += QB) {
    T acc[RS][QB];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      T f[QB];
      const T *fp = Fst + p * P + q0;
#pragma unroll
      for (int v = 0; v < FNV; ++v) {
        if constexpr (FVB == 16 && ES == 4) {
          const float4 t4 = *reinterpret_cast<const float4 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t4.x; f[v * FEPV + 1] = t4.y; f[v * FEPV + 2] = t4.z; f[v * FEPV + 3] = t4.w;
        } else if constexpr (FVB == 16 && ES == 8) {
          const double2 t2 = *reinterpret_cast<const double2 *>(fp + v * FEPV);
          f[v * FEPV + 0] = t2.x; f[v * FEPV + 1] = t2.y;
        } else {
#pragma unroll
          for (int e = 0; e < FEPV; ++e) f[v * FEPV + e] = fp[v * FEPV + e];
        }
      }
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int j = 0; j < QB; ++j) acc[r][j] = (p == 0) ? x[r][0] * f[j] : fma(x[r][p], f[j], acc[r][j]);
    }
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      unsigned char *o = buf + wb[r] + (uint32_t)q0 * strideQ;
#pragma unroll
      for (int j = 0; j < QB; ++j) *reinterpret_cast<T *>(o + (uint32_t)j * strideQ) = acc[r][j];
    }
  }
}

template <typename T, int P, int RS, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) kron_fused_warp_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                  const __grid_constant__ CUtensorMap tm_out,
                                                                  const FusedArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int SLICE_BYTES = P * ES;
  constexpr int VB = SLICE_BYTES < 16 ? SLICE_BYTES : 16;
  constexpr int NV = SLICE_BYTES / VB;
  constexpr int LINE = 128 / ES;
  constexpr int GE = 32 * RS * P;  // elements of one warp's share of the tile

  // [stages x tile][2 x output tile][factors][mbarriers], tiles 1024-aligned
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *obase = base + (size_t)a.stages * a.stage_bytes;
  T *Fs = reinterpret_cast<T *>(obase + (size_t)a.nout * a.stage_bytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(Fs) +
                                                ((a.nf * P * P * ES + 15) & ~15));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < a.nf * P * P; i += NT) {
    const int st = i / (P * P), e = i - st * (P * P);
    Fs[i] = reinterpret_cast<const T *>(a.F[st])[e];
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_in);
    prefetch_tmap(&tm_out);
  }

  const uint32_t C = (uint32_t)a.C, CP = C / P, R = (uint32_t)a.R;
  // warp phase: lane's slices lane + 32r of the warp's group
  constexpr bool PRE = RS * P <= 16;
  uint32_t rd0[RS][NV], rdg[RS][NV], wo[PRE ? RS : 1][PRE ? P : 1], wbase[RS], gx[RS];
  const uint32_t strideCP = CP * ES;
  const bool gm_on = C * ES >= 128;
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const uint32_t el = (uint32_t)warp * GE + (uint32_t)(lane + 32 * r) * P;
    const uint32_t gg = el / C, s = (el - gg * C) / P;
    gx[r] = gm_on ? gmix(gg) << 4 : 0u;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      rd0[r][v] = swz128(el * ES + v * VB);
      rdg[r][v] = swz_m(el * ES + v * VB, gx[r]);
    }
    wbase[r] = (gg * C + s) * ES;
    if constexpr (PRE) {
#pragma unroll
      for (int q = 0; q < P; ++q) wo[r][q] = swz_m((gg * C + q * CP + s) * ES, gx[r]);
    }
  }
  // last step: chunk-fastest slice order
  uint32_t rl[RS][NV], wl[RS];
  const bool chain = a.nf >= 2;
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const uint32_t idx = (uint32_t)tid + (uint32_t)r * NT;
    const uint32_t g = idx % R, rest = idx / R, s = rest % CP, row = rest / CP;
    const uint32_t gg = row * R + g;
    const uint32_t gxl = gm_on ? gmix(gg) << 4 : 0u;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t b = (gg * C + s * P) * ES + v * VB;
      rl[r][v] = chain ? swz_m(b, gxl) : swz128(b);
    }
    wl[r] = (row * (uint32_t)a.tileK + s * R + g) * ES;
  }
  const uint32_t strideQ = (uint32_t)a.Sl * ES;
  const bool noguard[RS] = {};
  __syncthreads();

  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      tma_load_3d(dst + (size_t)b * a.box_lines * 128, &tm_in, &bars[st], 0, line0 + b * a.box_lines, rb * a.tileM);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  for (int it = 0;; ++it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) break;
    const int st = it % a.stages;
    mbar_wait(&bars[st], (uint32_t)((it / a.stages) & 1));
    unsigned char *buf = base + (size_t)st * a.stage_bytes;
    unsigned char *ob = obase + (size_t)(a.nout == 2 ? (it & 1) : 0) * a.stage_bytes;
    T x[RS][P];
    if (chain) {
      // a5: steps 0 .. nf-2 stay inside the warp (in place, chunk-swizzled)
      load_slices<T, P, RS, NV, VB, false>(buf, rd0, noguard, x);
      for (int step = 0; step < a.nf - 1; ++step) {
        if (step > 0) load_slices<T, P, RS, NV, VB, false>(buf, rdg, noguard, x);
        __syncwarp();
        multiply_store_swz<T, P, RS, PRE>(buf, Fs + step * P * P, x, wo, wbase, gx, strideCP);
        __syncwarp();
      }
    }
    __syncthreads();  // warp-phase results visible; output buffer (it&1) released by the store of it-2
    load_slices<T, P, RS, NV, VB, false>(buf, rl, noguard, x);
    multiply_store_lin<T, P, RS>(ob, Fs + (a.nf - 1) * P * P, x, wl, strideQ);  // a6 source layout u*R + g
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
      tma_store_4d(&tm_out, ob, cb * a.R, 0, 0, rb * a.tileM);
      bulk_commit();
      issue_load(it + a.stages);  // this tile's stage is fully consumed
      if (a.nout == 2)
        bulk_wait_read<1>();  // the other output buffer is free for the next tile
      else
        bulk_wait_read<0>();  // the single output buffer is free for the next tile
    }
  }
  if (tid == 0) bulk_wait<0>();
}

// ------------------------------------------------------------------ instances

const FusedInstance kInstances[] = {
    // dtype, P, NT, RS, warp-chain
    // v2 (warp-local chain): ids 0..9
    {KRON_F32, 2, 256, 8, 1},  {KRON_F32, 4, 256, 4, 1},  {KRON_F32, 8, 256, 2, 1},
    {KRON_F32, 16, 256, 2, 1}, {KRON_F32, 32, 256, 1, 1}, {KRON_F64, 2, 256, 4, 1},
    {KRON_F64, 4, 256, 2, 1},  {KRON_F64, 8, 256, 1, 1},  {KRON_F64, 16, 256, 1, 1},
    {KRON_F64, 32, 128, 1, 1},
    // v1 (CTA-wide in-place chain, any chunk size): ids 10..19
    {KRON_F32, 2, 256, 8, 0},  {KRON_F32, 4, 256, 4, 0},  {KRON_F32, 8, 128, 4, 0},
    {KRON_F32, 16, 256, 2, 0}, {KRON_F32, 32, 128, 2, 0}, {KRON_F64, 2, 256, 4, 0},
    {KRON_F64, 4, 256, 2, 0},  {KRON_F64, 8, 256, 1, 0},  {KRON_F64, 16, 128, 2, 0},
    {KRON_F64, 32, 128, 1, 0},
};
constexpr int kNumInstances = sizeof(kInstances) / sizeof(kInstances[0]);

using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const FusedArgs);

KernelFn instance_kernel(int i) {
  switch (i) {
    case 0: return kron_fused_warp_kernel<float, 2, 8, 256, 2>;
    case 1: return kron_fused_warp_kernel<float, 4, 4, 256, 2>;
    case 2: return kron_fused_warp_kernel<float, 8, 2, 256, 2>;
    case 3: return kron_fused_warp_kernel<float, 16, 2, 256, 2>;
    case 4: return kron_fused_warp_kernel<float, 32, 1, 256, 2>;
    case 5: return kron_fused_warp_kernel<double, 2, 4, 256, 2>;
    case 6: return kron_fused_warp_kernel<double, 4, 2, 256, 2>;
    case 7: return kron_fused_warp_kernel<double, 8, 1, 256, 2>;
    case 8: return kron_fused_warp_kernel<double, 16, 1, 256, 2>;
    case 9: return kron_fused_warp_kernel<double, 32, 1, 128, 2>;
    case 10: return kron_fused_kernel<float, 2, 8, 256>;
    case 11: return kron_fused_kernel<float, 4, 4, 256>;
    case 12: return kron_fused_kernel<float, 8, 4, 128>;
    case 13: return kron_fused_kernel<float, 16, 2, 256>;
    case 14: return kron_fused_kernel<float, 32, 2, 128>;
    case 15: return kron_fused_kernel<double, 2, 4, 256>;
    case 16: return kron_fused_kernel<double, 4, 2, 256>;
    case 17: return kron_fused_kernel<double, 8, 1, 256>;
    case 18: return kron_fused_kernel<double, 16, 2, 128>;
    case 19: return kron_fused_kernel<double, 32, 1, 128>;
  }
  return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void load_encode() {
  std::call_once(g_encode_once, [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
}

}  // namespace

bool tmap_available() {
  load_encode();
  return g_encode != nullptr;
}

bool encode_tmap(CUtensorMap *m, int dtype, int rank, const void *gaddr, const uint64_t *dims, const uint64_t *strides,
                 const uint32_t *box, bool swizzle128) {
  load_encode();
  if (!g_encode) return false;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, dtype == KRON_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                        (cuuint32_t)rank, const_cast<void *>(gaddr), (const cuuint64_t *)dims,
                        (const cuuint64_t *)strides, (const cuuint32_t *)box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int fused_instance_count() { return kNumInstances; }
const FusedInstance &fused_instance(int i) { return kInstances[i]; }
int fused_find(int dtype, int P, int warp) {
  for (int i = 0; i < kNumInstances; ++i)
    if (kInstances[i].dtype == dtype && kInstances[i].P == P && kInstances[i].warp == warp) return i;
  return -1;
}

int launch_fused(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *const *Fgroup,
                 void *stream) {
  const FusedInstance &inst = kInstances[pp.variant];
  const int es = dtype == KRON_F32 ? 4 : 8;
  const int line = 128 / es;
  const int64_t W = pp.W_in, WC = W / pp.C, Wout = pp.W_out;

  FusedArgs a{};
  for (int i = 0; i < pp.nf; ++i) a.F[i] = Fgroup[i];
  a.nf = pp.nf;
  a.tileM = pp.tileM;
  a.tileK = (int)pp.tileK;
  a.R = pp.R;
  a.Sl = (int)(pp.tileK / pp.P);
  a.nslices = pp.tileM * a.Sl;
  a.C = (int)pp.C;
  a.tiles_k = (int)((WC + pp.R - 1) / pp.R);
  const int64_t tiles_m = (M + pp.tileM - 1) / pp.tileM;
  a.ntiles = tiles_m * a.tiles_k;
  const int lines = (int)(pp.tileK / line);
  a.box_lines = lines > 256 ? 256 : lines;
  a.nbox = lines / a.box_lines;
  a.tile_bytes = (uint32_t)(pp.tileM * pp.tileK * es);
  a.stage_bytes = (a.tile_bytes + 1023u) & ~1023u;
  a.stages = pp.stages;

  CUtensorMap tin, tout;
  {
    uint64_t dims[3] = {(uint64_t)line, (uint64_t)(W / line), (uint64_t)M};
    uint64_t strides[2] = {128, (uint64_t)W * es};
    uint32_t box[3] = {(uint32_t)line, (uint32_t)a.box_lines, (uint32_t)pp.tileM};
    if (!encode_tmap(&tin, dtype, 3, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
  }
  {
    const int64_t qlo = pp.Qc > 256 ? 256 : pp.Qc, qhi = pp.Qc / qlo;
    uint64_t dims[4] = {(uint64_t)WC, (uint64_t)qlo, (uint64_t)qhi, (uint64_t)M};
    uint64_t strides[3] = {(uint64_t)WC * es, (uint64_t)(WC * qlo * es), (uint64_t)Wout * es};
    uint32_t box[4] = {(uint32_t)pp.R, (uint32_t)qlo, (uint32_t)qhi, (uint32_t)pp.tileM};
    if (!encode_tmap(&tout, dtype, 4, out, dims, strides, box, false)) return (int)cudaErrorInvalidValue;
  }

  a.nout = pp.nout;
  const size_t smem = 1024 + (size_t)(a.stages + (inst.warp ? pp.nout : 0)) * a.stage_bytes +
                      (((size_t)pp.nf * pp.P * pp.P * es + 15) & ~15) + 8 * (size_t)a.stages;
  KernelFn k = instance_kernel(pp.variant);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, inst.NT, smem);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.ntiles) grid = a.ntiles;
  k<<<(unsigned)grid, inst.NT, smem, (cudaStream_t)stream>>>(tin, tout, a);
  return (int)cudaGetLastError();
}

}  // namespace kron
