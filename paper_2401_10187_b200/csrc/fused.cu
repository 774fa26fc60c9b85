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
#include <cstdlib>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

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
  void *Y;        // output matrix (kernels that store from registers)
  int64_t WC;     // W / C  (output column stride of a composite column u)
  int64_t Wout;   // output row width
  int64_t M;      // rows
  int tiles_k;    // tiles along a row
  int64_t ntiles;
  int nbox;       // input TMA boxes per tile (along dim1)
  int box_lines;  // 128-byte lines per input box
  uint32_t tile_bytes;
  uint32_t stage_bytes;
  int stages;
  PushArgs push;  // v9 / v6: the pass's output goes to per-destination buffers (distributed round, push.on)
  // distributed round input read in place from an all-to-all receive buffer (InRemap): local line l ->
  // run = l / rmp_rl, (e, src) = (run / rmp_GK, run % rmp_GK); 5-D map coordinates {0, l % rl, src, e, row}
  int rmp_rl;  // 0: plain 3-D [row][line][32] input map
  int rmp_GK;
};

// ------------------------------------------------------------------ constant-bank factors (round 2)
// The factors of a pass are copied (stream-ordered, device to device) into a constant-bank array before
// the launch; the kernels' FFMA2s then take their factor operand as a uniform register loaded by LDCU.128
// from the constant cache — `FFMA2 R, R.F32x2, UR.F32, R` (two slices' element p, one factor value
// broadcast).  Shared memory carries only the data and no register holds a factor: tools/microbench_cfma.cu
// measured 72 TFLOP/s (97% of the FP32 peak) for this loop shape with 1-3 16x16 factors (3 KB; 8 KB of
// factors drop to 50 TFLOP/s: the constant cache working set), profiles/r02_microbench_cfma.jsonl.
// The arrays sit at fixed addresses (compile-time LDCU offsets: a runtime slot offset makes ptxas fall back
// to per-thread LDC); one array per kernel family, reused in stream order (see cslot_acquire).
__constant__ float c_fac2[2 * 256];  // v10 pair (F1, F2)
__constant__ float c_fac3[3 * 256];  // v10 triple (F1, F2, F3)
__constant__ float c_fac32[1024];     // v12 P = 32 pair: F1 only (8 KB of factors thrash the constant cache)

// One input box of a fused pass (rows x 128-byte lines from `line`): the plain 3-D map, or the 5-D
// StoreGPUTile view of a receive buffer (Alg 2 line 685 done by the TMA engine's address generation).
__device__ __forceinline__ void load_in(const FusedArgs &a, void *dst, const CUtensorMap *m, uint64_t *bar, int line,
                                        int row) {
  if (a.rmp_rl) {
    const int run = line / a.rmp_rl, tl = line - run * a.rmp_rl;
    const int e = run / a.rmp_GK, src = run - e * a.rmp_GK;
    tma_load_5d(dst, m, bar, 0, tl, src, e, row);
  } else {
    tma_load_3d(dst, m, bar, 0, line, row);
  }
}

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

// acc[r][j] = sum_p x[r][p] * F[p][q0 + j] with F row-major (P x P) in shared memory, read as
// warp-uniform broadcasts.  fp32 uses Blackwell's paired FMA (FFMA2: two FMAs per instruction, x as a
// broadcast operand): profiles/r01_microbench_ffma2.jsonl measured 73 TFLOP/s for FFMA2 against
// 60 TFLOP/s for scalar FFMA in this loop shape, with half the issue slots.
template <typename T, int P, int RS, int QB>
__device__ __forceinline__ void mac_block(const T *Fst, int q0, const T (&x)[RS][P], T (&acc)[RS][QB]) {
  constexpr int ES = sizeof(T);
  if constexpr (ES == 4 && QB % 2 == 0) {
    float2 acc2[RS][QB / 2];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      float2 f2[QB / 2];
      const float *fp = reinterpret_cast<const float *>(Fst) + p * P + q0;
      if constexpr (QB % 4 == 0) {
#pragma unroll
        for (int v = 0; v < QB / 4; ++v) {
          const float4 t4 = *reinterpret_cast<const float4 *>(fp + 4 * v);
          f2[2 * v] = make_float2(t4.x, t4.y);
          f2[2 * v + 1] = make_float2(t4.z, t4.w);
        }
      } else {
#pragma unroll
        for (int v = 0; v < QB / 2; ++v) f2[v] = *reinterpret_cast<const float2 *>(fp + 2 * v);
      }
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const float2 xx = make_float2(x[r][p], x[r][p]);
#pragma unroll
        for (int j = 0; j < QB / 2; ++j) acc2[r][j] = p == 0 ? __fmul2_rn(xx, f2[j]) : __ffma2_rn(xx, f2[j], acc2[r][j]);
      }
    }
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int j = 0; j < QB / 2; ++j) {
        acc[r][2 * j] = acc2[r][j].x;
        acc[r][2 * j + 1] = acc2[r][j].y;
      }
  } else {
    constexpr int FVB = (QB * ES) < 16 ? QB * ES : 16;
    constexpr int FNV = QB * ES / FVB;
    constexpr int FEPV = FVB / ES;
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
        for (int j = 0; j < QB; ++j) acc[r][j] = p == 0 ? x[r][0] * f[j] : fma(x[r][p], f[j], acc[r][j]);
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
    mac_block<T, P, RS, QB>(Fst, q0, x, acc);
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
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &bars[st], line0 + b * a.box_lines, rb * a.tileM);
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
    mac_block<T, P, RS, QB>(Fst, q0, x, acc);
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
    mac_block<T, P, RS, QB>(Fst, q0, x, acc);
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
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &bars[st], line0 + b * a.box_lines, rb * a.tileM);
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

// acc[q] = sum_p x[p] * F[p][q] with the factor held in registers (fp32: as FFMA2 pairs).
template <typename T, int P>
struct RegFactor {
  static constexpr bool kPair = sizeof(T) == 4 && P % 2 == 0;
  typename std::conditional<kPair, float2, T>::type f[P][kPair ? P / 2 : P];
  __device__ __forceinline__ void load(const T *F) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if constexpr (kPair) {
#pragma unroll
        for (int j = 0; j < P / 2; ++j) f[p][j] = make_float2(F[p * P + 2 * j], F[p * P + 2 * j + 1]);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) f[p][q] = F[p * P + q];
      }
    }
  }
  __device__ __forceinline__ void mac(const T (&x)[P], T (&acc)[P]) const {
    if constexpr (kPair) {
      float2 a2[P / 2];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float2 xx = make_float2(x[p], x[p]);
#pragma unroll
        for (int j = 0; j < P / 2; ++j) a2[j] = p == 0 ? __fmul2_rn(xx, f[p][j]) : __ffma2_rn(xx, f[p][j], a2[j]);
      }
#pragma unroll
      for (int j = 0; j < P / 2; ++j) {
        acc[2 * j] = a2[j].x;
        acc[2 * j + 1] = a2[j].y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < P; ++q) acc[q] = x[0] * f[0][q];
#pragma unroll
      for (int p = 1; p < P; ++p)
#pragma unroll
        for (int q = 0; q < P; ++q) acc[q] = fma(x[p], f[p][q], acc[q]);
    }
  }
};

// ------------------------------------------------------------------ factor-pipelined chain (v3)
//
// Small factors (P*P values fit in registers: fp32 P <= 8, fp64 P <= 4).  The CTA is split into one
// producer warp (TMA loads) and one group of NWG warps PER FACTOR of the fused group (<= 3).  Group g
// keeps its factor F_{f-g} in registers for the whole kernel and applies it to every tile, in place on
// the stage buffer; tiles flow through the groups like a pipeline (mbarriers done[g][stage]), so the
// factor is never re-read from shared memory — only the data moves through shared memory (one read
// and one write per factor and element).
//   middle groups: a lane owns VS consecutive slices of one chunk (VS*P contiguous elements), so the
//     outputs of a column q are VS consecutive values: one 16-byte store per column;
//   last group: a thread owns VS consecutive chunks for one slice index (chunk-fastest order), so its
//     outputs are VS consecutive values of the final u*R + g layout: one 16-byte store per column into
//     the double-buffered output tile, which one TMA tensor store sends to HBM.
// Bank conflicts: the TMA 128B swizzle plus an XOR of the 16-byte granule with bitrev3(chunk) (chosen
// with a bank-conflict model over the three access patterns).
// linear maps over GF(2)^3 (3x3 bit matrices) picked by exhaustive search with the bank model
template <int P, int ES>
__device__ __forceinline__ uint32_t pipe_gx(uint32_t chunk) {
  const uint32_t g0 = chunk & 1u, g1 = (chunk >> 1) & 1u, g2 = (chunk >> 2) & 1u;
  if constexpr (P == 8 && ES == 4) return (g2 | (g1 << 1) | ((g0 ^ g1) << 2)) << 4;
  else return (g2 | (g1 << 1) | ((g0 ^ g2) << 2)) << 4;
}

// v3's chunk granule XOR: the last group's loads of one instruction cover chunks j*VS + i (j = 0..7 across a
// quarter-warp, i fixed), so the XOR must be injective on chunk / VS — round 1's 3x3 map over the chunk's low
// bits gave only four distinct values on even chunks (VS = 2: ncu counted 2x the ideal wavefronts on those
// LDS.128, profiles/r02_banks_B.json).  The middle groups' stores XOR a warp-constant value (one chunk per warp
// region), so any injective map keeps them conflict-free.
template <int VS>
__device__ __forceinline__ uint32_t pipe3_gx(uint32_t chunk) {
  return ((chunk / VS) & 7u) << 4;
}

template <typename T, int N>
struct VecIO;
template <>
struct VecIO<float, 2> {
  __device__ __forceinline__ static void st(unsigned char *p, const float (&v)[2]) {
    *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
  }
};
template <>
struct VecIO<float, 4> {
  __device__ __forceinline__ static void st(unsigned char *p, const float (&v)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct VecIO<double, 2> {
  __device__ __forceinline__ static void st(unsigned char *p, const double (&v)[2]) {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
  }
};

template <typename T, int P, int NWG, int VS, int G>
__device__ __forceinline__ void pipe_group(const FusedArgs &a, const CUtensorMap *tm_out, unsigned char *base,
                                           unsigned char *obase, uint64_t *full, uint64_t *empty, uint64_t *done,
                                           int wg, int lane, int tid);

template <typename T, int P, int NWG, int VS>
__global__ void __launch_bounds__(32 * (1 + NWG * 3), 1)
    kron_fused_pipe_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                           const FusedArgs a) {
  constexpr int ES = sizeof(T);               // VS: consecutive slices (middle) / chunks (last) per thread
  constexpr int LINE = 128 / ES;
  constexpr int NV = P * ES / 16 > 0 ? P * ES / 16 : 1;  // 16-byte loads per slice
  constexpr int EPV = 16 / ES > P ? P : 16 / ES;
  constexpr int VB = EPV * ES;
  constexpr int MAXNF = 3;
  static_assert(P * ES >= 8, "slice >= 8 bytes");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *obase = base + (size_t)a.stages * a.stage_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(obase + 2 * (size_t)a.stage_bytes);
  uint64_t *empty = full + a.stages;
  uint64_t *done = empty + a.stages;  // [MAXNF-1][stages]
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int nf = a.nf;

  const CUtensorMap *tin = &tm_in, *tout = &tm_out;
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      for (int g = 0; g < MAXNF - 1; ++g) mbar_init(&done[g * a.stages + s], NWG * 32);
    }
    fence_mbar_init();
    prefetch_tmap(tin);
    prefetch_tmap(tout);
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: TMA loads into the stage ring
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int64_t tile = blockIdx.x, it = 0; tile < a.ntiles; tile += gridDim.x, ++it) {
        if (it >= a.stages) mbar_wait(&empty[st], ph ^ 1u);
        const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
        const int lrow = rb * a.tileM;
        unsigned char *dst = base + (size_t)st * a.stage_bytes;
        mbar_arrive_expect_tx(&full[st], a.tile_bytes);
        const int line0 = cb * (a.tileK / LINE);
        for (int b = 0; b < a.nbox; ++b)
          load_in(a, dst + (size_t)b * a.box_lines * 128, tin, &full[st], line0 + b * a.box_lines, lrow);
        if (++st == a.stages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  const int g = (warp - 1) / NWG, wg = (warp - 1) % NWG;
  if (g >= nf) return;
  // one code path per group index so that the factor pointer (kernel parameter) and hence every
  // factor value is provably warp-uniform: the compiler keeps F in uniform registers
  if (g == 0) pipe_group<T, P, NWG, VS, 0>(a, tout, base, obase, full, empty, done, wg, lane, tid);
  else if (g == 1) pipe_group<T, P, NWG, VS, 1>(a, tout, base, obase, full, empty, done, wg, lane, tid);
  else pipe_group<T, P, NWG, VS, 2>(a, tout, base, obase, full, empty, done, wg, lane, tid);
}

template <typename T, int P, int NWG, int VS, int G>
__device__ __forceinline__ void pipe_group(const FusedArgs &a, const CUtensorMap *tm_out, unsigned char *base,
                                           unsigned char *obase, uint64_t *full, uint64_t *empty, uint64_t *done,
                                           int wg, int lane, int tid) {
  const int cta = (int)blockIdx.x, ncta = (int)gridDim.x;
  constexpr int ES = sizeof(T);
  constexpr int NV = P * ES / 16 > 0 ? P * ES / 16 : 1;  // 16-byte loads per slice
  constexpr int EPV = 16 / ES > P ? P : 16 / ES;
  constexpr int VB = EPV * ES;
  const int g = G, nf = a.nf;
  // this group's factor F_{first-g} lives in (uniform) registers for the whole kernel
  RegFactor<T, P> Fr;
  Fr.load(reinterpret_cast<const T *>(a.F[G]));
  const uint32_t C = (uint32_t)a.C, CP = C / P, R = (uint32_t)a.R;
  const uint32_t tile_elems = (uint32_t)a.tileM * (uint32_t)a.tileK;
  const bool gx_on = C * ES >= 128;  // the granule XOR must be constant over each 128-byte line

  if (g < nf - 1) {
    // ---------------- middle group: lane owns VS consecutive slices; warp regions of 32*VS*P elements
    constexpr uint32_t GE = 32u * VS * P;
    const uint32_t el = (uint32_t)lane * VS * P;            // first element of my slices in the region
    const uint32_t cl = el / C, s0 = (el - cl * C) / P;     // chunk within the region, first slice
    const uint32_t nreg = tile_elems / GE;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t tile = cta; tile < a.ntiles; tile += ncta) {
      mbar_wait(g == 0 ? &full[st] : &done[(g - 1) * a.stages + st], ph);
      unsigned char *buf = base + (size_t)st * a.stage_bytes;
#pragma unroll 1
      for (uint32_t grp = (uint32_t)wg; grp < nreg; grp += NWG) {
        unsigned char *gb = buf + grp * (GE * ES);
        const uint32_t chunk = grp * (GE / C) + cl;
        const uint32_t gx = gx_on ? pipe3_gx<VS>(chunk) : 0u;
        const uint32_t gxr = g == 0 ? 0u : gx;  // step 0 reads the plain TMA layout
        T x[VS][P];
#pragma unroll
        for (int r = 0; r < VS; ++r)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const uint32_t off = swz128((el + r * P) * ES + v * VB) ^ gxr;
            if constexpr (ES == 4 && EPV == 4) {
              const float4 t4 = *reinterpret_cast<const float4 *>(gb + off);
              x[r][4 * v] = t4.x; x[r][4 * v + 1] = t4.y; x[r][4 * v + 2] = t4.z; x[r][4 * v + 3] = t4.w;
            } else if constexpr (ES == 4 && EPV == 2) {
              const float2 t2 = *reinterpret_cast<const float2 *>(gb + off);
              x[r][0] = t2.x; x[r][1] = t2.y;
            } else {
              const double2 t2 = *reinterpret_cast<const double2 *>(gb + off);
              x[r][2 * v] = t2.x; x[r][2 * v + 1] = t2.y;
            }
          }
        __syncwarp();
        T acc[VS][P];
#pragma unroll
        for (int r = 0; r < VS; ++r) Fr.mac(x[r], acc[r]);
        const uint32_t ob = (cl * C + s0) * ES;  // chunk-local output index q*CP + s0
#pragma unroll
        for (int q = 0; q < P; ++q) {
          T v[VS];
#pragma unroll
          for (int r = 0; r < VS; ++r) v[r] = acc[r][q];
          VecIO<T, VS>::st(gb + (swz128(ob + (uint32_t)q * CP * ES) ^ gx), v);
        }
        __syncwarp();
      }
      mbar_arrive(&done[g * a.stages + st]);  // every lane releases its own in-place writes
      if (++st == a.stages) {
        st = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  // ---------------- last group: thread owns VS consecutive chunks for one slice (chunk-fastest)
  const int lt = tid - 32 * (1 + g * NWG);
  constexpr int LT = NWG * 32;
  const uint32_t nq = R / VS;                       // chunk groups per tile row
  const uint32_t slots = (uint32_t)a.tileM * nq * CP;
  const uint32_t strideQ = (uint32_t)a.Sl * ES;
  const bool chained = nf >= 2;
  // per-thread slot geometry (identical for every tile): first chunk and output offset
  constexpr int MAXSL = 4;
  const int nsl = (int)((slots + LT - 1) / LT);
  uint32_t sl_chunk[MAXSL], sl_s[MAXSL], sl_out[MAXSL];
#pragma unroll
  for (int k = 0; k < MAXSL; ++k) {
    const uint32_t slot = (uint32_t)lt + (uint32_t)k * LT;
    const uint32_t j = slot % nq, rest = slot / nq, s = rest % CP, row = rest / CP;
    sl_chunk[k] = row * R + j * VS;
    sl_s[k] = s;
    sl_out[k] = (row * (uint32_t)a.tileK + s * R + j * VS) * ES;
  }
  int st = 0;
  uint32_t ph = 0;
  for (int64_t tile = cta, it = 0; tile < a.ntiles; tile += ncta, ++it) {
    mbar_wait(nf == 1 ? &full[st] : &done[(nf - 2) * a.stages + st], ph);
    named_bar_sync(1, LT);  // the store that last read this output buffer has finished reading it
    const unsigned char *buf = base + (size_t)st * a.stage_bytes;
    unsigned char *obuf = obase + (size_t)(it & 1) * a.stage_bytes;
#pragma unroll
    for (int k = 0; k < MAXSL; ++k) {
      if (k >= nsl) break;
      const uint32_t s = sl_s[k];
      T acc[VS][P];
#pragma unroll
      for (int i = 0; i < VS; ++i) {
        const uint32_t chunk = sl_chunk[k] + i;
        const uint32_t gx = (chained && gx_on) ? pipe3_gx<VS>(chunk) : 0u;
        T x[P];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const uint32_t off = swz128((chunk * C + s * P) * ES + v * VB) ^ gx;
          if constexpr (ES == 4 && EPV == 4) {
            const float4 t4 = *reinterpret_cast<const float4 *>(buf + off);
            x[4 * v] = t4.x; x[4 * v + 1] = t4.y; x[4 * v + 2] = t4.z; x[4 * v + 3] = t4.w;
          } else if constexpr (ES == 4 && EPV == 2) {
            const float2 t2 = *reinterpret_cast<const float2 *>(buf + off);
            x[0] = t2.x; x[1] = t2.y;
          } else {
            const double2 t2 = *reinterpret_cast<const double2 *>(buf + off);
            x[2 * v] = t2.x; x[2 * v + 1] = t2.y;
          }
        }
        Fr.mac(x, acc[i]);
      }
      unsigned char *o = obuf + sl_out[k];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        T v[VS];
#pragma unroll
        for (int i = 0; i < VS; ++i) v[i] = acc[i][q];
        VecIO<T, VS>::st(o + (uint32_t)q * strideQ, v);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(2, LT);
    if (lt == 0) {
      mbar_arrive(&empty[st]);  // every group is done with this stage
      const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
      tma_store_4d(tm_out, obuf, cb * a.R, 0, 0, rb * a.tileM);
      bulk_commit();
      bulk_wait_read<1>();
    }
    if (++st == a.stages) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (lt == 0) bulk_wait<0>();
}

// ------------------------------------------------------------------ two-factor GEMM chunks (v4)
//
// Two square factors of size P = 16 / 32 (configs C and E).  A chunk (C = P^2 elements) is a P x P
// matrix X[s][p] (rows = slices), and the fused pair of sliced multiplies is the sandwich
//     OUT[q2][q1] = sum_s F2[s][q2] * Z[s][q1],   Z = X . F1            (u = q2*P + q1)
// i.e. two P x P x P matrix products per chunk, done with register-tiled FFMA2 (fp32) / DFMA (fp64):
//   GEMM1 (warp-local): each lane computes an RM x RN tile of Z for one chunk, reading X rows and F1
//     rows as 16-byte vectors, and writes Z back in place (row-major, chunk-swizzled);
//   GEMM2 (CTA-wide, chunk-fastest): lane = (chunk of an octet, q2 group) so that for every output the
//     8 lanes of a q2 group hold 8 consecutive chunks: their stores to u*(W/C) + g0 + g form full
//     32-byte sectors (the direct-index store of P:325-329, issued from registers).
// Loads of the tile use TMA (128B swizzle) through an mbarrier ring, as in the other fused kernels.
template <typename T, int P, int RM, int RN, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) kron_fused_gemm2_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                        const FusedArgs a) {
  constexpr int ES = sizeof(T);
  constexpr int LINE = 128 / ES;
  constexpr int C = P * P;
  constexpr int VA = 16 / ES;                 // p-values per 16-byte X load
  constexpr int L1 = (P / RM) * (P / RN);     // lane tiles per chunk
  constexpr int CPG = 32 / L1;                // chunks per warp in GEMM1
  static_assert(L1 <= 32 && 32 % L1 == 0, "GEMM1 lane tiling");
  static_assert(P % (4 * RM) == 0, "GEMM2: 4 q2 groups per warp");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  T *Fs = reinterpret_cast<T *>(base + (size_t)a.stages * a.stage_bytes);  // [2][P][P]
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(Fs) + 2 * P * P * ES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < 2 * P * P; i += NW * 32) {
    const int st = i / (P * P), e = i - st * (P * P);
    Fs[i] = reinterpret_cast<const T *>(a.F[st])[e];
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  const T *F1 = Fs, *F2 = Fs + P * P;
  const int nchunks = a.R;  // tileM == 1
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &bars[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  // GEMM1 lane geometry
  const int c1 = lane / L1, tau = lane % L1;
  const int sg = tau % (P / RM), q1g = tau / (P / RM);
  // GEMM2 lane geometry
  const int gl = lane & 7, q2s = lane >> 3;
  constexpr int U2_Q1 = P / RN, U2_Q2 = P / (4 * RM);
  const int units2 = (nchunks / 8) * U2_Q1 * U2_Q2;
  T *Y = reinterpret_cast<T *>(a.Y);

  for (int it = 0;; ++it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) break;
    const int st = it % a.stages;
    mbar_wait(&bars[st], (uint32_t)((it / a.stages) & 1));
    unsigned char *buf = base + (size_t)st * a.stage_bytes;

    // ---------------- GEMM1: Z = X . F1 per chunk (warp-local, in place)
    // swizzle bookkeeping: a row of P*ES bytes spans NL 128-byte lines; within a line the 128B TMA
    // swizzle is an XOR of the in-line offset, so each access is one LOP3 on a per-row line base.
    constexpr int NL = P * ES >= 128 ? P * ES / 128 : 1;
    for (int cg = warp; cg * CPG < nchunks; cg += NW) {
      const uint32_t gg = (uint32_t)(cg * CPG + c1);
      const uint32_t cbase = gg * C * ES;
      const uint32_t gx = pipe_gx<8, 4>(gg);
      uint32_t lb[RM][NL];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int l = 0; l < NL; ++l) lb[i][l] = swz128(cbase + (uint32_t)(sg + (P / RM) * i) * (P * ES) + l * 128);
      T acc[RM][RN];
#pragma unroll 2
      for (int p0 = 0; p0 < P; p0 += VA) {
        T xa[RM][VA];
#pragma unroll
        for (int i = 0; i < RM; ++i) {
          const uint32_t x = (uint32_t)p0 * ES;
          const unsigned char *src = buf + (((NL > 1 && (x >> 7)) ? lb[i][NL - 1] : lb[i][0]) ^ (x & 127u));
          if constexpr (ES == 4) {
            const float4 v = *reinterpret_cast<const float4 *>(src);
            xa[i][0] = v.x; xa[i][1] = v.y; xa[i][2] = v.z; xa[i][3] = v.w;
          } else {
            const double2 v = *reinterpret_cast<const double2 *>(src);
            xa[i][0] = v.x; xa[i][1] = v.y;
          }
        }
#pragma unroll
        for (int e = 0; e < VA; ++e) {
          T f[RN];
          const T *fr = F1 + (p0 + e) * P + q1g * RN;
#pragma unroll
          for (int j = 0; j < RN; j += VA) {
            if constexpr (ES == 4) {
              const float4 v = *reinterpret_cast<const float4 *>(fr + j);
              f[j] = v.x; f[j + 1] = v.y; f[j + 2] = v.z; f[j + 3] = v.w;
            } else {
              const double2 v = *reinterpret_cast<const double2 *>(fr + j);
              f[j] = v.x; f[j + 1] = v.y;
            }
          }
          const bool first = p0 == 0 && e == 0;
#pragma unroll
          for (int i = 0; i < RM; ++i) {
            if constexpr (ES == 4) {
              const float2 xx = make_float2(xa[i][e], xa[i][e]);
#pragma unroll
              for (int j = 0; j < RN; j += 2) {
                const float2 ff = make_float2(f[j], f[j + 1]);
                const float2 r2 = first ? __fmul2_rn(xx, ff) : __ffma2_rn(xx, ff, make_float2(acc[i][j], acc[i][j + 1]));
                acc[i][j] = r2.x;
                acc[i][j + 1] = r2.y;
              }
            } else {
#pragma unroll
              for (int j = 0; j < RN; ++j) acc[i][j] = first ? xa[i][e] * f[j] : fma(xa[i][e], f[j], acc[i][j]);
            }
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < RM; ++i) {
#pragma unroll
        for (int j = 0; j < RN; j += VA) {
          const uint32_t x = (uint32_t)(q1g * RN + j) * ES;
          unsigned char *dst = buf + ((((NL > 1 && (x >> 7)) ? lb[i][NL - 1] : lb[i][0]) ^ (x & 127u)) ^ gx);
          if constexpr (ES == 4)
            *reinterpret_cast<float4 *>(dst) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
          else
            *reinterpret_cast<double2 *>(dst) = make_double2(acc[i][j], acc[i][j + 1]);
        }
      }
      __syncwarp();
    }
    __syncthreads();

    // ---------------- GEMM2: OUT = F2^T . Z, chunk-fastest lanes, stores from registers
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    for (int u2 = warp; u2 < units2; u2 += NW) {
      const int oct = u2 / (U2_Q1 * U2_Q2), rest = u2 - oct * (U2_Q1 * U2_Q2);
      const int q1b = rest % U2_Q1, q2b = rest / U2_Q1;
      const uint32_t gg = (uint32_t)(oct * 8 + gl);
      const uint32_t gx = pipe_gx<8, 4>(gg);
      const int q2base = (q2b * 4 + q2s) * RM, q1base = q1b * RN;
      // Z row s, columns q1base..q1base+RN: a 32/64-byte aligned block inside one 128-byte line
      const uint32_t zb0 = gg * C * ES + (uint32_t)q1base * ES;
      T acc[RM][RN];
      if constexpr (ES == 4 && (P == 16 || P == 32)) {
        // fp32: the row-s / granule-h address is  gg*C*4 + line(s)*128 + (K ^ (v(s,h) << 4)), with
        // K = q1base*4 ^ gx a lane constant and v a compile-time 3-bit value (the 128B-swizzle line bits,
        // the half-line bit of 64-byte rows and h are disjoint), so eight per-unit offsets o[v] turn every
        // Z load into [register + immediate].
        constexpr int PE = P * ES;
        const uint32_t K = ((uint32_t)q1base * ES) ^ gx;
        const T *fr0 = F2 + q2base;
#pragma unroll 1
        for (int s0 = 0; s0 < P; s0 += 8) {
          // rows s0..s0+7: line(s) = line(s0) + line(s'), and the swizzle bits of line(s0) (0 or 4) XOR
          // into those of line(s') without carry, so one lane constant per block absorbs them
          const int line0 = (s0 * PE) >> 7;
          const uint32_t Kb = K ^ ((uint32_t)(line0 & 7) << 4);
          const uint32_t b0 = gg * C * ES + (uint32_t)line0 * 128;
#pragma unroll
          for (int sp = 0; sp < 8; ++sp) {
            const int line = (sp * PE) >> 7, a4 = ((sp * PE) & 127) >> 4;
            const float4 fv4 = *reinterpret_cast<const float4 *>(fr0 + (s0 + sp) * P);
            const float fv[4] = {fv4.x, fv4.y, fv4.z, fv4.w};
            float zv[8];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t v = (uint32_t)(a4 ^ h ^ (line & 7));
              const float4 t = *reinterpret_cast<const float4 *>(buf + b0 + (Kb ^ (v << 4)) + line * 128);
              zv[4 * h] = t.x; zv[4 * h + 1] = t.y; zv[4 * h + 2] = t.z; zv[4 * h + 3] = t.w;
            }
            const bool first = s0 == 0 && sp == 0;
#pragma unroll
            for (int i = 0; i < RM; ++i) {
#pragma unroll
              for (int j = 0; j < RN; j += 2) {
                const float2 zz = make_float2(zv[j], zv[j + 1]);
                const float2 r2 = first ? __fmul2_rn(make_float2(fv[i], fv[i]), zz)
                                        : __ffma2_rn(make_float2(fv[i], fv[i]), zz, make_float2(acc[i][j], acc[i][j + 1]));
                acc[i][j] = r2.x;
                acc[i][j + 1] = r2.y;
              }
            }
          }
        }
      } else {
#pragma unroll 4
      for (int s = 0; s < P; ++s) {
        T fv[RM], zv[RN];
        const T *fr = F2 + s * P + q2base;
#pragma unroll
        for (int i = 0; i < RM; i += VA) {
          if constexpr (ES == 4) {
            const float4 v = *reinterpret_cast<const float4 *>(fr + i);
            fv[i] = v.x; fv[i + 1] = v.y; fv[i + 2] = v.z; fv[i + 3] = v.w;
          } else {
            const double2 v = *reinterpret_cast<const double2 *>(fr + i);
            fv[i] = v.x; fv[i + 1] = v.y;
          }
        }
        const uint32_t zrow = swz128(zb0 + (uint32_t)s * (P * ES)) ^ gx;
#pragma unroll
        for (int j = 0; j < RN; j += VA) {
          const unsigned char *src = buf + (zrow ^ (uint32_t)(j * ES));
          if constexpr (ES == 4) {
            const float4 v = *reinterpret_cast<const float4 *>(src);
            zv[j] = v.x; zv[j + 1] = v.y; zv[j + 2] = v.z; zv[j + 3] = v.w;
          } else {
            const double2 v = *reinterpret_cast<const double2 *>(src);
            zv[j] = v.x; zv[j + 1] = v.y;
          }
        }
#pragma unroll
        for (int i = 0; i < RM; ++i) {
          if constexpr (ES == 4) {
            const float2 ff = make_float2(fv[i], fv[i]);
#pragma unroll
            for (int j = 0; j < RN; j += 2) {
              const float2 zz = make_float2(zv[j], zv[j + 1]);
              const float2 r2 = s == 0 ? __fmul2_rn(ff, zz) : __ffma2_rn(ff, zz, make_float2(acc[i][j], acc[i][j + 1]));
              acc[i][j] = r2.x;
              acc[i][j + 1] = r2.y;
            }
          } else {
#pragma unroll
            for (int j = 0; j < RN; ++j) acc[i][j] = s == 0 ? fv[i] * zv[j] : fma(fv[i], zv[j], acc[i][j]);
          }
        }
      }
      }
      // direct-index store: u = q2*P + q1 -> Y[row][u*(W/C) + cb*R + g]
      const int64_t gcol = (int64_t)cb * a.R + gg;
      if (gcol < a.WC && rb < a.M) {
        T *yb = Y + (int64_t)rb * a.Wout + gcol + (int64_t)(q2base * P + q1base) * a.WC;
        // every output of the unit sits (i*P + j) * WC elements past yb (< 2^32 bytes: one row of Y)
        const uint32_t wcb = (uint32_t)a.WC * (uint32_t)ES;
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j)
            *reinterpret_cast<T *>(reinterpret_cast<unsigned char *>(yb) + (uint64_t)(wcb * (uint32_t)(i * P + j))) =
                acc[i][j];
      }
    }
    __syncthreads();  // the stage is fully consumed
    if (tid == 0) issue_load(it + a.stages);
  }
}

// ------------------------------------------------------------------ constant-bank 16x16 chunk steps (v10)
//
// Every FFMA2 below takes its factor operand from a uniform register (LDCU from the constant bank): the
// factor index may depend only on loop counters, never on the lane, so each warp-level FFMA2 uses ONE
// factor value (or pair) — lanes differ only in the data they hold.  The calling branch must be provably
// warp-uniform (warp index via __shfl_sync) for the compiler to use the uniform datapath.
//
// cb_pair16: four 256-element chunks [d1][d2] (chunks g0 .. g0+3) of a 128B-swizzled stage, both factors of
// a 16x16 pair applied in place:
//   step 1 (F1 on d2): lane = row r = lane % 16 of chunks g0 + lane / 16 and g0 + lane / 16 + 2;
//          x = a row's 16 values (4 conflict-free LDS.128 on the TMA layout), out[q] = sum_p x[p] F1[p][q] as
//          128 FFMA2 per row with x broadcast and a factor PAIR (F1[p][q], F1[p][q+1]) from a uniform register
//          pair, written back over the row with the chunk's granule XOR gx(g) (so step 2's loads of
//          consecutive chunks fall in different bank halves);
//   step 2 (F2 on d1): lane = column pair (2j, 2j+1), j = lane % 8, of chunk g0 + lane / 8; x2[s] = the pair
//          in row s (LDS.64), OUT[q2][q1] = sum_s F2[s][q2] Z[s][q1] as 256 FFMA2 on the column pair with a
//          factor broadcast, written back over the same column pair (u = q2*16 + q1 at swz128(u*4) ^ gx).
// 32 FMAs per element, 8 LDS.128 + 8 STS.128 + 16 LDS.64 + 16 STS.64 per lane for 512 FFMA2, whose factor
// operands come from 128 LDCU.128.
__device__ __forceinline__ void cb_pair16(unsigned char *buf, uint32_t g0, int lane, const float *F1, const float *F2) {
  const float4 *F1v = reinterpret_cast<const float4 *>(F1), *F2v = reinterpret_cast<const float4 *>(F2);
  {
    const int sl = lane & 15;
    uint32_t rb[2], gx[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t g = g0 + (uint32_t)(lane >> 4) + 2u * h;
      rb[h] = g * 1024u;
      gx[h] = pipe_gx<8, 4>(g);
    }
    float x[2][16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float4 t = *reinterpret_cast<const float4 *>(buf + rb[h] + swz128((uint32_t)(sl * 16 + 4 * v) * 4u));
        x[h][4 * v] = t.x; x[h][4 * v + 1] = t.y; x[h][4 * v + 2] = t.z; x[h][4 * v + 3] = t.w;
      }
    float2 acc[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[h][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < 16; ++p)
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 f = F1v[p * 4 + j4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 xx = make_float2(x[h][p], x[h][p]);
          acc[h][2 * j4] = __ffma2_rn(xx, make_float2(f.x, f.y), acc[h][2 * j4]);
          acc[h][2 * j4 + 1] = __ffma2_rn(xx, make_float2(f.z, f.w), acc[h][2 * j4 + 1]);
        }
      }
    __syncwarp();  // the gx-XOR'd write-back of a row lands on its neighbour row's bytes
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<float4 *>(buf + rb[h] + (swz128((uint32_t)(sl * 16 + 4 * v) * 4u) ^ gx[h])) =
            make_float4(acc[h][2 * v].x, acc[h][2 * v].y, acc[h][2 * v + 1].x, acc[h][2 * v + 1].y);
  }
  __syncwarp();
  {
    const uint32_t g = g0 + (uint32_t)(lane >> 3), j = (uint32_t)(lane & 7);
    unsigned char *ch = buf + g * 1024u;
    const uint32_t gx = pipe_gx<8, 4>(g);
    float2 x2[16];
#pragma unroll
    for (int r = 0; r < 16; ++r)
      x2[r] = *reinterpret_cast<const float2 *>(ch + (swz128((uint32_t)(r * 16) * 4u + j * 8u) ^ gx));
    float2 acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 f = F2v[r * 4 + q4];
        acc[4 * q4] = __ffma2_rn(x2[r], make_float2(f.x, f.x), acc[4 * q4]);
        acc[4 * q4 + 1] = __ffma2_rn(x2[r], make_float2(f.y, f.y), acc[4 * q4 + 1]);
        acc[4 * q4 + 2] = __ffma2_rn(x2[r], make_float2(f.z, f.z), acc[4 * q4 + 2]);
        acc[4 * q4 + 3] = __ffma2_rn(x2[r], make_float2(f.w, f.w), acc[4 * q4 + 3]);
      }
#pragma unroll
    for (int q = 0; q < 16; ++q)
      *reinterpret_cast<float2 *>(ch + (swz128((uint32_t)(q * 16) * 4u + j * 8u) ^ gx)) = acc[q];
  }
}

// cb_top16: the third factor of a 16x16 triple on a 4096-element chunk of 16 subchunks (phase-1 layout:
// element (k, col) at k*1024 + (swz128(col*4) ^ gx(k))): lane = column pair c, c + 1; OUT[q][c] =
// sum_k F3[k][q] S[k][c] as 256 FFMA2 with a factor broadcast, in place (same layout, rows q; each lane owns
// its column pair in every row, so no lane waits for another).
__device__ __forceinline__ void cb_top16(unsigned char *cb, uint32_t c, const float *F3) {
  const float4 *F3v = reinterpret_cast<const float4 *>(F3);
  const uint32_t co = swz128(c * 4u);
  float2 x2[16];
#pragma unroll
  for (int k = 0; k < 16; ++k)
    x2[k] = *reinterpret_cast<const float2 *>(cb + (uint32_t)k * 1024u + (co ^ pipe_gx<8, 4>((uint32_t)k)));
  float2 acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 16; ++k)
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const float4 f = F3v[k * 4 + q4];
      acc[4 * q4] = __ffma2_rn(x2[k], make_float2(f.x, f.x), acc[4 * q4]);
      acc[4 * q4 + 1] = __ffma2_rn(x2[k], make_float2(f.y, f.y), acc[4 * q4 + 1]);
      acc[4 * q4 + 2] = __ffma2_rn(x2[k], make_float2(f.z, f.z), acc[4 * q4 + 2]);
      acc[4 * q4 + 3] = __ffma2_rn(x2[k], make_float2(f.w, f.w), acc[4 * q4 + 3]);
    }
#pragma unroll
  for (int q = 0; q < 16; ++q)
    *reinterpret_cast<float2 *>(cb + (uint32_t)q * 1024u + (co ^ pipe_gx<8, 4>((uint32_t)q))) = acc[q];
}

// cb_pair32 (v12): both factors of a 32 x 32 fp32 pair on two 1024-element chunks g0, g0+1 of a 128B-swizzled
// stage (row s of chunk g = one 128-byte line; element p at swz128(s*128 + 4p)).  A warp owns its two chunks:
//   step 1 (F1 on p): lane = rows r, r+16 (r = lane % 16) of chunk g0 + lane / 16: 8 LDS.128 per row
//          (a quarter-warp = 8 rows: distinct granules under the line XOR), out[q] = sum_p x[p] F1[p][q] as 512
//          FFMA2 per row pair with x broadcast and a factor PAIR from a uniform register (LDCU.128 from c_fac32),
//          written back over the row;
//   step 2 (F2 on s): lane = column pair (2j, 2j+1), j = lane % 16, of chunk g0 + lane / 16: x2[s] = the pair in
//          row s (LDS.64, a half-warp = one line), OUT[q2] = sum_s F2[s][q2] x2[s] as 1024 FFMA2 with the factor
//          value broadcast from a shared-memory row of F2 (LDS.128 at one address for the whole warp: one wavefront
//          per four FFMA2), written (after the warp's reads) at swz128(q2*128 + 8j) ^ gx(g): the chunk XOR makes
//          the chunk-fastest stream-out reads conflict-free.
// Only F1 sits in the constant bank: two 4 KB factors there run at 50 TFLOP/s in tools/microbench_cfma.cu (the
// constant cache), one at 71 TFLOP/s.
__device__ __forceinline__ void cb_pair32(unsigned char *buf, uint32_t g0, int lane, const float *F1,
                                          const float *F2s) {
  const float4 *F1v = reinterpret_cast<const float4 *>(F1);
  const uint32_t g = g0 + (uint32_t)(lane >> 4), j = (uint32_t)(lane & 15);
  unsigned char *ch = buf + g * 4096u;
  {
    float x[2][32];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float4 t = *reinterpret_cast<const float4 *>(ch + swz128((j + 16u * h) * 128u + (uint32_t)v * 16u));
        x[h][4 * v] = t.x; x[h][4 * v + 1] = t.y; x[h][4 * v + 2] = t.z; x[h][4 * v + 3] = t.w;
      }
    float2 acc[2][16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[h][k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < 32; ++p)
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 f = F1v[p * 8 + j4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 xx = make_float2(x[h][p], x[h][p]);
          acc[h][2 * j4] = __ffma2_rn(xx, make_float2(f.x, f.y), acc[h][2 * j4]);
          acc[h][2 * j4 + 1] = __ffma2_rn(xx, make_float2(f.z, f.w), acc[h][2 * j4 + 1]);
        }
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        *reinterpret_cast<float4 *>(ch + swz128((j + 16u * h) * 128u + (uint32_t)v * 16u)) =
            make_float4(acc[h][2 * v].x, acc[h][2 * v].y, acc[h][2 * v + 1].x, acc[h][2 * v + 1].y);
  }
  __syncwarp();
  {
    const uint32_t gx = pipe_gx<8, 4>(g);
    float2 x2[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) x2[r] = *reinterpret_cast<const float2 *>(ch + swz128((uint32_t)r * 128u + j * 8u));
    float2 acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        const float4 f = *reinterpret_cast<const float4 *>(F2s + r * 32 + q4 * 4);
        acc[4 * q4] = __ffma2_rn(x2[r], make_float2(f.x, f.x), acc[4 * q4]);
        acc[4 * q4 + 1] = __ffma2_rn(x2[r], make_float2(f.y, f.y), acc[4 * q4 + 1]);
        acc[4 * q4 + 2] = __ffma2_rn(x2[r], make_float2(f.z, f.z), acc[4 * q4 + 2]);
        acc[4 * q4 + 3] = __ffma2_rn(x2[r], make_float2(f.w, f.w), acc[4 * q4 + 3]);
      }
    __syncwarp();  // the XOR'd write-back lands on other lanes' column pairs
#pragma unroll
    for (int q = 0; q < 32; ++q)
      *reinterpret_cast<float2 *>(ch + (swz128((uint32_t)q * 128u + j * 8u) ^ gx)) = acc[q];
  }
}

// ------------------------------------------------------------------ fp32 two-factor chunks, warp-specialised (v6)
//
// The v4 sandwich OUT = F2^T . (X . F1) per P x P chunk (P = 16 / 32, fp32), with every chunk owned by
// one warp from start to finish: GEMM1 (A = X rows from the TMA tile, B = F1) writes Z in place, GEMM2
// (A = F2^T, B = Z) writes OUT in place, both with 4 x 8 register tiles of paired FFMA2 — no CTA barrier
// on the compute side; work units (one warp's chunks) are dealt round-robin across tile boundaries.
// Four store warps stream each finished tile out chunk-fastest (the direct-index store, P:325-329:
// Y[row][u*(W/C) + g0 + g]) while the compute warps work on the next tiles of the TMA ring (mbarriers:
// full = landed, cdone = computed, empty = streamed out -> refill).  Output runs are R*4 bytes; the
// measured write rate of such runs (tools/microbench_scatter.cu: 2.9 TB/s at 32 B, 4.5 TB/s at 128 B,
// profiles/r01_microbench_scatter.jsonl) is why P = 16 uses 64-chunk (256-byte) tiles.
// PUSH: distributed P2P round whose exchange is fused into this pass (NEXT-1): every output value is
// stored at its StoreGPUTile position in the destination rank's heap instead of into Y (push_dst).
// (32-bit index math: launch_fused refuses pushes with row widths >= 2^31 — a 64-bit division per value had made
// the pushing epilogues several times slower than the plain stores)
template <typename T>
__device__ __forceinline__ T *push_dst(const FusedArgs &a, int rb, int64_t col) {
  const uint32_t c = (uint32_t)col, B = (uint32_t)a.push.B, rho = (uint32_t)a.push.rho;
  const uint32_t d = c / B, e = c - d * B, run = e / rho;
  const uint32_t tcol = (run * (uint32_t)a.push.GK + (uint32_t)a.push.me) * rho + (e - run * rho);
  return reinterpret_cast<T *>(a.push.dst[d]) + (int64_t)rb * a.push.wd + tcol;
}

template <int P, int NCW, int RM, int RN, int VA, int KU = 1, bool PUSH = false, bool CB = false>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) kron_fused_gemm2ws_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                              const __grid_constant__ CUtensorMap tm_out,
                                                                              const FusedArgs a) {
  using T = float;
  constexpr int ES = 4, LINE = 32, C = P * P, PE = P * ES;
  constexpr int NSW = 4;
  constexpr int L1 = (P / RM) * (P / RN);  // lanes per chunk
  constexpr int CPG = CB ? (P == 16 ? 4 : 2) : 32 / L1;  // chunks per warp (one work unit)
  static_assert(!CB || P == 16 || P == 32, "constant-bank pairs are P = 16 / 32");
  const int UPT = a.R / CPG;               // work units per tile
  constexpr uint32_t CE = C * ES;          // chunk bytes (a multiple of 1024)
  static_assert(L1 <= 32 && 32 % L1 == 0, "lane tiling");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  T *F1s = reinterpret_cast<T *>(base + (size_t)a.stages * a.stage_bytes);  // [p][q1], plain
  unsigned char *F2Ts = reinterpret_cast<unsigned char *>(F1s + C);          // [q2][s], 128B-swizzled
  uint64_t *full = reinterpret_cast<uint64_t *>(F2Ts + CE);
  uint64_t *cdone = full + a.stages, *empty = cdone + a.stages;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // provably warp-uniform

  if constexpr (!CB) {
    const T *F1 = reinterpret_cast<const T *>(a.F[0]);
    const T *F2 = reinterpret_cast<const T *>(a.F[1]);
    for (int i = tid; i < C; i += (NCW + NSW) * 32) {
      const uint32_t r = (uint32_t)i / P, c = (uint32_t)i % P;
      F1s[i] = F1[i];
      *reinterpret_cast<T *>(F2Ts + swz128(c * PE + r * ES)) = F2[i];  // F2[s = r][q2 = c] -> F2T[c][r]
    }
  } else if constexpr (P == 32) {
    const T *F2 = reinterpret_cast<const T *>(a.F[1]);
    for (int i = tid; i < C; i += (NCW + NSW) * 32) F1s[i] = F2[i];  // v12: F2 rows, plain (broadcast reads)
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], UPT * 32);
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&full[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &full[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  if (CB && warp < NCW) {
    // v10 compute: each unit = four chunks through cb_pair16 (factors in the constant bank); v12 (P = 32): two
    // chunks through cb_pair32 (F1 in the constant bank, F2 broadcast from shared memory)
    for (int un = warp;; un += NCW) {
      const int it = un / UPT, cg = un % UPT;
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      mbar_wait(&full[st], (uint32_t)((it / a.stages) & 1));
      if constexpr (P == 16)
        cb_pair16(base + (size_t)st * a.stage_bytes, (uint32_t)(cg * CPG), lane, c_fac2, c_fac2 + 256);
      else
        cb_pair32(base + (size_t)st * a.stage_bytes, (uint32_t)(cg * CPG), lane, c_fac32, F1s);
      __syncwarp();
      mbar_arrive(&cdone[st]);  // every lane publishes its own writes
    }
  } else if (warp < NCW) {
    const int c1 = lane / L1, tau = lane % L1;
    const int sg = tau % (P / RM), q1g = tau / (P / RM);
    // A-operand rows sg + (P/RM)*i of a 128B-swizzled [P][P] matrix at a 1024-aligned base
    uint32_t arow[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) arow[i] = swz128((uint32_t)(sg + (P / RM) * i) * PE);
    // one warp-level P x P x P product: acc[i][j] = sum_k A[row_i][k] * B[k][q1g*RN + j], k in blocks of
    // 8 (compile-time offsets inside a block; loadB(k0, kk, f) gets the block base and the offset)
    auto gemm = [&](const unsigned char *A, auto loadB, T (&acc)[RM][RN]) {
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;
#pragma unroll KU
      for (int k0 = 0; k0 < P; k0 += 8) {
        uint32_t ab[RM];
#pragma unroll
        for (int i = 0; i < RM; ++i) ab[i] = arow[i] ^ (uint32_t)(k0 * ES);
#pragma unroll
        for (int kk = 0; kk < 8; kk += VA) {
          T xa[RM][VA];
#pragma unroll
          for (int i = 0; i < RM; ++i) {
            if constexpr (VA == 4) {
              const float4 v = *reinterpret_cast<const float4 *>(A + (ab[i] ^ (uint32_t)(kk * ES)));
              xa[i][0] = v.x; xa[i][1] = v.y; xa[i][2] = v.z; xa[i][3] = v.w;
            } else {
              const float2 v = *reinterpret_cast<const float2 *>(A + (ab[i] ^ (uint32_t)(kk * ES)));
              xa[i][0] = v.x; xa[i][1] = v.y;
            }
          }
#pragma unroll
          for (int e = 0; e < VA; ++e) {
            T f[RN];
            loadB(k0, kk + e, f);
#pragma unroll
            for (int i = 0; i < RM; ++i) {
              const float2 xx = make_float2(xa[i][e], xa[i][e]);
#pragma unroll
              for (int j = 0; j < RN; j += 2) {
                const float2 r2 = __ffma2_rn(xx, make_float2(f[j], f[j + 1]), make_float2(acc[i][j], acc[i][j + 1]));
                acc[i][j] = r2.x;
                acc[i][j + 1] = r2.y;
              }
            }
          }
        }
      }
    };
    // units are dealt round-robin over the compute warps across tile boundaries
    for (int un = warp;; un += NCW) {
      const int it = un / UPT, cg = un % UPT;
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      mbar_wait(&full[st], (uint32_t)((it / a.stages) & 1));
      unsigned char *buf = base + (size_t)st * a.stage_bytes;
      {
        const uint32_t gg = (uint32_t)(cg * CPG + c1);
        unsigned char *ch = buf + gg * CE;
        const uint32_t gx = pipe_gx<8, 4>(gg);
        T acc[RM][RN];
        // GEMM1: Z = X . F1
        gemm(ch, [&](int k0, int kk, T (&f)[RN]) {
          const T *fr = F1s + (k0 + kk) * P + q1g * RN;
#pragma unroll
          for (int j = 0; j < RN; j += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(fr + j);
            f[j] = v.x; f[j + 1] = v.y; f[j + 2] = v.z; f[j + 3] = v.w;
          }
        }, acc);
        __syncwarp();
        auto put = [&](uint32_t xr) {
#pragma unroll
          for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int j = 0; j < RN; j += 4)
              *reinterpret_cast<float4 *>(ch + ((arow[i] ^ (uint32_t)((q1g * RN + j) * ES)) ^ xr)) =
                  make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        };
        put(gx);  // Z (chunk-XOR'd: the chunks of one warp read Z rows in the same instruction)
        __syncwarp();
        // GEMM2: OUT[q2][q1] = sum_s F2T[q2][s] Z[s][q1]
        // Z row k = k0 + kk: ch + line(k)*128 + (Kq ^ (v << 4)): the 128B-swizzle bits of line(k0) and
        // line(kk) XOR without carry (k0 % 8 == 0), and the in-line bits of kk, j and q1g are disjoint
        const uint32_t Kq = (uint32_t)(q1g * RN * ES) ^ gx;
        gemm(F2Ts, [&](int k0, int kk, T (&f)[RN]) {
          const int line0 = (k0 * PE) >> 7, line = (kk * PE) >> 7, a4 = ((kk * PE) & 127) >> 4;
          const uint32_t Kb = Kq ^ ((uint32_t)(line0 & 7) << 4);
          const unsigned char *zb = ch + (line0 + line) * 128;
#pragma unroll
          for (int j = 0; j < RN; j += 4) {
            const uint32_t v = (uint32_t)(a4 ^ (j / 4) ^ (line & 7));
            const float4 t = *reinterpret_cast<const float4 *>(zb + (Kb ^ (v << 4)));
            f[j] = t.x; f[j + 1] = t.y; f[j + 2] = t.z; f[j + 3] = t.w;
          }
        }, acc);
        __syncwarp();
        put(gx);  // OUT[q2][q1] over Z[s = q2][q1]
      }
      __syncwarp();
      mbar_arrive(&cdone[st]);  // every lane: each publishes its own writes
    }
  } else {
    // ---------------- store warps: transpose the finished tile into a [u][g] staging tile (the
    // StoreFusedShMem layout) and send it with one TMA tensor store to Y[row][u*(W/C) + g0 + g];
    // 128-byte rows (R = 32) use the 128B swizzle, which the staging writes follow
    {
      // ---------------- store warps (direct): chunk-fastest stream-out from registers,
      // Y[row][u*(W/C) + cb*R + g]: 8 consecutive chunks = 32-byte runs
      const int sw = warp - NCW;
      T *Y = reinterpret_cast<T *>(a.Y);
      const int gl = lane & 7, uq = lane >> 3;
      for (int it = 0;; ++it) {
        const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
        if (tile >= a.ntiles) break;
        const int st = it % a.stages;
        const uint32_t par = (uint32_t)((it / a.stages) & 1);
        mbar_wait_sleep(&cdone[st], par);
        const unsigned char *buf = base + (size_t)st * a.stage_bytes;
        const int rb = (int)(tile / a.tiles_k), cbk = (int)(tile - (int64_t)rb * a.tiles_k);
        if (a.R % 32 == 0 && rb < a.M && (int64_t)(cbk + 1) * a.R <= a.WC) {
          // runs of >= 128 bytes: lane = chunk, so every store instruction writes one full 128-byte
          // line of a u row, and the R/32 lines of a row go out back to back
          T *yr = Y + (int64_t)rb * a.Wout + (int64_t)cbk * a.R + lane;
          const int64_t wc = a.WC;
          const uint32_t gxl = pipe_gx<8, 4>((uint32_t)lane);  // gx depends on g mod 8 only
#pragma unroll 1
          for (int u4 = sw; u4 < C / 4; u4 += NSW) {
            const uint32_t u = (uint32_t)(u4 * 4);
            T *p = yr + (int64_t)u * wc;
            for (int h = 0; h < a.R / 32; ++h) {
              const float4 v = *reinterpret_cast<const float4 *>(buf + (uint32_t)(h * 32 + lane) * CE +
                                                                 (swz128(u * ES) ^ gxl));
              if constexpr (PUSH) {
                const int64_t c0 = (int64_t)u * wc + (int64_t)cbk * a.R + h * 32 + lane;
                *push_dst<T>(a, rb, c0) = v.x;
                *push_dst<T>(a, rb, c0 + wc) = v.y;
                *push_dst<T>(a, rb, c0 + 2 * wc) = v.z;
                *push_dst<T>(a, rb, c0 + 3 * wc) = v.w;
              } else {
                p[h * 32] = v.x;
                p[h * 32 + wc] = v.y;
                p[h * 32 + 2 * wc] = v.z;
                p[h * 32 + 3 * wc] = v.w;
              }
            }
          }
        } else
        for (int oct = 0; oct < a.R / 8; ++oct) {
          const uint32_t gg = (uint32_t)(oct * 8 + gl);
          const uint32_t gx = pipe_gx<8, 4>(gg);
          const unsigned char *ch = buf + gg * CE;
          const int64_t gcol = (int64_t)cbk * a.R + gg;
          if (rb < a.M && gcol < a.WC) {
            T *yg = Y + (int64_t)rb * a.Wout + gcol;
            const int64_t wc = a.WC;
#pragma unroll 2
            for (int u16 = sw; u16 < C / 16; u16 += NSW) {
              const uint32_t u = (uint32_t)(u16 * 16 + uq * 4);
              const float4 v = *reinterpret_cast<const float4 *>(ch + (swz128(u * ES) ^ gx));
              if constexpr (PUSH) {
                const int64_t c0 = (int64_t)u * wc + gcol;
                *push_dst<T>(a, rb, c0) = v.x;
                *push_dst<T>(a, rb, c0 + wc) = v.y;
                *push_dst<T>(a, rb, c0 + 2 * wc) = v.z;
                *push_dst<T>(a, rb, c0 + 3 * wc) = v.w;
              } else {
                T *p = yg + (int64_t)u * wc;
                p[0] = v.x;
                p[wc] = v.y;
                p[2 * wc] = v.z;
                p[3 * wc] = v.w;
              }
            }
          }
        }
        __syncwarp();
        mbar_arrive(&empty[st]);
        if (sw == 0) {
          if (lane == 0) {
            mbar_wait_sleep(&empty[st], par);
            fence_proxy_async_smem();
            issue_load(it + a.stages);
          }
          __syncwarp();
        }
      }
    }
  }
}

// ------------------------------------------------------------------ fp32 16x16 factor triples on a CTA pair (v9)
//
// NEXT-2 (cluster / DSMEM fusion, "Fused <= floor(log_P TileK)" with the tile spanning a cluster):
// three 16 x 16 fp32 factors per pass, chunk C = 4096.  32-byte output runs need 8 chunks = 128 KB per
// tile, which leaves no room for a TMA ring in one CTA; here a cluster of two CTAs owns the 8-chunk tile
// (4 chunks = 64 KB each, three-stage ring each) and the stream-out gathers every 32-byte run from both
// CTAs' shared memory (lane pairs: one 16-byte half local, one over DSMEM), so each store instruction
// writes whole sectors (16-byte runs measured ~1.3 TB/s, tools/microbench.cu).
//   phase 1 (per 256-element subchunk [d2][d3], the v6 sandwich): S = F2^T . (X . F1), in place;
//   phase 2 (per 4096-chunk [d1][256]):  OUT[q3][col] = sum_d1 F3[d1][q3] . S[d1][col], in place by
//   64-column blocks (a warp reads and writes the same locations);
//   composite column u = q3*256 + q2*16 + q1 -> Y[row][u*(W/C) + 8*group + 4*rank + t], t < 4.
// Barriers per stage: full (TMA), p1[chunk] (phase 1 of that chunk done), cdone (phase 2 of the tile done
// in this CTA: every phase-2 lane), rdy (the peer's tile is done: one release.cluster arrive from the
// peer's signal warp after it acquired the peer's cdone), empty (this CTA's store lanes + the peer's last
// store warp, release.cluster: both CTAs' reads of this stage are done).  Warps: 12 compute, 3 store,
// 1 signal.
// compute-sanitizer racecheck / synccheck / memcheck clean (tools/sanitize.py).
// P2W: columns per lane in phase 2 (16: one unit = a 16 x 128 block, fewer shared loads per FMA than
// 8: E's v9 pass 11.73 -> 11.62 ms)
template <int NCW, bool PUSH = false, int P2W = 16, bool CB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((NCW + 4) * 32, 1)
    kron_fused_gemm3c_kernel(const __grid_constant__ CUtensorMap tm_in, const FusedArgs a) {
  using T = float;
  constexpr int P = 16, RM = 4, RN = 8, VA = 4, ES = 4, PE = P * ES, C1 = P * P;
  constexpr uint32_t CE = C1 * ES;                // subchunk bytes (1 KB)
  constexpr int NSW = 4, L1 = (P / RM) * (P / RN), CPG = 32 / L1;
  constexpr int SUB = 64;                         // subchunks per CTA tile (4 chunks of 4096)
  constexpr int U1 = CB ? SUB / 4 : SUB / CPG, U2 = CB ? 16 : 2 * 64 / P2W, UPT = U1 + U2;  // phase-2 units
  constexpr uint32_t TB = SUB * CE;               // 64 KB per CTA tile
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.stages;
  T *F1s = reinterpret_cast<T *>(base + (size_t)S * TB);     // [p][q1], plain
  unsigned char *F2Ts = reinterpret_cast<unsigned char *>(F1s + C1);  // [q2][p], 128B-swizzled
  unsigned char *F3Ts = F2Ts + CE;                                    // [q3][p], 128B-swizzled
  uint64_t *full = reinterpret_cast<uint64_t *>(F3Ts + CE);
  uint64_t *p1 = full + S, *cdone = p1 + 4 * S, *empty = cdone + S, *rdy = empty + S;
  unsigned *scnt = reinterpret_cast<unsigned *>(rdy + S);  // store warps done with the stage
  constexpr int NST = NSW - 1;  // store warps; the last warp of the group signals the peer
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // provably warp-uniform
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int64_t groups = a.tiles_k;  // 8-chunk groups per row

  if constexpr (!CB) {
    const T *F1 = reinterpret_cast<const T *>(a.F[0]);
    const T *F2 = reinterpret_cast<const T *>(a.F[1]);
    const T *F3 = reinterpret_cast<const T *>(a.F[2]);
    for (int i = tid; i < C1; i += (NCW + NSW) * 32) {
      const uint32_t r = (uint32_t)i / P, c = (uint32_t)i % P;
      F1s[i] = F1[i];
      *reinterpret_cast<T *>(F2Ts + swz128(c * PE + r * ES)) = F2[i];
      *reinterpret_cast<T *>(F3Ts + swz128(c * PE + r * ES)) = F3[i];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      for (int t = 0; t < 4; ++t) mbar_init(&p1[4 * s + t], (CB ? 4 : CPG == 4 ? 4 : 16 / CPG) * 32);
      mbar_init(&cdone[s], U2 * 32);       // every phase-2 lane of this CTA
      mbar_init(&rdy[s], 1);               // the peer's signal warp: its tile is computed
      mbar_init(&empty[s], NST * 32 + 1);  // every store lane of this CTA + the peer's last store warp
      scnt[s] = 0;
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  cluster_sync_all();  // barriers initialised in both CTAs before any remote arrive
  auto issue_load = [&](int it) {
    const int64_t tile = cid + (int64_t)it * ncl;
    if (tile >= a.ntiles) return;
    const int st = it % S;
    const int rb = (int)(tile / groups), gj = (int)(tile - (int64_t)rb * groups);
    unsigned char *dst = base + (size_t)st * TB;
    mbar_arrive_expect_tx(&full[st], TB);
    const int line0 = (gj * 8 + (int)rank * 4) * (4096 / 32);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &full[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < S; ++it) issue_load(it);

  if (CB && warp < NCW) {
    // v10 compute (factors in the constant bank): the compute warps form NCW / 4 groups of four; a group
    // owns one 4096-element chunk at a time (chunks dealt round-robin to the groups across the tiles of the
    // ring).  Warp i of the group runs phase 1 on subchunks 4i .. 4i+3 (cb_pair16), the group meets at a
    // named barrier, then warp i runs phase 2 on columns 64i .. 64i+63 (cb_top16).  Equal work per warp
    // and a hardware barrier: no warp idles on another chunk's phase 1 (round-1's unit order made a chunk's
    // phase-2 warps wait for its phase-1 warps; ncu put 14% of the stall samples on that wait).
    static_assert(NCW % 4 == 0, "groups of four compute warps");
    constexpr int NG = NCW / 4;
    const int grp = warp >> 2, wi = warp & 3;
    const float *F1c = c_fac3, *F2c = c_fac3 + C1, *F3c = c_fac3 + 2 * C1;
    for (int64_t ci = grp;; ci += NG) {
      const int it = (int)(ci >> 2), t = (int)(ci & 3);
      const int64_t tile = cid + (int64_t)it * ncl;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      unsigned char *buf = base + (size_t)st * TB;
      mbar_wait(&full[st], par);
      cb_pair16(buf, (uint32_t)(t * 16 + wi * 4), lane, F1c, F2c);
      named_bar_sync(1 + grp, 128);  // the chunk's four phase-1 units are in shared memory
      cb_top16(buf + (uint32_t)(t * 16) * CE, (uint32_t)(wi * 64 + 2 * lane), F3c);
      __syncwarp();
      mbar_arrive(&cdone[st]);  // every lane publishes its own writes (the signal warp relays to the peer)
    }
  } else if (warp < NCW) {
    // one warp-level P x P x P product with 128B-swizzled A rows arow[] (k in blocks of 8)
    auto gemm = [&](const unsigned char *A, const uint32_t (&arow)[RM], auto loadB, auto &acc) {
      constexpr int NN = sizeof(acc[0]) / sizeof(T);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < NN; ++j) acc[i][j] = 0.f;
#pragma unroll 2
      for (int k0 = 0; k0 < P; k0 += 8) {
        uint32_t ab[RM];
#pragma unroll
        for (int i = 0; i < RM; ++i) ab[i] = arow[i] ^ (uint32_t)(k0 * ES);
#pragma unroll
        for (int kk = 0; kk < 8; kk += VA) {
          T xa[RM][VA];
#pragma unroll
          for (int i = 0; i < RM; ++i) {
            const float4 v = *reinterpret_cast<const float4 *>(A + (ab[i] ^ (uint32_t)(kk * ES)));
            xa[i][0] = v.x; xa[i][1] = v.y; xa[i][2] = v.z; xa[i][3] = v.w;
          }
#pragma unroll
          for (int e = 0; e < VA; ++e) {
            T f[NN];
            loadB(k0, kk + e, f);
#pragma unroll
            for (int i = 0; i < RM; ++i) {
              const float2 xx = make_float2(xa[i][e], xa[i][e]);
#pragma unroll
              for (int j = 0; j < NN; j += 2) {
                const float2 r2 = __ffma2_rn(xx, make_float2(f[j], f[j + 1]), make_float2(acc[i][j], acc[i][j + 1]));
                acc[i][j] = r2.x;
                acc[i][j + 1] = r2.y;
              }
            }
          }
        }
      }
    };
    // phase-1 lane roles (as v6): c1 = subchunk of the unit, sg = row group, q1g = column group
    const int c1 = lane / L1, tau = lane % L1;
    const int sg = tau % (P / RM), q1g = tau / (P / RM);
    uint32_t arow[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) arow[i] = swz128((uint32_t)(sg + (P / RM) * i) * PE);
    // phase-2 lane roles: rows q3 = sg2 + 4i, 8 columns cg*8 .. +8 of the unit's 64-column block
    // (a quarter-warp = 8 lanes of one q3 row: its eight 16-byte column granules are distinct banks)
    const int sg2 = lane / 8, cg = lane % 8;
    uint32_t arow2[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) arow2[i] = swz128((uint32_t)(sg2 + 4 * i) * PE);

    for (int un = warp;; un += NCW) {
      const int it = un / UPT, wu = un % UPT;
      const int64_t tile = cid + (int64_t)it * ncl;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      unsigned char *buf = base + (size_t)st * TB;
      T acc[RM][RN];
      // unit order inside a tile (groups of 4 units): phase 1 of chunks 0, 1, 2, phase 2 of chunk 0, phase 1
      // of chunk 3, phase 2 of chunks 1, 2, 3 — a chunk's phase 2 starts about one wave of units after its
      // phase 1, so the p1 waits rarely block
      // (P2W = 16: phase-2 groups cover two chunks: p1 c0, p1 c1, p2 {c0,c1}, p1 c2, p1 c3, p2 {c2,c3})
      constexpr unsigned kOrder = P2W == 8 ? 0x76534210u : 0x532410u;  // nibble i = (p2 ? 4 : 0) + index
      const int og = (int)((kOrder >> (4 * (wu / 4))) & 15u);
      const int w = og < 4 ? og * 4 + wu % 4 : U1 + (og - 4) * 4 + wu % 4;
      if (w < U1) {
        mbar_wait(&full[st], par);
        const uint32_t gg = (uint32_t)(w * CPG + c1);
        unsigned char *ch = buf + gg * CE;
        const uint32_t gx = pipe_gx<8, 4>(gg);
        gemm(ch, arow, [&](int k0, int kk, T (&f)[RN]) {  // Z = X . F1
          const T *fr = F1s + (k0 + kk) * P + q1g * RN;
#pragma unroll
          for (int j = 0; j < RN; j += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(fr + j);
            f[j] = v.x; f[j + 1] = v.y; f[j + 2] = v.z; f[j + 3] = v.w;
          }
        }, acc);
        __syncwarp();
        auto put = [&]() {
#pragma unroll
          for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int j = 0; j < RN; j += 4)
              *reinterpret_cast<float4 *>(ch + ((arow[i] ^ (uint32_t)((q1g * RN + j) * ES)) ^ gx)) =
                  make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        };
        put();
        __syncwarp();
        const uint32_t Kq = (uint32_t)(q1g * RN * ES) ^ gx;
        gemm(F2Ts, arow, [&](int k0, int kk, T (&f)[RN]) {  // S = F2^T . Z
          const int line0 = (k0 * PE) >> 7, line = (kk * PE) >> 7, a4 = ((kk * PE) & 127) >> 4;
          const uint32_t Kb = Kq ^ ((uint32_t)(line0 & 7) << 4);
          const unsigned char *zb = ch + (line0 + line) * 128;
#pragma unroll
          for (int j = 0; j < RN; j += 4) {
            const uint32_t v = (uint32_t)(a4 ^ (j / 4) ^ (line & 7));
            const float4 t = *reinterpret_cast<const float4 *>(zb + (Kb ^ (v << 4)));
            f[j] = t.x; f[j + 1] = t.y; f[j + 2] = t.z; f[j + 3] = t.w;
          }
        }, acc);
        __syncwarp();
        put();
        __syncwarp();
        mbar_arrive(&p1[4 * st + (int)(gg / 16)]);
      } else {
        constexpr int UPC = 256 / (8 * P2W);  // phase-2 units per chunk
        const int w2 = w - U1, t = w2 / UPC, cb = w2 % UPC;
        mbar_wait(&p1[4 * st + t], par);
        const uint32_t cofs = swz128((uint32_t)(cb * 8 * P2W + cg * P2W) * ES);
        unsigned char *cbase = buf + (uint32_t)(t * 16) * CE;
        T acc2[RM][P2W];
        gemm(F3Ts, arow2, [&](int k0, int kk, T (&f)[P2W]) {  // OUT = F3^T . S over the 16 subchunks
          // subchunk t*16 + k: its granule XOR depends on k mod 8 only (t*16 = 0 mod 8)
          const uint32_t o = (uint32_t)(k0 + kk) * CE + (cofs ^ pipe_gx<8, 4>((uint32_t)(k0 + kk)));
#pragma unroll
          for (int g4 = 0; g4 < P2W / 4; ++g4) {
            const float4 v = *reinterpret_cast<const float4 *>(cbase + (o ^ (16u * g4)));
            f[4 * g4] = v.x; f[4 * g4 + 1] = v.y; f[4 * g4 + 2] = v.z; f[4 * g4 + 3] = v.w;
          }
        }, acc2);
        __syncwarp();  // every lane's reads of the column block are done before it is overwritten
#pragma unroll
        for (int i = 0; i < RM; ++i) {
          const uint32_t o = (uint32_t)(sg2 + 4 * i) * CE + (cofs ^ pipe_gx<8, 4>((uint32_t)(sg2 + 4 * i)));
#pragma unroll
          for (int g4 = 0; g4 < P2W / 4; ++g4)
            *reinterpret_cast<float4 *>(cbase + (o ^ (16u * g4))) =
                make_float4(acc2[i][4 * g4], acc2[i][4 * g4 + 1], acc2[i][4 * g4 + 2], acc2[i][4 * g4 + 3]);
        }
        __syncwarp();
        // the last phase-2 unit of the tile publishes it to both CTAs (one cluster-scope release per tile,
        // from a warp with no global stores in flight)
        mbar_arrive(&cdone[st]);  // every lane publishes its own writes (the signal warp relays to the peer)
      }
    }
  } else if (warp == NCW + NST) {
    // ---------------- signal warp: once this CTA's tile is computed (local acquire of every phase-2 lane's
    // release), ONE cluster-scope release-arrive on the peer's rdy barrier covers all of them (release is
    // cumulative).  A warp with no global stores in flight, so its fence does not wait on HBM writes; the
    // compute warps no longer pay a cluster fence each (ncu: 7.6% of the pass's stall samples).
    for (int it = 0;; ++it) {
      const int64_t tile = cid + (int64_t)it * ncl;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      mbar_wait_sleep(&cdone[st], (uint32_t)((it / S) & 1));
      if (lane == 0) mbar_arrive_cluster(&rdy[st], peer);
      __syncwarp();
    }
  } else {
    // ---------------- store warps: lane pair (i, h) gathers the 8-element run of composite column u from
    // CTA h's four chunks (h = this CTA: local; else DSMEM) and writes its 16-byte half of the 32-byte run
    const int sw = warp - NCW;
    T *Y = reinterpret_cast<T *>(a.Y);
    const int li = lane >> 1, h = lane & 1;
    for (int it = 0;; ++it) {
      const int64_t tile = cid + (int64_t)it * ncl;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      // both CTAs' tiles are computed: this CTA's (local barrier) and the peer's (its signal warp's
      // cluster-scope release, acquired here)
      mbar_wait_sleep(&cdone[st], par);
      mbar_wait_cluster(&rdy[st], par);
      const int rb = (int)(tile / groups), gj = (int)(tile - (int64_t)rb * groups);
      const uint32_t sb = mapa_shared(smem_u32(base + (size_t)st * TB), (uint32_t)h);
      if (rb < a.M) {
        T *yb = Y + (int64_t)rb * a.Wout + (int64_t)gj * 8 + h * 4;
        const int64_t wc = a.WC;
        // lane pair (li, h): four consecutive composite columns u0 .. u0+3 (one 16-byte granule per chunk)
#pragma unroll 2
        for (int ub = (int)rank * 2048 + sw * 64; ub < (int)rank * 2048 + 2048; ub += NST * 64) {
          const uint32_t u0 = (uint32_t)(ub + 4 * li), q3 = u0 >> 8;
          const uint32_t co = swz128((u0 & 255u) * ES);
          float4 v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t gg = (uint32_t)(t * 16) + q3;
            v[t] = ld_dsmem_f32x4(sb + gg * CE + (co ^ pipe_gx<8, 4>(gg)));
          }
          const float4 o4[4] = {make_float4(v[0].x, v[1].x, v[2].x, v[3].x), make_float4(v[0].y, v[1].y, v[2].y, v[3].y),
                                make_float4(v[0].z, v[1].z, v[2].z, v[3].z), make_float4(v[0].w, v[1].w, v[2].w, v[3].w)};
          if constexpr (!PUSH) {
            T *yu = yb + (int64_t)u0 * wc;
#pragma unroll
            for (int j = 0; j < 4; ++j) *reinterpret_cast<float4 *>(yu + j * wc) = o4[j];
          } else {
            // distributed round (NEXT-1, fused): the 16-byte run goes straight to its StoreGPUTile position
            // in the destination rank's next-round block over NVLink (runs of rho never split: rho % 4 == 0)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int64_t col = (int64_t)(u0 + j) * wc + (int64_t)gj * 8 + h * 4;
              *reinterpret_cast<float4 *>(push_dst<T>(a, rb, col)) = o4[j];
            }
          }
        }
      }
      __syncwarp();
      // the last store warp hands this CTA's stage back (its own reads and, through the peer's arrive, the
      // peer's DSMEM reads of it have returned) and refills it
      mbar_arrive(&empty[st]);  // every lane: its reads of this CTA's stage are done
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&scnt[st], 1u) == (unsigned)NST - 1) {
          scnt[st] = 0;
          __threadfence_block();
          mbar_arrive_cluster(&empty[st], peer);  // release: this CTA's DSMEM reads of the peer's stage
          mbar_wait_cluster(&empty[st], par);
          fence_proxy_async_smem();
          issue_load(it + S);
        }
      }
      __syncwarp();
    }
  }
  cluster_sync_all();  // neither CTA leaves while its peer may still read its shared memory
}

// ------------------------------------------------------------------ v11: tile-major hand-off between two fused passes
//
// A two-pass plan [group A, group B] whose second pass covers every remaining factor has C_B = W / C_A: pass
// B's chunk index is pass A's composite output column u and its in-chunk index is pass A's chunk index g
// (T[row][u*(W/C_A) + g], the direct-index layout).  With 16 KB chunks (config E's 16^3 triple)
// the direct-index store writes 32-byte runs at a 1 KB stride — measured 3.0-3.5 TB/s, which made v10's
// triple store-bound (10.6 ms for 34 GB).  v11 moves the permutation into pass B's TMA map instead:
//   pass A (kron_tri_tm_kernel) writes each 4-chunk tile as ONE contiguous 64 KB block
//       T''[row][g / 4][u][g % 4]                                   (fully coalesced 512-byte warp stores);
//   pass B (kron_pair_tm_kernel) loads its tile of R chunks u0 .. u0+R-1 through the 3-D map
//       {4u + g % 4, g / 4, row} with box {4R, C_B / 4, 1}          (1 KB contiguous runs per g / 4)
// so no extra pass runs and each value still crosses HBM once out and once in.  The values are those of the
// direct-index layout (same arithmetic, same order: results are bit-identical to the v10 plan); only the
// intermediate's element order differs.  Y (the last pass's output) keeps the paper's layout.
//
// kron_tri_tm_kernel: 16 x 16 fp32 factor triples, factors in the constant bank (cb_pair16 / cb_top16 as v10),
// one CTA per SM (no cluster, no DSMEM), tiles of 4 chunks (64 KB) through a 3-stage TMA ring; NCW compute warps
// in groups of four (one chunk per group), four store warps.
template <int NCW>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) kron_tri_tm_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                        const FusedArgs a) {
  constexpr uint32_t CE = 1024, TB = 64 * CE;  // 16 subchunks of 1 KB per chunk, 4 chunks per tile
  constexpr int NSW = 4, C = 4096;
  static_assert(NCW % 4 == 0, "groups of four compute warps");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.stages;
  uint64_t *full = reinterpret_cast<uint64_t *>(base + (size_t)S * TB);
  uint64_t *cdone = full + S, *empty = cdone + S;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // provably warp-uniform
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], 4 * 4 * 32);  // four chunks x four warps x 32 lanes
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % S;
    const int rb = (int)(tile / a.tiles_k), gq = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * TB;
    mbar_arrive_expect_tx(&full[st], TB);
    const int line0 = gq * (4 * C / 32);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &full[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < S; ++it) issue_load(it);

  if (warp < NCW) {
    // as v10: group grp owns one chunk at a time (chunks dealt round-robin across the tiles of the ring); warp
    // wi runs phase 1 on subchunks 4wi .. 4wi+3, the group meets at a named barrier, then phase 2 on columns
    // 64wi .. 64wi+63
    constexpr int NG = NCW / 4;
    const int grp = warp >> 2, wi = warp & 3;
    const float *F1c = c_fac3, *F2c = c_fac3 + 256, *F3c = c_fac3 + 512;
    for (int64_t ci = grp;; ci += NG) {
      const int it = (int)(ci >> 2), t = (int)(ci & 3);
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      unsigned char *buf = base + (size_t)st * TB;
      mbar_wait(&full[st], (uint32_t)((it / S) & 1));
      cb_pair16(buf, (uint32_t)(t * 16 + wi * 4), lane, F1c, F2c);
      named_bar_sync(1 + grp, 128);
      cb_top16(buf + (uint32_t)(t * 16) * CE, (uint32_t)(wi * 64 + 2 * lane), F3c);
      __syncwarp();
      mbar_arrive(&cdone[st]);
    }
  } else {
    // store warps: lane = composite column u; OUT of chunk t at t*16 KB + (u/256)*1 KB + (swz128(4*(u%256)) ^
    // gx(u/256)) (cb_top16's layout: 32 consecutive u = one permuted 128-byte line, conflict-free), the four
    // chunks' values form one float4 of T''[row][gq][u][0..3]: a warp writes 512 contiguous bytes
    const int sw = warp - NCW;
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      mbar_wait_sleep(&cdone[st], par);
      const unsigned char *buf = base + (size_t)st * TB;
      const int rb = (int)(tile / a.tiles_k), gq = (int)(tile - (int64_t)rb * a.tiles_k);
      if (rb < a.M) {
        // single GPU: one block T''[row][gq][u][4]; distributed round (push.on): the u range split over the GK
        // destinations, send[d][row][gq][u - d*Ud][4] (Ud = push.B composite columns per destination: the
        // round's destination-major send block in the tile-major order the next round's map reads)
        const int64_t Ud = a.push.on ? a.push.B : C;
        float4 *yb = reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.Y) + (int64_t)rb * a.Wout + (int64_t)gq * 4 * C);
#pragma unroll 4
        for (int ub = sw * 32; ub < C; ub += NSW * 32) {
          const uint32_t u = (uint32_t)(ub + lane), q3 = u >> 8;
          const uint32_t off = q3 * CE + (swz128((u & 255u) * 4u) ^ pipe_gx<8, 4>(q3));
          float4 v;
          v.x = *reinterpret_cast<const float *>(buf + off);
          v.y = *reinterpret_cast<const float *>(buf + 16 * CE + off);
          v.z = *reinterpret_cast<const float *>(buf + 32 * CE + off);
          v.w = *reinterpret_cast<const float *>(buf + 48 * CE + off);
          if (a.push.on) {
            const int d = ub / (int)Ud;  // warp-uniform: Ud is a multiple of 32
            float4 *sb = reinterpret_cast<float4 *>(a.push.dst[d]) + ((int64_t)rb * a.tiles_k + gq) * Ud;
            sb[u - (int64_t)d * Ud] = v;
          } else {
            yb[u] = v;
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
}

// tm_pair16: both factors of a 16 x 16 pair on eight 256-element chunks u0 .. u0+7 of a tile loaded in the
// tile-major order [g/4][u][g%4] (element g = 16r + c of chunk u at (4r + c/4)*1 KB + u*16 + (c%4)*4):
//   step 1 (F1 on c): lane = chunk u0 + lane%8, rows 4(lane/8) .. +3 (two at a time, as cb_pair16): a quarter-warp
//          reads / writes one 128-byte run of eight chunks' granules (LDS.128 / STS.128, conflict-free);
//   step 2 (F2 on r): lane = chunk u0 + lane%8, column pair 2(2k + (lane/8)%2) .. +1 with granule k = 2kk + lane/16;
//          16 LDS.64 over the rows, 256 FFMA2 with a factor broadcast, 16 STS.64 over the same words (OUT[q2][q1]
//          in place of Z[s = q2][q1]); each half-warp covers one 128-byte run (conflict-free).
// Same products and summation order as cb_pair16 (bit-identical results).
__device__ __forceinline__ void tm_pair16(unsigned char *buf, uint32_t u0, int lane, const float *F1, const float *F2) {
  const float4 *F1v = reinterpret_cast<const float4 *>(F1), *F2v = reinterpret_cast<const float4 *>(F2);
  const uint32_t cu = (u0 + (uint32_t)(lane & 7)) * 16u;
  {
    const int rg = lane >> 3;
#pragma unroll 1
    for (int i = 0; i < 2; ++i) {
      float x[2][16];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t r = (uint32_t)(rg * 4 + 2 * i + h);
          const float4 t = *reinterpret_cast<const float4 *>(buf + (4u * r + v) * 1024u + cu);
          x[h][4 * v] = t.x; x[h][4 * v + 1] = t.y; x[h][4 * v + 2] = t.z; x[h][4 * v + 3] = t.w;
        }
      float2 acc[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[h][j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int p = 0; p < 16; ++p)
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 f = F1v[p * 4 + j4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 xx = make_float2(x[h][p], x[h][p]);
            acc[h][2 * j4] = __ffma2_rn(xx, make_float2(f.x, f.y), acc[h][2 * j4]);
            acc[h][2 * j4 + 1] = __ffma2_rn(xx, make_float2(f.z, f.w), acc[h][2 * j4 + 1]);
          }
        }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t r = (uint32_t)(rg * 4 + 2 * i + h);
          *reinterpret_cast<float4 *>(buf + (4u * r + v) * 1024u + cu) =
              make_float4(acc[h][2 * v].x, acc[h][2 * v].y, acc[h][2 * v + 1].x, acc[h][2 * v + 1].y);
        }
    }
  }
  __syncwarp();  // step 2 reads other lanes' step-1 rows
  {
    const uint32_t s8 = (uint32_t)((lane >> 3) & 1) * 8u;
#pragma unroll 1
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t k = (uint32_t)(2 * kk + (lane >> 4));
      unsigned char *cb = buf + k * 1024u + cu + s8;
      float2 x2[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) x2[r] = *reinterpret_cast<const float2 *>(cb + (uint32_t)r * 4096u);
      float2 acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 f = F2v[r * 4 + q4];
          acc[4 * q4] = __ffma2_rn(x2[r], make_float2(f.x, f.x), acc[4 * q4]);
          acc[4 * q4 + 1] = __ffma2_rn(x2[r], make_float2(f.y, f.y), acc[4 * q4 + 1]);
          acc[4 * q4 + 2] = __ffma2_rn(x2[r], make_float2(f.z, f.z), acc[4 * q4 + 2]);
          acc[4 * q4 + 3] = __ffma2_rn(x2[r], make_float2(f.w, f.w), acc[4 * q4 + 3]);
        }
#pragma unroll
      for (int q = 0; q < 16; ++q) *reinterpret_cast<float2 *>(cb + (uint32_t)q * 4096u) = acc[q];
    }
  }
}

// kron_pair_tm_kernel: the 16 x 16 fp32 pair of pass B, input tile-major (see above), factors in the constant bank;
// tiles of R chunks (R * 1 KB) through a TMA ring; units of eight chunks dealt round-robin to NCW compute warps
// across tile boundaries; four store warps stream the tile out chunk-fastest to Y[row][u2*(W/C) + cb*R + u]
// (lane = chunk: every store instruction writes one 128-byte line).
template <int NCW>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) kron_pair_tm_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                         const FusedArgs a) {
  constexpr int NSW = 4, UC = 8;
  const int R = a.R, UPT = R / UC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.stages;
  uint64_t *full = reinterpret_cast<uint64_t *>(base + (size_t)S * a.stage_bytes);
  uint64_t *cdone = full + S, *empty = cdone + S;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // provably warp-uniform
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], UPT * 32);
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % S;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    mbar_arrive_expect_tx(&full[st], a.tile_bytes);
    // distributed round: the map has a 4th dimension, the source rank of the receive buffer (rmp_GK sources)
    if (a.rmp_GK) tma_load_4d(base + (size_t)st * a.stage_bytes, &tm_in, &full[st], cb * R * 4, 0, rb, 0);
    else tma_load_3d(base + (size_t)st * a.stage_bytes, &tm_in, &full[st], cb * R * 4, 0, rb);
  };
  if (tid == 0)
    for (int it = 0; it < S; ++it) issue_load(it);

  if (warp < NCW) {
    const float *F1c = c_fac2, *F2c = c_fac2 + 256;
    for (int un = warp;; un += NCW) {
      const int it = un / UPT, cg = un - (un / UPT) * UPT;
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      mbar_wait(&full[st], (uint32_t)((it / S) & 1));
      tm_pair16(base + (size_t)st * a.stage_bytes, (uint32_t)(cg * UC), lane, F1c, F2c);
      __syncwarp();
      mbar_arrive(&cdone[st]);
    }
  } else {
    const int sw = warp - NCW;
    float *Y = reinterpret_cast<float *>(a.Y);
    const int push_ush = a.push.on ? __ffs((int)(a.push.B / a.WC)) - 1 : 0;
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % S;
      const uint32_t par = (uint32_t)((it / S) & 1);
      mbar_wait_sleep(&cdone[st], par);
      const unsigned char *buf = base + (size_t)st * a.stage_bytes;
      const int rb = (int)(tile / a.tiles_k), cbk = (int)(tile - (int64_t)rb * a.tiles_k);
      if (rb < a.M) {
        const int64_t wc = a.WC;
        float *yr = Y + (int64_t)rb * a.Wout + (int64_t)cbk * R + lane;
        const int64_t push_row = (int64_t)rb * a.push.B;
        // granule gk = 4*q2 + q1/4 holds composite columns u2 = 4*gk .. 4*gk+3 of every chunk
#pragma unroll 1
        for (int gk = sw; gk < 64; gk += NSW) {
          float *p = yr + (int64_t)(4 * gk) * wc;
          for (int h = 0; h < R / 32; ++h) {
            const float4 v = *reinterpret_cast<const float4 *>(buf + (uint32_t)gk * 1024u + (uint32_t)(h * 32 + lane) * 16u);
            if (a.push.on) {
              // distributed round: column c = u2*wc + chunk goes to destination d = c / B of the send block
              // send[d][row][B] (the pack fused into the store, as the v6 / v10 PUSH epilogues with rho = B, GK = 1);
              // with B a multiple of wc (push.B = W / GK, wc = W / 256): d = u2 >> ush, B / wc = 2^ush composite
              // columns per destination (ush computed once per warp, no division in the loop)
              const float vv[4] = {v.x, v.y, v.z, v.w};
              const int d = (4 * gk) >> push_ush;  // the four columns 4gk .. 4gk+3 share a destination (B / wc >= 4)
              float *sd = reinterpret_cast<float *>(a.push.dst[d]) + push_row + (int64_t)cbk * R + h * 32 + lane +
                          (int64_t)((4 * gk) & ((1 << push_ush) - 1)) * wc;
#pragma unroll
              for (int j = 0; j < 4; ++j) sd[(int64_t)j * wc] = vv[j];
            } else {
              p[h * 32] = v.x;
              p[h * 32 + wc] = v.y;
              p[h * 32 + 2 * wc] = v.z;
              p[h * 32 + 3 * wc] = v.w;
            }
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
}

// ------------------------------------------------------------------ fp64 two-factor chunks on DMMA (v5)
//
// The v4 sandwich OUT = F2^T . (X . F1) per 32 x 32 chunk, fp64, on the FP64 tensor cores (mma.sync
// m16n8k4, SASS DMMA — tcgen05 has no f64 kind).  A warp owns a chunk: GEMM1 (64 DMMA) reads X rows
// from the TMA tile and F1 from shared memory, writes Z in place; GEMM2 (64 DMMA) reads F2^T and Z and
// writes OUT[q2][q1] in place.  All [32][32] fp64 matrices use 256-byte rows with the 128B swizzle on
// each 128-byte line, which makes every fragment gather bank-conflict free.  A CTA-wide pass then
// streams OUT chunk-fastest to Y[row][u*(W/C) + g0 + g]: 8 consecutive chunks = 64-byte runs.
__device__ __forceinline__ uint32_t rowswz32(uint32_t r, uint32_t c) {  // [rows][32 doubles], byte offset
  const uint32_t line = 2u * r + (c >> 4);
  return line * 128u + (((c & 15u) << 3) ^ ((line & 7u) << 4));
}
// The same [rows][32 doubles] rows with the 16-byte granule XOR'd by (r & 1) * 4 + ((r >> 1) & 1) * 2 instead of
// the TMA line pattern: with it the accumulator write-back (STS.128, lanes = 8 rows x 4 column pairs), the
// B-fragment gathers (LDS.64, 4 rows x 8 columns) and the chunk-fastest stream-out reads are all at ncu's ideal
// wavefront count (a GF(2) search with a bank model, tools/swizzle_search.py; with the TMA pattern the
// write-back took 2x its ideal wavefronts: profiles/r02_banks_C64.json).  Used for Z and OUT, which the kernel
// itself writes; X keeps the TMA layout (rowswz32).
__device__ __forceinline__ uint32_t rowswzZ(uint32_t r, uint32_t c) {
  const uint32_t line = 2u * r + (c >> 4);
  return line * 128u + (((c & 15u) << 3) ^ ((((r & 1u) << 2) | (r & 2u)) << 4));
}

// Warp-specialised: NCW compute warps (one chunk each per tile; with NCW = 2 * CPT two groups take
// alternate tiles; NCW = 16 gives every SM sub-partition four DMMA warps) never stop for the HBM stream-out, which NSW
// store warps do from the finished tile while the compute warps work on the next ones (mbarriers:
// full = TMA landed, cdone = chunks computed, empty = tile streamed out -> refill).
// Round 2: GEMM1 by row halves and GEMM2 by column halves, each half's results written right away (Z rows depend
// only on their own X rows; an OUT column half only on the Z columns of that half) — half the accumulator
// registers (96), so two tile groups of 8 compute warps fit (NCW = 16): C64 9.00 -> 8.75 ms
template <int NCW, int NSW, int CPT>
__global__ void __launch_bounds__((NCW + NSW) * 32, 1) kron_fused_dmma2_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                             const FusedArgs a) {
  constexpr int P = 32, C = P * P, LINE = 16;  // CPT = chunks per tile
  static_assert(NCW % CPT == 0, "compute warps come in groups of one tile");
  constexpr uint32_t CB = C * 8;  // chunk bytes
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *F1s = base + (size_t)a.stages * a.stage_bytes;  // [p][q1]
  unsigned char *F2Ts = F1s + CB;                                 // [q2][s] = F2[s][q2]
  uint64_t *full = reinterpret_cast<uint64_t *>(F2Ts + CB);
  uint64_t *cdone = full + a.stages, *empty = cdone + a.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;

  {
    const double *F1 = reinterpret_cast<const double *>(a.F[0]);
    const double *F2 = reinterpret_cast<const double *>(a.F[1]);
    for (int i = tid; i < C; i += (NCW + NSW) * 32) {
      const uint32_t r = (uint32_t)i / P, c = (uint32_t)i % P;
      *reinterpret_cast<double *>(F1s + rowswz32(r, c)) = F1[i];   // F1[p = r][q1 = c]
      *reinterpret_cast<double *>(F2Ts + rowswz32(c, r)) = F2[i];  // F2[s = r][q2 = c] -> F2T[c][r]
    }
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], CPT * 32);
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&full[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &full[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  if (warp < NCW) {
    // ---------------- compute warps: chunk (warp % CPT) of every (NCW / CPT)-th tile
    const int g = warp % CPT;
    const uint32_t gx = pipe_gx<8, 4>((uint32_t)g);
    for (int it = warp / CPT;; it += NCW / CPT) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      mbar_wait(&full[st], (uint32_t)((it / a.stages) & 1));
      unsigned char *cb0 = base + (size_t)st * a.stage_bytes + (uint32_t)g * CB;
      {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {  // GEMM1, rows 16mt..16mt+15 (they read only their own X rows)
          double acc1[4][4];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc1[nt][e] = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < P; k0 += 4) {
            const double a0 = *reinterpret_cast<const double *>(cb0 + rowswz32(mt * 16 + gq, k0 + tq));
            const double a1 = *reinterpret_cast<const double *>(cb0 + rowswz32(mt * 16 + gq + 8, k0 + tq));
            double b[4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) b[nt] = *reinterpret_cast<const double *>(F1s + rowswz32(k0 + tq, nt * 8 + gq));
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma_m16n8k4(acc1[nt], a0, a1, b[nt]);
          }
          __syncwarp();
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int v1 = 0; v1 < 2; ++v1)
              *reinterpret_cast<double2 *>(cb0 + rowswzZ(mt * 16 + gq + 8 * v1, nt * 8 + 2 * tq)) =
                  make_double2(acc1[nt][2 * v1], acc1[nt][2 * v1 + 1]);
        }
        __syncwarp();
#pragma unroll
        for (int nq = 0; nq < 2; ++nq) {  // GEMM2, columns 16nq..16nq+15 (OUT stays inside those columns' lines)
          double acc2[2][2][4];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) acc2[mt][nt][e] = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < P; k0 += 4) {
            double a0[2], a1[2], b[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              a0[mt] = *reinterpret_cast<const double *>(F2Ts + rowswz32(mt * 16 + gq, k0 + tq));
              a1[mt] = *reinterpret_cast<const double *>(F2Ts + rowswz32(mt * 16 + gq + 8, k0 + tq));
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              b[nt] = *reinterpret_cast<const double *>(cb0 + rowswzZ(k0 + tq, nq * 16 + nt * 8 + gq));
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) dmma_m16n8k4(acc2[mt][nt], a0[mt], a1[mt], b[nt]);
          }
          __syncwarp();
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
              for (int v1 = 0; v1 < 2; ++v1)
                *reinterpret_cast<double2 *>(cb0 + (rowswzZ(mt * 16 + gq + 8 * v1, nq * 16 + nt * 8 + 2 * tq) ^ gx)) =
                    make_double2(acc2[mt][nt][2 * v1], acc2[mt][nt][2 * v1 + 1]);
        }
        __syncwarp();
        mbar_arrive(&cdone[st]);  // every lane: each publishes its own writes
      }
    }
  } else {
    // ---------------- store warps: chunk-fastest stream-out, Y[row][u*(W/C) + cb*R + g]
    const int sw = warp - NCW;
    double *Y = reinterpret_cast<double *>(a.Y);
    constexpr int UPW = 32 / CPT;  // u values per warp instruction (CPT consecutive chunks each)
    const int g = lane % CPT;
    const uint32_t gx = pipe_gx<8, 4>((uint32_t)g);
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      const uint32_t par = (uint32_t)((it / a.stages) & 1);
      mbar_wait(&cdone[st], par);
      const unsigned char *buf = base + (size_t)st * a.stage_bytes + (uint32_t)g * CB;
      const int rb = (int)(tile / a.tiles_k), cbk = (int)(tile - (int64_t)rb * a.tiles_k);
      if (rb < a.M && (int64_t)cbk * a.R + g < a.WC) {
        double *yg = Y + (int64_t)rb * a.Wout + (int64_t)cbk * a.R + g;
#pragma unroll 4
        for (int w = sw; w < C / UPW; w += NSW) {
          const int u = w * UPW + lane / CPT;
          const double v = *reinterpret_cast<const double *>(buf + (rowswzZ((uint32_t)u / P, (uint32_t)u % P) ^ gx));
          yg[(int64_t)u * a.WC] = v;
        }
      }
      __syncwarp();
      mbar_arrive(&empty[st]);
      if (sw == 0) {
        if (lane == 0) {
          mbar_wait(&empty[st], par);
          fence_proxy_async_smem();
          issue_load(it + a.stages);
        }
        __syncwarp();
      }
    }
  }
}

// ------------------------------------------------------------------ fp64 non-square chunk pairs on DMMA (v7)
//
// Two consecutive 64 x 32 factors (the GP-style shape of config D2) fused in one pass: a chunk is a
// 64 x 64 matrix X[s][p] (C = 4096) and the pair is OUT[q2][q1] = sum_s F2[s][q2] * (X . F1)[s][q1]
// (32 x 32 = Qc = 1024 outputs, u = q2*32 + q1, P:519-523 with P != Q, reading G8).  A chunk is loaded
// as two TMA boxes of its p-halves, each a [64][32] matrix with 256-byte rows (the v5 layout, so the
// fragment gathers are conflict free).  Two warps share a chunk: warp h computes Z rows 32h..32h+31
// (GEMM1, 128 DMMA) and writes them over the p < 32 rows it consumed, then — after a pair barrier —
// OUT rows 16h..16h+15 (GEMM2, 64 DMMA) into the p >= 32 half.  Four store warps send each finished
// chunk to Y[row][u*(W/C) + g]; a CTA walks a contiguous range of chunks so consecutive chunks' stores
// land next to each other while their L2 lines are still resident.
__device__ __forceinline__ uint32_t rowswz64(uint32_t r, uint32_t c) {  // [rows][64 doubles], thread-filled
  // granule XOR 2*(r % 4) + (r / 4) % 2: the A-fragment gathers (4 rows x 4 consecutive doubles per half-warp)
  // hit 8 distinct granules (with r % 8 they paired up: 2x the ideal wavefronts, profiles/r02_banks_D2.json)
  return r * 512u + ((c * 8u) ^ ((((r & 3u) << 1) | ((r >> 2) & 1u)) << 4));
}

template <int NCW, int NSW>
__global__ void __launch_bounds__((NCW + NSW) * 32, 1) kron_fused_dmma2g_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                              const FusedArgs a) {
  constexpr int P = 64, Q = 32, C = P * P, CO = Q * Q;
  constexpr uint32_t CB = C * 8, HB = CB / 2;  // chunk bytes, p-half bytes
  static_assert(NCW % 2 == 0, "compute warps come in pairs");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *F1s = base + (size_t)a.stages * CB;  // [p][q1], rowswz32 (64 rows)
  unsigned char *F2Ts = F1s + P * Q * 8;              // [q2][s] = F2[s][q2], rowswz64 (32 rows)
  uint64_t *full = reinterpret_cast<uint64_t *>(F2Ts + P * Q * 8);
  uint64_t *cdone = full + a.stages, *empty = cdone + a.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  {
    const double *F1 = reinterpret_cast<const double *>(a.F[0]);
    const double *F2 = reinterpret_cast<const double *>(a.F[1]);
    for (int i = tid; i < P * Q; i += (NCW + NSW) * 32) {
      const uint32_t r = (uint32_t)i / Q, c = (uint32_t)i % Q;
      *reinterpret_cast<double *>(F1s + rowswz32(r, c)) = F1[i];   // F1[p = r][q1 = c]
      *reinterpret_cast<double *>(F2Ts + rowswz64(c, r)) = F2[i];  // F2[s = r][q2 = c] -> F2T[c][r]
    }
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], 2 * 32);
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  // a CTA walks the contiguous chunk range [t0, t1)
  const int64_t per = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t t1 = t0 + per < a.ntiles ? t0 + per : a.ntiles;
  auto issue_load = [&](int it) {
    const int64_t tile = t0 + it;
    if (tile >= t1) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), g = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * CB;
    mbar_arrive_expect_tx(&full[st], CB);
    tma_load_5d(dst, &tm_in, &full[st], 0, 0, 0, g, rb);
    tma_load_5d(dst + HB, &tm_in, &full[st], 0, 2, 0, g, rb);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  if (warp < NCW) {
    const int pair = warp >> 1, h = warp & 1;
    for (int it = pair; t0 + it < t1; it += NCW / 2) {
      const int st = it % a.stages;
      mbar_wait(&full[st], (uint32_t)((it / a.stages) & 1));
      unsigned char *cb0 = base + (size_t)st * CB;
      double acc[2][4][4];
      // ---- GEMM1 (rows 32h..32h+31): Z[s][q1] = sum_p X[s][p] F1[p][q1]; p-half hp at cb0 + hp*HB
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0;
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {
        const unsigned char *xb = cb0 + hp * HB;
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
          double a0[2], a1[2], b[4];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const uint32_t r = (uint32_t)(h * 32 + mt * 16 + gq);
            a0[mt] = *reinterpret_cast<const double *>(xb + rowswz32(r, k0 + tq));
            a1[mt] = *reinterpret_cast<const double *>(xb + rowswz32(r + 8, k0 + tq));
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
            b[nt] = *reinterpret_cast<const double *>(F1s + rowswz32(hp * 32 + k0 + tq, nt * 8 + gq));
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma_m16n8k4(acc[mt][nt], a0[mt], a1[mt], b[nt]);
        }
      }
      __syncwarp();
      // Z rows of this warp over the p < 32 half of the rows it consumed (same [64][32] layout)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int v1 = 0; v1 < 2; ++v1)
            *reinterpret_cast<double2 *>(cb0 + rowswzZ(h * 32 + mt * 16 + gq + 8 * v1, nt * 8 + 2 * tq)) =
                make_double2(acc[mt][nt][2 * v1], acc[mt][nt][2 * v1 + 1]);
      named_bar_sync(2 + pair, 64);  // both halves of Z written (and both GEMM1s done with the p >= 32 half)
      // ---- GEMM2 (rows q2 = 16h..16h+15): OUT[q2][q1] = sum_s F2T[q2][s] Z[s][q1]
      double acc2[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc2[nt][e] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 64; k0 += 4) {
        const uint32_t r = (uint32_t)(h * 16 + gq);
        const double a0 = *reinterpret_cast<const double *>(F2Ts + rowswz64(r, k0 + tq));
        const double a1 = *reinterpret_cast<const double *>(F2Ts + rowswz64(r + 8, k0 + tq));
        double b[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) b[nt] = *reinterpret_cast<const double *>(cb0 + rowswzZ(k0 + tq, nt * 8 + gq));
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_m16n8k4(acc2[nt], a0, a1, b[nt]);
      }
      // OUT rows into the p >= 32 half (no longer read by anyone); [32][32], rowswzZ
      unsigned char *ob = cb0 + HB;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1)
          *reinterpret_cast<double2 *>(ob + rowswzZ(h * 16 + gq + 8 * v1, nt * 8 + 2 * tq)) =
              make_double2(acc2[nt][2 * v1], acc2[nt][2 * v1 + 1]);
      __syncwarp();
      mbar_arrive(&cdone[st]);  // every lane: each publishes its own writes
    }
  } else {
    // ---------------- store warps: OUT[u] -> Y[row][u*(W/C) + g]
    const int sw = warp - NCW;
    double *Y = reinterpret_cast<double *>(a.Y);
    for (int it = 0; t0 + it < t1; ++it) {
      const int64_t tile = t0 + it;
      const int st = it % a.stages;
      const uint32_t par = (uint32_t)((it / a.stages) & 1);
      mbar_wait_sleep(&cdone[st], par);
      const unsigned char *ob = base + (size_t)st * CB + HB;
      const int rb = (int)(tile / a.tiles_k), g = (int)(tile - (int64_t)rb * a.tiles_k);
      double *yg = Y + (int64_t)rb * a.Wout + g;
#pragma unroll 4
      for (int u = sw * 32 + lane; u < CO; u += NSW * 32)
        yg[(int64_t)u * a.WC] = *reinterpret_cast<const double *>(ob + rowswzZ((uint32_t)u / Q, (uint32_t)u % Q));
      __syncwarp();
      mbar_arrive(&empty[st]);
      if (sw == 0) {
        if (lane == 0) {
          mbar_wait_sleep(&empty[st], par);
          fence_proxy_async_smem();
          issue_load(it + a.stages);
        }
        __syncwarp();
      }
    }
  }
}

// ------------------------------------------------------------------ fp32 chunk pairs, 3xTF32 tensor cores (v8)
//
// NEXT-4 (reported separately from the fp32 CUDA-core numbers): the v6 sandwich for P = 32 fp32 on the
// legacy warp MMA (mma.sync m16n8k8 TF32, SASS HMMA; measured 275 TF/s vs 74 TF/s FFMA2,
// profiles/r01_microbench_mma.jsonl) with the 3xTF32 split x = hi + lo per operand and
// acc += a_lo b_hi + a_hi b_lo + a_hi b_hi (fp32 accumulation): products keep ~22 significant bits,
// well inside the fp32 parity bar, and small-integer data stays bit-exact (lo = 0).  A warp owns a
// chunk: GEMM1 = X . F1 (A = X rows of the TMA tile, B = F1^T rows), Z^T written in place; GEMM2 =
// F2^T . Z (A = F2^T rows, B = Z^T rows), OUT written in place; every operand is a [32][32] matrix
// with 128-byte rows and the 128B swizzle, so all fragment gathers are conflict free.  Factor hi/lo
// splits are computed once per CTA.  Store warps as in v6.
__device__ __forceinline__ uint32_t sw32(uint32_t r, uint32_t c) {  // [32][32] fp32, 128B swizzle
  return r * 128u + ((c * 4u) ^ ((r & 7u) << 4));
}

template <int NCW, int NSW>
__global__ void __launch_bounds__((NCW + NSW) * 32, 1) kron_fused_tf32x3_kernel(const __grid_constant__ CUtensorMap tm_in,
                                                                              const FusedArgs a) {
  constexpr int P = 32, C = P * P, LINE = 32;
  constexpr uint32_t CE = C * 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char *FT = base + (size_t)a.stages * a.stage_bytes;  // [4][32][32] tf32: F1T hi, F1T lo, F2T hi, F2T lo
  uint64_t *full = reinterpret_cast<uint64_t *>(FT + 4 * CE);
  uint64_t *cdone = full + a.stages, *empty = cdone + a.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  {
    const float *F1 = reinterpret_cast<const float *>(a.F[0]);
    const float *F2 = reinterpret_cast<const float *>(a.F[1]);
    for (int i = tid; i < C; i += (NCW + NSW) * 32) {
      const uint32_t r = (uint32_t)i / P, c = (uint32_t)i % P;
      uint32_t hi, lo;
      tf32_split(F1[i], hi, lo);  // F1[p = r][q1 = c] -> F1T[c][r]
      *reinterpret_cast<uint32_t *>(FT + sw32(c, r)) = hi;
      *reinterpret_cast<uint32_t *>(FT + CE + sw32(c, r)) = lo;
      tf32_split(F2[i], hi, lo);  // F2[s = r][q2 = c] -> F2T[c][r]
      *reinterpret_cast<uint32_t *>(FT + 2 * CE + sw32(c, r)) = hi;
      *reinterpret_cast<uint32_t *>(FT + 3 * CE + sw32(c, r)) = lo;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&cdone[s], a.R * 32);  // one arrival per lane per chunk
      mbar_init(&empty[s], NSW * 32);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_in);
  }
  __syncthreads();
  auto issue_load = [&](int it) {
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= a.ntiles) return;
    const int st = it % a.stages;
    const int rb = (int)(tile / a.tiles_k), cb = (int)(tile - (int64_t)rb * a.tiles_k);
    unsigned char *dst = base + (size_t)st * a.stage_bytes;
    mbar_arrive_expect_tx(&full[st], a.tile_bytes);
    const int line0 = cb * (a.tileK / LINE);
    for (int b = 0; b < a.nbox; ++b)
      load_in(a, dst + (size_t)b * a.box_lines * 128, &tm_in, &full[st], line0 + b * a.box_lines, rb);
  };
  if (tid == 0)
    for (int it = 0; it < a.stages; ++it) issue_load(it);

  if (warp < NCW) {
    // one warp-level 32 x 32 x 32 product, 3xTF32: acc[mt][nt] = A[32][32] . B, with A rows and
    // B^T rows both stored [32][32] swizzled; A split on the fly (xsplit) or pre-split (a_hi/a_lo)
    auto gemm = [&](const unsigned char *Ah, const unsigned char *Al, bool asplit, const unsigned char *Bh,
                    const unsigned char *Bl, bool bsplit, float (&acc)[2][4][4]) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
#pragma unroll 2
      for (int k0 = 0; k0 < P; k0 += 8) {
        uint32_t ah[2][4], al[2][4], bh[4][2], bl[4][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t r = (uint32_t)(mt * 16 + g + 8 * (e & 1)), c = (uint32_t)(k0 + t + 4 * (e >> 1));
            if (asplit) {
              tf32_split(*reinterpret_cast<const float *>(Ah + sw32(r, c)), ah[mt][e], al[mt][e]);
            } else {
              ah[mt][e] = *reinterpret_cast<const uint32_t *>(Ah + sw32(r, c));
              al[mt][e] = *reinterpret_cast<const uint32_t *>(Al + sw32(r, c));
            }
          }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t r = (uint32_t)(nt * 8 + g), c = (uint32_t)(k0 + t + 4 * e);
            if (bsplit) {
              tf32_split(*reinterpret_cast<const float *>(Bh + sw32(r, c)), bh[nt][e], bl[nt][e]);
            } else {
              bh[nt][e] = *reinterpret_cast<const uint32_t *>(Bh + sw32(r, c));
              bl[nt][e] = *reinterpret_cast<const uint32_t *>(Bl + sw32(r, c));
            }
          }
        // the three products of the split, small terms first; 8 independent accumulators per term
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[mt][nt], al[mt], bh[nt][0], bh[nt][1]);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[mt][nt], ah[mt], bl[nt][0], bl[nt][1]);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[mt][nt], ah[mt], bh[nt][0], bh[nt][1]);
      }
    };
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      mbar_wait(&full[st], (uint32_t)((it / a.stages) & 1));
      unsigned char *buf = base + (size_t)st * a.stage_bytes;
      for (int gg = warp; gg < a.R; gg += NCW) {
        unsigned char *ch = buf + (uint32_t)gg * CE;
        const uint32_t gx = pipe_gx<8, 4>((uint32_t)gg);
        float acc[2][4][4];
        // GEMM1: Z[s][q1] = sum_p X[s][p] F1[p][q1]  (A = X rows, B^T = F1T rows)
        gemm(ch, nullptr, true, FT, FT + CE, false, acc);
        __syncwarp();
        // Z^T[q1][s] in place (B^T operand of GEMM2)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t s = (uint32_t)(mt * 16 + g + 8 * (e >> 1)), q1 = (uint32_t)(nt * 8 + 2 * t + (e & 1));
              *reinterpret_cast<float *>(ch + sw32(q1, s)) = acc[mt][nt][e];
            }
        __syncwarp();
        // GEMM2: OUT[q2][q1] = sum_s F2T[q2][s] Z[s][q1]  (A = F2T rows, B^T = Z^T rows)
        gemm(FT + 2 * CE, FT + 3 * CE, false, ch, nullptr, true, acc);
        __syncwarp();
        // OUT[q2][q1] in place, chunk-XOR'd for the store warps' chunk-fastest reads
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const uint32_t q2 = (uint32_t)(mt * 16 + g + 8 * v), q1 = (uint32_t)(nt * 8 + 2 * t);
              *reinterpret_cast<float2 *>(ch + (swz128(q2 * 128u + q1 * 4u) ^ gx)) =
                  make_float2(acc[mt][nt][2 * v], acc[mt][nt][2 * v + 1]);
            }
        __syncwarp();
        mbar_arrive(&cdone[st]);  // every lane: R * 32 arrivals per tile
      }
    }
  } else {
    // ---------------- store warps: chunk-fastest stream-out (as v6), Y[row][u*(W/C) + cb*R + g]
    const int sw = warp - NCW;
    float *Y = reinterpret_cast<float *>(a.Y);
    const int gl = lane & 7, uq = lane >> 3;
    for (int it = 0;; ++it) {
      const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
      if (tile >= a.ntiles) break;
      const int st = it % a.stages;
      const uint32_t par = (uint32_t)((it / a.stages) & 1);
      mbar_wait_sleep(&cdone[st], par);
      const unsigned char *buf = base + (size_t)st * a.stage_bytes;
      const int rb = (int)(tile / a.tiles_k), cbk = (int)(tile - (int64_t)rb * a.tiles_k);
      for (int oct = 0; oct < a.R / 8; ++oct) {
        const uint32_t gg = (uint32_t)(oct * 8 + gl);
        const uint32_t gx = pipe_gx<8, 4>(gg);
        const unsigned char *ch = buf + gg * CE;
        const int64_t gcol = (int64_t)cbk * a.R + gg;
        if (rb < a.M && gcol < a.WC) {
          float *yg = Y + (int64_t)rb * a.Wout + gcol;
          const int64_t wc = a.WC;
#pragma unroll 2
          for (int u16 = sw; u16 < C / 16; u16 += NSW) {
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
          issue_load(it + a.stages);
        }
        __syncwarp();
      }
    }
  }
}

// ------------------------------------------------------------------ instances

const FusedInstance kInstances[] = {
    // dtype, P, NT (threads doing the last step), RS (slices per thread, last step), kind, rsw
    // v3 factor-pipelined (factors in registers): ids 0..4
    // (P = 8: 32 KB tiles, so the last group's output runs are 16 chunks = 64 bytes; 16 KB tiles (32-byte
    //  runs) measured 0.82 ms on config B vs 0.74 ms)
    {KRON_F32, 2, 128, 16, 2, 4}, {KRON_F32, 4, 128, 8, 2, 4}, {KRON_F32, 8, 128, 8, 2, 2},
    {KRON_F64, 2, 128, 8, 2, 2},  {KRON_F64, 4, 128, 4, 2, 2},
    // v4 two-factor GEMM chunks (nf == 2 only): ids 25..26 appended at the end
    // v2 (warp-local chain): ids 5..14
    {KRON_F32, 2, 256, 8, 1, 8},  {KRON_F32, 4, 256, 4, 1, 4},  {KRON_F32, 8, 256, 2, 1, 2},
    {KRON_F32, 16, 256, 2, 1, 2}, {KRON_F32, 32, 256, 1, 1, 1}, {KRON_F64, 2, 256, 4, 1, 4},
    {KRON_F64, 4, 256, 2, 1, 2},  {KRON_F64, 8, 256, 1, 1, 1},  {KRON_F64, 16, 256, 1, 1, 1},
    {KRON_F64, 32, 128, 1, 1, 1},
    // v1 (CTA-wide in-place chain, any chunk size): ids 15..24
    {KRON_F32, 2, 256, 8, 0, 0},  {KRON_F32, 4, 256, 4, 0, 0},  {KRON_F32, 8, 128, 4, 0, 0},
    {KRON_F32, 16, 256, 2, 0, 0}, {KRON_F32, 32, 128, 2, 0, 0}, {KRON_F64, 2, 256, 4, 0, 0},
    {KRON_F64, 4, 256, 2, 0, 0},  {KRON_F64, 8, 256, 2, 0, 0},  {KRON_F64, 16, 128, 2, 0, 0},
    {KRON_F64, 32, 128, 1, 0, 0},
    // v4: two-factor chunk GEMMs (tile = 256 * RS * P elements = 8192)
    {KRON_F32, 16, 256, 2, 3, 0}, {KRON_F32, 32, 256, 1, 3, 0},
    {KRON_F64, 16, 256, 1, 3, 0}, {KRON_F64, 32, 256, 1, 3, 0},
    // id 29: retired (round 1's experimental L2-fused pair of factor pipelines, measured slower than two
    // passes on config B; removed in round 2).  Kept as a never-selected slot so the ids below stay put.
    {KRON_F32, 8, 64, 8, -1, 2},
    // v5: fp64 two-factor chunks on DMMA (P = 32, tile = 256 * RS * P = 8 chunks = 64-byte output runs;
    //     4-chunk tiles (32-byte runs) measured 9.42 ms on C64 vs 8.93 ms): id 30
    {KRON_F64, 32, 256, 1, 5, 0},
    // v6: fp32 two-factor chunks, warp-specialised (tile = 8192 elements): ids 31..32
    // (P = 16: 64-chunk tiles = 256-byte output runs; P = 32: 8-chunk tiles = 32-byte runs)
    {KRON_F32, 16, 512, 2, 6, 0}, {KRON_F32, 32, 256, 1, 6, 0},
    // v7: fp64 64 x 32 factor pairs on DMMA (one chunk of 4096 per tile): id 33
    {KRON_F64, 64, 64, 1, 7, 0},
    // v8: fp32 P = 32 pairs, 3xTF32 tensor-core mode (KRON_F32_3XTF32 only): id 34
    // (16-chunk tiles: 64-byte output runs)
    {KRON_F32, 32, 512, 1, 8, 0},
    // v6 P = 16 with 32-chunk tiles (128-byte runs, twice the ring stages): id 35 (autotuner candidate)
    {KRON_F32, 16, 256, 2, 6, 0},
    // v9: fp32 16 x 16 factor triples on a 2-CTA cluster (NEXT-2): id 36
    {KRON_F32, 16, 256, 2, 10, 0},
    // v10 (round 2): the v6 P = 16 pair and the v9 triple with their factors in the constant bank
    // (cb_pair16 / cb_top16 compute warps, same TMA rings and stream-out): ids 37 (pair), 38 (triple)
    {KRON_F32, 16, 512, 2, 11, 0}, {KRON_F32, 16, 256, 2, 12, 0},
    // tcgen05 tensor-core pairs (tc.cu, TF32 / 3xTF32 modes only): ids 39 (P = 16), 40 (P = 32)
    {KRON_F32, 16, 512, 1, 13, 0}, {KRON_F32, 32, 512, 1, 13, 0},
    // v12 (round 2): the fp32 P = 32 pair in the v6 frame with F1 in the constant bank (cb_pair32): id 41
    // (16-chunk tiles = 64-byte output runs, 3 x 64 KB stages)
    {KRON_F32, 32, 512, 1, 11, 0},
    // v12 with 8-chunk tiles (32-byte runs, 6 x 32 KB stages): id 42 (autotuner candidate, policy.short_tiles)
    {KRON_F32, 32, 256, 1, 11, 0},
};
constexpr int kNumInstances = sizeof(kInstances) / sizeof(kInstances[0]);

using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const FusedArgs);
using Kernel4Fn = void (*)(const CUtensorMap, const FusedArgs);

Kernel4Fn instance_kernel4(int i) {
  switch (i) {
    case 30: return kron_fused_dmma2_kernel<16, 4, 8>;
    case 33: return kron_fused_dmma2g_kernel<8, 4>;
    case 34: return kron_fused_tf32x3_kernel<8, 4>;
    case 36: return kron_fused_gemm3c_kernel<12>;
    case 38: return kron_fused_gemm3c_kernel<12, false, 16, true>;
    case 25: return kron_fused_gemm2_kernel<float, 16, 4, 8, 8, 2>;
    case 26: return kron_fused_gemm2_kernel<float, 32, 4, 8, 8, 2>;
    case 27: return kron_fused_gemm2_kernel<double, 16, 4, 8, 8, 1>;
    case 28: return kron_fused_gemm2_kernel<double, 32, 4, 8, 8, 1>;
  }
  return nullptr;
}

KernelFn instance_pipe(int i) {
  switch (i) {
    case 0: return kron_fused_pipe_kernel<float, 2, 4, 4>;
    case 1: return kron_fused_pipe_kernel<float, 4, 4, 4>;
    case 2: return kron_fused_pipe_kernel<float, 8, 4, 2>;
    case 3: return kron_fused_pipe_kernel<double, 2, 4, 2>;
    case 4: return kron_fused_pipe_kernel<double, 4, 4, 2>;
  }
  return nullptr;
}

KernelFn instance_kernel(int i) {
  switch (i) {
    // two k-blocks of the chunk GEMMs unrolled together (KU = 2): E 8.50 -> 7.96 ms per pass, C32 3.27 -> 3.20
    // P = 32: 8 x 8 lane tiles on 8 compute warps (162 registers): C32 3.20 -> 3.10 ms per pass; P = 16 keeps
    // 4 x 8 tiles on 12 warps (8 x 8 measured 7.6 -> 8.4 ms on E's pair pass)
    case 31: case 35: return kron_fused_gemm2ws_kernel<16, 12, 4, 8, 4, 2>;
    case 37: return kron_fused_gemm2ws_kernel<16, 12, 4, 8, 4, 2, false, true>;
    case 41: case 42: return kron_fused_gemm2ws_kernel<32, 8, 8, 8, 4, 2, false, true>;
    case 32: return kron_fused_gemm2ws_kernel<32, 8, 8, 8, 4, 2>;
    case 5: return kron_fused_warp_kernel<float, 2, 8, 256, 2>;
    case 6: return kron_fused_warp_kernel<float, 4, 4, 256, 2>;
    case 7: return kron_fused_warp_kernel<float, 8, 2, 256, 2>;
    case 8: return kron_fused_warp_kernel<float, 16, 2, 256, 2>;
    case 9: return kron_fused_warp_kernel<float, 32, 1, 256, 2>;
    case 10: return kron_fused_warp_kernel<double, 2, 4, 256, 2>;
    case 11: return kron_fused_warp_kernel<double, 4, 2, 256, 2>;
    case 12: return kron_fused_warp_kernel<double, 8, 1, 256, 2>;
    case 13: return kron_fused_warp_kernel<double, 16, 1, 256, 2>;
    case 14: return kron_fused_warp_kernel<double, 32, 1, 128, 2>;
    case 15: return kron_fused_kernel<float, 2, 8, 256>;
    case 16: return kron_fused_kernel<float, 4, 4, 256>;
    case 17: return kron_fused_kernel<float, 8, 4, 128>;
    case 18: return kron_fused_kernel<float, 16, 2, 256>;
    case 19: return kron_fused_kernel<float, 32, 2, 128>;
    case 20: return kron_fused_kernel<double, 2, 4, 256>;
    case 21: return kron_fused_kernel<double, 4, 2, 256>;
    case 22: return kron_fused_kernel<double, 8, 2, 256>;
    case 23: return kron_fused_kernel<double, 16, 2, 128>;
    case 24: return kron_fused_kernel<double, 32, 1, 128>;
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

bool encode_tmap_sw(CUtensorMap *m, int dtype, int rank, const void *gaddr, const uint64_t *dims,
                    const uint64_t *strides, const uint32_t *box, int swizzle_bytes) {
  load_encode();
  if (!g_encode) return false;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(m, dtype == KRON_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                        (cuuint32_t)rank, const_cast<void *>(gaddr), (const cuuint64_t *)dims,
                        (const cuuint64_t *)strides, (const cuuint32_t *)box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_tmap(CUtensorMap *m, int dtype, int rank, const void *gaddr, const uint64_t *dims, const uint64_t *strides,
                 const uint32_t *box, bool swizzle128) {
  return encode_tmap_sw(m, dtype, rank, gaddr, dims, strides, box, swizzle128 ? 128 : 0);
}


// Host-side launch bookkeeping is cached per (kernel, block, smem): cudaFuncSetAttribute and the
// occupancy query cost microseconds, which dominate small problems (Table 4 sizes).
namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void *, int>, size_t> g_attr;  // dynamic-smem limit set per (kernel, device)

// caller holds g_attr_mu; the attribute only ever grows, so launches with any smaller smem stay valid
int set_smem_attr_locked(const void *fn, size_t smem, int dev) {
  size_t &cur = g_attr[std::make_pair(fn, dev)];
  if (smem > cur) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    cur = smem;
  }
  return 0;
}
}  // namespace

int set_smem_attr(const void *fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  return set_smem_attr_locked(fn, smem, dev);
}

int kernel_slots(const void *fn, int threads, size_t smem) {
  static std::map<std::tuple<const void *, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, threads, smem, dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (set_smem_attr_locked(fn, smem, dev) != 0) return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) return -1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int slots = per_sm * sms;
  cache[key] = slots;
  return slots;
}

// Constant-bank factor arrays (v10): one per kernel family and device.  A launch copies its factors into
// the array on its stream (device to device) after waiting for the array's previous user (an event
// recorded after that kernel), so launches on different streams never overwrite each other's factors; on
// one stream the wait is implied by stream order (the copy follows the previous kernel anyway).  Inside a
// stream capture the waits / records are skipped (an uncaptured event cannot be waited on); a captured
// graph carries its own copy nodes, ordered before its kernels.
namespace {
struct CSlot {
  std::mutex mu;
  cudaEvent_t ev = nullptr;
  bool used = false;
};
CSlot g_cslots[64][3];  // kind 0: c_fac2, 1: c_fac3, 2: c_fac32

int cslot_acquire(cudaStream_t s, int kind, const void *const *F, int nf, int pp, bool *capturing) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (kind == 2) nf = 1;  // v12: only F1 goes to the constant bank
  if (dev < 0 || dev >= 64 || nf * pp > (kind == 2 ? 1024 : kind ? 768 : 512)) return (int)cudaErrorInvalidValue;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) return (int)cudaGetLastError();
  *capturing = cs != cudaStreamCaptureStatusNone;
  CSlot &S = g_cslots[dev][kind];
  {
    std::lock_guard<std::mutex> lk(S.mu);
    if (!S.ev && cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming) != cudaSuccess) return (int)cudaGetLastError();
    if (S.used && !*capturing && cudaStreamWaitEvent(s, S.ev, 0) != cudaSuccess) return (int)cudaGetLastError();
  }
  for (int i = 0; i < nf; ++i) {
    const cudaError_t e = kind == 2 ? cudaMemcpyToSymbolAsync(c_fac32, F[i], (size_t)pp * sizeof(float), 0,
                                                              cudaMemcpyDeviceToDevice, s)
                          : kind ? cudaMemcpyToSymbolAsync(c_fac3, F[i], (size_t)pp * sizeof(float),
                                                         (size_t)i * pp * sizeof(float), cudaMemcpyDeviceToDevice, s)
                               : cudaMemcpyToSymbolAsync(c_fac2, F[i], (size_t)pp * sizeof(float),
                                                         (size_t)i * pp * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

void cslot_release(cudaStream_t s, int kind, bool capturing) {
  if (capturing) return;
  int dev = 0;
  cudaGetDevice(&dev);
  CSlot &S = g_cslots[dev][kind];
  std::lock_guard<std::mutex> lk(S.mu);
  if (cudaEventRecord(S.ev, s) == cudaSuccess) S.used = true;
}
}  // namespace

int fused_instance_count() { return kNumInstances; }
const FusedInstance &fused_instance(int i) { return kInstances[i]; }
int fused_find(int dtype, int P, int warp) {
  for (int i = 0; i < kNumInstances; ++i)
    if (kInstances[i].dtype == dtype && kInstances[i].P == P && kInstances[i].warp == warp) return i;
  return -1;
}

int fused_box_lines(const PassPlan &pp, int dtype) {
  const int line = dtype == KRON_F32 ? 32 : 16;
  const int lines = (int)(pp.tileK / line);
  return lines > 256 ? 256 : lines;
}

int launch_fused(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *const *Fgroup,
                 void *stream, const PushArgs *push, const InRemap *rin) {
  const FusedInstance &inst = kInstances[pp.variant];
  if (pp.tc_mode) return launch_tc(pp, M, in, out, Fgroup, stream);
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
  a.box_lines = fused_box_lines(pp, dtype);
  a.nbox = lines / a.box_lines;
  a.tile_bytes = (uint32_t)(pp.tileM * pp.tileK * es);
  a.stage_bytes = (a.tile_bytes + 1023u) & ~1023u;
  a.stages = pp.stages;

  if (rin && rin->on && inst.warp == 7) return (int)cudaErrorInvalidValue;
  if (pp.tm_out || pp.tm_in) {
    // v11 tile-major hand-off (E-shaped [16^3 triple, 16^2 pair] plans, see kron_tri_tm_kernel).  Distributed
    // rounds (kron_matmul_dist): the triple pushes into the destination-major send blocks (push->B = composite
    // columns per destination), the pair reads the receive blocks through a 4-D map (rin->GK sources) and pushes
    // its outputs into the next send blocks (push->B = values per row and destination)
    if (dtype != KRON_F32 || pp.P != 16 || (rin && rin->on && !pp.tm_in)) return (int)cudaErrorInvalidValue;
    if (push && push->on) {
      if (push->GK != 1 || push->rho != push->B || push->B < 1) return (int)cudaErrorInvalidValue;
      a.push = *push;
    }
    CUtensorMap tin;
    a.Y = out;
    a.WC = WC;
    a.Wout = Wout;
    a.M = M;
    Kernel4Fn kt;
    size_t smem;
    int threads;
    if (pp.tm_out) {
      if (pp.nf != 3 || WC % 4) return (int)cudaErrorInvalidValue;
      if (a.push.on && (pp.Qc % a.push.B || a.push.B % 32 || pp.Qc / a.push.B > kMaxPush)) return (int)cudaErrorInvalidValue;
      a.tiles_k = (int)(WC / 4);
      a.ntiles = M * a.tiles_k;
      a.box_lines = 256;
      a.nbox = 2;  // 4 chunks = 512 lines of 128 bytes
      uint64_t dims[3] = {(uint64_t)line, (uint64_t)(W / line), (uint64_t)M};
      uint64_t strides[2] = {128, (uint64_t)W * es};
      uint32_t box[3] = {(uint32_t)line, 256u, 1u};
      if (!encode_tmap(&tin, dtype, 3, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
      smem = 1024 + (size_t)a.stages * 65536 + 24 * (size_t)a.stages;
      // 16 compute warps (4 per SM sub-partition): E's triple 8.13 ms vs 8.34 with 12 and 8.92 with 8
      threads = 32 * (16 + 4);
      kt = kron_tri_tm_kernel<16>;
    } else {
      // T''[row][g/4][u][g%4], u < WC (this pass's chunks), g < C = 256 (the producer's chunks): box {4, R, 64, 1}
      if (pp.nf != 2 || pp.C != 256 || pp.R != 64 || WC % pp.R) return (int)cudaErrorInvalidValue;
      if (a.push.on) {
        const int64_t upd = a.push.B / WC;  // composite columns per destination: a power of two >= 4
        if (a.push.B % WC || (pp.Qc * WC) % a.push.B || upd < 4 || (upd & (upd - 1)) || pp.Qc / upd > kMaxPush)
          return (int)cudaErrorInvalidValue;
      }
      a.tiles_k = (int)(WC / pp.R);
      a.ntiles = M * a.tiles_k;
      a.tile_bytes = (uint32_t)pp.R * 1024u;
      a.stage_bytes = a.tile_bytes;
      // (u, g%4) merged into one contiguous dimension: a box row is 4R floats = 1 KB (a 16-byte inner box dimension
      // measured 7.9 ms on E's pair pass vs 6.9 ms for the direct-index kernel)
      if (rin && rin->on) {
        // receive blocks recv[src][row][gq][u][4], gq < 64 / GK: box {4R, 64 / GK, 1, GK} lands as [g/4][u][g%4]
        // with g/4 = src * (64 / GK) + gq — the single-GPU tile layout
        const int64_t GK = rin->GK, Gs = 64 / GK;
        if (GK < 1 || 64 % GK || W % GK) return (int)cudaErrorInvalidValue;
        uint64_t dims[4] = {(uint64_t)WC * 4, (uint64_t)Gs, (uint64_t)M, (uint64_t)GK};
        uint64_t strides[3] = {(uint64_t)WC * 16, (uint64_t)(W / GK) * es, (uint64_t)M * (uint64_t)(W / GK) * es};
        uint32_t box[4] = {(uint32_t)pp.R * 4, (uint32_t)Gs, 1, (uint32_t)GK};
        if (!encode_tmap(&tin, dtype, 4, in, dims, strides, box, false)) return (int)cudaErrorInvalidValue;
        a.rmp_GK = (int)GK;
      } else {
        uint64_t dims[3] = {(uint64_t)WC * 4, 64, (uint64_t)M};
        uint64_t strides[2] = {(uint64_t)WC * 16, (uint64_t)W * es};
        uint32_t box[3] = {(uint32_t)pp.R * 4, 64, 1};
        if (!encode_tmap(&tin, dtype, 3, in, dims, strides, box, false)) return (int)cudaErrorInvalidValue;
      }
      smem = 1024 + (size_t)a.stages * a.stage_bytes + 24 * (size_t)a.stages;
      threads = 32 * (12 + 4);
      kt = kron_pair_tm_kernel<12>;
    }
    const int kind = pp.tm_out ? 1 : 0;
    bool capturing = false;
    const int err = cslot_acquire((cudaStream_t)stream, kind, Fgroup, pp.nf, 256, &capturing);
    if (err != 0) return err;
    const int slots = kernel_slots((const void *)kt, threads, smem);
    int lerr = (int)cudaErrorInvalidConfiguration;
    if (slots >= 1) {
      int64_t grid = slots;
      if (grid > a.ntiles) grid = a.ntiles;
      kt<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(tin, a);
      lerr = (int)cudaGetLastError();
    }
    cslot_release((cudaStream_t)stream, kind, capturing);
    return lerr;
  }
  if (inst.warp == 7) {
    // 5-D map over X[m][g][s][p/16][p%16]; box = one p-half of one chunk ([64][2][16] = 16 KB)
    CUtensorMap t5;
    uint64_t dims[5] = {16, 4, 64, (uint64_t)WC, (uint64_t)M};
    uint64_t strides[4] = {128, 512, 32768, (uint64_t)W * 8};
    uint32_t box[5] = {16, 2, 64, 1, 1};
    if (!encode_tmap(&t5, dtype, 5, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
    a.Y = out;
    a.WC = WC;
    a.Wout = Wout;
    a.M = M;
    const size_t smem7 = 1024 + (size_t)a.stages * 32768 + 2 * 64 * 32 * 8 + 24 * (size_t)a.stages;
    Kernel4Fn k7 = instance_kernel4(pp.variant);
    const int slots = kernel_slots((const void *)k7, 32 * (8 + 4), smem7);
    if (slots < 1) return (int)cudaErrorInvalidConfiguration;
    int64_t grid = slots;
    if (grid > a.ntiles) grid = a.ntiles;
    k7<<<(unsigned)grid, 32 * (8 + 4), smem7, (cudaStream_t)stream>>>(t5, a);
    return (int)cudaGetLastError();
  }
  CUtensorMap tin, tout;
  if (rin && rin->on) {
    // receive buffer recv[src][m][e*rho + t] (B = W/GK values per row and source) seen in local-column order
    // (e*GK + src)*rho + t: dims {line, rho/line, GK, B/rho, M}; a box covers whole runs or lies in one
    const int64_t rl = rin->rho / line, GK = rin->GK, B = W / GK, bl = a.box_lines;
    if (rin->rho % line || W % (rin->rho * GK)) return (int)cudaErrorInvalidValue;
    uint64_t dims[5] = {(uint64_t)line, (uint64_t)rl, (uint64_t)GK, (uint64_t)(B / rin->rho), (uint64_t)M};
    uint64_t strides[4] = {128, (uint64_t)(M * B * es), (uint64_t)(rin->rho * es), (uint64_t)(B * es)};
    uint32_t box[5] = {(uint32_t)line, 1, 1, 1, (uint32_t)pp.tileM};
    if (bl <= rl) {
      if (rl % bl) return (int)cudaErrorInvalidValue;
      box[1] = (uint32_t)bl;
    } else {
      const int64_t nr = bl / rl;
      if (bl % rl || (nr <= GK ? GK % nr : nr % GK)) return (int)cudaErrorInvalidValue;
      box[1] = (uint32_t)rl;
      box[2] = (uint32_t)(nr <= GK ? nr : GK);
      box[3] = (uint32_t)(nr <= GK ? 1 : nr / GK);
    }
    if (!encode_tmap(&tin, dtype, 5, in, dims, strides, box, true)) return (int)cudaErrorInvalidValue;
    a.rmp_rl = (int)rl;
    a.rmp_GK = (int)GK;
  } else {
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
  a.Y = out;
  a.WC = WC;
  a.Wout = Wout;
  a.M = M;
  size_t smem;
  int threads = inst.NT;
  if (inst.warp == 5 || inst.warp == 8) {
    smem = 1024 + (size_t)a.stages * a.stage_bytes + (inst.warp == 8 ? 4 : 2) * (size_t)pp.P * pp.P * es +
           24 * (size_t)a.stages;
    threads = 32 * ((inst.warp == 5 ? 16 : 8) + 4);  // v5: two tile groups of 8 compute warps
  } else if (inst.warp == 6 || inst.warp == 11) {
    smem = 1024 + (size_t)a.stages * a.stage_bytes + 2 * (size_t)pp.P * pp.P * es + 24 * (size_t)a.stages;
    threads = 32 * ((pp.P == 32 ? 8 : 12) + 4);  // compute warps of the instance (see instance_kernel)
  } else if (inst.warp == 3) {
    smem = 1024 + (size_t)a.stages * a.stage_bytes + 2 * (size_t)pp.P * pp.P * es + 8 * (size_t)a.stages;
  } else if (inst.warp == 2) {
    smem = 1024 + (size_t)(a.stages + 2) * a.stage_bytes + 8 * 4 * (size_t)a.stages;
    threads = 32 * (1 + 3 * (inst.NT / 32));  // producer warp + one warp group per factor (max 3)
  } else {
    smem = 1024 + (size_t)(a.stages + (inst.warp ? pp.nout : 0)) * a.stage_bytes +
           (((size_t)pp.nf * pp.P * pp.P * es + 15) & ~15) + 8 * (size_t)a.stages;
  }
  if (push && push->on) {
    if ((inst.warp != 10 && inst.warp != 6 && inst.warp != 11 && inst.warp != 12) || push->GK > kMaxPush)
      return (int)cudaErrorInvalidValue;
    if (Wout >= (int64_t(1) << 31) || push->wd >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;  // push_dst
    a.push = *push;
  }
  // v10: this launch's factors go to a constant-bank slot first (stream-ordered)
  const int cslot = inst.warp == 12 ? 1 : inst.warp == 11 ? (pp.P == 32 ? 2 : 0) : -1;
  bool capturing = false;
  if (cslot >= 0) {
    const int err = cslot_acquire((cudaStream_t)stream, cslot, Fgroup, pp.nf, pp.P * pp.P, &capturing);
    if (err != 0) return err;
  }
  if (inst.warp == 10 || inst.warp == 12) {
    // cluster pair: grid = 2 x clusters (one CTA per SM), a.ntiles = 8-chunk groups
    smem = 1024 + (size_t)a.stages * 65536 + 3 * 1024 + 80 * (size_t)a.stages;
    threads = 32 * (12 + 4);
    Kernel4Fn k10 = inst.warp == 12 ? (a.push.on ? kron_fused_gemm3c_kernel<12, true, 16, true> : instance_kernel4(pp.variant))
                                    : (a.push.on ? kron_fused_gemm3c_kernel<12, true> : instance_kernel4(pp.variant));
    const int aerr = set_smem_attr((const void *)k10, 227 * 1024);  // per (kernel, device)
    if (aerr != 0) return aerr;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t ncl = sms / 2;  // one CTA per SM (the smem footprint), clusters of two
    if (ncl > a.ntiles) ncl = a.ntiles;
    k10<<<(unsigned)(2 * ncl), threads, smem, (cudaStream_t)stream>>>(tin, a);
    const int lerr = (int)cudaGetLastError();
    if (cslot >= 0) cslot_release((cudaStream_t)stream, cslot, capturing);
    return lerr;
  }
  if (inst.warp == 3 || inst.warp == 5 || inst.warp == 8) {
    Kernel4Fn k4 = instance_kernel4(pp.variant);
    const int slots = kernel_slots((const void *)k4, threads, smem);
    if (slots < 1) return (int)cudaErrorInvalidConfiguration;
    int64_t grid = slots;
    if (grid > a.ntiles) grid = a.ntiles;
    k4<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(tin, a);
    return (int)cudaGetLastError();
  }
  if (inst.warp == 2) {
    KernelFn kp = instance_pipe(pp.variant);
    const int slots = kernel_slots((const void *)kp, threads, smem);
    if (slots < 1) return (int)cudaErrorInvalidConfiguration;
    int64_t grid = slots;
    if (grid > a.ntiles) grid = a.ntiles;
    kp<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(tin, tout, a);
    return (int)cudaGetLastError();
  }
  KernelFn k = instance_kernel(pp.variant);
  if (a.push.on) {  // v6 / v10 pair with the fused exchange (same tiling, push epilogue)
    k = inst.warp == 11 ? (pp.P == 32 ? kron_fused_gemm2ws_kernel<32, 8, 8, 8, 4, 2, true, true>
                                      : kron_fused_gemm2ws_kernel<16, 12, 4, 8, 4, 2, true, true>)
        : pp.P == 32    ? kron_fused_gemm2ws_kernel<32, 8, 8, 8, 4, 2, true>
                        : kron_fused_gemm2ws_kernel<16, 12, 4, 8, 4, 2, true>;
  }
  const int slots = kernel_slots((const void *)k, threads, smem);
  if (slots < 1) return (int)cudaErrorInvalidConfiguration;
  int64_t grid = slots;
  if (grid > a.ntiles) grid = a.ntiles;
  k<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(tin, tout, a);
  const int lerr = (int)cudaGetLastError();
  if (cslot >= 0) cslot_release((cudaStream_t)stream, cslot, capturing);
  return lerr;
}

}  // namespace kron
