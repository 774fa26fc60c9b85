// kron_internal.h — host-side plan structures and kernel launchers shared by the libkron sources.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda.h>

#include "../../include/kron.h"

namespace kron {

enum Kind { KIND_GENERIC = 0, KIND_FUSED = 1, KIND_GEMM = 2, KIND_CHAIN = 3 };
enum Buf { BUF_X = 0, BUF_Y = 1, BUF_WS0 = 2, BUF_WS1 = 3 };

constexpr int kMaxFactors = 64;
constexpr int kMaxFused = 8;

// One kernel launch: applies factors F^{first}, F^{first-1}, ..., F^{first-nf+1} (1-based).
struct PassPlan {
  int kind = KIND_GENERIC;
  int first = 0;  // 1-based index of the first factor this pass applies (processing order N -> 1)
  int nf = 1;     // factors fused in this pass
  int P = 0, Q = 0;           // factor shape (uniform within a fused group; P == Q for KIND_FUSED)
  int64_t W_in = 0, W_out = 0;  // row widths entering / leaving the pass
  int64_t C = 1, Qc = 1;      // chunk = prod P over the group, composite columns = prod Q
  // fused-kernel tiling: a tile is tileM rows x tileK = R*C columns
  int R = 0, tileM = 1;
  int64_t tileK = 0;
  int variant = -1;  // fused: kernel instance id; gemm: instance id
  int stages = 2;
  int nout = 0;  // output staging buffers (warp-chain fused kernel)
  int src = BUF_X, dst = BUF_Y;
  int tc_mode = 0;  // fused pair on the tcgen05 tensor cores (tc.cu): 1 TF32, 2 3xTF32; 0 otherwise
  // v11 tile-major hand-off (fused.cu, kron_tri_tm_kernel): this pass writes its output as T''[row][g/4][u][g%4]
  // (tm_out) / reads its input through the matching 4-D map (tm_in) instead of the direct-index layout
  int tm_out = 0, tm_in = 0;
};

struct Plan {
  int N = 0;
  int64_t M = 0;
  int dtype = 0;
  std::vector<int64_t> W;  // W[f], f = 0..N (W[N] = K, W[0] = L)
  std::vector<PassPlan> passes;
  int nws = 0;             // workspace buffers (0, 1 or 2)
  int64_t ws_elems = 0;    // elements per workspace buffer
};

// Builds the plan (host only).  Returns KRON_OK or a validation error.
// Knobs the autotuner searches over; the default policy is the static planner.
struct PlanPolicy {
  int kcap = kMaxFused;       // largest fused group
  unsigned kinds = 0xFFFFu;    // allowed kernel families (bit = FusedInstance::warp; bit 14 = chain.cu; bit 15 = fp32 sgemm)
  int chain_rdiv = 1;         // chain passes: tile of R / chain_rdiv chunks (autotuner tile-size candidates)
  bool dmma = true;           // fp64 large-P passes on DMMA (else register-tiled DFMA)
  bool short_tiles = false;   // v6 fp32 P = 16: 32-chunk tiles (128-byte runs, deeper ring) instead of 64-chunk
  bool handoff = true;        // v11 tile-major hand-off between the passes of [16^3 triple, 16^2 pair] plans
  bool operator==(const PlanPolicy &o) const {
    return kcap == o.kcap && kinds == o.kinds && dmma == o.dmma && short_tiles == o.short_tiles &&
           chain_rdiv == o.chain_rdiv && handoff == o.handoff;
  }
};
kron_status_t make_plan(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype, Plan *out,
                        int64_t lead = 1, const PlanPolicy &policy = PlanPolicy());
size_t plan_ws_bytes(const Plan &plan);
// Distributed rounds (Algorithm 2).  Two hooks let a round's local passes do the exchange's
// data movement themselves, so no separate pack / StoreGPUTile pass touches HBM:
//
// PushArgs — the LAST pass of a plan writes every output value to a per-destination buffer instead of Y.
// Output column c of the local block goes to rank d = c / B at column ((e / rho) * GK + me) * rho + e % rho,
// e = c % B, of a row of width wd.  P2P (backend 2): dst[d] = peer d's heap half, rho = the round's run
// length (StoreGPUTile over NVLink, NEXT-1).  NCCL / virtual (backends 0, 1): dst[d] = this rank's
// destination-major send block d, rho = B, GK = 1, me = 0, wd = B (the pack fused into the epilogue).
constexpr int kMaxPush = 8;
struct PushArgs {
  void *dst[kMaxPush] = {};
  int64_t B = 0, rho = 0, wd = 0;
  int GK = 0, me = 0, on = 0;
};
// InRemap — the FIRST pass of a plan reads its input in place from an all-to-all receive buffer
// recv[src][m][e*rho + t] through a 5-D tensor map whose coordinate order is the StoreGPUTile layout
// (local column (e*GK + src)*rho + t, Alg 2): the remap happens in the TMA engine.
struct InRemap {
  int64_t rho = 0;
  int GK = 0, on = 0;
};
bool plan_push_ok(const Plan &plan, const PushArgs &push);
bool plan_remap_ok(const Plan &plan, const InRemap &rin);
void keep_pool_cached();  // default mem pool keeps freed blocks (stream-ordered workspaces)
// Enqueue passes [i0, i1) (i1 < 0: all) of `plan` (F indexed like the plan's P/Q arrays); ws >= plan_ws_bytes.
kron_status_t plan_run(const Plan &plan, const void *X, const void *const *F, void *Y, void *ws, void *stream,
                       const PushArgs *push = nullptr, const InRemap *rin = nullptr, int i0 = 0, int i1 = -1);
kron_status_t validate(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype);

// ---- fused small-P kernel family (fused.cu)
struct FusedInstance {
  int dtype;  // 0 f32, 1 f64
  int P;
  int NT;     // threads per CTA
  int RS;     // slices per thread
  int warp;   // 2: factor-pipelined kernel, 1: warp-local chain kernel, 0: CTA-wide in-place chain
  int rsw;    // slices per lane in the warp-owned (intermediate) steps; 32*rsw*P % chunk == 0 needed
  int64_t elems() const { return (int64_t)NT * RS * P; }
};
int fused_instance_count();
const FusedInstance &fused_instance(int i);
int fused_find(int dtype, int P, int warp);  // instance id or -1

// ---- launchers (device code lives in the .cu files).  Return cudaError_t as int.
int launch_generic(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F,
                   void *stream);
int launch_fused(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *const *Fgroup,
                 void *stream, const PushArgs *push = nullptr, const InRemap *rin = nullptr);
// input-box geometry of a fused pass (lines of 128 bytes per TMA box); shared by launch_fused and plan_remap_ok
int fused_box_lines(const PassPlan &pp, int dtype);
int launch_gemm(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *F, void *stream);
// fused passes of any square P without TMA (chain.cu, NEXT-3)
bool chain_geometry(int P, int k, int dtype, int64_t W, int rdiv, PassPlan *pp);
int launch_chain(const PassPlan &pp, int dtype, int64_t M, const void *in, void *out, const void *const *Fgroup,
                 void *stream);
// tcgen05 fp32 pair (tc.cu, NEXT-4): geometry for P = 16 / 32 pairs in mode 1 (TF32) / 2 (3xTF32), and launch
bool tc_geometry(int P, int mode, int64_t W, PassPlan *pp);
int launch_tc(const PassPlan &pp, int64_t M, const void *in, void *out, const void *const *Fgroup, void *stream);
bool gemm_supported(int dtype, int64_t M, int64_t W, int P, int Q);
bool sgemm_supported(int64_t M, int64_t W, int P, int Q);  // fp32 large-P pass on kron_sgemm_kernel

// resident CTA slots (SMs x CTAs per SM) for a kernel launch shape; sets the dynamic-smem attribute.
// Cached per (kernel, block, smem, device).  fused.cu
int kernel_slots(const void *fn, int threads, size_t smem);
// raise the kernel's dynamic-smem limit on the current device (cached per (kernel, device)); cudaError_t
int set_smem_attr(const void *fn, size_t smem);

// tensor-map encoder (driver entry point fetched through the runtime); fused.cu
bool tmap_available();
bool encode_tmap_sw(CUtensorMap *m, int dtype, int rank, const void *gaddr, const uint64_t *dims,
                    const uint64_t *strides, const uint32_t *box, int swizzle_bytes);  // 0 / 32 / 64 / 128
bool encode_tmap(CUtensorMap *m, int dtype, int rank, const void *gaddr, const uint64_t *dims, const uint64_t *strides,
                 const uint32_t *box, bool swizzle128);

}  // namespace kron
