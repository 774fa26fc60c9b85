// api.cu — the libkron C-ABI (include/kron.h): validation, the pass planner (Algorithm 1 loop +
// fusion groups), the plan cache, workspace handling and dispatch.
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kron_internal.h"

namespace kron {

namespace {

int es_of(int dtype) { return dtype == KRON_F64 ? 8 : 4; }

bool mul_ok(int64_t a, int64_t b, int64_t lim, int64_t *out) {
  if (a != 0 && b > lim / a) return false;
  *out = a * b;
  return true;
}

// Tile geometry of a fused group: C = P^k chunk, R chunks per tile row
// (output runs of R*s >= 32 bytes), tileK = R*C columns, tileM rows; all TMA box constraints.
bool fused_geometry(const FusedInstance &inst, int k, int64_t W, int64_t M, PassPlan *pp) {
  const int es = es_of(inst.dtype), line = 128 / es;
  const int p = inst.P;
  int64_t C = 1;
  for (int i = 0; i < k; ++i) C *= p;
  const int64_t E = inst.elems();
  if (W % line || W % C || (C > E && inst.warp != 10 && inst.warp != 12)) return false;
  const int64_t WC = W / C;
  if ((WC * es) % 16) return false;
  if (inst.warp == 10 || inst.warp == 12) {
    // v9 / v10 cluster pair: three factors, 8-chunk tiles split 4 + 4 over two CTAs (32-byte runs)
    if (k != 3 || p != 16 || inst.dtype != KRON_F32 || W % (8 * C)) return false;
    pp->kind = KIND_FUSED;
    pp->nf = 3;
    pp->P = pp->Q = p;
    pp->C = pp->Qc = C;
    pp->R = 8;
    pp->tileK = 4 * C;  // per CTA
    pp->tileM = 1;
    pp->stages = 3;
    pp->nout = 0;
    return true;
  }
  int64_t R = E / C;
  if (R > WC) R = WC;
  if (R > 256) R = 256;
  if (R * es < 32 || (R * es) % 16) return false;
  const int64_t tileK = R * C;
  if (tileK % line) return false;
  const int64_t lines = tileK / line;
  if (lines > 256 && lines % 256) return false;
  int64_t tileM = E / tileK;
  if (inst.warp) {
    // the warp-chain kernel always works on full tiles (rows past M are TMA zero-fill / clipped)
    if (E % tileK || tileM > 256) return false;
  } else {
    if (tileM > M) tileM = M;
    if (tileM > 256) tileM = 256;
    if (tileM < 1) tileM = 1;
  }
  if (tileM > 1 && lines > 256) return false;
  if (C > 256 && (C % 256 || C / 256 > 256)) return false;
  if (inst.warp && ((int64_t)32 * inst.rsw * p) % C) return false;  // warp share = whole chunks
  if (inst.warp == 3) {
    // two-factor chunk GEMMs: exactly two factors, one tile row of whole chunk octets
    if (k != 2 || tileM != 1 || R % 8 || (R * C) != E) return false;
    if (W * es >= (int64_t(1) << 32)) return false;  // 32-bit in-row store offsets
  }
  if (inst.warp == 6 || inst.warp == 8 || inst.warp == 11) {
    // warp-specialised fp32 chunk pairs: two factors, one tile row of whole chunk octets
    if (k != 2 || tileM != 1 || R % 8 || (R * C) != E) return false;
  }
  if (inst.warp == 5) {
    // DMMA chunk pairs: exactly two factors, one tile row of 8 chunks (64-byte fp64 runs)
    if (k != 2 || tileM != 1 || R != 8 || (R * C) != E) return false;
  }
  if (inst.warp == 2 || inst.warp == 4) {
    if (k > 3) return false;                                   // one warp group per factor
    if (R % inst.rsw || (k >= 2 && C < (int64_t)inst.rsw * p)) return false;  // 16-byte chunk/slice vectors
    if (tileM * R / inst.rsw * (C / p) > 4 * inst.NT) return false;        // <= 4 last-step slots per thread
  }
  const int64_t stage = (tileM * tileK * es + 1023) / 1024 * 1024;
  int stages, nout = 0;
  if (inst.warp == 5 || inst.warp == 6 || inst.warp == 8 || inst.warp == 11) {
    // one warp-specialised CTA per SM (v8 keeps hi/lo splits of both factors)
    stages = (int)((220 * 1024 - (inst.warp == 8 ? 4 : inst.warp == 11 ? 0 : 2) * (int64_t)p * p * es) / stage);
    if (stages > 8) stages = 8;
  } else if (inst.warp == 3) {
    stages = stage <= 32 * 1024 ? 3 : 2;
  } else if (inst.warp == 4) {
    if (tileM != 1) return false;
    nout = 2;
    stages = 4;  // two co-resident CTAs (one per pass) per SM
  } else if (inst.warp == 2) {
    nout = 2;
    // deep ring: one CTA per SM, as many stages as the 227 KB allow next to the two output tiles
    // (config B: 5 x 32 KB stages, 0.743 -> 0.726 ms vs 4)
    stages = (int)((227 * 1024 - 1024 - 2 * stage - 512) / stage);
    if (stages > 8) stages = 8;
    if (stages < k + 1) return false;
  } else if (inst.warp == 1) {
    stages = 2;
    nout = stage <= 16 * 1024 ? 2 : 1;  // keep >= 2 CTAs per SM
  } else {
    stages = stage <= 32 * 1024 ? 3 : 2;
  }
  const int64_t smem = 1024 + (stages + nout) * stage + (int64_t)k * p * p * es + 16 + 32 * stages;
  if (smem > 227 * 1024) return false;
  pp->kind = KIND_FUSED;
  pp->nf = k;
  pp->P = pp->Q = p;
  pp->C = C;
  pp->Qc = C;
  pp->R = (int)R;
  pp->tileK = tileK;
  pp->tileM = (int)tileM;
  pp->stages = stages;
  pp->nout = nout;
  return true;
}

struct PlanKey {
  int dev;
  int64_t M;
  int dtype;
  std::vector<int32_t> P, Q;
  bool operator<(const PlanKey &o) const {
    if (dev != o.dev) return dev < o.dev;
    if (M != o.M) return M < o.M;
    if (dtype != o.dtype) return dtype < o.dtype;
    if (P != o.P) return P < o.P;
    return Q < o.Q;
  }
};

std::mutex g_cache_mu;
std::map<PlanKey, std::shared_ptr<const Plan>> g_cache;

kron_status_t cached_plan(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype,
                          std::shared_ptr<const Plan> *out) {
  int dev = 0;
  cudaGetDevice(&dev);
  PlanKey key{dev, M, dtype, std::vector<int32_t>(P, P + N), std::vector<int32_t>(Q, Q + N)};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *out = it->second;
    return KRON_OK;
  }
  auto plan = std::make_shared<Plan>();
  kron_status_t st = make_plan(M, N, P, Q, dtype, plan.get());
  if (st != KRON_OK) return st;
  g_cache.emplace(key, plan);
  *out = plan;
  return KRON_OK;
}

thread_local char g_err_detail[256] = "";

kron_status_t cuda_fail(int err, const char *what) {
  snprintf(g_err_detail, sizeof(g_err_detail), "%s: %s", what, cudaGetErrorName((cudaError_t)err));
  return KRON_ERR_CUDA;
}

kron_status_t run_plan(const Plan &plan, const void *X, const void *const *F, void *Y, void *ws, void *stream,
                       void *const *events = nullptr, const PushArgs *push = nullptr, const InRemap *rin = nullptr,
                       int i0 = 0, int i1 = -1) {
  const size_t es = es_of(plan.dtype);
  const int np = (int)plan.passes.size();
  if (i1 < 0 || i1 > np) i1 = np;
  int ip = 0;
  void *bufs[4] = {const_cast<void *>(X), Y, ws,
                   ws ? static_cast<char *>(ws) + (size_t)plan.ws_elems * es : nullptr};
  for (int i = i0; i < i1; ++i) {
    const PassPlan &pp = plan.passes[i];
    const void *in = bufs[pp.src];
    void *out = bufs[pp.dst];
    int err = 0;
    if (events && cudaEventRecord((cudaEvent_t)events[ip], (cudaStream_t)stream) != cudaSuccess) return KRON_ERR_CUDA;
    ++ip;
    const bool lastp = i == np - 1, firstp = i == 0;
    if (pp.kind == KIND_FUSED) {
      if (!tmap_available()) return KRON_ERR_CUDA;
      const void *grp[kMaxFused];
      for (int k = 0; k < pp.nf; ++k) grp[k] = F[pp.first - 1 - k];
      err = launch_fused(pp, plan.dtype, plan.M, in, out, grp, stream, lastp ? push : nullptr,
                         firstp ? rin : nullptr);
    } else if (pp.kind == KIND_CHAIN) {
      const void *grp[kMaxFused];
      for (int k = 0; k < pp.nf; ++k) grp[k] = F[pp.first - 1 - k];
      err = launch_chain(pp, plan.dtype, plan.M, in, out, grp, stream);
    } else if (pp.kind == KIND_GEMM) {
      err = launch_gemm(pp, plan.dtype, plan.M, in, out, F[pp.first - 1], stream);
    } else {
      err = launch_generic(pp, plan.dtype, plan.M, in, out, F[pp.first - 1], stream);
    }
    if (err != 0)
      return cuda_fail(err, pp.kind == KIND_FUSED ? "fused pass launch"
                            : pp.kind == KIND_CHAIN ? "chain pass launch"
                            : pp.kind == KIND_GEMM ? "gemm pass launch" : "generic pass launch");
  }
  if (events && cudaEventRecord((cudaEvent_t)events[ip], (cudaStream_t)stream) != cudaSuccess) return KRON_ERR_CUDA;
  return KRON_OK;
}

size_t ws_bytes_of(const Plan &plan) {
  return (size_t)plan.nws * (size_t)plan.ws_elems * (size_t)es_of(plan.dtype);
}

}  // namespace

// kron_matmul() reserves its workspace with cudaMallocAsync on the caller's stream.  Keep freed blocks
// in the device's default memory pool (release threshold = max) so repeated calls do not re-map GiBs
// of workspace every time.
void keep_pool_cached() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

size_t plan_ws_bytes(const Plan &plan) { return ws_bytes_of(plan); }

kron_status_t plan_run(const Plan &plan, const void *X, const void *const *F, void *Y, void *ws, void *stream,
                       const PushArgs *push, const InRemap *rin, int i0, int i1) {
  if ((push && push->on && !plan_push_ok(plan, *push)) || (rin && rin->on && !plan_remap_ok(plan, *rin)))
    return KRON_ERR_UNSUPPORTED;
  return run_plan(plan, X, F, Y, ws, stream, nullptr, push, rin, i0, i1);
}

// The pushing epilogues exist in the v9 cluster kernel (16-byte runs: rho, B and the row width must keep
// every float4 inside one run and 16-byte aligned) and the v6 fp32 chunk-pair kernels (scalar stores).
bool plan_push_ok(const Plan &plan, const PushArgs &push) {
  if (plan.passes.empty() || push.GK < 1 || push.GK > kMaxPush || push.B < 1 || push.rho < 1) return false;
  const PassPlan &pp = plan.passes.back();
  if (pp.kind != KIND_FUSED || pp.tm_in || pp.tm_out) return false;
  if (pp.W_out % push.B || push.B % push.rho || pp.W_out / push.B > kMaxPush) return false;
  const FusedInstance &fi = fused_instance(pp.variant);
  if (fi.warp == 10 || fi.warp == 12) return push.rho % 4 == 0 && push.B % 4 == 0 && push.wd % 4 == 0;
  return (fi.warp == 6 || fi.warp == 11) && fi.dtype == KRON_F32 && (fi.P == 16 || fi.P == 32);
}

// The remapped input view needs every TMA box of the first pass to cover whole runs of rho elements, or
// lie inside one: fused kernels with the standard 3-D line-box loads (all but v7), rho a multiple of a
// 128-byte line.
bool plan_remap_ok(const Plan &plan, const InRemap &rin) {
  if (plan.passes.empty() || rin.GK < 1 || rin.rho < 1) return false;
  const PassPlan &pp = plan.passes.front();
  if (pp.kind != KIND_FUSED || pp.tm_in || pp.tm_out || fused_instance(pp.variant).warp == 7) return false;
  const int64_t line = 128 / es_of(plan.dtype);
  if (rin.rho % line || pp.W_in % (rin.rho * rin.GK)) return false;
  const int64_t rl = rin.rho / line, bl = fused_box_lines(pp, plan.dtype);
  if (bl < 1) return false;
  if (bl <= rl) return rl % bl == 0;
  if (bl % rl) return false;
  const int64_t nr = bl / rl;
  return nr <= rin.GK ? rin.GK % nr == 0 : nr % rin.GK == 0;
}

kron_status_t validate(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype) {
  if (M < 0 || N < 1 || N > kMaxFactors || !P || !Q) return KRON_ERR_INVALID_ARG;
  if (dtype != KRON_F32 && dtype != KRON_F64 && dtype != KRON_F32_3XTF32 && dtype != KRON_F32_TF32)
    return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (P[i] < 1 || Q[i] < 1) return KRON_ERR_INVALID_ARG;
  const int64_t lim = (int64_t)1 << 50;  // elements per row; beyond any HBM
  int64_t K = 1, L = 1;
  for (int i = 0; i < N; ++i) {
    if (!mul_ok(K, P[i], lim, &K) || !mul_ok(L, Q[i], lim, &L)) return KRON_ERR_SHAPE;
  }
  // every intermediate must fit the address space: M * width * s < 2^60
  int64_t W = K, maxw = K;
  for (int f = N; f >= 1; --f) {
    W = W / P[f - 1];
    if (!mul_ok(W, Q[f - 1], lim, &W)) return KRON_ERR_SHAPE;
    if (W > maxw) maxw = W;
  }
  int64_t tot;
  if (!mul_ok(maxw, M > 0 ? M : 1, (int64_t)1 << 57, &tot)) return KRON_ERR_SHAPE;
  return KRON_OK;
}

kron_status_t make_plan(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype, Plan *plan, int64_t lead,
                        const PlanPolicy &policy) {
  kron_status_t st = validate(M, N, P, Q, dtype);
  // tensor-core modes (fp32 data, reported separately): P = 16 / 32 square pairs go to the tcgen05 pair kernel
  // (3xTF32 also to round 1's mma.sync kernel for P = 32 when the tcgen05 kernel is masked), everything else
  // runs as KRON_F32
  const bool tf32x3 = dtype == KRON_F32_3XTF32;
  const int tcm = dtype == KRON_F32_3XTF32 ? 2 : dtype == KRON_F32_TF32 ? 1 : 0;
  if (tcm) dtype = KRON_F32;
  if (st != KRON_OK) return st;
  if (lead < 1) return KRON_ERR_INVALID_ARG;
  plan->N = N;
  plan->M = M;
  plan->dtype = dtype;
  plan->W.assign(N + 1, 0);
  int64_t K = 1;
  for (int i = 0; i < N; ++i) K *= P[i];
  // W[N] = K (Alg 1).  lead > 1: the rows hold `lead` independent blocks of K columns — an
  // implicit most-significant identity factor I_lead that is never applied (a distributed rank's
  // local block, Alg 2).
  plan->W[N] = K * lead;
  for (int f = N; f >= 1; --f) plan->W[f - 1] = plan->W[f] / P[f - 1] * Q[f - 1];  // line 307 / 319
  plan->passes.clear();

  const int64_t Mp = M > 0 ? M : 1;
  int f = N;  // next factor to apply (processing order N -> 1, Alg 1)
  while (f >= 1) {
    const int p = P[f - 1], q = Q[f - 1];
    const int64_t W = plan->W[f];
    const bool dmma_ok = policy.dmma && !getenv("KRON_NO_DMMA");
    // KRON_KINDS_MASK (experiments only): restrict the kernel families of every plan (hex bit mask)
    static const unsigned env_mask = getenv("KRON_KINDS_MASK") ? (unsigned)strtoul(getenv("KRON_KINDS_MASK"), nullptr, 16)
                                                               : ~0u;
    auto allowed = [&](int kind) { return (policy.kinds >> kind) & (env_mask >> kind) & 1u; };
    const int inst_d = (p == q && dmma_ok && allowed(5)) ? fused_find(dtype, p, 5) : -1;
    const int inst_t = (tf32x3 && p == q && allowed(8)) ? fused_find(dtype, p, 8) : -1;
    const int inst_tc = (tcm && p == q && allowed(13)) ? fused_find(dtype, p, 13) : -1;
    const int inst_3 = (p == q && allowed(10)) ? fused_find(dtype, p, 10) : -1;
    const int inst_3c = (p == q && allowed(12)) ? fused_find(dtype, p, 12) : -1;  // v10 triple
    int inst_sc = (p == q && allowed(11)) ? fused_find(dtype, p, 11) : -1;  // v10 pair (P = 16) / v12 pair (P = 32)
    if (inst_sc >= 0 && dtype == KRON_F32 && p == 32 && policy.short_tiles) inst_sc = 42;  // autotuner candidate
    int inst_s = (p == q && allowed(6)) ? fused_find(dtype, p, 6) : -1;
    if (inst_s >= 0 && policy.short_tiles && dtype == KRON_F32 && p == 16) inst_s = 35;
    // v4 chunk-pair GEMMs: not for fp64 P = 16, where the warp-chain kernel (v2) is faster (Table 3's fp64 16^6:
    // 4.41 -> 3.89 ms, found by the autotuner, profiles/r02_sweeps/table3.jsonl); v4 stays an autotuner candidate
    const int inst_g = (p == q && allowed(3) && !(dtype == KRON_F64 && p == 16 && policy.kinds == 0xFFFFu))
                           ? fused_find(dtype, p, 3)
                           : -1;
    const int inst_p = (p == q && allowed(2)) ? fused_find(dtype, p, 2) : -1;
    const int inst_w = (p == q && allowed(1)) ? fused_find(dtype, p, 1) : -1;
    const int inst_c = (p == q) ? fused_find(dtype, p, 0) : -1;  // always allowed: any chunk size
    // fp64 64 x 32 factor pairs (GP-style, config D2): one fused DMMA pass per pair (v7)
    if (dtype == KRON_F64 && p == 64 && q == 32 && f >= 2 && P[f - 2] == 64 && Q[f - 2] == 32 && dmma_ok &&
        allowed(7) && policy.kcap >= 2 && W % 4096 == 0) {
      const int iv = fused_find(dtype, 64, 7);
      if (iv >= 0) {
        PassPlan pp;
        pp.kind = KIND_FUSED;
        pp.variant = iv;
        pp.first = f;
        pp.nf = 2;
        pp.P = 64;
        pp.Q = 32;
        pp.C = 4096;
        pp.Qc = 1024;
        pp.R = 1;
        pp.tileM = 1;
        pp.tileK = 4096;
        pp.stages = 6;
        pp.W_in = W;
        pp.W_out = W / 4096 * 1024;
        plan->passes.push_back(pp);
        f -= 2;
        continue;
      }
    }
    if (inst_c >= 0) {
      int run = 1;  // consecutive factors of the same square shape
      while (f - run >= 1 && P[f - run - 1] == p && Q[f - run - 1] == p && run < 64) ++run;
      // largest group either kernel can tile; prefer the warp-chain kernel for each group size
      auto pick = [&](int k, PassPlan *pp) -> int {
        if (inst_tc >= 0 && k == 2 && tc_geometry(p, tcm, W, pp)) return inst_tc;
        if (inst_3c >= 0 && fused_geometry(fused_instance(inst_3c), k, W, Mp, pp)) return inst_3c;
        if (inst_3 >= 0 && fused_geometry(fused_instance(inst_3), k, W, Mp, pp)) return inst_3;
        if (inst_t >= 0 && fused_geometry(fused_instance(inst_t), k, W, Mp, pp)) return inst_t;
        if (inst_d >= 0 && fused_geometry(fused_instance(inst_d), k, W, Mp, pp)) return inst_d;
        if (inst_sc >= 0 && fused_geometry(fused_instance(inst_sc), k, W, Mp, pp)) return inst_sc;
        if (inst_s >= 0 && fused_geometry(fused_instance(inst_s), k, W, Mp, pp)) return inst_s;
        if (inst_g >= 0 && fused_geometry(fused_instance(inst_g), k, W, Mp, pp)) return inst_g;
        if (inst_p >= 0 && fused_geometry(fused_instance(inst_p), k, W, Mp, pp)) return inst_p;
        if (inst_w >= 0 && fused_geometry(fused_instance(inst_w), k, W, Mp, pp)) return inst_w;
        if (fused_geometry(fused_instance(inst_c), k, W, Mp, pp)) return inst_c;
        return -1;
      };
      int kmax = 0;
      PassPlan probe;
      for (int k = 1; k <= run && k <= kMaxFused && k <= policy.kcap; ++k)
        if (pick(k, &probe) >= 0) kmax = k;
      if (kmax >= 1) {
        // fewest passes, then balanced group sizes ("ceil(N/Fused) iterations")
        const int npass = (run + kmax - 1) / kmax;
        const int base = run / npass, extra = run % npass;
        for (int i = 0; i < npass; ++i) {
          const int k = base + (i < extra ? 1 : 0);
          PassPlan pp;
          pp.variant = pick(k, &pp);
          pp.first = f;
          pp.W_in = W;
          pp.W_out = W;  // square factors keep the width
          plan->passes.push_back(pp);
          f -= k;
        }
        continue;
      }
    }
    // any square P (odd sizes, rows a TMA map cannot describe): fused chain passes without TMA (chain.cu)
    if (p == q && p <= 16 && allowed(14)) {
      int run = 1;
      while (f - run >= 1 && P[f - run - 1] == p && Q[f - run - 1] == p && run < 64) ++run;
      int kmax = 0;
      PassPlan probe;
      for (int k = 2; k <= run && k <= kMaxFused && k <= policy.kcap; ++k)
        if (chain_geometry(p, k, dtype, W, policy.chain_rdiv, &probe)) kmax = k;
      if (kmax >= 2) {
        // fewest passes, then balanced group sizes; any size the balanced split cannot tile falls back
        // to kmax-sized groups
        const int npass = (run + kmax - 1) / kmax;
        const int base = run / npass, extra = run % npass;
        bool ok = true;
        std::vector<int> sizes;
        for (int i = 0; i < npass; ++i) {
          const int k = base + (i < extra ? 1 : 0);
          ok &= k == 1 || chain_geometry(p, k, dtype, W, policy.chain_rdiv, &probe);
          sizes.push_back(k);
        }
        if (!ok) {
          sizes.clear();
          for (int left = run; left > 0; left -= kmax) sizes.push_back(left < kmax ? left : kmax);
        }
        int done = 0;
        for (int k : sizes) {
          PassPlan cp;
          if (k >= 2 && chain_geometry(p, k, dtype, W, policy.chain_rdiv, &cp)) {
            cp.first = f;
            cp.W_in = W;
            cp.W_out = W;
            plan->passes.push_back(cp);
            f -= k;
            done += k;
          } else {
            break;  // the rest goes through the single-factor passes below
          }
        }
        if (done > 0) continue;
      }
    }
    PassPlan pp;
    pp.first = f;
    pp.nf = 1;
    pp.P = p;
    pp.Q = q;
    pp.C = p;
    pp.Qc = q;
    pp.W_in = W;
    pp.W_out = plan->W[f - 1];
    pp.kind = gemm_supported(dtype, Mp, W, p, q) ? KIND_GEMM : KIND_GENERIC;
    pp.variant = (pp.kind == KIND_GEMM && dtype == KRON_F64 && policy.dmma && p % 16 == 0 && q % 16 == 0) ? 1 : 0;
    if (pp.kind == KIND_GEMM && dtype == KRON_F32 && allowed(15) && sgemm_supported(Mp, W, p, q)) pp.variant = 2;
    plan->passes.push_back(pp);
    f -= 1;
  }

  // buffers (Alg 1, 318): the last pass writes Y, X is never written; interior
  // intermediates ping-pong between the workspace and Y when Y is wide enough, else two workspaces.
  const int np = (int)plan->passes.size();
  int64_t max_interior = 0;
  for (int i = 0; i + 1 < np; ++i)
    if (plan->passes[i].W_out > max_interior) max_interior = plan->passes[i].W_out;
  const bool y_alt = max_interior <= plan->W[0];
  plan->nws = np <= 1 ? 0 : (y_alt || np == 2 ? 1 : 2);
  plan->ws_elems = np <= 1 ? 0 : (M * max_interior + 63) / 64 * 64;  // keep the second buffer 256B-aligned
  for (int i = np - 1, k = 0; i >= 0; --i, ++k) {
    int dst;
    if (k == 0) dst = BUF_Y;
    else if (y_alt) dst = (k % 2 == 1) ? BUF_WS0 : BUF_Y;
    else dst = (k % 2 == 1) ? BUF_WS0 : BUF_WS1;
    plan->passes[i].dst = dst;
  }
  for (int i = 0; i < np; ++i) plan->passes[i].src = i == 0 ? BUF_X : plan->passes[i - 1].dst;

  // v11 tile-major hand-off (fused.cu, kron_tri_tm_kernel): a [16^3 triple, 16^2 pair] plan whose pair covers
  // every remaining factor (C_B = W / C_A) passes its intermediate in tile order; single-GPU plans only (lead == 1:
  // the distributed rounds' push / remap layouts assume the direct-index intermediate)
  static const bool no_handoff = getenv("KRON_NO_HANDOFF") != nullptr;
  if (np == 2 && lead == 1 && policy.handoff && !no_handoff) {
    PassPlan &A = plan->passes[0], &B = plan->passes[1];
    if (A.kind == KIND_FUSED && B.kind == KIND_FUSED && !A.tc_mode && !B.tc_mode &&
        fused_instance(A.variant).warp == 12 && fused_instance(B.variant).warp == 11 && A.C == 4096 && B.C == 256 &&
        A.W_out == B.W_in && A.C * B.C == A.W_out && (A.W_out / A.C) % 4 == 0 && B.R == 64 &&
        (B.W_in / B.C) % B.R == 0) {
      A.tm_out = 1;
      B.tm_in = 1;
    }
  }
  return KRON_OK;
}

}  // namespace kron

using namespace kron;

extern "C" {

const char *kron_last_error_detail(void) { return g_err_detail; }

const char *kron_status_string(kron_status_t s) {
  switch (s) {
    case KRON_OK: return "KRON_OK";
    case KRON_ERR_INVALID_ARG: return "KRON_ERR_INVALID_ARG";
    case KRON_ERR_SHAPE: return "KRON_ERR_SHAPE";
    case KRON_ERR_UNSUPPORTED: return "KRON_ERR_UNSUPPORTED";
    case KRON_ERR_NO_MEMORY: return "KRON_ERR_NO_MEMORY";
    case KRON_ERR_CUDA: return "KRON_ERR_CUDA";
    case KRON_ERR_NCCL: return "KRON_ERR_NCCL";
    case KRON_ERR_DIST_LAYOUT: return "KRON_ERR_DIST_LAYOUT";
  }
  return "KRON_ERR_UNKNOWN";
}

kron_status_t kron_matmul_workspace_size(int64_t M, int32_t N, const int32_t *P, const int32_t *Q,
                                         kron_dtype_t dtype, size_t *bytes) {
  if (!bytes) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> plan;
  kron_status_t st = cached_plan(M, N, P, Q, (int)dtype, &plan);
  if (st != KRON_OK) return st;
  *bytes = M == 0 ? 0 : ws_bytes_of(*plan);
  return KRON_OK;
}

kron_status_t kron_matmul_ws(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                             const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                             size_t workspace_bytes, void *stream) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X || !F || !Y) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> plan;
  st = cached_plan(M, N, P, Q, (int)dtype, &plan);
  if (st != KRON_OK) return st;
  const size_t need = ws_bytes_of(*plan);
  if (need > 0 && (!workspace || workspace_bytes < need)) return KRON_ERR_SHAPE;
  return run_plan(*plan, X, F, Y, workspace, stream);
}

struct kron_graph_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

kron_status_t kron_graph_create(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                                const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                                size_t workspace_bytes, kron_graph_t **out) {
  if (!out) return KRON_ERR_INVALID_ARG;
  *out = nullptr;
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_ERR_INVALID_ARG;
  if (!X || !F || !Y) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> plan;
  st = cached_plan(M, N, P, Q, (int)dtype, &plan);
  if (st != KRON_OK) return st;
  const size_t need = ws_bytes_of(*plan);
  if (need > 0 && (!workspace || workspace_bytes < need)) return KRON_ERR_SHAPE;
  // capture the plan's launches on a private stream (thread-local capture mode: other threads' CUDA
  // calls are unaffected); one-time launch bookkeeping (function attributes) happens during capture
  cudaStream_t cs;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
    return cuda_fail((int)cudaGetLastError(), "graph capture stream");
  auto *g = new kron_graph_s();
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    st = run_plan(*plan, X, F, Y, workspace, cs);
    e = cudaStreamEndCapture(cs, &g->graph);
    if (st == KRON_OK && e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  }
  cudaStreamDestroy(cs);
  if (st == KRON_OK && e != cudaSuccess) st = cuda_fail((int)e, "graph capture / instantiate");
  if (st != KRON_OK) {
    cudaGetLastError();
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return st;
  }
  *out = g;
  return KRON_OK;
}

kron_status_t kron_graph_launch(kron_graph_t *g, void *stream) {
  if (!g || !g->exec) return KRON_ERR_INVALID_ARG;
  const cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
  return e == cudaSuccess ? KRON_OK : cuda_fail((int)e, "graph launch");
}

kron_status_t kron_graph_destroy(kron_graph_t *g) {
  if (!g) return KRON_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return KRON_OK;
}

kron_status_t kron_matmul_ws_events(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                                    const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                                    size_t workspace_bytes, void *const *events, int32_t nevents, void *stream) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X || !F || !Y || !events) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> plan;
  st = cached_plan(M, N, P, Q, (int)dtype, &plan);
  if (st != KRON_OK) return st;
  if (nevents < (int32_t)plan->passes.size() + 1) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < (int)plan->passes.size() + 1; ++i)
    if (!events[i]) return KRON_ERR_INVALID_ARG;
  const size_t need = ws_bytes_of(*plan);
  if (need > 0 && (!workspace || workspace_bytes < need)) return KRON_ERR_SHAPE;
  return run_plan(*plan, X, F, Y, workspace, stream, events);
}

kron_status_t kron_matmul(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                          const void *const *F, void *Y, kron_dtype_t dtype, void *stream) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X || !F || !Y) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> plan;
  st = cached_plan(M, N, P, Q, (int)dtype, &plan);
  if (st != KRON_OK) return st;
  const size_t need = ws_bytes_of(*plan);
  void *ws = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (need > 0) {
    keep_pool_cached();
    if (cudaMallocAsync(&ws, need, s) != cudaSuccess) {
      cudaGetLastError();
      return KRON_ERR_NO_MEMORY;
    }
  }
  st = run_plan(*plan, X, F, Y, ws, stream);
  if (ws) cudaFreeAsync(ws, s);
  return st;
}

kron_status_t kron_matmul_host(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                               const void *const *F, void *Y, kron_dtype_t dtype, int64_t chunk_rows,
                               void *stream) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X || !F || !Y || chunk_rows < 0) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  const size_t es = (size_t)es_of((int)dtype);
  int64_t K = 1, L = 1;
  for (int i = 0; i < N; ++i) {
    K *= P[i];
    L *= Q[i];
  }
  // rows are independent (Alg 1): stream row chunks of ~64 MB through two device slots
  int64_t Mc = chunk_rows;
  if (Mc == 0) Mc = (int64_t)((64u << 20) / ((size_t)(K > L ? K : L) * es));
  if (Mc < 1) Mc = 1;
  if (Mc > M) Mc = M;
  const int64_t nchunks = (M + Mc - 1) / Mc, Mt = M - (nchunks - 1) * Mc;
  std::shared_ptr<const Plan> pc, pt;
  if ((st = cached_plan(Mc, N, P, Q, (int)dtype, &pc)) != KRON_OK) return st;
  if ((st = cached_plan(Mt, N, P, Q, (int)dtype, &pt)) != KRON_OK) return st;
  const size_t wsb = std::max(ws_bytes_of(*pc), ws_bytes_of(*pt));
  size_t fbytes = 0;
  std::vector<size_t> foff(N);
  for (int i = 0; i < N; ++i) {
    foff[i] = fbytes;
    fbytes += (((size_t)P[i] * Q[i] * es + 255) / 256) * 256;
  }
  const size_t xb = (size_t)Mc * K * es, yb = (size_t)Mc * L * es;
  const size_t xs = (xb + 255) / 256 * 256, ys = (yb + 255) / 256 * 256, wss = (wsb + 255) / 256 * 256;
  cudaStream_t sc = (cudaStream_t)stream, sin = nullptr, sout = nullptr;
  char *dev = nullptr;
  keep_pool_cached();
  if (cudaMallocAsync((void **)&dev, fbytes + 2 * xs + 2 * ys + wss, sc) != cudaSuccess) {
    cudaGetLastError();
    return KRON_ERR_NO_MEMORY;
  }
  char *Fd = dev, *Xs[2] = {dev + fbytes, dev + fbytes + xs}, *Ys[2] = {dev + fbytes + 2 * xs, dev + fbytes + 2 * xs + ys};
  char *ws = wsb ? dev + fbytes + 2 * xs + 2 * ys : nullptr;
  cudaEvent_t ev0, evF, ev_in[2], ev_comp[2], ev_out[2];
  cudaError_t e = cudaSuccess;
  auto ck = [&](cudaError_t r) {
    if (e == cudaSuccess && r != cudaSuccess) e = r;
  };
  ck(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking));
  ck(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking));
  ck(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
  ck(cudaEventCreateWithFlags(&evF, cudaEventDisableTiming));
  for (int b = 0; b < 2; ++b) {
    ck(cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming));
    ck(cudaEventCreateWithFlags(&ev_comp[b], cudaEventDisableTiming));
    ck(cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming));
  }
  if (e != cudaSuccess) {
    cudaFreeAsync(dev, sc);
    return cuda_fail((int)e, "host-path streams / events");
  }
  // the copy streams start after the caller's prior work and the allocation
  ck(cudaEventRecord(ev0, sc));
  ck(cudaStreamWaitEvent(sin, ev0, 0));
  ck(cudaStreamWaitEvent(sout, ev0, 0));
  std::vector<const void *> Fdev(N);
  for (int i = 0; i < N; ++i) {
    Fdev[i] = Fd + foff[i];
    ck(cudaMemcpyAsync(Fd + foff[i], F[i], (size_t)P[i] * Q[i] * es, cudaMemcpyHostToDevice, sin));
  }
  ck(cudaEventRecord(evF, sin));
  ck(cudaStreamWaitEvent(sc, evF, 0));
  for (int64_t c = 0; c < nchunks && e == cudaSuccess && st == KRON_OK; ++c) {
    const int b = (int)(c & 1);
    const int64_t r0 = c * Mc, rows = c + 1 < nchunks ? Mc : Mt;
    // H2D of chunk c once compute c-2 is done with slot b
    if (c >= 2) ck(cudaStreamWaitEvent(sin, ev_comp[b], 0));
    ck(cudaMemcpyAsync(Xs[b], static_cast<const char *>(X) + (size_t)r0 * K * es, (size_t)rows * K * es,
                       cudaMemcpyHostToDevice, sin));
    ck(cudaEventRecord(ev_in[b], sin));
    // the passes of chunk c once its rows landed and D2H c-2 has drained slot b
    ck(cudaStreamWaitEvent(sc, ev_in[b], 0));
    if (c >= 2) ck(cudaStreamWaitEvent(sc, ev_out[b], 0));
    st = run_plan(c + 1 < nchunks ? *pc : *pt, Xs[b], Fdev.data(), Ys[b], ws, sc);
    ck(cudaEventRecord(ev_comp[b], sc));
    // D2H of chunk c
    ck(cudaStreamWaitEvent(sout, ev_comp[b], 0));
    ck(cudaMemcpyAsync(static_cast<char *>(Y) + (size_t)r0 * L * es, Ys[b], (size_t)rows * L * es,
                       cudaMemcpyDeviceToHost, sout));
    ck(cudaEventRecord(ev_out[b], sout));
  }
  // the caller's stream completes with the last copies; buffers are released stream-ordered after them
  for (int b = 0; b < 2; ++b) ck(cudaStreamWaitEvent(sc, ev_out[b], 0));
  ck(cudaEventRecord(ev0, sin));
  ck(cudaStreamWaitEvent(sc, ev0, 0));
  cudaFreeAsync(dev, sc);
  cudaEventDestroy(ev0);
  cudaEventDestroy(evF);
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(ev_in[b]);
    cudaEventDestroy(ev_comp[b]);
    cudaEventDestroy(ev_out[b]);
  }
  cudaStreamDestroy(sin);
  cudaStreamDestroy(sout);
  if (st != KRON_OK) return st;
  return e == cudaSuccess ? KRON_OK : cuda_fail((int)e, "host-path copies");
}

// Candidate plans for the autotuner: fusion-depth caps x kernel-family masks x fp64 DMMA,
// duplicates removed; the static plan (no cap, all families, DMMA) is always candidate 0.
std::vector<Plan> autotune_candidates(int64_t M, int N, const int32_t *P, const int32_t *Q, int dtype) {
  // candidate policies: fusion-depth caps x kernel families x DMMA; duplicate plans removed
  const unsigned all = 0xFFFFu;
  const unsigned v10 = (1u << 11) | (1u << 12);  // constant-bank kernels vs their round-1 shared-memory twins
  const unsigned kinds[] = {all, all & ~v10, all & ~(1u << 12), all & ~(1u << 11), all & ~((1u << 10) | (1u << 12)),
                            all & ~(1u << 13), all & ~((1u << 13) | v10), all & ~(1u << 2), all & ~((1u << 5) | (1u << 6) | (1u << 7)),
                            all & ~((1u << 3) | (1u << 5) | (1u << 6) | (1u << 7)), (1u << 0) | (1u << 1)};
  const int caps[] = {kMaxFused, 3, 2, 1};
  std::vector<Plan> cands;
  auto same = [](const Plan &a, const Plan &b) {
    if (a.passes.size() != b.passes.size()) return false;
    for (size_t i = 0; i < a.passes.size(); ++i) {
      const PassPlan &x = a.passes[i], &y = b.passes[i];
      if (x.kind != y.kind || x.variant != y.variant || x.first != y.first || x.nf != y.nf || x.tileK != y.tileK ||
          x.R != y.R || x.tm_out != y.tm_out || x.tm_in != y.tm_in ||
          x.tileM != y.tileM || x.stages != y.stages)
        return false;
    }
    return true;
  };
  for (int ho = 1; ho >= 0; --ho)
  for (int rd : {1, 2, 4})
  for (int st = 0; st <= 1; ++st)
  for (int dm = 1; dm >= 0; --dm)
    for (unsigned km : kinds)
      for (int cap : caps) {
        PlanPolicy pol;
        pol.kcap = cap;
        pol.kinds = km;
        pol.dmma = dm == 1;
        pol.short_tiles = st == 1;
        pol.chain_rdiv = rd;
        pol.handoff = ho == 1;
        Plan pl;
        if (make_plan(M, N, P, Q, dtype, &pl, 1, pol) != KRON_OK) continue;
        bool dup = false;
        for (const Plan &c : cands) dup |= same(c, pl);
        if (!dup) cands.push_back(pl);
      }
  return cands;
}

kron_status_t kron_autotune_candidates(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                       int32_t *ncand) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (!ncand) return KRON_ERR_INVALID_ARG;
  *ncand = M == 0 ? 0 : (int32_t)autotune_candidates(M, N, P, Q, (int)dtype).size();
  return KRON_OK;
}

kron_status_t kron_plan_cache_clear(void) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.clear();
  return KRON_OK;
}

kron_status_t kron_autotune(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                            const void *const *F, void *Y, kron_dtype_t dtype, int32_t reps, void *stream,
                            int32_t *ncand, float *best_ms) {
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X || !F || !Y || reps < 1) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  std::vector<Plan> cands = autotune_candidates(M, N, P, Q, (int)dtype);
  if (cands.empty()) return KRON_ERR_UNSUPPORTED;
  size_t wsmax = 0;
  for (const Plan &c : cands) wsmax = std::max(wsmax, ws_bytes_of(c));
  cudaStream_t s = (cudaStream_t)stream;
  void *ws = nullptr;
  keep_pool_cached();
  if (wsmax && cudaMallocAsync(&ws, wsmax, s) != cudaSuccess) {
    cudaGetLastError();
    return KRON_ERR_NO_MEMORY;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int best = -1;
  float best_t = 0.f;
  // two sweeps over the candidates (the second in reverse order, so clock drift over the sweep does not favour
  // one end), each run timed on its own; a candidate's time is its fastest run.  A candidate replaces the static
  // plan (candidate 0) only when it is more than 2% faster: near-ties stay on the static plan
  std::vector<float> tmin(cands.size(), 1e30f);
  for (int sweep = 0; sweep < 2 && st == KRON_OK; ++sweep)
    for (size_t n = 0; n < cands.size() && st == KRON_OK; ++n) {
      const size_t i = sweep == 0 ? n : cands.size() - 1 - n;
      if (sweep == 0) {
        st = run_plan(cands[i], X, F, Y, ws, stream);  // warm-up (also primes kernel attributes)
        if (st != KRON_OK) break;
      }
      for (int r = 0; r < reps && st == KRON_OK; ++r) {
        cudaEventRecord(e0, s);
        st = run_plan(cands[i], X, F, Y, ws, stream);
        cudaEventRecord(e1, s);
        if (cudaEventSynchronize(e1) != cudaSuccess) st = cuda_fail((int)cudaGetLastError(), "autotune timing");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (st == KRON_OK && ms < tmin[i]) tmin[i] = ms;
      }
    }
  if (st == KRON_OK) {
    best = 0;
    best_t = tmin[0];
    for (size_t i = 1; i < cands.size(); ++i)
      if (tmin[i] < best_t && tmin[i] < 0.98f * tmin[0]) {
        best = (int)i;
        best_t = tmin[i];
      }
  }
  // leave Y holding the result of the chosen plan
  if (st == KRON_OK) st = run_plan(cands[best], X, F, Y, ws, stream);
  if (ws) cudaFreeAsync(ws, s);
  cudaStreamSynchronize(s);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != KRON_OK) return st;
  int dev = 0;
  cudaGetDevice(&dev);
  PlanKey key{dev, M, (int)dtype, std::vector<int32_t>(P, P + N), std::vector<int32_t>(Q, Q + N)};
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[key] = std::make_shared<Plan>(cands[best]);
  }
  if (ncand) *ncand = (int32_t)cands.size();
  if (best_ms) *best_ms = best_t;
  return KRON_OK;
}

kron_status_t kron_plan_describe(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                 int32_t cap, int32_t *npasses, int32_t *first, int32_t *nfactors, int32_t *kind) {
  if (!npasses) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> pl;
  kron_status_t st = cached_plan(M, N, P, Q, (int)dtype, &pl);
  if (st != KRON_OK) return st;
  const Plan &plan = *pl;
  *npasses = (int32_t)plan.passes.size();
  for (int i = 0; i < (int)plan.passes.size() && i < cap; ++i) {
    if (first) first[i] = plan.passes[i].first;
    if (nfactors) nfactors[i] = plan.passes[i].nf;
    if (kind) kind[i] = plan.passes[i].kind;
  }
  return KRON_OK;
}

kron_status_t kron_plan_kernel(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                               int32_t pass, char *name, int32_t len) {
  if (!name || len < 1) return KRON_ERR_INVALID_ARG;
  std::shared_ptr<const Plan> pl;
  kron_status_t st = cached_plan(M, N, P, Q, (int)dtype, &pl);
  if (st != KRON_OK) return st;
  if (pass < 0 || pass >= (int32_t)pl->passes.size()) return KRON_ERR_INVALID_ARG;
  const PassPlan &pp = pl->passes[pass];
  const char *k = "sliced_generic_kernel";
  if (pp.kind == KIND_CHAIN) {
    k = "kron_chain_kernel";
  } else if (pp.kind == KIND_GEMM) {
    k = pp.variant == 1 ? "kron_dmma_kernel" : pp.variant == 2 ? "kron_sgemm_kernel" : "kron_gemm_kernel";
  } else if (pp.kind == KIND_FUSED) {
    static const char *names[] = {"kron_fused_kernel",       "kron_fused_warp_kernel",  "kron_fused_pipe_kernel",
                                  "kron_fused_gemm2_kernel", "kron_fused_pipe_kernel",  "kron_fused_dmma2_kernel",
                                  "kron_fused_gemm2ws_kernel", "kron_fused_dmma2g_kernel", "kron_fused_tf32x3_kernel",
                                  "kron_fused_kernel",         "kron_fused_gemm3c_kernel",
                                  "kron_fused_gemm2ws_kernel", "kron_fused_gemm3c_kernel",
                                  "kron_tc_pair_kernel"};
    const int w = fused_instance(pp.variant).warp;
    k = (w >= 0 && w < 14) ? names[w] : "kron_fused_kernel";
    if (pp.tm_out) k = "kron_tri_tm_kernel";
    if (pp.tm_in) k = "kron_pair_tm_kernel";
  }
  snprintf(name, (size_t)len, "%s", k);
  return KRON_OK;
}

kron_status_t kron_plan_cost(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                             double *hbm_bytes, double *flops) {
  std::shared_ptr<const Plan> pl;
  kron_status_t st = cached_plan(M, N, P, Q, (int)dtype, &pl);
  if (st != KRON_OK) return st;
  const Plan &plan = *pl;
  const double es = es_of((int)dtype);
  double b = 0, fl = 0;
  for (const PassPlan &pp : plan.passes) b += es * (double)M * (double)(pp.W_in + pp.W_out);
  for (int i = 0; i < N; ++i) b += es * (double)P[i] * Q[i];
  for (int f = 1; f <= N; ++f) fl += 2.0 * (double)M * (double)plan.W[f] * Q[f - 1];
  if (hbm_bytes) *hbm_bytes = b;
  if (flops) *flops = fl;
  return KRON_OK;
}

}  // extern "C"
