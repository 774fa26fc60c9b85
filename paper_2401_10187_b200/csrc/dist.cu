// dist.cu — distributed Kron-Matmul, Algorithm 2: host round planner and grid rule.
// (The context / exchange implementation is added in a later milestone.)
#include <cuda_runtime.h>

#include <vector>

#include "kron_internal.h"

namespace kron {

// Round plan (reading G11): each round applies the most factors its local column block allows —
// the round's chunk C = prod P must divide the local width W/GK (local slices are global slices,
// P:645-647), and GK must divide the round's composite column count prod Q so that every rank
// sends one contiguous part of W'/GK^2 values to every peer (Fig 8).  Fewest rounds first,
// then balanced round sizes for uniform shapes.
kron_status_t dist_round_plan(int64_t M, int N, const int32_t *P, const int32_t *Q, int GM, int GK,
                              std::vector<int> *rounds, std::vector<int64_t> *ledger) {
  kron_status_t st = validate(M, N, P, Q, KRON_F64);
  if (st != KRON_OK) return st;
  if (GM < 1 || GK < 1) return KRON_ERR_INVALID_ARG;
  if (M % GM) return KRON_ERR_DIST_LAYOUT;
  std::vector<int64_t> W(N + 1);
  W[N] = 1;
  for (int i = 0; i < N; ++i) W[N] *= P[i];
  for (int f = N; f >= 1; --f) W[f - 1] = W[f] / P[f - 1] * Q[f - 1];
  auto feasible = [&](int f, int k) {  // factors f, f-1, ..., f-k+1 in one round
    if (W[f] % GK) return false;
    const int64_t wl = W[f] / GK;
    int64_t C = 1, Qc = 1;
    for (int i = 0; i < k; ++i) {
      C *= P[f - 1 - i];
      Qc *= Q[f - 1 - i];
    }
    return wl % C == 0 && Qc % GK == 0;
  };
  std::vector<int> greedy;
  for (int f = N; f >= 1;) {
    int best = 0;
    for (int k = 1; k <= f; ++k)
      if (feasible(f, k)) best = k;
    if (best == 0) return KRON_ERR_DIST_LAYOUT;
    greedy.push_back(best);
    f -= best;
  }
  if (W[0] % GK) return KRON_ERR_DIST_LAYOUT;
  std::vector<int> plan = greedy;
  bool uniform = true;
  for (int i = 1; i < N; ++i) uniform &= (P[i] == P[0] && Q[i] == Q[0]);
  if (uniform && greedy.size() > 1) {
    const int nr = (int)greedy.size(), base = N / nr, extra = N % nr;
    std::vector<int> bal;
    bool ok = true;
    for (int j = 0, f = N; j < nr; ++j) {
      const int k = base + (j < extra ? 1 : 0);
      ok &= feasible(f, k);
      bal.push_back(k);
      f -= k;
    }
    if (ok) plan = bal;
  }
  if (rounds) *rounds = plan;
  if (ledger) {
    ledger->clear();
    int f = N;
    for (int k : plan) {
      f -= k;
      ledger->push_back(M * W[f] / GK * (GK - 1));  // M * W_j * (1 - 1/GK)  (reading G12)
    }
  }
  return KRON_OK;
}

kron_status_t grid_rule(int G, int *GM, int *GK) {
  if (G < 1 || !GM || !GK) return KRON_ERR_INVALID_ARG;
  int s = 0;
  while ((s + 1) * (s + 1) <= G) ++s;
  if (s * s == G) {
    *GM = *GK = s;
    return KRON_OK;
  }
  int lg = 0;
  while ((1 << (lg + 1)) <= G) ++lg;
  if ((1 << lg) != G) return KRON_ERR_INVALID_ARG;  // rule yields 2^a * 2^b != G
  *GM = 1 << ((lg + 1) / 2);  // 2^ceil(log2 sqrt G)
  *GK = 1 << (lg / 2);        // 2^floor(log2 sqrt G)
  return KRON_OK;
}

}  // namespace kron

using namespace kron;

struct kron_dist_ctx {
  int backend = 0;
};

extern "C" {

kron_status_t kron_dist_grid_rule(int32_t G, int32_t *GM, int32_t *GK) { return grid_rule(G, GM, GK); }

kron_status_t kron_dist_plan(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, int32_t GM, int32_t GK,
                             int32_t cap, int32_t *nrounds, int32_t *rounds, int64_t *ledger) {
  if (!nrounds) return KRON_ERR_INVALID_ARG;
  std::vector<int> r;
  std::vector<int64_t> l;
  kron_status_t st = dist_round_plan(M, N, P, Q, GM, GK, &r, &l);
  if (st != KRON_OK) return st;
  *nrounds = (int32_t)r.size();
  for (int i = 0; i < (int)r.size() && i < cap; ++i) {
    if (rounds) rounds[i] = r[i];
    if (ledger) ledger[i] = l[i];
  }
  return KRON_OK;
}

kron_status_t kron_dist_nccl_unique_id(void *) { return KRON_ERR_NCCL; }

kron_status_t kron_dist_ctx_create(int32_t, const void *, int32_t, int32_t, int32_t, int32_t, kron_dist_ctx_t **out) {
  if (out) *out = nullptr;
  return KRON_ERR_UNSUPPORTED;
}

kron_status_t kron_dist_ctx_destroy(kron_dist_ctx_t *ctx) {
  delete ctx;
  return KRON_OK;
}

kron_status_t kron_dist_ctx_grid(const kron_dist_ctx_t *, int32_t *, int32_t *) { return KRON_ERR_UNSUPPORTED; }

kron_status_t kron_matmul_dist(int64_t, int32_t, const int32_t *, const int32_t *, const void *, const void *const *,
                               void *, kron_dtype_t, kron_dist_ctx_t *, void *) {
  return KRON_ERR_UNSUPPORTED;
}

}  // extern "C"
