// dist.cu — distributed Kron-Matmul, Algorithm 2, one rank per GPU.
//
// Grid {GM, GK}: rank r = gM*GK + gK holds X[gM rows][gK column block].  Rows never
// communicate.  Within a row group the K dimension is split: each ROUND applies as many
// factors as the local column block allows (Local = floor(log_P GTileK), line 666),
// using the single-GPU fused / GEMM passes on the local block, then ONE all-to-all regroups the
// slices (lines 676-692, reading G13) and StoreGPUTile places the received runs (line 685):
//
//   after a round with chunk C = prod P and Qc = prod Q of its factors, local run u (length
//   rho = W/(C*GK)) of source gK belongs to global column (u*GK + gK)*rho; destination
//   d = u div (Qc/GK) receives runs e = u mod (Qc/GK) and stores them at local (e*GK + gK)*rho.
//
// The exchange is ncclAlltoAll on a row-group communicator (ncclCommSplit(color = gM)); NCCL is
// loaded with dlopen so libkron itself needs no NCCL at link time.  A "virtual" backend drives all
// ranks of the grid from one process on one GPU, exchanging with device-to-device copies: it runs the
// same planner, local passes, pack and StoreGPUTile kernels, and is how the distributed data path is
// tested on a single B200.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "kron_internal.h"

namespace kron {

// ------------------------------------------------------------------ round planner (host)

// Reading G11: each round applies the most factors its local column block allows — the round's chunk
// C = prod P must divide the local width W/GK (local slices are global slices), and GK must
// divide the round's composite column count prod Q so that every rank sends one contiguous part of
// W'/GK^2 values per row to every peer (Fig 8).  Fewest rounds first, then balanced sizes.
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
  *GM = 1 << ((lg + 1) / 2);                         // 2^ceil(log2 sqrt G)
  *GK = 1 << (lg / 2);                               // 2^floor(log2 sqrt G)
  return KRON_OK;
}

// ------------------------------------------------------------------ pack / StoreGPUTile kernels

namespace {

// send[d][m][e] = out[m][d*B + e]      (destination-major send buffer, B = W'/GK)
template <typename T>
__global__ void __launch_bounds__(256) dist_pack_kernel(const T *__restrict__ in, T *__restrict__ send, int64_t rows,
                                                        int64_t Wl, int64_t B) {
  const int64_t n = rows * Wl;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / Wl, c = i - m * Wl;
    const int64_t d = c / B, e = c - d * B;
    send[(d * rows + m) * B + e] = in[i];
  }
}

// StoreGPUTile (Alg 2): out[m][(e*GK + src)*rho + t] = recv[src][m][e*rho + t]
template <typename T>
__global__ void __launch_bounds__(256) dist_store_gpu_tile_kernel(const T *__restrict__ recv, T *__restrict__ out,
                                                                  int64_t rows, int64_t Wl, int64_t rho, int GK) {
  const int64_t n = rows * Wl, B = Wl / GK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / Wl, c = i - m * Wl;
    const int64_t run = c / rho, t = c - run * rho;
    const int64_t e = run / GK, src = run - e * GK;
    out[i] = recv[(src * rows + m) * B + e * rho + t];
  }
}

// The same StoreGPUTile copy by whole runs (rho >= 64): one CTA per run, 16-byte copies when the runs are
// 16-byte aligned — the per-element kernel above spends three 64-bit divisions per value (config E's final
// remap, rho = 2048: 5.4 ms for 8.6 GB through the virtual backend)
template <typename T>
__global__ void __launch_bounds__(256) dist_store_gpu_tile_runs_kernel(const T *__restrict__ recv, T *__restrict__ out,
                                                                       int64_t rows, int64_t Wl, int64_t rho, int GK,
                                                                       int vec) {
  const int64_t B = Wl / GK, nrun = Wl / rho, total = rows * nrun;
  for (int64_t r = blockIdx.x; r < total; r += gridDim.x) {
    const int64_t m = r / nrun, run = r - m * nrun;
    const int64_t e = run / GK, src = run - e * GK;
    const T *sp = recv + (src * rows + m) * B + e * rho;
    T *dp = out + m * Wl + run * rho;
    if (vec) {
      const int n4 = (int)(rho * (int64_t)sizeof(T) / 16);
      for (int i = threadIdx.x; i < n4; i += blockDim.x)
        reinterpret_cast<float4 *>(dp)[i] = reinterpret_cast<const float4 *>(sp)[i];
    } else {
      for (int i = threadIdx.x; i < (int)rho; i += blockDim.x) dp[i] = sp[i];
    }
  }
}

int launch_pack(int dtype, const void *in, void *send, int64_t rows, int64_t Wl, int64_t B, cudaStream_t s) {
  const int64_t n = rows * Wl;
  if (n == 0) return 0;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (dtype == KRON_F32)
    dist_pack_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float *)in, (float *)send, rows, Wl, B);
  else
    dist_pack_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double *)in, (double *)send, rows, Wl, B);
  return (int)cudaGetLastError();
}

int launch_store_gpu_tile(int dtype, const void *recv, void *out, int64_t rows, int64_t Wl, int64_t rho, int GK,
                          cudaStream_t s) {
  const int64_t n = rows * Wl;
  if (n == 0) return 0;
  if (rho >= 64 && Wl % rho == 0 && rho < (int64_t(1) << 30)) {
    const size_t es = dtype == KRON_F32 ? 4 : 8;
    const int vec = ((uintptr_t)recv % 16 == 0 && (uintptr_t)out % 16 == 0 && (rho * (int64_t)es) % 16 == 0 &&
                     ((Wl / GK) * (int64_t)es) % 16 == 0 && (Wl * (int64_t)es) % 16 == 0)
                        ? 1
                        : 0;
    int64_t blocks = rows * (Wl / rho);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (dtype == KRON_F32)
      dist_store_gpu_tile_runs_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float *)recv, (float *)out, rows,
                                                                              Wl, rho, GK, vec);
    else
      dist_store_gpu_tile_runs_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double *)recv, (double *)out,
                                                                               rows, Wl, rho, GK, vec);
    return (int)cudaGetLastError();
  }
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (dtype == KRON_F32)
    dist_store_gpu_tile_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float *)recv, (float *)out, rows, Wl,
                                                                       rho, GK);
  else
    dist_store_gpu_tile_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double *)recv, (double *)out, rows,
                                                                        Wl, rho, GK);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ P2P exchange over peer memory (NEXT-1)
//
// The paper notes that lines 676-690 of Algorithm 2 can run as ONE kernel when the GPUs can access each
// other's memory.  Backend 2 does that: every rank's round output lives in a symmetric heap
// (cudaMalloc + CUDA IPC, mapped by the peers of its row group over NVLink / NVSwitch), and after a
// device-side flag barrier each rank PULLS its values straight from the peers' heaps into their
// StoreGPUTile position of its next-round block (or of Y_local after the last round):
//
//   dst[m][(e*GK + src)*rho + t] = out_src[m][me*B + e*rho + t]          (B = W'/GK, t < rho)
//
// which is the pack kernel, the all-to-all and the StoreGPUTile kernel of backend 0 in one pass (one
// HBM read at the source, one write at the destination, no send / receive buffers).  The round outputs
// alternate between two halves of the heap, so one barrier per round suffices: when a rank passes the
// barrier of round j every peer has finished its round j-1 pulls, which is the half round j+1 rewrites.

constexpr int kMaxPeers = 64;
constexpr size_t kP2PHeader = 4096;       // heap header: u64 flag per row-group peer, then the timeout word
constexpr size_t kP2PTimeoutOff = 8 * kMaxPeers;
struct PeerPtrs {
  const char *p[kMaxPeers];
};

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Row-group barrier: lane i signals peer i (flag slot `me` of its heap) with the epoch, then waits until
// peer i has signalled this rank.  The wait is bounded (~`spin_ns`): on timeout it counts the miss in
// the heap's timeout word (kron_dist_p2p_timeouts) instead of hanging the device.
__global__ void p2p_barrier_kernel(PeerPtrs heaps, unsigned long long *my_flags, int GK, int me,
                                   unsigned long long epoch, unsigned *timeouts, long long spin_ns) {
  const int i = threadIdx.x;
  if (i >= GK || i == me) return;
  __threadfence_system();  // this rank's earlier kernels (its round output) before the signal
  st_release_sys(reinterpret_cast<unsigned long long *>(const_cast<char *>(heaps.p[i])) + me, epoch);
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(my_flags + i) < epoch) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > spin_ns) {
      atomicAdd(timeouts, 1u);
      break;
    }
    __nanosleep(64);
  }
}

// Pull + StoreGPUTile.  V = elements per vector (16 bytes when rho*es and the offsets allow, else 1).
// I: the index type — 32-bit when rows * Wl / V < 2^31 (the divisions per vector are then 32-bit: a 64-bit
// division is several times the cost)
template <typename T, int V, typename I>
__global__ void __launch_bounds__(256) p2p_pull_kernel(PeerPtrs outs, T *__restrict__ dst, int64_t rows, int64_t Wl,
                                                       int64_t rho, int GK, int me) {
  using Vec = typename std::conditional<V == 1, T, uint4>::type;
  const I wv = (I)(Wl / V), B = (I)(Wl / GK), rv = (I)(rho / V), n = (I)(rows * (Wl / V)), gk = (I)GK;
  const I stride = (I)gridDim.x * (I)blockDim.x;
  for (I i0 = (I)blockIdx.x * (I)blockDim.x + (I)threadIdx.x; i0 < n; i0 += 4 * stride) {
    Vec v[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // four independent remote loads in flight per thread
      const I i = i0 + (I)u * stride;
      ok[u] = i < n;
      if (ok[u]) {
        const I m = i / wv, c = i - m * wv;
        const I run = c / rv, t = c - run * rv;
        const I e = run / gk, src = run - e * gk;
        const Vec *s = reinterpret_cast<const Vec *>(outs.p[src]) + (int64_t)m * wv + (int64_t)me * (B / V) + e * rv + t;
        v[u] = *s;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) reinterpret_cast<Vec *>(dst)[(int64_t)i0 + (int64_t)u * stride] = v[u];
  }
}

int launch_p2p_pull(int dtype, const PeerPtrs &outs, void *dst, int64_t rows, int64_t Wl, int64_t rho, int GK, int me,
                    cudaStream_t s) {
  const int64_t n = rows * Wl;
  if (n == 0) return 0;
  const int es = dtype == KRON_F32 ? 4 : 8;
  const int V = 16 / es;
  bool vec = (rho * es) % 16 == 0 && (Wl * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  for (int g = 0; g < GK; ++g) vec &= (reinterpret_cast<uintptr_t>(outs.p[g]) & 15) == 0;
  int64_t blocks = (n / (vec ? V : 1) + 1023) / 1024;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  const bool small = n < (int64_t(1) << 31) - 4 * 148 * 8 * 256;  // 32-bit indices cannot overflow
  if (dtype == KRON_F32) {
    if (small) {
      if (vec) p2p_pull_kernel<float, 4, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (float *)dst, rows, Wl, rho, GK, me);
      else p2p_pull_kernel<float, 1, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (float *)dst, rows, Wl, rho, GK, me);
    } else {
      if (vec) p2p_pull_kernel<float, 4, int64_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (float *)dst, rows, Wl, rho, GK, me);
      else p2p_pull_kernel<float, 1, int64_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (float *)dst, rows, Wl, rho, GK, me);
    }
  } else {
    if (small) {
      if (vec) p2p_pull_kernel<double, 2, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (double *)dst, rows, Wl, rho, GK, me);
      else p2p_pull_kernel<double, 1, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (double *)dst, rows, Wl, rho, GK, me);
    } else {
      if (vec) p2p_pull_kernel<double, 2, int64_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (double *)dst, rows, Wl, rho, GK, me);
      else p2p_pull_kernel<double, 1, int64_t><<<(unsigned)blocks, 256, 0, s>>>(outs, (double *)dst, rows, Wl, rho, GK, me);
    }
  }
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ NCCL via dlopen

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
  ncclResult_t (*AlltoAll)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi &nccl() {
  std::call_once(g_nccl_once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
      g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (g_nccl.h) break;
    }
    if (!g_nccl.h) return;
#define KRON_SYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(g_nccl.h, name))
    KRON_SYM(GetUniqueId, "ncclGetUniqueId");
    KRON_SYM(CommInitRank, "ncclCommInitRank");
    KRON_SYM(CommSplit, "ncclCommSplit");
    KRON_SYM(CommDestroy, "ncclCommDestroy");
    KRON_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    KRON_SYM(AlltoAll, "ncclAlltoAll");
    KRON_SYM(GroupStart, "ncclGroupStart");
    KRON_SYM(GroupEnd, "ncclGroupEnd");
    KRON_SYM(Send, "ncclSend");
    KRON_SYM(Recv, "ncclRecv");
    KRON_SYM(CommAbort, "ncclCommAbort");
#undef KRON_SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommSplit && g_nccl.CommDestroy &&
                (g_nccl.AlltoAll || (g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.Send && g_nccl.Recv));
  });
  return g_nccl;
}

}  // namespace
}  // namespace kron

using namespace kron;

struct kron_dist_ctx {
  int backend = 0;  // 0 NCCL, 1 virtual, 2 P2P (peer memory)
  int world = 1, rank = 0, GM = 1, GK = 1, gM = 0, gK = 0;
  // backends 0 / 1: row chunks per round (chunk c's all-to-all overlaps chunk c+1's local passes) and the
  // fused data layout (the round's last pass writes the send buffer, the next round's first pass reads the
  // receive buffer through the StoreGPUTile-ordered tensor map)
  int nchunks = 2;
  bool fused = true;
  bool push = true;  // backend 2: fuse the exchange into the round's last pass where the kernel has a push epilogue
  ncclComm_t world_comm = nullptr, row_comm = nullptr;
  cudaStream_t comm = nullptr;  // backend 0: all-to-all stream (created on first use on the calling device)
  std::vector<cudaEvent_t> ev;  // backend 0: [start | per chunk: computed, exchanged]
  // backend 2: symmetric heap = [flags: u64 per row-group peer | timeout word] [out half 0] [out half 1]
  char *heap = nullptr;
  size_t heap_bytes = 0;                 // usable bytes (both halves)
  char *peer_heap[kron::kMaxPeers] = {};  // row-group peers' heaps (index gK; own heap at this->gK)
  bool connected = false;
  unsigned long long epoch = 0;  // barrier epoch (identical on every rank: calls are collective)
  unsigned parity = 0;           // which heap half the next round writes
};

namespace kron {
namespace {

// All-to-all inside the row group: recv[src] <- send_src[me].  blk = elements per peer.
kron_status_t exchange_nccl(kron_dist_ctx *ctx, int dtype, const void *send, void *recv, size_t blk, cudaStream_t s) {
  const NcclApi &api = nccl();
  const ncclDataType_t dt = dtype == KRON_F32 ? ncclFloat32 : ncclFloat64;
  const size_t es = dtype == KRON_F32 ? 4 : 8;
  if (api.AlltoAll) {
    if (api.AlltoAll(send, recv, blk, dt, ctx->row_comm, s) != ncclSuccess) return KRON_ERR_NCCL;
    return KRON_OK;
  }
  if (api.GroupStart() != ncclSuccess) return KRON_ERR_NCCL;
  for (int p = 0; p < ctx->GK; ++p) {
    api.Send(static_cast<const char *>(send) + p * blk * es, blk, dt, p, ctx->row_comm, s);
    api.Recv(static_cast<char *>(recv) + p * blk * es, blk, dt, p, ctx->row_comm, s);
  }
  if (api.GroupEnd() != ncclSuccess) return KRON_ERR_NCCL;
  return KRON_OK;
}

// asynchronous NCCL errors of earlier calls on this context (non-blocking)
kron_status_t nccl_async_status(kron_dist_ctx *ctx) {
  if (ctx->backend != 0) return KRON_OK;
  const NcclApi &api = nccl();
  if (!api.CommGetAsyncError) return KRON_OK;
  for (ncclComm_t c : {ctx->world_comm, ctx->row_comm}) {
    if (!c) continue;
    ncclResult_t r = ncclSuccess;
    if (api.CommGetAsyncError(c, &r) != ncclSuccess || (r != ncclSuccess && r != ncclInProgress)) return KRON_ERR_NCCL;
  }
  return KRON_OK;
}

struct RankBufs {
  void *cur = nullptr, *out = nullptr, *send = nullptr, *recv = nullptr, *ws = nullptr;
};

// One round of Algorithm 2 (lines 670-692): `k` factors applied locally to the [rows][wl_in] block.
struct RoundPlan {
  Plan plan[2];  // [0]: full row chunk, [1]: the ragged last chunk
  int first = 0, k = 0;
  int64_t wl_in = 0, wl_out = 0, rho = 0;
  bool fpush = false;   // backends 0/1: the last pass writes the destination-major send buffer
  bool fremap = false;  // backends 0/1: the first pass reads the previous round's receive buffer in place
  int tm = 0;           // backends 0/1, config-E rounds [16^3, 16^2]: v11 tile-major layouts (1 triple, 2 pair)
};

// v11 hand-off through the exchange (fused.cu kron_tri_tm_kernel): rounds [16^3 triple, 16^2 pair] on fp32 — the
// triple writes the send blocks tile-major (each destination's u range), the pair reads the receive blocks through
// a 4-D map whose box lands in the single-GPU tile layout, and pushes its outputs into the final send blocks; the
// values and the exchanged volume are those of the direct-index rounds.  plans[j][v]: round j's local plans (full
// and ragged row chunk); wl_in[j]: round j's local input width.
bool tile_major_rounds(int dtype, int N, const int32_t *P, const int32_t *Q, int GK, const std::vector<int> &rounds,
                       const Plan *const (*plans)[2], const int64_t *wl_in, bool fused, bool p2p) {
  static const bool no_handoff = getenv("KRON_NO_HANDOFF") != nullptr;
  bool tm = !p2p && fused && !no_handoff && dtype == KRON_F32 && rounds.size() == 2 && rounds[0] == 3 &&
            rounds[1] == 2 && GK <= kMaxPush && 64 % GK == 0;
  for (int i = 0; i < N && tm; ++i) tm &= P[i] == 16 && Q[i] == 16;
  for (int j = 0; j < 2 && tm; ++j)
    for (int v = 0; v < 2; ++v) {
      const Plan &pl = *plans[j][v];
      tm &= pl.passes.size() == 1 && pl.passes[0].kind == KIND_FUSED && !pl.passes[0].tc_mode &&
            fused_instance(pl.passes[0].variant).warp == (j == 0 ? 12 : 11) && pl.passes[0].R == (j == 0 ? 8 : 64);
    }
  return tm && (wl_in[0] / 4096) % 4 == 0 && 4096 % (32 * GK) == 0 && (wl_in[1] / 256) % 64 == 0;
}

inline char *at(void *p, int64_t elems, size_t es) { return static_cast<char *>(p) + (size_t)elems * es; }
inline const char *at(const void *p, int64_t elems, size_t es) { return static_cast<const char *>(p) + (size_t)elems * es; }

}  // namespace
}  // namespace kron

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

kron_status_t kron_dist_nccl_unique_id(void *out128) {
  if (!out128) return KRON_ERR_INVALID_ARG;
  const NcclApi &api = nccl();
  if (!api.ok) return KRON_ERR_NCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return KRON_ERR_NCCL;
  memcpy(out128, &id, sizeof(id));
  return KRON_OK;
}

kron_status_t kron_dist_ctx_create(int32_t backend, const void *nccl_unique_id, int32_t world_size, int32_t rank,
                                   int32_t GM, int32_t GK, kron_dist_ctx_t **out) {
  if (!out || world_size < 1 || backend < 0 || backend > 2) return KRON_ERR_INVALID_ARG;
  *out = nullptr;
  if (GM == 0 && GK == 0) {
    kron_status_t st = grid_rule(world_size, &GM, &GK);
    if (st != KRON_OK) return st;
  }
  if (GM < 1 || GK < 1 || GM * GK != world_size) return KRON_ERR_INVALID_ARG;
  auto *ctx = new kron_dist_ctx;
  ctx->backend = backend;
  ctx->world = world_size;
  ctx->GM = GM;
  ctx->GK = GK;
  // the P2P push mode is fixed here, once (every rank of a context must use the same protocol)
  ctx->push = getenv("KRON_P2P_NO_PUSH") == nullptr;
  if (backend == 0) {
    if (!nccl_unique_id || rank < 0 || rank >= world_size) {
      delete ctx;
      return KRON_ERR_INVALID_ARG;
    }
    const NcclApi &api = nccl();
    if (!api.ok) {
      delete ctx;
      return KRON_ERR_NCCL;
    }
    ctx->rank = rank;
    ctx->gM = rank / GK;
    ctx->gK = rank % GK;
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    if (api.CommInitRank(&ctx->world_comm, world_size, id, rank) != ncclSuccess ||
        api.CommSplit(ctx->world_comm, ctx->gM, ctx->gK, &ctx->row_comm, nullptr) != ncclSuccess) {
      if (ctx->world_comm) api.CommDestroy(ctx->world_comm);
      delete ctx;
      return KRON_ERR_NCCL;
    }
  }
  if (backend == 2) {
    if (rank < 0 || rank >= world_size || GK > kMaxPeers) {
      delete ctx;
      return KRON_ERR_INVALID_ARG;
    }
    ctx->rank = rank;
    ctx->gM = rank / GK;
    ctx->gK = rank % GK;
  }
  *out = ctx;
  return KRON_OK;
}

kron_status_t kron_dist_ctx_set(kron_dist_ctx_t *ctx, int32_t option, int32_t value) {
  if (!ctx) return KRON_ERR_INVALID_ARG;
  switch (option) {
    case KRON_DIST_OPT_CHUNKS:
      if (value < 1 || value > 64) return KRON_ERR_INVALID_ARG;
      ctx->nchunks = value;
      return KRON_OK;
    case KRON_DIST_OPT_FUSED_LAYOUT: ctx->fused = value != 0; return KRON_OK;
    case KRON_DIST_OPT_P2P_PUSH: ctx->push = value != 0; return KRON_OK;
  }
  return KRON_ERR_INVALID_ARG;
}

static void p2p_release(kron_dist_ctx_t *ctx) {
  for (int g = 0; g < ctx->GK && g < kMaxPeers; ++g) {
    if (ctx->peer_heap[g] && ctx->peer_heap[g] != ctx->heap) cudaIpcCloseMemHandle(ctx->peer_heap[g]);
    ctx->peer_heap[g] = nullptr;
  }
  if (ctx->heap) cudaFree(ctx->heap);
  ctx->heap = nullptr;
  ctx->heap_bytes = 0;
  ctx->connected = false;
}

kron_status_t kron_dist_ctx_destroy(kron_dist_ctx_t *ctx) {
  if (!ctx) return KRON_OK;
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->comm);
    cudaStreamDestroy(ctx->comm);
  }
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  if (ctx->backend == 0) {
    const NcclApi &api = nccl();
    if (ctx->row_comm) api.CommDestroy(ctx->row_comm);
    if (ctx->world_comm) api.CommDestroy(ctx->world_comm);
  }
  if (ctx->backend == 2) p2p_release(ctx);
  delete ctx;
  return KRON_OK;
}

kron_status_t kron_dist_sync(kron_dist_ctx_t *ctx, void *stream, int32_t timeout_ms) {
  if (!ctx) return KRON_ERR_INVALID_ARG;
  cudaEvent_t done;
  if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess) return KRON_ERR_CUDA;
  if (cudaEventRecord(done, (cudaStream_t)stream) != cudaSuccess) {
    cudaEventDestroy(done);
    return KRON_ERR_CUDA;
  }
  const auto t0 = std::chrono::steady_clock::now();
  kron_status_t st = KRON_OK;
  for (unsigned sleep_us = 10;; sleep_us = std::min(sleep_us * 2, 2000u)) {
    const cudaError_t q = cudaEventQuery(done);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      st = KRON_ERR_CUDA;
      break;
    }
    if ((st = nccl_async_status(ctx)) != KRON_OK) break;
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms >= 0 && ms > timeout_ms) {
      st = ctx->backend == 0 ? KRON_ERR_NCCL : KRON_ERR_CUDA;
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
  }
  if (st == KRON_OK) st = nccl_async_status(ctx);
  if (st == KRON_OK && ctx->backend == 2 && ctx->heap) {
    uint32_t to = 0;
    if (cudaMemcpy(&to, ctx->heap + kP2PTimeoutOff, sizeof(to), cudaMemcpyDeviceToHost) != cudaSuccess) st = KRON_ERR_CUDA;
    else if (to) st = KRON_ERR_CUDA;  // a barrier gave up: the result is not trustworthy
  }
  if (st == KRON_ERR_NCCL && ctx->backend == 0) {
    // a stuck or failed collective: abort the communicators so the stream drains (the context is unusable)
    const NcclApi &api = nccl();
    if (api.CommAbort) {
      if (ctx->row_comm) api.CommAbort(ctx->row_comm);
      if (ctx->world_comm) api.CommAbort(ctx->world_comm);
      ctx->row_comm = ctx->world_comm = nullptr;
    }
  }
  cudaEventDestroy(done);
  return st;
}

kron_status_t kron_dist_p2p_heap_bytes(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                       int32_t GM, int32_t GK, size_t *bytes) {
  if (!bytes) return KRON_ERR_INVALID_ARG;
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  std::vector<int> rounds;
  st = dist_round_plan(M, N, P, Q, GM, GK, &rounds, nullptr);
  if (st != KRON_OK) return st;
  std::vector<int64_t> W(N + 1);
  W[N] = 1;
  for (int i = 0; i < N; ++i) W[N] *= P[i];
  for (int f = N; f >= 1; --f) W[f - 1] = W[f] / P[f - 1] * Q[f - 1];
  int64_t mw = 0;
  int f = N;
  for (int k : rounds) {
    f -= k;
    mw = std::max(mw, W[f] / GK);
  }
  const int64_t half = ((M / GM) * mw * (dtype == KRON_F64 ? 8 : 4) + 255) / 256 * 256;
  *bytes = GK > 1 ? (size_t)(2 * half) : 0;
  return KRON_OK;
}

kron_status_t kron_dist_p2p_reserve(kron_dist_ctx_t *ctx, size_t bytes, void *ipc_handle_out) {
  if (!ctx || ctx->backend != 2 || !ipc_handle_out) return KRON_ERR_INVALID_ARG;
  p2p_release(ctx);
  bytes = (bytes + 511) / 512 * 512;
  if (cudaMalloc(&ctx->heap, kP2PHeader + bytes) != cudaSuccess) {
    cudaGetLastError();
    ctx->heap = nullptr;
    return KRON_ERR_NO_MEMORY;
  }
  cudaIpcMemHandle_t h;
  if (cudaMemset(ctx->heap, 0, kP2PHeader) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
      cudaIpcGetMemHandle(&h, ctx->heap) != cudaSuccess) {
    cudaGetLastError();
    p2p_release(ctx);
    return KRON_ERR_CUDA;
  }
  memcpy(ipc_handle_out, &h, sizeof(h));
  ctx->heap_bytes = bytes;
  ctx->epoch = 0;
  ctx->parity = 0;
  return KRON_OK;
}

kron_status_t kron_dist_p2p_connect(kron_dist_ctx_t *ctx, const void *ipc_handles) {
  if (!ctx || ctx->backend != 2 || !ctx->heap || !ipc_handles) return KRON_ERR_INVALID_ARG;
  for (int g = 0; g < ctx->GK; ++g) {
    if (g == ctx->gK) {
      ctx->peer_heap[g] = ctx->heap;
      continue;
    }
    if (ctx->peer_heap[g]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char *>(ipc_handles) + (size_t)(ctx->gM * ctx->GK + g) * sizeof(h), sizeof(h));
    void *p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return KRON_ERR_CUDA;
    }
    ctx->peer_heap[g] = static_cast<char *>(p);
  }
  ctx->connected = true;
  return KRON_OK;
}

kron_status_t kron_dist_p2p_timeouts(kron_dist_ctx_t *ctx, uint32_t *count) {
  if (!ctx || ctx->backend != 2 || !count) return KRON_ERR_INVALID_ARG;
  *count = 0;
  if (!ctx->heap) return KRON_OK;
  if (cudaMemcpy(count, ctx->heap + kP2PTimeoutOff, sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return KRON_ERR_CUDA;
  return KRON_OK;
}

kron_status_t kron_dist_ctx_grid(const kron_dist_ctx_t *ctx, int32_t *GM, int32_t *GK) {
  if (!ctx || !GM || !GK) return KRON_ERR_INVALID_ARG;
  *GM = ctx->GM;
  *GK = ctx->GK;
  return KRON_OK;
}

kron_status_t kron_dist_round_info(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                   const kron_dist_ctx_t *ctx, int32_t cap, int32_t *nrounds, int32_t *fused_send,
                                   int32_t *fused_recv) {
  if (!ctx || !nrounds) return KRON_ERR_INVALID_ARG;
  std::vector<int> rounds;
  kron_status_t st = dist_round_plan(M, N, P, Q, ctx->GM, ctx->GK, &rounds, nullptr);
  if (st != KRON_OK) return st;
  *nrounds = (int32_t)rounds.size();
  const int GK = ctx->GK;
  std::vector<int64_t> W(N + 1);
  W[N] = 1;
  for (int i = 0; i < N; ++i) W[N] *= P[i];
  for (int f = N; f >= 1; --f) W[f - 1] = W[f] / P[f - 1] * Q[f - 1];
  const int64_t Ml = M / ctx->GM, nc = std::max<int64_t>(1, std::min<int64_t>(ctx->nchunks, Ml));
  const int64_t rows = (Ml + nc - 1) / nc;
  int f = N;
  int64_t prev_rho = 0;
  for (int j = 0; j < (int)rounds.size(); ++j) {
    const int k = rounds[j];
    int64_t C = 1;
    for (int i = 0; i < k; ++i) C *= P[f - 1 - i];
    const int64_t wl_in = W[f] / GK, wl_out = W[f - k] / GK;
    Plan plan;
    st = make_plan(std::max<int64_t>(rows, 1), k, P + (f - k), Q + (f - k), (int)dtype, &plan, wl_in / C);
    if (st != KRON_OK) return st;
    PushArgs pa;
    pa.B = pa.rho = pa.wd = wl_out / GK;
    pa.GK = 1;
    pa.on = 1;
    InRemap ri;
    ri.rho = prev_rho;
    ri.GK = GK;
    ri.on = 1;
    if (j < cap) {
      if (fused_send) fused_send[j] = GK > 1 && GK <= kMaxPush && ctx->fused && ctx->backend != 2 && plan_push_ok(plan, pa);
      if (fused_recv) fused_recv[j] = GK > 1 && j > 0 && ctx->fused && ctx->backend != 2 && plan_remap_ok(plan, ri);
    }
    prev_rho = wl_in / C;
    f -= k;
  }
  return KRON_OK;
}

kron_status_t kron_dist_round_layouts(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                      const kron_dist_ctx_t *ctx, int32_t cap, int32_t *nrounds, int32_t *layout) {
  if (!ctx || !nrounds || (cap > 0 && !layout)) return KRON_ERR_INVALID_ARG;
  std::vector<int32_t> fs(64), fr(64);
  kron_status_t st = kron_dist_round_info(M, N, P, Q, dtype, ctx, 64, nrounds, fs.data(), fr.data());
  if (st != KRON_OK) return st;
  std::vector<int> rounds;
  if ((st = dist_round_plan(M, N, P, Q, ctx->GM, ctx->GK, &rounds, nullptr)) != KRON_OK) return st;
  bool tm = false;
  if (rounds.size() == 2 && ctx->GK > 1) {
    // the same check kron_matmul_dist makes, on the plans of the full and the ragged row chunk
    const int GK = ctx->GK;
    std::vector<int64_t> W(N + 1);
    W[N] = 1;
    for (int i = 0; i < N; ++i) W[N] *= P[i];
    for (int f = N; f >= 1; --f) W[f - 1] = W[f] / P[f - 1] * Q[f - 1];
    const int64_t Ml = M / ctx->GM, nc = std::max<int64_t>(1, std::min<int64_t>(ctx->nchunks, Ml));
    const int64_t rows0 = (Ml + nc - 1) / nc, nchunk = (Ml + rows0 - 1) / rows0, rows_last = Ml - (nchunk - 1) * rows0;
    Plan pl[2][2];
    int64_t wl[2];
    int f = N;
    for (int j = 0; j < 2 && st == KRON_OK; ++j) {
      const int k = rounds[j];
      int64_t C = 1;
      for (int i = 0; i < k; ++i) C *= P[f - 1 - i];
      wl[j] = W[f] / GK;
      for (int v = 0; v < 2 && st == KRON_OK; ++v)
        st = make_plan(std::max<int64_t>(v == 0 ? rows0 : rows_last, 1), k, P + (f - k), Q + (f - k), (int)dtype,
                       &pl[j][v], wl[j] / C);
      f -= k;
    }
    if (st != KRON_OK) return st;
    const Plan *const pls[2][2] = {{&pl[0][0], &pl[0][1]}, {&pl[1][0], &pl[1][1]}};
    tm = tile_major_rounds((int)dtype, N, P, Q, GK, rounds, pls, wl, ctx->fused, ctx->backend == 2);
  }
  for (int j = 0; j < *nrounds && j < cap; ++j) layout[j] = tm ? 2 : (fs[j] || fr[j]) ? 1 : 0;
  return KRON_OK;
}

}  // extern "C"

namespace kron {
namespace {

// ---- backend 2: P2P rounds (NEXT-1).  Returns the status; `bufs0` = this rank's scratch.
kron_status_t dist_p2p(kron_dist_ctx_t *ctx, const std::vector<int> &rounds, std::vector<RoundPlan> &rp, int dtype,
                       const void *X, const void *const *F, void *Y, RankBufs &b, size_t half, int64_t Ml,
                       cudaStream_t s) {
  const int GK = ctx->GK;
  kron_status_t st = KRON_OK;
  PeerPtrs heaps{};
  for (int g = 0; g < GK; ++g) heaps.p[g] = ctx->peer_heap[g];
  auto barrier = [&]() {
    const unsigned long long ep = ++ctx->epoch;
    p2p_barrier_kernel<<<1, 64, 0, s>>>(heaps, reinterpret_cast<unsigned long long *>(ctx->heap), GK, ctx->gK, ep,
                                        reinterpret_cast<unsigned *>(ctx->heap + kP2PTimeoutOff),
                                        (long long)20 * 1000 * 1000 * 1000);
    return cudaGetLastError() == cudaSuccess;
  };
  int in_half = -1;  // heap half holding this round's input block (after a push round), else -1
  for (size_t j = 0; j < rounds.size() && st == KRON_OK; ++j) {
    const RoundPlan &R = rp[j];
    const Plan &plan = R.plan[0];
    const void *const *Fj = F + (R.first - R.k);
    const bool last = j + 1 == rounds.size();
    const int64_t B = R.wl_out / GK;  // values per row sent to each peer
    // this round writes the heap half its input does not occupy
    const int out_half = in_half >= 0 ? 1 - in_half : (int)ctx->parity;
    const size_t off = kP2PHeader + (size_t)out_half * half;
    const void *in = j == 0 ? X : (in_half >= 0 ? (const void *)(ctx->heap + kP2PHeader + (size_t)in_half * half)
                                                : (const void *)b.cur);
    ctx->parity = 1u - (unsigned)out_half;
    PushArgs pa;
    for (int g = 0; g < GK; ++g) pa.dst[g] = ctx->peer_heap[g] + off;
    pa.B = B;
    pa.rho = R.rho;
    pa.wd = R.wl_out;
    pa.GK = GK;
    pa.me = ctx->gK;
    pa.on = 1;
    if (!last && ctx->push && GK <= kMaxPush && plan_push_ok(plan, pa)) {
      // FUSED exchange: the round's last pass stores every value straight into its StoreGPUTile position
      // in the destination rank's heap half (peer memory over NVLink), so the transfer overlaps the
      // arithmetic tile by tile.  The passes before it run first — their intermediates may live in this
      // rank's own heap half, which no peer writes before this rank reaches the barrier — then a barrier
      // (every peer is done with the half it is about to receive) and the pushing pass, then a barrier
      // (every value addressed to this rank has landed).
      const int np = (int)plan.passes.size();
      if (np > 1 && (st = plan_run(plan, in, Fj, ctx->heap + off, b.ws, s, nullptr, nullptr, 0, np - 1)) != KRON_OK)
        break;
      if (!barrier()) { st = KRON_ERR_CUDA; break; }
      if ((st = plan_run(plan, in, Fj, ctx->heap + off, b.ws, s, &pa, nullptr, np - 1, np)) != KRON_OK) break;
      if (!barrier()) { st = KRON_ERR_CUDA; break; }
      in_half = out_half;  // the next round reads its block from this rank's own heap half
      continue;
    }
    // lines 670-674 into this rank's heap half, barrier, then lines 676-690 + 685 as one pull kernel
    if ((st = plan_run(plan, in, Fj, ctx->heap + off, b.ws, s)) != KRON_OK) break;
    PeerPtrs outs{};
    for (int g = 0; g < GK; ++g) outs.p[g] = ctx->peer_heap[g] + off;
    if (!barrier()) { st = KRON_ERR_CUDA; break; }
    void *dst = last ? Y : b.cur;
    if (launch_p2p_pull(dtype, outs, dst, Ml, R.wl_out, R.rho, GK, ctx->gK, s) != 0) st = KRON_ERR_CUDA;
    in_half = -1;
  }
  return st;
}

}  // namespace
}  // namespace kron

extern "C" {

kron_status_t kron_matmul_dist(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X_local,
                               const void *const *F, void *Y_local, kron_dtype_t dtype, kron_dist_ctx_t *ctx,
                               void *stream) {
  if (!ctx) return KRON_ERR_INVALID_ARG;
  kron_status_t st = validate(M, N, P, Q, (int)dtype);
  if (st != KRON_OK) return st;
  if (dtype == KRON_F32_3XTF32) return KRON_ERR_UNSUPPORTED;  // the distributed path is fp32 / fp64 only
  const int GM = ctx->GM, GK = ctx->GK;
  std::vector<int> rounds;
  st = dist_round_plan(M, N, P, Q, GM, GK, &rounds, nullptr);
  if (st != KRON_OK) return st;
  if (M == 0) return KRON_OK;
  if (!X_local || !F || !Y_local) return KRON_ERR_INVALID_ARG;
  for (int i = 0; i < N; ++i)
    if (!F[i]) return KRON_ERR_INVALID_ARG;
  const int nranks = ctx->backend == 1 ? GM * GK : 1;
  const void *const *Xv = ctx->backend == 1 ? static_cast<const void *const *>(X_local) : &X_local;
  void *const *Yv = ctx->backend == 1 ? static_cast<void *const *>(Y_local) : &Y_local;
  for (int r = 0; r < nranks; ++r)
    if (!Xv[r] || !Yv[r]) return KRON_ERR_INVALID_ARG;
  if ((st = nccl_async_status(ctx)) != KRON_OK) return st;  // a collective of an earlier call failed
  if (ctx->backend == 0 && !ctx->row_comm) return KRON_ERR_NCCL;  // aborted by kron_dist_sync

  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_cached();
  const size_t es = dtype == KRON_F32 ? 4 : 8;
  const int64_t Ml = M / GM;
  std::vector<int64_t> W(N + 1);
  W[N] = 1;
  for (int i = 0; i < N; ++i) W[N] *= P[i];
  for (int f = N; f >= 1; --f) W[f - 1] = W[f] / P[f - 1] * Q[f - 1];

  // Row-only grid: every rank is an independent single-GPU Kron-Matmul (no communication).
  if (GK == 1) {
    Plan plan;
    st = make_plan(Ml, N, P, Q, (int)dtype, &plan);
    if (st != KRON_OK) return st;
    const size_t wsb = plan_ws_bytes(plan);
    void *ws = nullptr;
    if (wsb && cudaMallocAsync(&ws, wsb, s) != cudaSuccess) return KRON_ERR_NO_MEMORY;
    for (int r = 0; r < nranks && st == KRON_OK; ++r) st = plan_run(plan, Xv[r], F, Yv[r], ws, stream);
    if (ws) cudaFreeAsync(ws, s);
    return st;
  }

  const bool p2p = ctx->backend == 2;
  // row chunks (backends 0 / 1): chunk c's all-to-all overlaps chunk c+1's local passes (rows are
  // independent); P2P rounds run whole
  const int64_t nc = p2p ? 1 : std::max<int64_t>(1, std::min<int64_t>(ctx->nchunks, Ml));
  const int64_t rows0 = (Ml + nc - 1) / nc, nchunk = (Ml + rows0 - 1) / rows0, rows_last = Ml - (nchunk - 1) * rows0;

  // local plans per round (identical on every rank: shape-only)
  std::vector<RoundPlan> rp(rounds.size());
  int64_t max_w = 0;
  size_t ws_max = 0;
  bool need_cur = false, need_out = false;
  {
    int f = N;
    for (size_t j = 0; j < rounds.size(); ++j) {
      RoundPlan &R = rp[j];
      R.k = rounds[j];
      int64_t C = 1;
      for (int i = 0; i < R.k; ++i) C *= P[f - 1 - i];
      R.first = f;
      R.wl_in = W[f] / GK;
      R.wl_out = W[f - R.k] / GK;
      R.rho = R.wl_in / C;
      // factors f-k+1 .. f (most significant first) on the local block with lead = wl_in / C
      for (int v = 0; v < 2; ++v) {
        st = make_plan(v == 0 ? rows0 : rows_last, R.k, P + (f - R.k), Q + (f - R.k), (int)dtype, &R.plan[v],
                       R.wl_in / C);
        if (st != KRON_OK) return st;
        ws_max = std::max(ws_max, plan_ws_bytes(R.plan[v]));
      }
      if (!p2p && ctx->fused) {
        PushArgs pa;
        pa.B = pa.rho = pa.wd = R.wl_out / GK;
        pa.GK = 1;
        pa.on = 1;
        InRemap ri;
        ri.rho = j > 0 ? rp[j - 1].rho : 0;
        ri.GK = GK;
        ri.on = 1;
        R.fpush = GK <= kMaxPush && plan_push_ok(R.plan[0], pa) && plan_push_ok(R.plan[1], pa);
        R.fremap = j > 0 && plan_remap_ok(R.plan[0], ri) && plan_remap_ok(R.plan[1], ri);
      }
      need_out |= !R.fpush;
      need_cur |= j > 0 && !R.fremap;
      max_w = std::max(max_w, std::max(R.wl_in, R.wl_out));
      f -= R.k;
    }
    bool tm = false;
    if (rounds.size() == 2) {
      const Plan *const pls[2][2] = {{&rp[0].plan[0], &rp[0].plan[1]}, {&rp[1].plan[0], &rp[1].plan[1]}};
      const int64_t wl[2] = {rp[0].wl_in, rp[1].wl_in};
      tm = tile_major_rounds((int)dtype, N, P, Q, GK, rounds, pls, wl, ctx->fused, p2p);
    }
    if (tm) {
      rp[0].tm = 1;
      rp[1].tm = 2;
      need_out = false;
      need_cur = false;
    }
  }
  const size_t buf_bytes = (size_t)Ml * max_w * es;
  size_t half = 0;
  if (p2p) {
    // the round outputs live in the symmetric heap (two halves); see kron_dist_p2p_heap_bytes
    size_t need = 0;
    st = kron_dist_p2p_heap_bytes(M, N, P, Q, dtype, GM, GK, &need);
    if (st != KRON_OK) return st;
    if (!ctx->connected) return KRON_ERR_INVALID_ARG;
    if (need > ctx->heap_bytes) return KRON_ERR_NO_MEMORY;
    half = need / 2;
    need_cur = true;
    need_out = false;
  }
  std::vector<RankBufs> bufs(nranks);
  bool oom = false;
  for (int r = 0; r < nranks; ++r) {
    if (need_cur) oom |= cudaMallocAsync(&bufs[r].cur, buf_bytes, s) != cudaSuccess;
    if (!p2p) {
      if (need_out) oom |= cudaMallocAsync(&bufs[r].out, buf_bytes, s) != cudaSuccess;
      oom |= cudaMallocAsync(&bufs[r].send, buf_bytes, s) != cudaSuccess;
      oom |= cudaMallocAsync(&bufs[r].recv, buf_bytes, s) != cudaSuccess;
    }
    if (ws_max) oom |= cudaMallocAsync(&bufs[r].ws, ws_max, s) != cudaSuccess;
  }
  auto free_all = [&] {
    for (auto &b : bufs)
      for (void *p : {b.cur, b.out, b.send, b.recv, b.ws})
        if (p) cudaFreeAsync(p, s);
  };
  if (oom) {
    cudaGetLastError();
    free_all();
    return KRON_ERR_NO_MEMORY;
  }
  if (p2p) {
    st = dist_p2p(ctx, rounds, rp, (int)dtype, Xv[0], F, Yv[0], bufs[0], half, Ml, s);
    free_all();
    return st;
  }

  // ---- backends 0 (NCCL) and 1 (virtual): per round and row chunk
  //   lines 670-674: local passes; the last one writes the destination-major send block send[d][rows][B]
  //                  (fused pack) or the plain block + a pack kernel
  //   lines 676-692: one all-to-all within the row group (NCCL on the context's comm stream, overlapping the
  //                  next chunk's passes; virtual: device copies)
  //   line 685:      StoreGPUTile — done by the next round's first pass through the remapped tensor map
  //                  (fused), else by a kernel into the next round's block; after the last round into Y_local
  const bool nccl_be = ctx->backend == 0;
  cudaStream_t sc = s;
  cudaEvent_t *ev = nullptr;
  if (nccl_be) {
    if (!ctx->comm && cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking) != cudaSuccess) st = KRON_ERR_CUDA;
    while (st == KRON_OK && ctx->ev.size() < (size_t)(1 + 2 * nchunk)) {
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) st = KRON_ERR_CUDA;
      else ctx->ev.push_back(e);
    }
    if (st != KRON_OK) {
      free_all();
      return st;
    }
    sc = ctx->comm;
    ev = ctx->ev.data();
    // the comm stream starts after the caller's prior work and the stream-ordered allocations
    if (cudaEventRecord(ev[0], s) != cudaSuccess || cudaStreamWaitEvent(sc, ev[0], 0) != cudaSuccess) st = KRON_ERR_CUDA;
  }
  const int64_t Kl = W[N] / GK, Ll = W[0] / GK;
  for (size_t j = 0; j < rounds.size() && st == KRON_OK; ++j) {
    const RoundPlan &R = rp[j];
    const void *const *Fj = F + (R.first - R.k);
    const int64_t B = R.wl_out / GK;
    for (int64_t c = 0; c < nchunk && st == KRON_OK; ++c) {
      const int64_t r0 = c * rows0, rows = c + 1 < nchunk ? rows0 : rows_last;
      const Plan &plan = R.plan[c + 1 < nchunk ? 0 : 1];
      const size_t blk = (size_t)rows * B;  // values per peer
      if (j > 0 && nccl_be && cudaStreamWaitEvent(s, ev[2 + 2 * c], 0) != cudaSuccess) st = KRON_ERR_CUDA;
      for (int r = 0; r < nranks && st == KRON_OK; ++r) {
        RankBufs &b = bufs[r];
        if (R.tm) {
          // v11 rounds: one kernel each, exchange layouts written / read by the kernels themselves
          PassPlan pp = plan.passes[0];
          const void *grp[kMaxFused];
          for (int k = 0; k < pp.nf; ++k) grp[k] = Fj[pp.first - 1 - k];
          char *send = at(b.send, r0 * R.wl_out, es);
          PushArgs pa;
          for (int d = 0; d < GK; ++d) pa.dst[d] = send + (size_t)d * blk * es;
          pa.B = pa.rho = R.tm == 1 ? pp.Qc / GK : B;
          pa.wd = pa.B;
          pa.GK = 1;
          pa.me = 0;
          pa.on = 1;
          InRemap ri;
          int err;
          if (R.tm == 1) {
            pp.tm_out = 1;
            err = launch_fused(pp, (int)dtype, rows, at(Xv[r], r0 * Kl, es), send, grp, s, &pa, nullptr);
          } else {
            pp.tm_in = 1;
            ri.rho = rp[j - 1].rho;
            ri.GK = GK;
            ri.on = 1;
            err = launch_fused(pp, (int)dtype, rows, at(b.recv, r0 * R.wl_in, es), send, grp, s, &pa, &ri);
          }
          if (err != 0) st = KRON_ERR_CUDA;
          continue;
        }
        // this chunk's input: X, the previous round's receive block (remapped view) or its StoreGPUTile copy
        const void *in;
        InRemap ri;
        if (j == 0) {
          in = at(Xv[r], r0 * Kl, es);
        } else if (R.fremap) {
          in = at(b.recv, r0 * R.wl_in, es);
          ri.rho = rp[j - 1].rho;
          ri.GK = GK;
          ri.on = 1;
        } else {
          void *cur = at(b.cur, r0 * R.wl_in, es);
          if (launch_store_gpu_tile((int)dtype, at(b.recv, r0 * R.wl_in, es), cur, rows, R.wl_in, rp[j - 1].rho, GK,
                                    s) != 0) {
            st = KRON_ERR_CUDA;
            break;
          }
          in = cur;
        }
        char *send = at(b.send, r0 * R.wl_out, es);
        if (R.fpush) {
          PushArgs pa;
          for (int d = 0; d < GK; ++d) pa.dst[d] = send + (size_t)d * blk * es;
          pa.B = pa.rho = pa.wd = B;
          pa.GK = 1;
          pa.me = 0;
          pa.on = 1;
          // intermediates (if any) ping-pong through ws and this chunk's receive block region is not touched;
          // Y of the plan (never written by a pushing last pass) is the send block itself
          st = plan_run(plan, in, Fj, send, b.ws, s, &pa, R.fremap ? &ri : nullptr);
        } else {
          void *outb = at(b.out, r0 * R.wl_out, es);
          st = plan_run(plan, in, Fj, outb, b.ws, s, nullptr, R.fremap ? &ri : nullptr);
          if (st == KRON_OK && launch_pack((int)dtype, outb, send, rows, R.wl_out, B, s) != 0) st = KRON_ERR_CUDA;
        }
      }
      if (st != KRON_OK) break;
      if (nccl_be) {
        if (cudaEventRecord(ev[1 + 2 * c], s) != cudaSuccess || cudaStreamWaitEvent(sc, ev[1 + 2 * c], 0) != cudaSuccess) {
          st = KRON_ERR_CUDA;
          break;
        }
        st = exchange_nccl(ctx, (int)dtype, at(bufs[0].send, r0 * R.wl_out, es), at(bufs[0].recv, r0 * R.wl_out, es),
                           blk, sc);
        if (st == KRON_OK && cudaEventRecord(ev[2 + 2 * c], sc) != cudaSuccess) st = KRON_ERR_CUDA;
      } else {
        for (int gm = 0; gm < GM && st == KRON_OK; ++gm)
          for (int src = 0; src < GK; ++src)
            for (int dst = 0; dst < GK; ++dst) {
              const int rs = gm * GK + src, rd = gm * GK + dst;
              if (cudaMemcpyAsync(at(bufs[rd].recv, r0 * R.wl_out + (int64_t)src * (int64_t)blk, es),
                                  at(bufs[rs].send, r0 * R.wl_out + (int64_t)dst * (int64_t)blk, es), blk * es,
                                  cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                st = KRON_ERR_CUDA;
            }
      }
    }
  }
  // line 685 after the last round: StoreGPUTile into Y_local (natural column block gK*L/GK ...)
  const RoundPlan &RL = rp.back();
  for (int64_t c = 0; c < nchunk && st == KRON_OK; ++c) {
    const int64_t r0 = c * rows0, rows = c + 1 < nchunk ? rows0 : rows_last;
    if (nccl_be && cudaStreamWaitEvent(s, ev[2 + 2 * c], 0) != cudaSuccess) st = KRON_ERR_CUDA;
    for (int r = 0; r < nranks && st == KRON_OK; ++r)
      if (launch_store_gpu_tile((int)dtype, at(bufs[r].recv, r0 * RL.wl_out, es), at(Yv[r], r0 * Ll, es), rows,
                                RL.wl_out, RL.rho, GK, s) != 0)
        st = KRON_ERR_CUDA;
  }
  if (st != KRON_OK && nccl_be) {
    // keep the buffers alive until whatever was enqueued on the comm stream has finished
    for (int64_t c = 0; c < nchunk; ++c) cudaStreamWaitEvent(s, ev[2 + 2 * c], 0);
  }
  free_all();
  return st;
}

}  // extern "C"
