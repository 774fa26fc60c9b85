/* include/kron.h — C-ABI of libkron, the B200 (sm_100a) Kron-Matmul library.
 *
 * Operation ("Kron-Matmul"):
 *     Y[M x prod_i Q_i] = X[M x prod_i P_i] . (F^1 (x) F^2 (x) ... (x) F^N)
 * computed as one sliced multiply per factor, F^N first (Algorithm 1):
 *     T'[m, q*(W/P) + s] = sum_p T[m, s*P + p] * F[p, q]           (W = width of T)
 * with consecutive factors fused in shared memory and results stored directly at
 * their next-iteration positions, so no transpose ever runs.
 *
 * Conventions shared by every entry point
 *   Layout     all matrices dense, row-major, leading dimension = column count, same dtype.
 *   Factors    P[i], Q[i] (host arrays, length N) give F[i] = F^{i+1} as a P[i] x Q[i] matrix;
 *              F[0] = F^1 is the MOST significant factor of the Kronecker product.
 *              F is a host array of N device pointers.
 *   Pointers   X, F[i], Y, workspace, X_local, Y_local are DEVICE pointers on the current device.
 *   Ownership  the caller owns X, F and Y.  X and F are read-only; Y is write-only and must not
 *              overlap X or any F[i].  kron_matmul() allocates its workspace stream-ordered
 *              (cudaMallocAsync on `stream`) and frees it stream-ordered; kron_matmul_ws() uses
 *              caller memory instead.
 *   Streams    `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *              work is enqueued on it; the call returns without synchronising.
 *   Errors     argument / shape problems are reported synchronously, BEFORE any work is
 *              enqueued.  Kernel faults are asynchronous (CUDA semantics) and surface at the
 *              next synchronising call.  The library never aborts and never prints.
 *   M = 0      a successful no-op.
 *   Threads    reentrant and thread-safe across distinct streams (the plan cache is locked).
 */
#ifndef KRON_H_
#define KRON_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* KRON_F32_3XTF32: fp32 data (same layout and buffers as KRON_F32) computed in the separately reported
 * 3xTF32 tensor-core mode: P = 32 factor pairs run on the warp MMA with the
 * split x = hi + lo per operand (~22-bit products, fp32 accumulation); every other pass uses the fp32
 * CUDA-core kernels.  Not the default: KRON_F32 is the reference fp32 arithmetic. */
typedef enum { KRON_F32 = 0, KRON_F64 = 1, KRON_F32_3XTF32 = 2, KRON_F32_TF32 = 3 } kron_dtype_t;

typedef enum {
  KRON_OK = 0,
  KRON_ERR_INVALID_ARG = 1, /* null pointer, N < 1, P_i < 1, Q_i < 1, bad dtype, M < 0, bad grid  */
  KRON_ERR_SHAPE = 2,       /* prod P or prod Q overflows int64 / exceeds addressable memory, or  */
                            /* a caller buffer (workspace) is too small                           */
  KRON_ERR_UNSUPPORTED = 3, /* no kernel for this configuration (not returned for valid shapes)   */
  KRON_ERR_NO_MEMORY = 4,   /* workspace allocation failed                                        */
  KRON_ERR_CUDA = 5,        /* a CUDA launch / API call failed                                    */
  KRON_ERR_NCCL = 6,        /* NCCL unavailable or an NCCL call failed (distributed path)         */
  KRON_ERR_DIST_LAYOUT = 7  /* distributed shape does not partition: GM !| M, GK !| K or L, or no */
                            /* legal round plan exists                                            */
} kron_status_t;

/* Human-readable name of a status code (static storage; never NULL). */
const char *kron_status_string(kron_status_t s);

/* Detail of the most recent KRON_ERR_CUDA / KRON_ERR_NCCL returned on the calling thread (the CUDA or
 * NCCL error name and the failing step), or "" if none.  Thread-local static storage.            */
const char *kron_last_error_detail(void);

/* ---------------------------------------------------------------------------------------------
 * Single GPU — Algorithm 1 + fusion.
 *
 * kron_matmul: Y = X . (F^1 (x) ... (x) F^N).  M >= 0, N >= 1, P[i], Q[i] >= 1.
 * The library plans the factor passes (cached per (device, M, shapes, dtype)), reserves its
 * workspace stream-ordered on `stream`, and enqueues one kernel per pass.                      */
kron_status_t kron_matmul(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                          const void *const *F, void *Y, kron_dtype_t dtype, void *stream);

/* Bytes of workspace kron_matmul_ws() needs for this problem (0 when none). */
kron_status_t kron_matmul_workspace_size(int64_t M, int32_t N, const int32_t *P, const int32_t *Q,
                                         kron_dtype_t dtype, size_t *bytes);

/* kron_matmul with a caller-owned device workspace of `workspace_bytes` bytes (>= the size
 * above; KRON_ERR_SHAPE otherwise).  The workspace must not overlap X, F or Y.               */
kron_status_t kron_matmul_ws(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                             const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                             size_t workspace_bytes, void *stream);

/* kron_matmul_ws with per-pass timing hooks (used by bench.py's roofline): events[i] (cudaEvent_t
 * handles passed as void*) is recorded on `stream` right before pass i is launched and
 * events[npasses] after the last pass; nevents must be >= npasses + 1 (KRON_ERR_INVALID_ARG).     */
kron_status_t kron_matmul_ws_events(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                                    const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                                    size_t workspace_bytes, void *const *events, int32_t nevents, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Planner introspection (host only; no GPU needed).  Describes the pass plan kron_matmul uses:
 * pass i applies factors F^{first[i]}, F^{first[i]-1}, ..., F^{first[i]-nfactors[i]+1}
 * (1-based, processing order N -> 1) with kernel family kind[i] (0 generic, 1 fused small-P,
 * 2 GEMM-style large-P).  Arrays have room for `cap` passes; *npasses receives the count.     */
kron_status_t kron_plan_describe(int64_t M, int32_t N, const int32_t *P, const int32_t *Q,
                                 kron_dtype_t dtype, int32_t cap, int32_t *npasses, int32_t *first,
                                 int32_t *nfactors, int32_t *kind);

/* Host-buffer Kron-Matmul (the end-to-end path): X, F[i] and Y are HOST pointers (page-locked memory
 * strongly recommended: pageable memory makes the copies synchronous).  Rows are independent
 * (Algorithm 1), so the call streams chunks of `chunk_rows` rows (0 = ~64 MB per chunk) through
 * two device slots: the host->device copy of chunk c+1, the passes of chunk c and the device->host copy
 * of chunk c-1 overlap on two internal copy streams and `stream`.  Device memory (factors, two slots,
 * workspace) is allocated and freed stream-ordered.  Everything is ordered after prior work on `stream`
 * and `stream` completes with the last copy; the call returns without synchronising (Y is valid after
 * the stream synchronises).  Errors as kron_matmul; chunk_rows < 0 -> KRON_ERR_INVALID_ARG. */
kron_status_t kron_matmul_host(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                               const void *const *F, void *Y, kron_dtype_t dtype, int64_t chunk_rows,
                               void *stream);

/* CUDA-graph form of kron_matmul_ws for repeated calls on the same buffers (small, launch-bound
 * problems: the paper's Table 4 shapes).  kron_graph_create captures the plan's kernel launches for
 * these exact device pointers (X, F[i], Y, workspace; contents may change between launches, the
 * pointers may not) into an instantiated graph; kron_graph_launch enqueues one Kron-Matmul on `stream`
 * at graph-replay cost; kron_graph_destroy frees it.  Same argument rules as kron_matmul_ws; M = 0 is
 * KRON_ERR_INVALID_ARG here (nothing to capture).  The graph owns no device memory. */
typedef struct kron_graph_s kron_graph_t;
kron_status_t kron_graph_create(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                                const void *const *F, void *Y, kron_dtype_t dtype, void *workspace,
                                size_t workspace_bytes, kron_graph_t **graph);
kron_status_t kron_graph_launch(kron_graph_t *graph, void *stream);
kron_status_t kron_graph_destroy(kron_graph_t *graph);

/* Autotuning ("performs auto-tuning over a range of tile size parameter values for the
 * given shape ... find the kernel with the least execution time").  Candidate plans (fusion group
 * caps x kernel-family choices x fp64 DMMA on/off x tile-major hand-off on/off x chain tile sizes;
 * duplicates removed) are each run once untimed, then timed run by run between CUDA events on `stream`
 * with the caller's X, F and Y (Y receives the correct result) in two sweeps over the candidates
 * (forward, then reverse), `reps` runs each; a candidate's time is its fastest run, and it replaces the
 * static plan only when more than 2% faster.  The winner is installed in the plan cache for (device,
 * M, shapes, dtype), so subsequent kron_matmul / kron_matmul_ws calls use it.  Synchronous (waits for
 * `stream`).  *ncand receives the number of distinct candidates and *best_ms the winner's time (both
 * optional).                                                                                      */
kron_status_t kron_autotune(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X,
                            const void *const *F, void *Y, kron_dtype_t dtype, int32_t reps, void *stream,
                            int32_t *ncand, float *best_ms);

/* Number of distinct candidate plans kron_autotune would time for this problem (host only). */
kron_status_t kron_autotune_candidates(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                       int32_t *ncand);

/* Drop every cached (static or autotuned) plan. */
kron_status_t kron_plan_cache_clear(void);

/* Kernel (family) that runs pass `pass` of the plan kron_matmul uses, as a NUL-terminated name in
 * name[0..len) (e.g. "kron_fused_pipe_kernel", "kron_dmma_kernel").  Host only. */
kron_status_t kron_plan_kernel(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                               int32_t pass, char *name, int32_t len);

/* Algorithmic HBM bytes and FLOPs of the plan:
 *   bytes = sum_passes s*M*(W_in + W_out) + sum_f s*P_f*Q_f,   flops = sum_f 2*M*W_f*Q_f.      */
kron_status_t kron_plan_cost(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                             double *hbm_bytes, double *flops);

/* ---------------------------------------------------------------------------------------------
 * Distributed — Algorithm 2 on a {GM, GK} grid of ranks (one process per GPU).
 *
 * Rank r has grid coordinates {gM, gK} = {r / GK, r % GK}.  It holds
 *     X_local = X[gM*M/GM : +M/GM][gK*K/GK : +K/GK]          (M/GM x K/GK, row-major)
 * and receives
 *     Y_local = Y[gM*M/GM : +M/GM][gK*L/GK : +L/GK]          (M/GM x L/GK, row-major).
 * Factors are replicated on every rank.  Each round performs as many sliced multiplies
 * as the local column block allows and then ONE all-to-all among the GK ranks of
 * the row group regroups the slices (lines 676-692; reading G13).
 *
 * Context creation.  `backend` selects the exchange:
 *     0  NCCL: `nccl_unique_id` points to the 128-byte ncclUniqueId created by rank 0 and
 *        broadcast by the caller (e.g. over a torch ProcessGroup); world_size = GM*GK ranks,
 *        one per GPU; `rank` is this process's rank.  The row-group communicator is
 *        ncclCommSplit(world, color = gM, key = gK).  Per round and per row chunk (rows are
 *        independent): the local passes, whose LAST pass writes the destination-major
 *        send block send[d][rows][W'/GK] directly from its epilogue where the kernel has one (the
 *        fp32 16x16 cluster kernel and the fp32 16x16 / 32x32 chunk-pair kernels; else a pack
 *        kernel); ONE ncclAlltoAll on the context's own stream, so chunk c's exchange overlaps chunk
 *        c+1's passes; and StoreGPUTile (line 685), which the NEXT round's first pass performs
 *        itself by reading the receive buffer through a 5-D tensor map in StoreGPUTile order (any
 *        fused kernel but the 64x32 pair; else a remap kernel).  After the last round one remap
 *        kernel writes Y_local.  Every value crosses HBM once per round at the source and once at the
 *        destination besides the local passes' own traffic.
 *     1  virtual: ONE process drives all GM*GK ranks on the current device; the exchange is a
 *        device-to-device copy (used to test the distributed data path on a single GPU) and the
 *        rounds use exactly backend 0's buffers, chunks, fused send / receive layouts and kernels.
 *        nccl_unique_id and rank are ignored.
 *     2  P2P (peer memory, "a single CUDA kernel ... when GPUs support P2P"): one rank per
 *        process (`rank` = this process's rank, nccl_unique_id ignored).  Before the first call the
 *        ranks reserve a symmetric heap (kron_dist_p2p_reserve), exchange its 64-byte CUDA IPC
 *        handles (e.g. all_gather over a torch ProcessGroup) and map the row-group peers' heaps
 *        (kron_dist_p2p_connect).  A round whose last local pass is the fp32 16x16 cluster kernel or
 *        an fp32 16x16 / 32x32 chunk-pair kernel (and that is not the last round) FUSES the exchange
 *        into that pass: its store warps write every value straight into its StoreGPUTile position
 *        in the destination rank's heap (peer stores over NVLink / NVSwitch), between two
 *        device-side flag barriers (the round's earlier passes run before the first barrier).  Every
 *        other round writes its local output into this rank's heap, meets the row group at a flag
 *        barrier, and runs ONE pull kernel that reads every value it owns straight from the peers'
 *        heaps into its StoreGPUTile position.  Ranks may share a GPU (IPC within one device), which
 *        is how it is tested on one B200.  Whether rounds push is fixed at context creation
 *        (KRON_P2P_NO_PUSH in the environment then, or kron_dist_ctx_set) so all ranks agree.
 * GM = GK = 0 selects the grid by the paper's rule.                               */
typedef struct kron_dist_ctx kron_dist_ctx_t;

kron_status_t kron_dist_ctx_create(int32_t backend, const void *nccl_unique_id, int32_t world_size,
                                   int32_t rank, int32_t GM, int32_t GK, kron_dist_ctx_t **out);
kron_status_t kron_dist_ctx_destroy(kron_dist_ctx_t *ctx);
/* Context options (host only; set the same value on every rank before the calls that use it):
 *   KRON_DIST_OPT_CHUNKS        row chunks per round, 1..64 (backends 0 / 1; default 2)
 *   KRON_DIST_OPT_FUSED_LAYOUT  0 / 1: fused send / receive layouts (backends 0 / 1; default 1 — 0 forces
 *                               the separate pack and remap kernels, for testing)
 *   KRON_DIST_OPT_P2P_PUSH      0 / 1: backend 2's fused push rounds (default 1 unless KRON_P2P_NO_PUSH
 *                               was set when the context was created)
 * Errors: null ctx, unknown option or value out of range -> KRON_ERR_INVALID_ARG. */
enum { KRON_DIST_OPT_CHUNKS = 1, KRON_DIST_OPT_FUSED_LAYOUT = 2, KRON_DIST_OPT_P2P_PUSH = 3 };
kron_status_t kron_dist_ctx_set(kron_dist_ctx_t *ctx, int32_t option, int32_t value);
/* Wait (host) until `stream` has drained, polling the context's asynchronous errors meanwhile:
 * NCCL (ncclCommGetAsyncError) -> KRON_ERR_NCCL; still not done after timeout_ms (< 0: no bound)
 * -> KRON_ERR_NCCL for backend 0 (its communicators are aborted: the context is unusable) or
 * KRON_ERR_CUDA otherwise; a P2P barrier that gave up (kron_dist_p2p_timeouts) -> KRON_ERR_CUDA.
 * kron_matmul_dist itself never blocks; it returns KRON_ERR_NCCL up front when an earlier
 * collective of the context failed. */
kron_status_t kron_dist_sync(kron_dist_ctx_t *ctx, void *stream, int32_t timeout_ms);
/* Per round (host only, up to `cap`): whether backends 0 / 1 write the send buffer from the last
 * pass (fused_send[j]) and read the receive buffer in place in the first pass (fused_recv[j]). */
kron_status_t kron_dist_round_info(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                   const kron_dist_ctx_t *ctx, int32_t cap, int32_t *nrounds, int32_t *fused_send,
                                   int32_t *fused_recv);
/* Per round (host only, up to `cap`): the exchange layout backends 0 / 1 use — 0 plain block + pack /
 * StoreGPUTile kernels, 1 fused direct-index send / receive layouts (above), 2 the v11 tile-major layouts
 * (config E's rounds [16^3, 16^2]: the triple writes the send blocks tile-major, the pair reads the receive
 * blocks through a 4-D map).  Same errors as kron_dist_round_info. */
kron_status_t kron_dist_round_layouts(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                      const kron_dist_ctx_t *ctx, int32_t cap, int32_t *nrounds, int32_t *layout);
/* Grid actually used by the context. */
kron_status_t kron_dist_ctx_grid(const kron_dist_ctx_t *ctx, int32_t *GM, int32_t *GK);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (rank 0 calls this, then broadcasts it). */
kron_status_t kron_dist_nccl_unique_id(void *out128);

/* Backend 2 (P2P) symmetric heap.
 * kron_dist_p2p_heap_bytes: heap bytes kron_matmul_dist needs for this problem on a {GM,GK} grid
 *   (two halves of M/GM x max round output width / GK elements; 0 when GK = 1).  Host only.
 * kron_dist_p2p_reserve: (re)allocates this rank's heap of `bytes` usable bytes plus a 4 KB header
 *   (barrier flags, timeout word) with cudaMalloc on the current device, zeroes the header, and writes
 *   its cudaIpcMemHandle_t (64 bytes) to `ipc_handle_out`.  Collective in effect: every rank of the
 *   context calls it, and no rank may still be using the previous heaps (synchronize + barrier first).
 *   Errors: wrong backend / null -> KRON_ERR_INVALID_ARG; allocation -> KRON_ERR_NO_MEMORY;
 *   IPC export -> KRON_ERR_CUDA.
 * kron_dist_p2p_connect: `ipc_handles` = world_size x 64 bytes in rank order (all ranks' handles);
 *   opens the heaps of this rank's row-group peers (cudaIpcOpenMemHandle, lazy peer access).
 *   Errors: no heap reserved -> KRON_ERR_INVALID_ARG; IPC open failure -> KRON_ERR_CUDA.
 * kron_matmul_dist on backend 2 returns KRON_ERR_INVALID_ARG before connect and KRON_ERR_NO_MEMORY
 *   when the heap is smaller than kron_dist_p2p_heap_bytes.  Calls on one context must be issued in
 *   stream order on each rank (heap halves and barrier epochs continue across calls).
 * kron_dist_p2p_timeouts: synchronously reads how many barrier waits gave up (~20 s bound instead of
 *   hanging the device when a peer never arrives); 0 in a healthy run.                          */
kron_status_t kron_dist_p2p_heap_bytes(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, kron_dtype_t dtype,
                                       int32_t GM, int32_t GK, size_t *bytes);
kron_status_t kron_dist_p2p_reserve(kron_dist_ctx_t *ctx, size_t bytes, void *ipc_handle_out);
kron_status_t kron_dist_p2p_connect(kron_dist_ctx_t *ctx, const void *ipc_handles);
kron_status_t kron_dist_p2p_timeouts(kron_dist_ctx_t *ctx, uint32_t *count);

/* Collective over the context's ranks: every rank calls it with identical M, N, P, Q, dtype.
 * NCCL and P2P backends: X_local / Y_local are this rank's blocks.
 * Virtual backend: X_local / Y_local are host arrays of GM*GK device pointers, one per rank.
 * dtype KRON_F32 or KRON_F64 (KRON_F32_3XTF32 -> KRON_ERR_UNSUPPORTED).
 * Errors: GM !| M, GK !| K, GK !| L or no legal round plan -> KRON_ERR_DIST_LAYOUT (shape-only,
 * so every rank returns the same status).  NCCL failures -> KRON_ERR_NCCL.                    */
kron_status_t kron_matmul_dist(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, const void *X_local,
                               const void *const *F, void *Y_local, kron_dtype_t dtype, kron_dist_ctx_t *ctx,
                               void *stream);

/* Round plan of the distributed path (host only).  On return rounds[j] = number of factors the
 * j-th round applies locally (sum = N), *nrounds the count; ledger[j] (optional) = values sent
 * between distinct ranks in round j summed over all ranks = M * W_j * (GK-1)/GK (reading G12). */
kron_status_t kron_dist_plan(int64_t M, int32_t N, const int32_t *P, const int32_t *Q, int32_t GM, int32_t GK,
                             int32_t cap, int32_t *nrounds, int32_t *rounds, int64_t *ledger);

/* Grid rule of P:654-655 ({sqrt G, sqrt G}, else {2^ceil(log2 sqrt G), 2^floor(log2 sqrt G)}). */
kron_status_t kron_dist_grid_rule(int32_t G, int32_t *GM, int32_t *GK);

#ifdef __cplusplus
}
#endif
#endif /* KRON_H_ */
