/* oracle/kron_oracle.c — the CPU ORACLE for Kron-Matmul (arxiv 2401.10187, FastKron).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * the CUDA path (paper_2401_10187_b200/), and neither imports the other.
 *
 * Plain, slow, obviously-correct fp64 implementations, each following the paper's text:
 *   O1 oracle_kron_product / oracle_naive   — Kronecker definition and the naive
 *                                             algorithm "computes the Kronecker matrix and then
 *                                             matrix multiply".
 *   O2 oracle_sliced_multiply / oracle_alg1 — Algorithm 1, one sliced multiply per
 *                                             factor, F^N first, two swapped intermediates.
 *   O3 oracle_alg2                           — Algorithm 2 simulated on G virtual
 *                                             GPUs with an exact communication ledger.
 *   index maps                               — Fig 7 StoreFusedShMem and Fig 5
 *                                             shift caching, under the DESIGN.md
 *                                             readings G6/G7 of their %-truncated lines.
 * Readings of ambiguous passages are marked G<n>.
 * All accumulation is fp64 in a fixed order; build with -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math).  Pins: tests/test_oracle.py (-m "not gpu").
 *
 * Conventions: matrices are dense row-major; factor i (0-based) is F^{i+1}, P[i] x Q[i];
 * F[0] = F^1 is the MOST significant factor (reading G4).
 * Return codes: 0 ok, 1 invalid argument, 2 too large / shape error, 3 out of memory.
 */
#include <stdint.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- O1: definition */

/* G = F^1 (x) ... (x) F^N by the block definition: entry
 *   G[r, c] = prod_i F^i[r_i, c_i],  r = sum_i r_i * prod_{j>i} P_j,  c likewise with Q,
 * i.e. mixed-radix digits with F^1 most significant. */
int oracle_kron_product(int N, const int *P, const int *Q, const double *const *F, double *G) {
  if (N < 1 || !P || !Q || !F || !G) return 1;
  int64_t K = 1, L = 1;
  for (int i = 0; i < N; ++i) {
    if (P[i] < 1 || Q[i] < 1 || !F[i]) return 1;
    K *= P[i];
    L *= Q[i];
    if (K * L > ((int64_t)1 << 30)) return 2;
  }
  for (int64_t r = 0; r < K; ++r) {
    for (int64_t c = 0; c < L; ++c) {
      double v = 1.0;
      int64_t rr = r, cc = c;
      for (int i = N - 1; i >= 0; --i) { /* least significant digit belongs to F^N */
        int ri = (int)(rr % P[i]), ci = (int)(cc % Q[i]);
        rr /= P[i];
        cc /= Q[i];
        v *= F[i][(int64_t)ri * Q[i] + ci];
      }
      G[r * L + c] = v;
    }
  }
  return 0;
}

/* O1 naive Kron-Matmul: Y = X . G with G materialised.  Guarded to K*L <= 2^26. */
int oracle_naive(int64_t M, int N, const int *P, const int *Q, const double *X, const double *const *F, double *Y) {
  if (M < 0 || N < 1 || !P || !Q || !F || (M > 0 && (!X || !Y))) return 1;
  int64_t K = 1, L = 1;
  for (int i = 0; i < N; ++i) {
    if (P[i] < 1 || Q[i] < 1) return 1;
    K *= P[i];
    L *= Q[i];
    if (K * L > ((int64_t)1 << 26)) return 2;
  }
  double *G = (double *)malloc(sizeof(double) * (size_t)(K * L));
  if (!G) return 3;
  int rc = oracle_kron_product(N, P, Q, F, G);
  if (rc) { free(G); return rc; }
  for (int64_t m = 0; m < M; ++m)
    for (int64_t c = 0; c < L; ++c) {
      double acc = 0.0;
      for (int64_t r = 0; r < K; ++r) acc += X[m * K + r] * G[r * L + c];
      Y[m * L + c] = acc;
    }
  free(G);
  return 0;
}

/* ---------------------------------------------------------------- O2: Algorithm 1 */

/* One sliced multiply (Alg 1) on `rows` rows of width K:
 *   Lout = (K / P) * Q                                      (line 307)
 *   for j in [0, Lout):  rowSlice = (j * P) mod K           (line 309)
 *                        kCol     = j div (K / P)           (line 310, reading G1)
 *                        Y1[i][j] = sum_k Y0[i][rowSlice + k] * F[k][kCol]   (lines 311-315)
 * 0-based indices (reading G3).  Requires P | K. */
int oracle_sliced_multiply(int64_t rows, int64_t K, int P, int Q, const double *Y0, const double *F, double *Y1) {
  if (rows < 0 || K < 1 || P < 1 || Q < 1 || K % P != 0 || !F || (rows > 0 && (!Y0 || !Y1))) return 1;
  int64_t S = K / P, Lout = S * Q;
  for (int64_t i = 0; i < rows; ++i) {
    const double *y0 = Y0 + i * K;
    double *y1 = Y1 + i * Lout;
    for (int64_t j = 0; j < Lout; ++j) {
      int64_t rowSlice = (j * P) % K;
      int64_t kCol = j / S;
      double acc = 0.0;
      for (int k = 0; k < P; ++k) acc += y0[rowSlice + k] * F[(int64_t)k * Q + kCol];
      y1[j] = acc;
    }
  }
  return 0;
}

/* Widths of the intermediates: W[N] = K = prod P (the input); for f = N..1 the sliced multiply
 * with F^f maps width W[f] to W[f-1] = W[f] / P_f * Q_f; W[0] = L = prod Q.  (Alg 1,
 * 307, 319; the buffer size of line 301 is max_f W[f], reading G2.) */
int oracle_widths(int N, const int *P, const int *Q, int64_t *W) {
  if (N < 1 || !P || !Q || !W) return 1;
  int64_t K = 1;
  for (int i = 0; i < N; ++i) {
    if (P[i] < 1 || Q[i] < 1) return 1;
    if (K > ((int64_t)1 << 40) / P[i]) return 2;
    K *= P[i];
  }
  W[N] = K;
  for (int f = N; f >= 1; --f) {
    if (W[f] % P[f - 1] != 0) return 2;
    W[f - 1] = W[f] / P[f - 1] * Q[f - 1];
  }
  return 0;
}

/* O2: Algorithm 1 on the selected rows (rows == NULL: all M rows).  Rows are
 * independent in Alg 1 (the loop of line 306), so a row subset is an exact check of those rows.
 * Xrows holds the selected rows of X packed (nrows x K); Y receives nrows x L.
 * OpenMP parallelises over rows only, so the result does not depend on the thread count. */
int oracle_alg1(int64_t nrows, int N, const int *P, const int *Q, const double *Xrows, const double *const *F,
                double *Y) {
  if (nrows < 0 || N < 1 || !P || !Q || !F || (nrows > 0 && (!Xrows || !Y))) return 1;
  int64_t W[65];
  if (N > 64) return 1;
  int rc = oracle_widths(N, P, Q, W);
  if (rc) return rc;
  int64_t maxw = 0;
  for (int f = 0; f <= N; ++f) maxw = W[f] > maxw ? W[f] : maxw; /* line 301, reading G2 */
  int err = 0;
#pragma omp parallel reduction(| : err)
  {
    double *Y1 = (double *)malloc(sizeof(double) * (size_t)maxw);
    double *Y2 = (double *)malloc(sizeof(double) * (size_t)maxw);
    if (!Y1 || !Y2) {
      err |= 1;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (int64_t i = 0; i < nrows; ++i) {
        memcpy(Y1, Xrows + i * W[N], sizeof(double) * (size_t)W[N]); /* line 302: Y1 = X */
        int64_t Kc = W[N];                                           /* line 303 */
        double *cur = Y1, *nxt = Y2;
        for (int f = N; f >= 1; --f) { /* line 304: f = N -> 1 */
          oracle_sliced_multiply(1, Kc, P[f - 1], Q[f - 1], cur, F[f - 1], nxt);
          double *t = cur; cur = nxt; nxt = t; /* line 318: swap intermediates */
          Kc = W[f - 1];                       /* line 319: K = L */
        }
        memcpy(Y + i * W[0], cur, sizeof(double) * (size_t)W[0]); /* line 321 */
      }
    }
    free(Y1);
    free(Y2);
  }
  return err ? 3 : 0;
}

/* ---------------------------------------------------------------- index maps */

/* Fig 7 StoreFusedShMem, reading G7 of the %-truncated lines 564/568/571:
 *   XgSlics = K/P; XsSlics = TileK/P; XgFuseSlics = K/P^Fused; XsFuseSlics = TileK/P^Fused
 *   c = e mod TileK
 *   slice      = (c div XsSlics) * XgSlics
 *   fusedSlice = ((c mod XsSlics) div XsFuseSlics) * XgFuseSlics
 *   elem       = bidy * XsFuseSlics + c mod XsFuseSlics
 *   col        = slice + fusedSlice + elem
 * Returns the global column of shared-memory element c of thread block `bidy` (square P x P
 * factors, as in the paper's example).  Fixture: P=4, K=256, TileK=128, Fused=2, c=41 -> 81. */
int64_t oracle_fused_store_col(int64_t K, int P, int64_t TileK, int Fused, int64_t bidy, int64_t c) {
  int64_t pf = 1;
  for (int i = 0; i < Fused; ++i) pf *= P;
  int64_t XgSlics = K / P, XsSlics = TileK / P, XgFuseSlics = K / pf, XsFuseSlics = TileK / pf;
  c = c % TileK;
  int64_t slice = (c / XsSlics) * XgSlics;
  int64_t fusedSlice = ((c % XsSlics) / XsFuseSlics) * XgFuseSlics;
  int64_t elem = bidy * XsFuseSlics + c % XsFuseSlics;
  return slice + fusedSlice + elem;
}

/* Fig 5 ShiftGToS, reading G6: element k of the row tile goes to shared position
 *   elem = k mod TileP, slice = k div TileP, shift = slice div RegK,
 *   pos  = slice * TileP + (elem + shift) mod TileP.
 * (The paper's printed "Xs[14]" for slice 4 contradicts this rule, which gives 18: reading G9.) */
int64_t oracle_shift_pos(int64_t k, int TileP, int RegK) {
  int64_t elem = k % TileP, slice = k / TileP, shift = slice / RegK;
  return slice * TileP + (elem + shift) % TileP;
}

/* ---------------------------------------------------------------- O3: Algorithm 2 */

/* Grid rule: {sqrt G, sqrt G} for square G, else {2^ceil(log2 sqrt G), 2^floor(log2 sqrt G)}.
 * Returns 0 and writes GM, GK, or 2 when the rule gives GM*GK != G (reading G14). */
int oracle_grid(int G, int *GM, int *GK) {
  if (G < 1 || !GM || !GK) return 1;
  int s = 0;
  while ((s + 1) * (s + 1) <= G) ++s;
  if (s * s == G) { *GM = s; *GK = s; return 0; }
  /* log2 sqrt G = log2(G)/2 */
  int lg = 0;
  while ((1 << (lg + 1)) <= G) ++lg;
  int exact_pow2 = (1 << lg) == G;
  /* ceil/floor of log2(G)/2 for a power of two G = 2^lg (lg odd here) */
  if (!exact_pow2) return 2;
  *GM = 1 << ((lg + 1) / 2);
  *GK = 1 << (lg / 2);
  return (*GM) * (*GK) == G ? 0 : 2;
}

/* O3: Algorithm 2 on a {GM, GK} grid of simulated GPUs, rows independent.
 *
 * Each GPU {gM, gK} holds the block X[gM*GTileM : +GTileM][gK*GTileK : +GTileK] (line 668).
 * Rounds: round j performs local[j] sliced multiplies (lines 670-674) with F^f, F^{f-1}, ...
 * (f running N -> 1) on the local block, then the GPUs with the same gM share their parts
 * (lines 676-692) and StoreGPUTile places each received element (line 685).
 *
 * StoreGPUTile is not printed ("similar to StoreFusedShMem").  Reading G13/G15: every
 * element travels to the GPU that owns its column of the globally distributed intermediate
 * (natural block distribution, width/GK columns per GPU) and is stored at its column there.
 * The simulator tracks, for every local element, its column in the global intermediate, using
 * only the sliced-multiply rule "local slice s of width P at local index q*S_loc + s is global
 * slice sigma, stored at global q*(W/P) + sigma" (Alg 1 line 309-315 on a contiguous slice);
 * a local slice that is not a contiguous, P-aligned run of global columns makes the round
 * illegal (return 4).  Ledger: values sent between distinct GPUs per round (line 683/690).
 *
 * X: M x K (full, fp64);  Y: M x L (gathered result);  ledger[j] (optional) gets round j's
 * total values sent.  Returns 0 ok, 1 bad args, 2 layout (GM !| M, GK !| width), 3 oom, 4 illegal. */
int oracle_alg2(int64_t M, int N, const int *P, const int *Q, const double *X, const double *const *F, int GM,
                int GK, int nrounds, const int *local, double *Y, int64_t *ledger) {
  if (M < 1 || N < 1 || !P || !Q || !X || !F || !Y || GM < 1 || GK < 1 || nrounds < 1 || !local) return 1;
  int64_t W[65];
  if (N > 64) return 1;
  int rc = oracle_widths(N, P, Q, W);
  if (rc) return rc;
  int tot = 0;
  for (int j = 0; j < nrounds; ++j) {
    if (local[j] < 1) return 1;
    tot += local[j];
  }
  if (tot != N) return 1;
  if (M % GM) return 2;
  int64_t GTileM = M / GM;
  int G = GM * GK;
  int64_t maxw = 0;
  for (int f = 0; f <= N; ++f) maxw = W[f] > maxw ? W[f] : maxw;
  /* per-GPU buffers: values and their global column */
  double **val = (double **)calloc((size_t)G, sizeof(double *));
  double **tmp = (double **)calloc((size_t)G, sizeof(double *));
  int64_t **col = (int64_t **)calloc((size_t)G, sizeof(int64_t *));
  int64_t **tcol = (int64_t **)calloc((size_t)G, sizeof(int64_t *));
  int ret = 0;
  if (!val || !tmp || !col || !tcol) { ret = 3; goto done; }
  for (int g = 0; g < G; ++g) {
    int64_t n = GTileM * (maxw / GK + 1);
    val[g] = (double *)malloc(sizeof(double) * (size_t)n);
    tmp[g] = (double *)malloc(sizeof(double) * (size_t)n);
    col[g] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    tcol[g] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!val[g] || !tmp[g] || !col[g] || !tcol[g]) { ret = 3; goto done; }
  }
  /* line 664-668: blocks */
  if (W[N] % GK) { ret = 2; goto done; }
  {
    int64_t wl = W[N] / GK;
    for (int gM = 0; gM < GM; ++gM)
      for (int gK = 0; gK < GK; ++gK) {
        int g = gM * GK + gK;
        for (int64_t i = 0; i < GTileM; ++i)
          for (int64_t c = 0; c < wl; ++c) {
            val[g][i * wl + c] = X[(gM * GTileM + i) * W[N] + gK * wl + c];
            col[g][i * wl + c] = gK * wl + c;
          }
      }
  }
  {
    int f = N;
    for (int j = 0; j < nrounds; ++j) {
      int64_t wl = W[f] / GK; /* local width entering the round */
      if (W[f] % GK) { ret = 2; goto done; }
      /* lines 670-674: local sliced multiplies */
      for (int b = 0; b < local[j]; ++b, --f) {
        int p = P[f - 1], q = Q[f - 1];
        int64_t Wg = W[f]; /* global width before this multiply */
        if (wl % p) { ret = 4; goto done; }
        int64_t S = wl / p, wl2 = S * q;
        for (int g = 0; g < G; ++g) {
          for (int64_t i = 0; i < GTileM; ++i) {
            const int64_t *c0 = col[g] + i * wl;
            /* legality: each local slice must be a P-aligned contiguous global slice */
            for (int64_t s = 0; s < S; ++s) {
              if (c0[s * p] % p) { ret = 4; goto done; }
              for (int k = 1; k < p; ++k)
                if (c0[s * p + k] != c0[s * p] + k) { ret = 4; goto done; }
            }
          }
          oracle_sliced_multiply(GTileM, wl, p, q, val[g], F[f - 1], tmp[g]);
          for (int64_t i = 0; i < GTileM; ++i)
            for (int64_t jj = 0; jj < wl2; ++jj) {
              int64_t s = jj % S, kq = jj / S;
              int64_t sigma = col[g][i * wl + s * p] / p; /* global slice index */
              tcol[g][i * wl2 + jj] = kq * (Wg / p) + sigma;
            }
          double *t = val[g]; val[g] = tmp[g]; tmp[g] = t;
          int64_t *tc = col[g]; col[g] = tcol[g]; tcol[g] = tc;
        }
        wl = wl2;
      }
      /* lines 676-692: share parts among GPUs with the same gM; StoreGPUTile (reading G13/G15) */
      int64_t Wn = W[f], wn = Wn / GK;
      if (Wn % GK) { ret = 2; goto done; }
      int64_t sent = 0;
      for (int gM = 0; gM < GM; ++gM) {
        for (int gK = 0; gK < GK; ++gK) {
          int g = gM * GK + gK;
          for (int64_t i = 0; i < GTileM; ++i)
            for (int64_t c = 0; c < wl; ++c) {
              int64_t gc = col[g][i * wl + c];
              int dst = (int)(gc / wn);
              int gd = gM * GK + dst;
              if (dst != gK) ++sent;
              tmp[gd][i * wn + (gc - dst * wn)] = val[g][i * wl + c];
              tcol[gd][i * wn + (gc - dst * wn)] = gc;
            }
        }
      }
      for (int g = 0; g < G; ++g) {
        double *t = val[g]; val[g] = tmp[g]; tmp[g] = t;
        int64_t *tc = col[g]; col[g] = tcol[g]; tcol[g] = tc;
      }
      if (ledger) ledger[j] = sent;
    }
    /* gather: GPU {gM,gK} now holds Y[gM rows][gK*L/GK : +L/GK] */
    int64_t wl = W[0] / GK;
    for (int gM = 0; gM < GM; ++gM)
      for (int gK = 0; gK < GK; ++gK) {
        int g = gM * GK + gK;
        for (int64_t i = 0; i < GTileM; ++i)
          for (int64_t c = 0; c < wl; ++c) Y[(gM * GTileM + i) * W[0] + gK * wl + c] = val[g][i * wl + c];
      }
  }
done:
  for (int g = 0; g < G && val && tmp && col && tcol; ++g) {
    free(val[g]);
    free(tmp[g]);
    free(col[g]);
    free(tcol[g]);
  }
  free(val);
  free(tmp);
  free(col);
  free(tcol);
  return ret;
}

/* OpenMP thread count for the row-parallel loops (infrastructure only: rows are independent, so the
 * result does not depend on it).  n > 0 sets it; returns the count the next parallel region uses. */
int oracle_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}
