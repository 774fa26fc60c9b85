/* synth/synth.c — seeded, counter-based synthetic input generator (host side).
 *
 * Test/bench infrastructure shared by BOTH the oracle side and the CUDA side; it holds
 * none of the Kron-Matmul arithmetic.
 * Any process can regenerate any element of any tensor from (seed, tensor_id, index):
 *
 *     h = splitmix64(splitmix64(seed) ^ (tensor_id << 56) ^ index)
 *
 * tensor_id 0 = X, i = F^i (1-based).  Modes (values exactly representable in fp32, so
 * fp32 and fp64 runs see identical data):
 *     0 urand : (h >> 40) * 2^-24              in [0,1)
 *     1 srand : 2*urand - 1                    in [-1,1)
 *     2 int   : (h mod 5) - 2                  in {-2..2}   (fp64 bit-exact tests)
 *     3 int1  : (h mod 3) - 1                  in {-1,0,1}  (fp32 bit-exact tests)
 * The device twin is synth/synth_dev.cu; tests pin the two to each other and to the
 * published splitmix64 reference outputs.
 */
#include <stdint.h>
#include <stddef.h>

uint64_t synth_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline double synth_value(uint64_t key, uint64_t idx, int mode) {
  uint64_t h = synth_splitmix64(key ^ idx);
  switch (mode) {
    case 0: return (double)(h >> 40) * (1.0 / 16777216.0);
    case 1: return 2.0 * ((double)(h >> 40) * (1.0 / 16777216.0)) - 1.0;
    case 2: return (double)(int)(h % 5u) - 2.0;
    case 3: return (double)(int)(h % 3u) - 1.0;
    default: return 0.0;
  }
}

static inline uint64_t synth_key(uint64_t seed, uint64_t tensor_id) {
  return synth_splitmix64(seed) ^ (tensor_id << 56);
}

/* Fill n consecutive elements starting at linear index `first` of tensor `tensor_id`. */
int synth_fill_f64(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t tensor_id, int mode) {
  if (!out || n < 0 || mode < 0 || mode > 3) return 1;
  uint64_t key = synth_key(seed, tensor_id);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = synth_value(key, (uint64_t)(first + i), mode);
  return 0;
}

int synth_fill_f32(float *out, int64_t n, int64_t first, uint64_t seed, uint64_t tensor_id, int mode) {
  if (!out || n < 0 || mode < 0 || mode > 3) return 1;
  uint64_t key = synth_key(seed, tensor_id);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = (float)synth_value(key, (uint64_t)(first + i), mode);
  return 0;
}

/* Rows `rows[0..nrows)` of an (implicit) row-major matrix with `cols` columns, packed. */
int synth_fill_rows_f64(double *out, const int64_t *rows, int64_t nrows, int64_t cols, uint64_t seed,
                        uint64_t tensor_id, int mode) {
  if (!out || !rows || nrows < 0 || cols < 0) return 1;
  uint64_t key = synth_key(seed, tensor_id);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      out[r * cols + c] = synth_value(key, (uint64_t)(rows[r] * cols + c), mode);
  return 0;
}
