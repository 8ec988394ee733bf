/* inputs.c — the benchmark's synthetic gradients (SURVEY.md §8(d) inputs),
 * host C so that the CPU reference arm, the golden generator and the device
 * arm all start from the same f32 bytes.  Not part of the encode/decode path:
 * it only fills host arrays that are then uploaded once.
 *
 *   g_w[i] = (float) CounterRng(hash64(w, hash64(0xBE7C, seed))).normal()
 *
 * is the reference CLI's bench generator (tools/gradpack_main.cpp:279-281)
 * extended with the rank; CounterRng (include/gradpack/rng.hpp:40-70) is
 * counter based — draw j (0-based) of a stream is mix64(seed + (j+1)·γ) — so
 * element i is a pure function of (seed, i) (draws 2i and 2i+1 of normal(),
 * rng.hpp:62-67) and any slice can be produced on its own thread.  log / cos
 * are libm's, as in the reference build; compiled without FP contraction.
 *
 * NCF-style natural sparsity: 64-wide row q is zero when draw q
 * of CounterRng(hash64(w, hash64(0x0DCF, seed))).unit() is < 0.4.
 */
#include <math.h>
#include <stdint.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline double unit_at(uint64_t seed, uint64_t j) { /* draw j of CounterRng(seed).unit() */
  return (double)(mix64(seed + (j + 1) * GAMMA) >> 11) * 0x1.0p-53;
}

/* out[k] = normal() number first + k of CounterRng(seed), as f32 */
void gpi_fill_normal_f32(uint64_t seed, uint64_t first, float* out, uint64_t n) {
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (uint64_t k = 0; k < n; ++k) {
    const uint64_t i = first + k;
    const double u1 = 1.0 - unit_at(seed, 2 * i);
    const double u2 = unit_at(seed, 2 * i + 1);
    out[k] = (float)(sqrt(-2.0 * log(u1)) * cos(two_pi * u2));
  }
}

/* zero g[k] (global element first + k) whose row (first + k) / row_width has
 * unit() < frac in CounterRng(seed) */
void gpi_zero_rows(uint64_t seed, uint64_t first, float* g, uint64_t n, uint64_t row_width, double frac) {
  uint64_t k = 0;
  while (k < n) {
    const uint64_t i = first + k;
    const uint64_t row = i / row_width;
    uint64_t end = (row + 1) * row_width - first;
    if (end > n) end = n;
    if (unit_at(seed, row) < frac)
      for (uint64_t j = k; j < end; ++j) g[j] = 0.0f;
    k = end;
  }
}

uint64_t gpi_hash64(uint64_t x, uint64_t seed) { return mix64(x ^ (seed + GAMMA)); }
