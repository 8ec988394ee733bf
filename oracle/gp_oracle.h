/*
 * gp_oracle.h — CPU restatement of gradpack's encode → decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so, and
 * only as the checker or the timed CPU baseline — never as the product path.
 *
 * Every function restates a reference function (file:line under
 * /root/reference/proj) in plain C11.  Parity of this restatement is pinned two
 * ways (tests/test_oracle.py): against the reference's own known-answer
 * vectors, and against the unmodified reference sources built
 * into oracle/_ref/ (see oracle/Makefile).
 *
 * Conventions: gradients are f32 (the GPU path's input type); the reference
 * holds them as double, which is exact for f32-origin data.  Outputs returned
 * through pointer-to-pointer are malloc'd; release them with gpo_free().
 * Every function returns a gp_status code (include/gradpack_b200.h); the
 * message of the last failure on this thread is gpo_last_error().
 */
#ifndef GP_ORACLE_H_
#define GP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/gradpack_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpo_volume_report {
  uint64_t index_bits, value_bits, reorder_bits, metadata_bits, total_bits;
  double ratio_dense, ratio_sparse;
} gpo_volume_report;

const char* gpo_last_error(void);
void gpo_free(void* p);

uint64_t gpo_mix64(uint64_t z);
uint64_t gpo_hash64(uint64_t x, uint64_t seed);
/* CounterRng::below sequence: fills out[0..n) with successive below(bound) draws. */
int gpo_rng_below_seq(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out);
/* (float) CounterRng(seed).normal() stream (rng.hpp:65-69). */
void gpo_fill_normal_f32(uint64_t seed, float* out, uint64_t n);
uint64_t gpo_pipeline_seed(uint64_t seed, int worker, int step); /* harness.cpp:201-203 */

uint32_t gpo_crc32c(const uint8_t* data, size_t n);
int gpo_bloom_params(double eps, uint64_t r, uint64_t* m, uint32_t* k);

int gpo_top_r(const float* g, uint64_t d, uint64_t r, uint32_t* support);

/* Bit-exact codec components. */
int gpo_bitmap_bytes(const uint32_t* support, uint64_t r, uint64_t d, uint8_t* out);
int gpo_rle_encode(const uint32_t* support, uint64_t r, uint64_t d, uint8_t** out, size_t* len);
int gpo_bloom_build(const uint32_t* support, uint64_t r, double eps, uint64_t seed_a,
                    uint64_t seed_b, uint8_t** filter, size_t* len);
int gpo_positive_scan(const uint8_t* filter, size_t len, uint64_t d, uint32_t** pos, uint64_t* n);
/* index_method 5 (P1) or 6 (P2); seed = pipeline seed of the container. */
int gpo_bloom_select(const uint8_t* filter, size_t len, uint64_t d, uint64_t r, int index_method,
                     uint32_t** selected);
/* conflict_sets (bloom.cpp:156-173) in CSR form, in (size, bit) order. */
int gpo_conflict_sets(const uint8_t* filter, size_t len, uint64_t d, uint64_t** bits,
                      uint64_t** offsets, uint32_t** members, uint64_t* nsets);
/* value_compress (curvefit.cpp:432-493): fit payload bytes (serialize_fit) and
 * the reorder map (empty when identity). */
int gpo_value_compress(const double* v, uint64_t n, int degree, int max_segments,
                       uint8_t** fit, size_t* fit_len, uint32_t** map, uint64_t* map_len);

/* Pipeline. support/values describe the SparseGradient; dense may be NULL. */
int gpo_compress_pack(uint64_t d, const uint32_t* support, const double* values, uint64_t r,
                      const float* dense, const gp_pipeline_config* cfg, uint8_t** out,
                      size_t* len);
/* top_r + compress_gradient(sg, cfg, &dense) + pack (harness.cpp:242-251). */
int gpo_encode_dense(const float* g, uint64_t d, uint64_t r, const gp_pipeline_config* cfg,
                     uint8_t** out, size_t* len);
/* unpack + decompress_gradient. */
int gpo_decode(const uint8_t* bytes, size_t len, uint64_t* d, uint32_t** support,
               double** values, uint64_t* n);
/* unpack + decompress + dense[support] += scale * value, in f64 (to_dense). */
int gpo_decode_accumulate(const uint8_t* bytes, size_t len, double* dense, uint64_t d,
                          double scale);
int gpo_volume(const uint8_t* bytes, size_t len, gpo_volume_report* rep);

#ifdef __cplusplus
}
#endif
#endif /* GP_ORACLE_H_ */
