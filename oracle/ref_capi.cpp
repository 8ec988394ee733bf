// ref_capi.cpp — extern "C" bridge over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles /root/reference/proj/src/*.cpp (never copied into
// this repo) against oracle/ref_shim/ and links this file into
// oracle/_ref/libgpref.so.  The entry points mirror gp_oracle.h one for one
// (gpr_* ↔ gpo_*), so the tests can run the real reference and the C
// restatement on identical inputs, and bench.py --impl reference can time the
// reference's own code path on the host cores.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gradpack/bloom.hpp"
#include "gradpack/codecs.hpp"
#include "gradpack/container.hpp"
#include "gradpack/curvefit.hpp"
#include "gradpack/errors.hpp"
#include "gradpack/gradient.hpp"
#include "gradpack/pipeline.hpp"
#include "gradpack/rng.hpp"
#include "gradpack/sparsify.hpp"

#include "../include/gradpack_b200.h"

using namespace gradpack;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return GP_OK;
  } catch (const TruncatedError& e) {
    g_err = e.what();
    return GP_TRUNCATED;
  } catch (const ChecksumError& e) {
    g_err = e.what();
    return GP_CHECKSUM;
  } catch (const UnknownMethodError& e) {
    g_err = e.what();
    return GP_UNKNOWN_METHOD;
  } catch (const CorruptPayloadError& e) {
    g_err = e.what();
    return GP_CORRUPT_PAYLOAD;
  } catch (const DecodeError& e) {
    g_err = e.what();
    return GP_DECODE;
  } catch (const FitError& e) {
    g_err = e.what();
    return GP_FIT;
  } catch (const Error& e) {
    g_err = e.what();
    return GP_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GP_ERROR;
  }
}

template <typename T>
T* out_copy(const T* p, std::size_t n) {
  T* o = static_cast<T*>(std::malloc(n ? n * sizeof(T) : 1));
  if (n) std::memcpy(o, p, n * sizeof(T));
  return o;
}

PipelineConfig to_cfg(const gp_pipeline_config* c) {
  PipelineConfig p;
  p.index_method = static_cast<IndexMethod>(c->index_method);
  p.value_method = static_cast<ValueMethod>(c->value_method);
  p.fpr = c->fpr;
  p.pd_variant = static_cast<PdVariant>(c->pd_variant);
  p.degree = c->degree;
  p.max_segments = c->max_segments;
  p.quant_bits = c->quant_bits;
  p.quant_bucket = c->quant_bucket;
  p.slot_codec = static_cast<ByteCodec>(c->slot_codec);
  p.seed = c->seed;
  return p;
}

Vector dense_of(const float* g, std::uint64_t d) {
  Vector v(static_cast<Index>(d));
  for (std::uint64_t i = 0; i < d; ++i) v(static_cast<Index>(i)) = static_cast<double>(g[i]);
  return v;
}

}  // namespace

extern "C" {

const char* gpr_last_error(void) { return g_err.c_str(); }
void gpr_free(void* p) { std::free(p); }

int gpr_top_r(const float* g, std::uint64_t d, std::uint64_t r, std::uint32_t* support) {
  return guarded([&] {
    const Vector v = dense_of(g, d);
    const SparseGradient sg = top_r(v, static_cast<Index>(r));
    std::memcpy(support, sg.support.data(), sg.support.size() * 4);
  });
}

// random_r (sparsify.cpp:48-58) over a zero vector: the support only
int gpr_random_r(std::uint64_t d, std::uint64_t r, std::uint64_t seed, std::uint32_t* support) {
  return guarded([&] {
    const Vector v = Vector::Zero(static_cast<Index>(d));
    CounterRng rng(seed);
    const SparseGradient sg = random_r(v, static_cast<Index>(r), rng);
    std::memcpy(support, sg.support.data(), sg.support.size() * 4);
  });
}

int gpr_bloom_params(double eps, std::uint64_t r, std::uint64_t* m, std::uint32_t* k) {
  return guarded([&] {
    const BloomParams p = bloom_params(eps, r);
    *m = p.m;
    *k = p.k;
  });
}

std::uint32_t gpr_crc32c(const std::uint8_t* data, std::size_t n) {
  return crc32c(std::span<const std::uint8_t>(data, n));
}

int gpr_bloom_build(const std::uint32_t* support, std::uint64_t r, double eps, std::uint64_t sa,
                    std::uint64_t sb, std::uint8_t** filter, std::size_t* len) {
  return guarded([&] {
    const BloomFilter f = build_filter(std::span<const std::uint32_t>(support, r), eps, sa, sb);
    const std::vector<std::uint8_t> b = f.serialize();
    *len = b.size();
    *filter = out_copy(b.data(), b.size());
  });
}

int gpr_positive_scan(const std::uint8_t* filter, std::size_t len, std::uint64_t d,
                      std::uint32_t** pos, std::uint64_t* n) {
  return guarded([&] {
    ByteReader rd(std::span<const std::uint8_t>(filter, len));
    const BloomFilter f = BloomFilter::deserialize(rd);
    const std::vector<std::uint32_t> p = positive_scan(f, static_cast<Index>(d));
    *n = p.size();
    *pos = out_copy(p.data(), p.size());
  });
}

int gpr_bloom_select(const std::uint8_t* filter, std::size_t len, std::uint64_t d, std::uint64_t r,
                     int index_method, std::uint32_t** selected) {
  return guarded([&] {
    ByteReader rd(std::span<const std::uint8_t>(filter, len));
    const BloomFilter f = BloomFilter::deserialize(rd);
    const std::vector<std::uint32_t> p = positive_scan(f, static_cast<Index>(d));
    CounterRng rng(derive_selection_seed(f.seed_a(), f.seed_b()));
    const std::vector<std::uint32_t> s =
        index_method == GP_INDEX_BLOOM_P1 ? p1_select(p, static_cast<Index>(r), rng)
                                          : p2_select(p, f, static_cast<Index>(r), rng);
    *selected = out_copy(s.data(), s.size());
  });
}

int gpr_conflict_sets(const std::uint8_t* filter, std::size_t len, std::uint64_t d,
                      std::uint64_t** bits, std::uint64_t** offsets, std::uint32_t** members,
                      std::uint64_t* nsets) {
  return guarded([&] {
    ByteReader rd(std::span<const std::uint8_t>(filter, len));
    const BloomFilter f = BloomFilter::deserialize(rd);
    const std::vector<std::uint32_t> p = positive_scan(f, static_cast<Index>(d));
    const std::vector<ConflictSet> sets = conflict_sets(p, f);
    std::vector<std::uint64_t> b, o;
    std::vector<std::uint32_t> m;
    for (const ConflictSet& s : sets) {
      b.push_back(s.bit);
      o.push_back(m.size());
      m.insert(m.end(), s.members.begin(), s.members.end());
    }
    o.push_back(m.size());
    *nsets = sets.size();
    *bits = out_copy(b.data(), b.size());
    *offsets = out_copy(o.data(), o.size());
    *members = out_copy(m.data(), m.size());
  });
}

int gpr_value_compress(const double* v, std::uint64_t n, int degree, int max_segments,
                       std::uint8_t** fit, std::size_t* fit_len, std::uint32_t** map,
                       std::uint64_t* map_len) {
  return guarded([&] {
    ValueCodecConfig vc;
    vc.degree = degree;
    vc.max_segments = max_segments;
    const CompressedValues cv =
        value_compress(Eigen::Map<const Vector>(v, static_cast<Index>(n)), vc);
    const std::vector<std::uint8_t> b = serialize_fit(cv.model);
    *fit_len = b.size();
    *fit = out_copy(b.data(), b.size());
    *map_len = cv.reorder.size();
    *map = out_copy(cv.reorder.data(), cv.reorder.size());
  });
}

int gpr_compress_pack(std::uint64_t d, const std::uint32_t* support, const double* values,
                      std::uint64_t r, const float* dense, const gp_pipeline_config* cfg,
                      std::uint8_t** out, std::size_t* len) {
  return guarded([&] {
    SparseGradient sg;
    sg.dim = static_cast<Index>(d);
    sg.support.assign(support, support + r);
    sg.values.resize(static_cast<Index>(r));
    for (std::uint64_t i = 0; i < r; ++i)
      sg.values(static_cast<Index>(i)) = values ? values[i] : static_cast<double>(dense[support[i]]);
    Vector dv;
    if (dense) dv = dense_of(dense, d);
    const Container c = compress_gradient(sg, to_cfg(cfg), dense ? &dv : nullptr);
    const std::vector<std::uint8_t> b = pack(c);
    *len = b.size();
    *out = out_copy(b.data(), b.size());
  });
}

// top_r + compress_gradient(sg, cfg, &input) + pack: the encode span of
// Simulation::step (harness.cpp:235-252).
int gpr_encode_dense(const float* g, std::uint64_t d, std::uint64_t r,
                     const gp_pipeline_config* cfg, std::uint8_t** out, std::size_t* len) {
  return guarded([&] {
    const Vector dv = dense_of(g, d);
    const SparseGradient sg = top_r(dv, static_cast<Index>(r));
    const Container c = compress_gradient(sg, to_cfg(cfg), &dv);
    const std::vector<std::uint8_t> b = pack(c);
    *len = b.size();
    *out = out_copy(b.data(), b.size());
  });
}

// compress_gradient(sg, cfg, dense) + pack with f64 values and an optional
// f64 dense vector: the reference's own value type (pipeline.hpp:53-54).
int gpr_encode_sparse64(std::uint64_t d, const std::uint32_t* support, const double* values, std::uint64_t r,
                        const double* dense, const gp_pipeline_config* cfg, std::uint8_t** out, std::size_t* len) {
  return guarded([&] {
    SparseGradient sg;
    sg.dim = static_cast<Index>(d);
    sg.support.assign(support, support + r);
    sg.values.resize(static_cast<Index>(r));
    for (std::uint64_t i = 0; i < r; ++i) sg.values(static_cast<Index>(i)) = values[i];
    Vector dv;
    if (dense) {
      dv.resize(static_cast<Index>(d));
      for (std::uint64_t i = 0; i < d; ++i) dv(static_cast<Index>(i)) = dense[i];
    }
    const Container c = compress_gradient(sg, to_cfg(cfg), dense ? &dv : nullptr);
    const std::vector<std::uint8_t> b = pack(c);
    *len = b.size();
    *out = out_copy(b.data(), b.size());
  });
}

// One worker's compensated step of Simulation::step in the reference's own
// f64 arithmetic (harness.cpp:230, :242-251, :257-258, :269-271):
// input = g + residual; wire = pack(compress_gradient(top_r(input, r), cfg,
// &input)); residual = input - to_dense(decompress_gradient(unpack(wire))).
int gpr_ef_step64(const float* g, double* residual, std::uint64_t d, std::uint64_t r,
                  const gp_pipeline_config* cfg, std::uint8_t** out, std::size_t* len) {
  return guarded([&] {
    Vector res(static_cast<Index>(d));
    for (std::uint64_t i = 0; i < d; ++i) res(static_cast<Index>(i)) = residual[i];
    const Vector gv = dense_of(g, d);
    const Vector input = gv + res;
    const SparseGradient sg = top_r(input, static_cast<Index>(r));
    const std::vector<std::uint8_t> wire = pack(compress_gradient(sg, to_cfg(cfg), &input));
    const Vector decoded = to_dense(decompress_gradient(unpack(wire)));
    const Vector next = input - decoded;
    for (std::uint64_t i = 0; i < d; ++i) residual[i] = next(static_cast<Index>(i));
    *len = wire.size();
    *out = out_copy(wire.data(), wire.size());
  });
}

int gpr_decode(const std::uint8_t* bytes, std::size_t len, std::uint64_t* d, std::uint32_t** support,
               double** values, std::uint64_t* n) {
  return guarded([&] {
    const Container c = unpack(std::span<const std::uint8_t>(bytes, len));
    const SparseGradient sg = decompress_gradient(c);
    *d = static_cast<std::uint64_t>(sg.dim);
    *n = sg.support.size();
    *support = out_copy(sg.support.data(), sg.support.size());
    *values = out_copy(sg.values.data(), static_cast<std::size_t>(sg.values.size()));
  });
}

// unpack + decompress_gradient + to_dense accumulate (harness.cpp:257-258, :274-284)
int gpr_decode_accumulate(const std::uint8_t* bytes, std::size_t len, double* dense, std::uint64_t d,
                          double scale) {
  return guarded([&] {
    const Container c = unpack(std::span<const std::uint8_t>(bytes, len));
    const SparseGradient sg = decompress_gradient(c);
    if (static_cast<std::uint64_t>(sg.dim) != d) throw Error("decode_accumulate: dimension mismatch");
    const Vector dv = to_dense(sg);
    for (std::uint64_t i = 0; i < d; ++i) dense[i] += scale * dv(static_cast<Index>(i));
  });
}

int gpr_volume(const std::uint8_t* bytes, std::size_t len, std::uint64_t* out7) {
  return guarded([&] {
    const Container c = unpack(std::span<const std::uint8_t>(bytes, len));
    const VolumeReport v = volume(c);
    out7[0] = v.index_bits;
    out7[1] = v.value_bits;
    out7[2] = v.reorder_bits;
    out7[3] = v.metadata_bits;
    out7[4] = v.total_bits;
    std::memcpy(&out7[5], &v.ratio_dense, 8);
    std::memcpy(&out7[6], &v.ratio_sparse, 8);
  });
}

}  // extern "C"
