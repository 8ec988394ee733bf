// pipeline_b200.cpp — the B200 route for gradpack's pipeline: the adapter a
// gradpack maintainer adds in place of src/pipeline.cpp.  It defines the
// reference's own entry points (pipeline.hpp:41-59) with the reference's own
// types, so the reference's callers and tests link against it unchanged:
//
//   compress_gradient(sg, cfg, dense)   → gp_encode_sparse on the device
//                                         (f64 values, optional f64 dense),
//                                         then the reference's unpack() turns
//                                         the packed bytes into its Container
//   decompress_gradient(c)              → the reference's pack() of the
//                                         Container, then gp_decode_sparse
//   derive_*_seed                       → pipeline.cpp:21-26 (host arithmetic)
//
// Device errors come back as the gp_status of the first failing check, in the
// reference's order, and are rethrown as the matching errors.hpp class.
// One context and its staging buffers are kept per process and grown on
// demand (no allocation on the steady path).
//
// Built against the reference headers by oracle/Makefile (_ref/test_*_b200:
// the reference's own test sources linked with this file instead of
// pipeline.cpp) — see INTEGRATION.md §2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gradpack/container.hpp"
#include "gradpack/errors.hpp"
#include "gradpack/pipeline.hpp"

#include "../include/gradpack_b200.h"

namespace gradpack {

namespace {

[[noreturn]] void rethrow(int code, const std::string& msg) {
  switch (code) {
    case GP_DECODE: throw DecodeError(msg);
    case GP_TRUNCATED: throw TruncatedError(msg);
    case GP_CHECKSUM: throw ChecksumError(msg);
    case GP_UNKNOWN_METHOD: throw UnknownMethodError(msg);
    case GP_CORRUPT_PAYLOAD: throw CorruptPayloadError(msg);
    case GP_FIT: throw FitError(msg);
    default: throw Error(msg);
  }
}

std::uint64_t hash64_h(std::uint64_t x, std::uint64_t seed) {  // rng.hpp mix64 over x ^ (seed + gamma)
  std::uint64_t z = x ^ (seed + 0x9E3779B97F4A7C15ULL);
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// One device context + staging buffers for this process.
struct Session {
  std::mutex mu;
  gp_ctx* ctx = nullptr;
  std::uint64_t max_d = 0;
  cudaStream_t s = nullptr;
  void* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // support, values, dense, container, scalars
  std::size_t cap[5] = {0, 0, 0, 0, 0};

  void* grow(int i, std::size_t bytes) {
    if (cap[i] < bytes) {
      cudaFree(buf[i]);
      buf[i] = nullptr;
      if (cudaMalloc(&buf[i], std::max<std::size_t>(bytes, 256)) != cudaSuccess) throw Error("b200: cudaMalloc failed");
      cap[i] = std::max<std::size_t>(bytes, 256);
    }
    return buf[i];
  }

  void need(std::uint64_t d) {
    if (!s && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) throw Error("b200: no CUDA stream");
    if (ctx && d <= max_d) return;
    if (ctx) gp_ctx_destroy(ctx);
    ctx = nullptr;
    max_d = std::max<std::uint64_t>(d, 1u << 16);
    if (gp_ctx_create(0, max_d, &ctx) != GP_OK) throw Error("b200: gp_ctx_create failed");
  }

  void check(int rc) {
    if (rc == GP_OK) rc = gp_ctx_status(ctx, s);  // device-latched errors, reference order
    if (rc != GP_OK) rethrow(rc, std::string("b200: ") + gp_last_error(ctx));
  }
};

Session& session() {
  static Session S;
  return S;
}

gp_pipeline_config to_c(const PipelineConfig& c) {
  gp_pipeline_config o;
  gp_pipeline_config_default(&o);
  o.index_method = static_cast<std::uint8_t>(c.index_method);
  o.value_method = static_cast<std::uint8_t>(c.value_method);
  o.pd_variant = static_cast<std::uint8_t>(c.pd_variant);
  o.slot_codec = static_cast<std::uint8_t>(c.slot_codec);
  o.degree = c.degree;
  o.max_segments = c.max_segments;
  o.quant_bits = c.quant_bits;
  o.quant_bucket = c.quant_bucket;
  o.fpr = c.fpr;
  o.seed = c.seed;
  return o;
}

}  // namespace

// pipeline.cpp:21-26
std::uint64_t derive_filter_seed_a(std::uint64_t seed) { return hash64_h(0xA, seed); }
std::uint64_t derive_filter_seed_b(std::uint64_t seed) { return hash64_h(0xB, seed); }
std::uint64_t derive_selection_seed(std::uint64_t seed_a, std::uint64_t seed_b) { return hash64_h(seed_a, seed_b); }
std::uint64_t derive_quant_seed(std::uint64_t seed) { return hash64_h(0xC, seed); }

Container compress_gradient(const SparseGradient& sg, const PipelineConfig& config, const Vector* dense) {
  // the host-side argument checks of compress_gradient (pipeline.cpp:148-150);
  // support order and range are validated on the device (gradient.cpp:19-30)
  if (static_cast<std::size_t>(sg.values.size()) != sg.support.size())
    throw Error("gradient: support/value length mismatch");
  if (dense != nullptr && dense->size() != sg.dim) throw Error("pipeline: dense gradient dimension mismatch");
  if (sg.dim < 1) throw Error("gradient: dim must be >= 1");
  Session& S = session();
  std::lock_guard<std::mutex> lock(S.mu);
  const std::uint64_t d = static_cast<std::uint64_t>(sg.dim), r = sg.support.size();
  S.need(d);
  const gp_pipeline_config cfg = to_c(config);
  auto* sup = static_cast<std::uint32_t*>(S.grow(0, 4 * r));
  auto* val = static_cast<double*>(S.grow(1, 8 * r));
  double* dn = nullptr;
  if (r) {
    cudaMemcpyAsync(sup, sg.support.data(), 4 * r, cudaMemcpyHostToDevice, S.s);
    cudaMemcpyAsync(val, sg.values.data(), 8 * r, cudaMemcpyHostToDevice, S.s);
  }
  if (dense) {
    dn = static_cast<double*>(S.grow(2, 8 * d));
    cudaMemcpyAsync(dn, dense->data(), 8 * d, cudaMemcpyHostToDevice, S.s);
  }
  const std::uint64_t cap = gp_max_container_bytes(d, std::max<std::uint64_t>(r, 1), &cfg);
  auto* out = static_cast<std::uint8_t*>(S.grow(3, cap));
  auto* len = static_cast<std::uint64_t*>(S.grow(4, 64));
  S.check(gp_encode_sparse(S.ctx, d, r ? sup : nullptr, r ? val : nullptr, r, dn, &cfg, out, cap, len, S.s));
  std::uint64_t n = 0;
  cudaMemcpyAsync(&n, len, 8, cudaMemcpyDeviceToHost, S.s);
  cudaStreamSynchronize(S.s);
  std::vector<std::uint8_t> bytes(n);
  cudaMemcpyAsync(bytes.data(), out, n, cudaMemcpyDeviceToHost, S.s);
  cudaStreamSynchronize(S.s);
  return unpack(bytes);
}

SparseGradient decompress_gradient(const Container& c) {
  const std::vector<std::uint8_t> bytes = pack(c);
  Session& S = session();
  std::lock_guard<std::mutex> lock(S.mu);
  // the decoded support never exceeds d; r bounds every selection but naive's (|P| <= d)
  const std::uint64_t dcap = std::max<std::uint64_t>(std::min<std::uint64_t>(c.d, 0xFFFFFFFFull), 1);
  S.need(dcap);
  auto* in = static_cast<std::uint8_t*>(S.grow(3, bytes.size()));
  auto* sup = static_cast<std::uint32_t*>(S.grow(0, 4 * dcap));
  auto* val = static_cast<double*>(S.grow(1, 8 * dcap));
  auto* sc = static_cast<std::uint64_t*>(S.grow(4, 64));
  cudaMemcpyAsync(in, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, S.s);
  S.check(gp_decode_sparse(S.ctx, in, bytes.size(), sup, val, dcap, sc, sc + 1, S.s));
  std::uint64_t h[2] = {0, 0};
  cudaMemcpyAsync(h, sc, 16, cudaMemcpyDeviceToHost, S.s);
  cudaStreamSynchronize(S.s);
  SparseGradient out;
  out.dim = static_cast<Index>(h[1]);
  out.support.resize(h[0]);
  out.values.resize(static_cast<Index>(h[0]));
  if (h[0]) {
    cudaMemcpyAsync(out.support.data(), sup, 4 * h[0], cudaMemcpyDeviceToHost, S.s);
    cudaMemcpyAsync(out.values.data(), val, 8 * h[0], cudaMemcpyDeviceToHost, S.s);
    cudaStreamSynchronize(S.s);
  }
  return out;
}

}  // namespace gradpack
