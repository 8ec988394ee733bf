// gradpack_b200.hpp — C++ face of the C-ABI for gradpack's callers.
//
// Header-only, over include/gradpack_b200.h.  It restores what a C++ caller of
// the reference expects: the exception hierarchy of errors.hpp:21-53, a
// PipelineConfig with the reference defaults (pipeline.hpp:28-39), and the
// compressor calls with HOST buffers —
//   compress_dense      = top_r + compress_gradient(sg, cfg, &dense) + pack
//                         (harness.cpp:242-251)
//   compress_gradient   = compress_gradient(sg, cfg, &dense) + pack for a given
//                         support (pipeline.hpp:53-54, container.hpp:65)
//   decompress_gradient = unpack + decompress_gradient (container.hpp:66,
//                         pipeline.hpp:59)
//   volume              = volume (container.hpp:85)
// Every byte is produced on the device; these wrappers only stage host memory.
#ifndef GRADPACK_B200_HPP_
#define GRADPACK_B200_HPP_

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gradpack_b200.h"

namespace gradpack_b200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DecodeError : Error {
  using Error::Error;
};
struct TruncatedError : DecodeError {
  using DecodeError::DecodeError;
};
struct ChecksumError : DecodeError {
  using DecodeError::DecodeError;
};
struct UnknownMethodError : DecodeError {
  using DecodeError::DecodeError;
};
struct CorruptPayloadError : DecodeError {
  using DecodeError::DecodeError;
};
struct FitError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};
struct UnsupportedMethodError : Error {
  using Error::Error;
};
struct CapacityError : Error {
  using Error::Error;
};

[[noreturn]] inline void throw_status(int code, const std::string& msg) {
  switch (code) {
    case GP_DECODE: throw DecodeError(msg);
    case GP_TRUNCATED: throw TruncatedError(msg);
    case GP_CHECKSUM: throw ChecksumError(msg);
    case GP_UNKNOWN_METHOD: throw UnknownMethodError(msg);
    case GP_CORRUPT_PAYLOAD: throw CorruptPayloadError(msg);
    case GP_FIT: throw FitError(msg);
    case GP_CUDA: throw CudaError(msg);
    case GP_UNSUPPORTED: throw UnsupportedMethodError(msg);
    case GP_CAPACITY: throw CapacityError(msg);
    default: throw Error(msg);
  }
}

using PipelineConfig = gp_pipeline_config;

inline PipelineConfig default_config() {
  PipelineConfig c;
  gp_pipeline_config_default(&c);
  return c;
}

struct SparseGradient {
  uint64_t dim = 0;
  std::vector<uint32_t> support;  // strictly increasing, all < dim
  std::vector<double> values;     // values[i] belongs to support[i]
};

// RAII device buffer (fixed size)
template <typename T>
class DeviceBuffer {
 public:
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n && cudaMalloc(&p_, n * sizeof(T)) != cudaSuccess) throw CudaError("cudaMalloc failed");
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_;
};

// A device buffer that only grows: the host-buffer calls below stage through
// the Context's buffers, so repeated calls allocate nothing once warm.
class GrowBuffer {
 public:
  GrowBuffer() = default;
  ~GrowBuffer() {
    if (p_) cudaFree(p_);
  }
  GrowBuffer(const GrowBuffer&) = delete;
  GrowBuffer& operator=(const GrowBuffer&) = delete;
  void* reserve(size_t bytes) {
    if (bytes > cap_) {
      if (p_) cudaFree(p_);
      p_ = nullptr;
      cap_ = 0;
      const size_t want = bytes < 256 ? 256 : bytes + bytes / 4;  // headroom: fewer regrowths
      if (cudaMalloc(&p_, want) != cudaSuccess) throw CudaError("cudaMalloc failed");
      cap_ = want;
    }
    return p_;
  }
  size_t capacity() const { return cap_; }

 private:
  void* p_ = nullptr;
  size_t cap_ = 0;
};

class Context {
 public:
  explicit Context(uint64_t max_d, int device = 0) {
    const int rc = gp_ctx_create(device, max_d, &ctx_);
    if (rc != GP_OK) throw_status(rc, "gp_ctx_create failed");
  }
  ~Context() { gp_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  gp_ctx* get() const { return ctx_; }

  // staging slots of the host-buffer calls: 0 input vector, 1 support, 2 values,
  // 3 container, 4 small scalars
  template <typename T>
  T* stage(int slot, size_t n) { return static_cast<T*>(staging_[slot].reserve(n * sizeof(T))); }

  // raise a launch-time status immediately
  void check(int rc) const {
    if (rc != GP_OK) throw_status(rc, gp_last_error(ctx_));
  }
  // synchronise the stream and raise the first latched device status
  void sync(cudaStream_t s = nullptr) const { check(gp_ctx_status(ctx_, s)); }

 private:
  gp_ctx* ctx_ = nullptr;
  GrowBuffer staging_[5];
};

namespace detail {
inline void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
inline std::vector<uint8_t> fetch(const uint8_t* out, const uint64_t* len) {
  uint64_t n = 0;
  cuda_ok(cudaMemcpy(&n, len, sizeof(n), cudaMemcpyDeviceToHost), "length");
  std::vector<uint8_t> bytes(n);
  cuda_ok(cudaMemcpy(bytes.data(), out, n, cudaMemcpyDeviceToHost), "container");
  return bytes;
}
}  // namespace detail

// top_r + compress_gradient(sg, cfg, &dense) + pack of a host gradient.
inline std::vector<uint8_t> compress_dense(Context& ctx, const float* grad, uint64_t d, uint64_t r,
                                           const PipelineConfig& cfg) {
  float* g = ctx.stage<float>(0, d);
  detail::cuda_ok(cudaMemcpy(g, grad, d * sizeof(float), cudaMemcpyHostToDevice), "gradient");
  const uint64_t cap = gp_max_container_bytes(d, r, &cfg);
  uint8_t* out = ctx.stage<uint8_t>(3, cap);
  uint64_t* len = ctx.stage<uint64_t>(4, 2);
  ctx.check(gp_encode_topr(ctx.get(), g, d, r, &cfg, out, cap, len, nullptr));
  ctx.sync();
  return detail::fetch(out, len);
}

// compress_gradient(sg, cfg, &dense) + pack for a caller-chosen support.
inline std::vector<uint8_t> compress_gradient(Context& ctx, const float* dense, uint64_t d,
                                              const std::vector<uint32_t>& support, const PipelineConfig& cfg) {
  float* g = ctx.stage<float>(0, d);
  uint32_t* s = ctx.stage<uint32_t>(1, support.size());
  detail::cuda_ok(cudaMemcpy(g, dense, d * sizeof(float), cudaMemcpyHostToDevice), "dense");
  detail::cuda_ok(cudaMemcpy(s, support.data(), support.size() * 4, cudaMemcpyHostToDevice), "support");
  const uint64_t cap = gp_max_container_bytes(d, support.size(), &cfg);
  uint8_t* out = ctx.stage<uint8_t>(3, cap);
  uint64_t* len = ctx.stage<uint64_t>(4, 2);
  ctx.check(gp_encode_support(ctx.get(), g, d, s, support.size(), &cfg, out, cap, len, nullptr));
  ctx.sync();
  return detail::fetch(out, len);
}

// compress_gradient(sg, cfg, dense) + pack with the reference's f64 values
// (and optionally its f64 dense vector): bit-identical for any double.
inline std::vector<uint8_t> compress_sparse(Context& ctx, const SparseGradient& sg, const PipelineConfig& cfg,
                                            const double* dense = nullptr) {
  const uint64_t d = sg.dim, r = sg.support.size();
  if (sg.values.size() != r) throw Error("gradient: support/value length mismatch");
  uint32_t* s = ctx.stage<uint32_t>(1, r);
  double* v = ctx.stage<double>(2, r);
  if (r) {
    detail::cuda_ok(cudaMemcpy(s, sg.support.data(), r * 4, cudaMemcpyHostToDevice), "support");
    detail::cuda_ok(cudaMemcpy(v, sg.values.data(), r * 8, cudaMemcpyHostToDevice), "values");
  }
  double* dn = nullptr;
  if (dense) {
    dn = ctx.stage<double>(0, d);
    detail::cuda_ok(cudaMemcpy(dn, dense, d * 8, cudaMemcpyHostToDevice), "dense");
  }
  const uint64_t cap = gp_max_container_bytes(d, r ? r : 1, &cfg);
  uint8_t* out = ctx.stage<uint8_t>(3, cap);
  uint64_t* len = ctx.stage<uint64_t>(4, 2);
  ctx.check(gp_encode_sparse(ctx.get(), d, r ? s : nullptr, r ? v : nullptr, r, dn, &cfg, out, cap, len, nullptr));
  ctx.sync();
  return detail::fetch(out, len);
}

// unpack + decompress_gradient.
inline SparseGradient decompress_gradient(Context& ctx, const std::vector<uint8_t>& container, uint64_t cap) {
  uint8_t* in = ctx.stage<uint8_t>(3, container.size() ? container.size() : 1);
  detail::cuda_ok(cudaMemcpy(in, container.data(), container.size(), cudaMemcpyHostToDevice), "container");
  uint32_t* sup = ctx.stage<uint32_t>(1, cap);
  double* val = ctx.stage<double>(2, cap);
  uint64_t* meta = ctx.stage<uint64_t>(4, 2);
  ctx.check(gp_decode_sparse(ctx.get(), in, container.size(), sup, val, cap, meta, meta + 1, nullptr));
  ctx.sync();
  uint64_t m[2];
  detail::cuda_ok(cudaMemcpy(m, meta, sizeof(m), cudaMemcpyDeviceToHost), "meta");
  SparseGradient sg;
  sg.dim = m[1];
  sg.support.resize(m[0]);
  sg.values.resize(m[0]);
  detail::cuda_ok(cudaMemcpy(sg.support.data(), sup, m[0] * 4, cudaMemcpyDeviceToHost), "support");
  detail::cuda_ok(cudaMemcpy(sg.values.data(), val, m[0] * 8, cudaMemcpyDeviceToHost), "values");
  return sg;
}

inline gp_volume_report volume(const std::vector<uint8_t>& container) {
  gp_volume_report v;
  const int rc = gp_volume(container.data(), container.size(), &v);
  if (rc != GP_OK) throw_status(rc, "volume");
  return v;
}

}  // namespace gradpack_b200

#endif  // GRADPACK_B200_HPP_
