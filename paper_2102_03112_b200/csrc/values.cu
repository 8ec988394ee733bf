// values.cu — value payloads and the decode scatter.
//   gather_values (pipeline.cpp:38-54): v[j] = dense[sel[j]] for Bloom selections
//   id 0 raw f32 / id 5 raw f64 (pipeline.cpp:58-68, :97-112)
//   K18 decode_accumulate: dense[support[i]] += scale * value[i] — the
//   per-peer term of the harness mean (harness.cpp:274-284) fused with
//   to_dense (gradient.cpp:38-42).  Supports are unique per container, so the
//   scatter needs no atomics; peers are accumulated in rank order.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

__global__ void gather_values(const float* __restrict__ dense, const uint32_t* __restrict__ sel, const Plan* plan,
                              float* __restrict__ values, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    values[i] = dense[sel[i]];
}

// 4 values per thread per step, blockDim apart (each store instruction stays
// coalesced) with all four loads issued ahead of the stores: one value per
// thread leaves too few bytes in flight for HBM.
// f64 gather for compress_gradient(sg, cfg, dense) with Vector values
// (pipeline.cpp:38-54): dense[idx] when the dense vector is given, otherwise
// the sparse gradient's value at idx (binary search of the support) or 0
__global__ void gather_values64(const double* __restrict__ dense, const uint32_t* __restrict__ sup,
                                const double* __restrict__ sval, uint64_t r, const uint32_t* __restrict__ sel,
                                const Plan* plan, double* __restrict__ values, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t x = sel[i];
    if (dense) {
      values[i] = dense[x];
    } else {
      uint64_t lo = 0, hi = r;  // lower_bound
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (sup[mid] < x) lo = mid + 1; else hi = mid;
      }
      values[i] = lo < r && sup[lo] == x ? sval[lo] : 0.0;
    }
  }
}

__global__ void values_raw_encode(const ValSrc values, Plan* plan, uint8_t* out, int f64,
                                  const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  uint8_t* p = out + 49 + plan->il;
  const uint64_t step = 4ull * gridDim.x * blockDim.x;
  for (uint64_t i0 = 4ull * blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += step) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + static_cast<uint64_t>(q) * blockDim.x;
      v[q] = i < n ? values[i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + static_cast<uint64_t>(q) * blockDim.x;
      if (i >= n) break;
      if (f64)  // put_f64(values(i))
        st_u64_unaligned(p + 8 * i, static_cast<uint64_t>(__double_as_longlong(v[q])));
      else      // put_f32(static_cast<float>(values(i)))
        st_u32_unaligned(p + 4 * i, __float_as_uint(__double2float_rn(v[q])));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->vl = (f64 ? 8 : 4) * n;
    plan->rl = 0;
  }
}

// decode_values length checks for the raw kinds (pipeline.cpp:98-99, :107-108)
__global__ void values_raw_check(Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint8_t vm = plan->value_method;
  const uint64_t n = plan->n_values;
  if (vm == GP_VALUE_NONE && plan->vl != 4 * n) latch(status, GP_CORRUPT_PAYLOAD);
  if (vm == GP_VALUE_RAW_F64 && plan->vl != 8 * n) latch(status, GP_CORRUPT_PAYLOAD);
}

// value i of the decoded container: raw payload bytes or the fit evaluation
__device__ __forceinline__ double value_at(const uint8_t* vp, uint8_t vm, const double* fitv, uint64_t i) {
  if (vm == GP_VALUE_NONE) return static_cast<double>(__uint_as_float(ld_u32_unaligned(vp + 4 * i)));
  if (vm == GP_VALUE_RAW_F64) return __longlong_as_double(static_cast<long long>(ld_u64_unaligned(vp + 8 * i)));
  if (vm == GP_VALUE_DEFLATE_SLOT) return static_cast<double>(__uint_as_float(ld_u32_unaligned(vp + 9 + 4 * i)));
  return fitv[i];
}

__global__ void decode_scatter(const uint8_t* __restrict__ in, const Plan* plan, const uint32_t* __restrict__ sel,
                               const double* __restrict__ fitv, float* dense, uint64_t dense_d, float scale,
                               uint32_t* out_support, double* out_values, uint64_t cap, uint64_t* d_count,
                               uint64_t* d_dim, double* dense64, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->fused_bitmap) return;  // bitmap containers on the fused path: dense.cu bm_scatter
  // the container's d must equal the caller's dense length: to_dense builds a
  // d-vector (gradient.cpp:38-42) and the mean adds equal-length vectors
  // (harness.cpp:274-284); a mismatch is caller misuse, never a stray write
  if ((dense || dense64) && plan->d != dense_d) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_ERROR);
    return;
  }
  const uint64_t n = plan->n_sel;       // coordinates written (|P| for naive)
  const uint64_t nv = plan->n_values;   // values carried (naive: r, zero-filled past it)
  if (out_support && n > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_CAPACITY);
    return;
  }
  // an inflated Deflate slot was widened into fitv (inflate.cu)
  const uint8_t vm = plan->value_method == GP_VALUE_DEFLATE_SLOT && plan->slot_id == 1
                         ? static_cast<uint8_t>(GP_VALUE_FIT_POLY)
                         : plan->value_method;
  const uint8_t* vp = in + plan->off_value;
  // 4 coordinates per thread per step, blockDim apart (coalesced per
  // instruction): selections, values and the dense reads of all four are
  // issued before the dependent read-modify-writes
  const uint64_t step = 4ull * gridDim.x * blockDim.x;
  for (uint64_t i0 = 4ull * blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += step) {
    uint32_t s[4];
    double v[4];
    float dv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + static_cast<uint64_t>(q) * blockDim.x;
      s[q] = i < n ? sel[i] : 0u;
      v[q] = i < n && i < nv ? value_at(vp, vm, fitv, i) : 0.0;
    }
    if (dense) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + static_cast<uint64_t>(q) * blockDim.x < n) dv[q] = dense[s[q]];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + static_cast<uint64_t>(q) * blockDim.x;
      if (i >= n) break;
      if (dense) dense[s[q]] = fmaf(scale, static_cast<float>(v[q]), dv[q]);
      if (dense64)  // the f64 error-feedback residual: e = input - decoded (scale = -1, exact)
        dense64[s[q]] = __dadd_rn(dense64[s[q]], __dmul_rn(static_cast<double>(scale), v[q]));
      if (out_support) {
        out_support[i] = s[q];
        out_values[i] = v[q];
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (d_count) *d_count = n;
    if (d_dim) *d_dim = plan->d;
  }
}

}  // namespace

void launch_gather_values(gp_ctx* ctx, const float* dense, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, gather_values, grid_for(ctx, n_bound, 256), 256, 0, s, dense, w.sel, w.plan, w.values, w.status);
}

void launch_gather_values64(gp_ctx* ctx, const double* dense, const uint32_t* sup, const double* sval, uint64_t r,
                            uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, gather_values64, grid_for(ctx, n_bound, 256), 256, 0, s, dense, sup, sval, r, w.sel, w.plan, w.f64a,
            w.status);
}

void launch_values_raw(gp_ctx* ctx, uint8_t* out, bool f64, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, values_raw_encode, grid_for(ctx, n_bound, 256), 256, 0, s, ValSrc{w.values, ctx->vals64}, w.plan,
            out, f64 ? 1 : 0, w.status);
}

void launch_values_raw_check(gp_ctx* ctx, cudaStream_t s) {
  GP_LAUNCH(ctx, values_raw_check, 1, 1, 0, s, ctx->ws.plan, ctx->ws.status);
}

void launch_decode_scatter(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, float* dense, uint64_t dense_d,
                           float scale,
                           uint32_t* out_support, double* out_values, uint64_t cap, uint64_t* d_count,
                           uint64_t* d_dim, cudaStream_t s, double* dense64) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, decode_scatter, grid_for(ctx, n_bound, 256), 256, 0, s, in, w.plan, w.sel, w.f64a, dense, dense_d,
            scale, out_support, out_values, cap, d_count, d_dim, dense64, w.status);
}

}  // namespace gp
