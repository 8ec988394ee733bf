// values_quant.cu — the stochastic quantizer (value id 3) and the byte-codec
// slot with the Store codec (value id 4), encode and decode, bit-exact.
//
// quantize (codecs.cpp:290-325) + serialize_quant (:327-333): per bucket of
// `bucket` values the f32 scale 2*max|v|; code = floor(u) + [unit() < frac(u)]
// with u = (v/scale + 0.5)*levels clamped to [0, levels] in f64 (no
// contraction); codes packed LSB-first at `bits` each.  The CounterRng stream
// (seed hash64(0xC, seed), pipeline.cpp:26) is consumed once per value of a
// bucket with scale > 0, so value i draws number i - (values of zero-scale
// buckets before it): a bucket scan, then every value is independent.
//   quant_scales : warp per bucket — scale, zero-bucket length
//   quant_zscan  : one block — exclusive scan of the zero-bucket lengths
//   quant_codes  : thread per value — its code (u32 scratch)
//   quant_pack   : thread per payload byte — gathers its <= 8 code bit runs
// Decode (parse_quant :335-351 + dequantize :339-355, pipeline.cpp:124-129):
//   quant_parse validates in the reference's order (truncation, bit range,
//   bucket, trailing bytes); quant_values evaluates scale*(code/levels - 0.5).
// Store slot (byte_compress/byte_decompress codecs.cpp:244-288 with
// ByteCodec::Store, pipeline.cpp:85-90, :130-139): [0 u8][4n u64][n f32].
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

__global__ void quant_scales(const ValSrc values, Plan* plan, uint8_t* out, uint32_t bucket,
                             uint32_t* __restrict__ zlen, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  const uint64_t nb = (n + bucket - 1) / bucket;
  uint8_t* p = out + 49 + plan->il + 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t b = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; b < nb; b += warps) {
    const uint64_t lo = b * bucket, hi = lo + bucket < n ? lo + bucket : n;
    double mx = 0.0;  // cwiseAbs().maxCoeff() (codecs.cpp:306)
    for (uint64_t i = lo + lane; i < hi; i += 32) mx = fmax(mx, fabs(values[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane == 0) {
      const float scale = __double2float_rn(2.0 * mx);
      st_u32_unaligned(p + 4 * b, __float_as_uint(scale));
      zlen[b] = scale > 0.0f ? 0u : static_cast<uint32_t>(hi - lo);
    }
  }
}

// exclusive scan of zlen[0, nb) in place (one block of 1024)
__global__ void __launch_bounds__(1024) quant_zscan(const Plan* plan, uint32_t bucket, uint32_t* zlen,
                                                    const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[40];
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  const uint64_t nb = (n + bucket - 1) / bucket;
  uint64_t run = 0;
  for (uint64_t b0 = 0; b0 < nb; b0 += 1024) {
    const uint64_t b = b0 + threadIdx.x;
    const uint64_t v = b < nb ? zlen[b] : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum<uint64_t, 1024>(v, sh, tot);
    if (b < nb) zlen[b] = static_cast<uint32_t>(run + ex);
    run += tot;
    __syncthreads();
  }
}

__global__ void quant_codes(const ValSrc values, const Plan* plan, const uint8_t* __restrict__ out,
                            uint32_t bits, uint32_t bucket, const uint32_t* __restrict__ zbefore,
                            uint32_t* __restrict__ codes, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  const uint8_t* sp = out + 49 + plan->il + 5;
  const uint64_t levels = (1ull << bits) - 1;
  const double lv = static_cast<double>(levels);
  const uint64_t seed = hash64(0xC, plan->seed);  // derive_quant_seed (pipeline.cpp:26)
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b = i / bucket;
    const float scale = __uint_as_float(ld_u32_unaligned(sp + 4 * b));
    uint64_t code = 0;
    if (scale > 0.0f) {
      double u = __dmul_rn(__dadd_rn(__ddiv_rn(values[i], static_cast<double>(scale)), 0.5), lv);
      u = u < 0.0 ? 0.0 : (u > lv ? lv : u);
      const double lo = floor(u);
      const double frac = __dsub_rn(u, lo);
      code = static_cast<uint64_t>(lo);
      const uint64_t draw = rng_at(seed, i - zbefore[b]);
      const double unit = static_cast<double>(draw >> 11) * 0x1.0p-53;
      if (unit < frac) ++code;
      if (code > levels) code = levels;
    }
    codes[i] = static_cast<uint32_t>(code);
  }
}

__global__ void quant_pack(const uint32_t* __restrict__ codes, Plan* plan, uint8_t* out, uint32_t bits,
                           uint32_t bucket, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  const uint64_t nb = (n + bucket - 1) / bucket;
  const uint64_t nbytes = (n * bits + 7) / 8;
  uint8_t* p = out + 49 + plan->il;
  uint8_t* cp = p + 5 + 4 * nb;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < nbytes;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b0 = 8 * j, b1 = b0 + 8;  // this byte's bit range
    uint32_t byte = 0;
    for (uint64_t c = b0 / bits; c < n && c * bits < b1; ++c) {
      const uint64_t cs = c * bits;  // code c occupies [cs, cs + bits)
      const uint64_t code = codes[c];
      // bits of the code that land in [b0, b1)
      const int64_t shift = static_cast<int64_t>(cs) - static_cast<int64_t>(b0);
      const uint64_t v = shift >= 0 ? (code << shift) : (code >> (-shift));
      byte |= static_cast<uint32_t>(v & 0xFFu);
    }
    cp[j] = static_cast<uint8_t>(byte);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p[0] = static_cast<uint8_t>(bits);
    st_u32_unaligned(p + 1, bucket);
    plan->vl = 5 + 4 * nb + nbytes;
    plan->rl = 0;
  }
}

// parse_quant (codecs.cpp:335-351) + the trailing check (pipeline.cpp:127)
__global__ void quant_parse(const uint8_t* __restrict__ in, Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t vl = plan->vl, count = plan->n_values;
  const uint8_t* p = in + plan->off_value;
  if (vl < 1) return latch(status, GP_TRUNCATED);
  const uint32_t bits = p[0];
  if (bits < 1 || bits > 16) return latch(status, GP_CORRUPT_PAYLOAD);
  if (vl < 5) return latch(status, GP_TRUNCATED);
  const uint32_t bucket = ld_u32_unaligned(p + 1);
  if (bucket < 1) return latch(status, GP_CORRUPT_PAYLOAD);
  const uint64_t nb = (count + bucket - 1) / bucket;
  if ((vl - 5) / 4 < nb) return latch(status, GP_TRUNCATED);
  const uint64_t code_bytes = (count * bits + 7) / 8;
  if (vl - 5 - 4 * nb < code_bytes) return latch(status, GP_TRUNCATED);
  if (vl - 5 - 4 * nb != code_bytes) return latch(status, GP_CORRUPT_PAYLOAD);
  plan->q_bits = bits;
  plan->q_bucket = bucket;
}

__global__ void quant_values(const uint8_t* __restrict__ in, const Plan* plan, double* __restrict__ vals,
                             const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t count = plan->n_values;
  const uint32_t bits = plan->q_bits, bucket = plan->q_bucket;
  const uint8_t* p = in + plan->off_value;
  const uint64_t nb = (count + bucket - 1) / bucket;
  const uint8_t* cp = p + 5 + 4 * nb;
  const double lv = static_cast<double>((1ull << bits) - 1);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = i * bits;
    // <= 16 bits starting at bit s: at most 3 bytes
    uint32_t w = 0;
    const uint64_t last = (s + bits - 1) / 8;
    for (uint64_t q = s / 8; q <= last; ++q) w |= static_cast<uint32_t>(cp[q]) << (8 * (q - s / 8));
    const uint32_t code = (w >> (s % 8)) & ((1u << bits) - 1u);
    const double scale = static_cast<double>(__uint_as_float(ld_u32_unaligned(p + 5 + 4 * (i / bucket))));
    vals[i] = __dmul_rn(scale, __dsub_rn(__ddiv_rn(static_cast<double>(code), lv), 0.5));
  }
}

__global__ void slot_encode(const ValSrc values, Plan* plan, uint8_t* out, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_values;
  uint8_t* p = out + 49 + plan->il;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    st_u32_unaligned(p + 9 + 4 * i, __float_as_uint(__double2float_rn(values[i])));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p[0] = 0;  // ByteCodec::Store
    st_u64_unaligned(p + 1, 4 * n);
    plan->vl = 9 + 4 * n;
    plan->rl = 0;
  }
}

// byte_decompress (codecs.cpp:268-288) + pipeline.cpp:131-133
__global__ void slot_parse(const uint8_t* __restrict__ in, Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t vl = plan->vl, count = plan->n_values;
  const uint8_t* p = in + plan->off_value;
  if (vl < 9) return latch(status, GP_TRUNCATED);
  const uint8_t id = p[0];
  const uint64_t raw_len = ld_u64_unaligned(p + 1);
  if (id > 1) return latch(status, GP_UNKNOWN_METHOD);
  plan->slot_id = id;
  // Deflate (id 1): an inflate that is not exactly 4·count bytes fails either
  // in uncompress or in pipeline.cpp:132-133 — CorruptPayloadError both ways
  if (id == 0 && vl - 9 != raw_len) return latch(status, GP_CORRUPT_PAYLOAD);
  if (raw_len != 4 * count) return latch(status, GP_CORRUPT_PAYLOAD);
}

}  // namespace

void launch_values_quant(gp_ctx* ctx, uint8_t* out, int bits, uint32_t bucket, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t nb_bound = (n_bound + bucket - 1) / bucket;
  const ValSrc vals{w.values, ctx->vals64};
  GP_LAUNCH(ctx, quant_scales, grid_for(ctx, nb_bound * 32, 256), 256, 0, s, vals, w.plan, out, bucket, w.u32b,
            w.status);
  GP_LAUNCH(ctx, quant_zscan, 1, 1024, 0, s, w.plan, bucket, w.u32b, w.status);
  GP_LAUNCH(ctx, quant_codes, grid_for(ctx, n_bound, 256), 256, 0, s, vals, w.plan, out,
            static_cast<uint32_t>(bits), bucket, w.u32b, w.u32a, w.status);
  GP_LAUNCH(ctx, quant_pack, grid_for(ctx, (n_bound * bits + 7) / 8, 256), 256, 0, s, w.u32a, w.plan, out,
            static_cast<uint32_t>(bits), bucket, w.status);
}

void launch_decode_quant(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, quant_parse, 1, 1, 0, s, in, w.plan, w.status);
  GP_LAUNCH(ctx, quant_values, grid_for(ctx, n_bound, 256), 256, 0, s, in, w.plan, w.f64a, w.status);
}

void launch_values_slot(gp_ctx* ctx, uint8_t* out, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, slot_encode, grid_for(ctx, n_bound, 256), 256, 0, s, ValSrc{w.values, ctx->vals64}, w.plan, out,
            w.status);
}

void launch_decode_slot(gp_ctx* ctx, const uint8_t* in, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, slot_parse, 1, 1, 0, s, in, w.plan, w.status);
}

}  // namespace gp
