// container.cu — K16/K17: the "DRC1" envelope (FORMAT.md:21-44,
// container.cpp:58-127) and its CRC-32C.
//
// CRC-32C (reflected Castagnoli, init/xorout 0xFFFFFFFF, container.cpp:30-48)
// is computed chunk-parallel: every thread folds a 1 KiB chunk with a
// shared-memory table, chunk CRCs are merged pairwise with the zlib
// combination rule crc(AB) = x^(8|B|) * crc(A) xor crc(B) over GF(2), first
// inside each block and then across blocks by one block.  The payloads are
// covered as one contiguous range (they follow the header back to back).
//
// Decode validation reproduces unpack's order exactly: magic, version,
// header truncation, body length, CRC, method ids, flags, reorder
// consistency, r <= d — checks after the CRC are computed by the parse kernel
// but only latched after the CRC verdict.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr uint32_t kPoly = 0x82F63B78u;
constexpr int kChunk = 1024;
constexpr int kCrcBlock = 256;

__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
  // a * b mod P in the reflected representation (bit 31 = x^0)
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(8 n) mod P via square-and-multiply on x^(2^k)
__device__ uint32_t x8nmodp(uint64_t n) {
  uint32_t p = 1u << 31;      // x^0
  uint32_t sq = 1u << 23;     // x^8
  while (n) {
    if (n & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

__device__ __forceinline__ uint32_t crc_combine(uint32_t a, uint32_t b, uint64_t len_b) {
  return multmodp(x8nmodp(len_b), a) ^ b;
}

__device__ void load_table(uint32_t* t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = static_cast<uint32_t>(i);
    for (int j = 0; j < 8; ++j) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
    t[i] = c;
  }
  __syncthreads();
}

// Per block: 256 chunks of 1 KiB.  Writes the block CRC to part[blockIdx].
// The range is [base + off, base + off + len) with off/len from device words.
__global__ void __launch_bounds__(kCrcBlock) crc_chunks(const uint8_t* __restrict__ base, const uint64_t* off_p,
                                                        uint64_t off_h, const uint64_t* len_a, const uint64_t* len_b,
                                                        const uint64_t* len_c, uint64_t len_h, uint32_t* part,
                                                        const uint32_t* status) {
  __shared__ uint32_t table[256];
  __shared__ uint32_t crc_s[kCrcBlock];
  __shared__ uint64_t len_s[kCrcBlock];
  if (failed(status)) return;
  load_table(table);
  const uint64_t off = off_p ? *off_p : off_h;
  const uint64_t len = len_a ? (*len_a + (len_b ? *len_b : 0) + (len_c ? *len_c : 0)) : len_h;
  const uint64_t nblocks = (len + static_cast<uint64_t>(kChunk) * kCrcBlock - 1) / (static_cast<uint64_t>(kChunk) * kCrcBlock);
  const uint8_t* data = base + off;
  for (uint64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const uint64_t start = (blk * kCrcBlock + threadIdx.x) * static_cast<uint64_t>(kChunk);
    const uint64_t end = start + kChunk < len ? start + kChunk : len;
    uint32_t c = 0xFFFFFFFFu;
    for (uint64_t i = start; i < end; ++i) c = (c >> 8) ^ table[(c ^ data[i]) & 0xFFu];
    crc_s[threadIdx.x] = start < end ? (c ^ 0xFFFFFFFFu) : 0u;
    len_s[threadIdx.x] = start < end ? end - start : 0;
    __syncthreads();
    for (int stride = 1; stride < kCrcBlock; stride <<= 1) {
      const int i = threadIdx.x;
      if ((i % (2 * stride)) == 0 && i + stride < kCrcBlock) {
        const uint64_t lb = len_s[i + stride];
        if (lb) crc_s[i] = crc_combine(crc_s[i], crc_s[i + stride], lb);
        len_s[i] += lb;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) part[blk] = crc_s[0];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) crc_merge(const uint32_t* __restrict__ part, const uint64_t* len_a,
                                                  const uint64_t* len_b, const uint64_t* len_c, uint64_t len_h,
                                                  uint32_t* out, const uint32_t* status) {
  __shared__ uint32_t crc_s[1024];
  __shared__ uint64_t len_s[1024];
  if (failed(status)) return;
  const uint64_t len = len_a ? (*len_a + (len_b ? *len_b : 0) + (len_c ? *len_c : 0)) : len_h;
  const uint64_t span = static_cast<uint64_t>(kChunk) * kCrcBlock;
  const uint64_t nblocks = (len + span - 1) / span;
  uint32_t acc = 0;
  uint64_t acc_len = 0;
  // fold 1024-wide groups of block CRCs left to right
  for (uint64_t g = 0; g < nblocks; g += 1024) {
    const uint64_t b = g + threadIdx.x;
    crc_s[threadIdx.x] = b < nblocks ? part[b] : 0u;
    len_s[threadIdx.x] = b < nblocks ? (b + 1 < nblocks ? span : len - b * span) : 0;
    __syncthreads();
    for (int stride = 1; stride < 1024; stride <<= 1) {
      const int i = threadIdx.x;
      if ((i % (2 * stride)) == 0 && i + stride < 1024) {
        const uint64_t lb = len_s[i + stride];
        if (lb) crc_s[i] = crc_combine(crc_s[i], crc_s[i + stride], lb);
        len_s[i] += lb;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      acc = acc_len ? crc_combine(acc, crc_s[0], len_s[0]) : crc_s[0];
      acc_len += len_s[0];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = len == 0 ? 0u : acc;
}

// Header (container.cpp:62-73) + CRC trailer (:77-80); lengths from the plan.
__global__ void finish_container(uint8_t* out, uint64_t cap, uint64_t* d_len, Plan* plan,
                                 const uint32_t* crc, uint32_t* status) {
  if (failed(status)) return;
  const uint64_t total = 49 + plan->il + plan->vl + plan->rl + 4;
  if (total > cap) {
    latch(status, GP_CAPACITY);
    return;
  }
  const int t = threadIdx.x;
  if (t == 0) {
    out[0] = 'D';
    out[1] = 'R';
    out[2] = 'C';
    out[3] = '1';
    out[4] = 1;
    out[5] = 0;
    out[6] = plan->index_method;
    out[7] = plan->value_method;
    out[8] = plan->rl ? 1 : 0;
    st_u64_unaligned(out + 9, plan->d);
    st_u64_unaligned(out + 17, plan->r);
    st_u64_unaligned(out + 25, plan->il);
    st_u64_unaligned(out + 33, plan->vl);
    st_u64_unaligned(out + 41, plan->rl);
    st_u32_unaligned(out + total - 4, *crc);
    plan->total_len = total;
    if (d_len) *d_len = total;
  }
}

// unpack (container.cpp:84-127) up to, but not including, the CRC verdict.
__global__ void parse_container(const uint8_t* __restrict__ in, uint64_t len_host, const uint64_t* len_dev,
                                uint64_t max_d, Plan* plan, const gp_pipeline_config hint, int use_hint,
                                uint32_t* status) {
  if (failed(status)) return;
  const uint64_t len = len_dev ? *len_dev : len_host;
  if (len_dev && len > len_host) return latch(status, GP_CAPACITY);  // len_host is the buffer capacity
  if (len < 4) return latch(status, GP_TRUNCATED);
  if (in[0] != 'D' || in[1] != 'R' || in[2] != 'C' || in[3] != '1') return latch(status, GP_CORRUPT_PAYLOAD);
  if (len < 6) return latch(status, GP_TRUNCATED);
  const uint32_t version = in[4] | (in[5] << 8);
  if (version != 1) return latch(status, GP_DECODE);
  if (len < 49) return latch(status, GP_TRUNCATED);
  const uint8_t index_id = in[6], value_id = in[7], flags = in[8];
  const uint64_t d = ld_u64_unaligned(in + 9), r = ld_u64_unaligned(in + 17);
  const uint64_t il = ld_u64_unaligned(in + 25), vl = ld_u64_unaligned(in + 33), rl = ld_u64_unaligned(in + 41);
  const uint64_t body = il + vl + rl + 4;  // u64 wrap-around, as in the reference
  const uint64_t rem = len - 49;
  if (rem < body) return latch(status, GP_TRUNCATED);
  if (rem > body) return latch(status, GP_CORRUPT_PAYLOAD);
  // bounds of the individual spans (guards against wrapped sums)
  if (il > rem || vl > rem || rl > rem) return latch(status, GP_TRUNCATED);
  plan->d = d;
  plan->r = r;
  plan->il = il;
  plan->vl = vl;
  plan->rl = rl;
  plan->off_index = 49;
  plan->off_value = 49 + il;
  plan->off_reorder = 49 + il + vl;
  plan->index_method = index_id;
  plan->value_method = value_id;
  plan->flags = flags;
  plan->crc_stored = ld_u32_unaligned(in + 49 + il + vl + rl);
  // post-CRC checks, in container.cpp order, then pipeline.cpp:224-225
  uint32_t post = 0;
  if (index_id > GP_INDEX_BLOOM_NAIVE || value_id > GP_VALUE_RAW_F64) post = GP_UNKNOWN_METHOD;
  else if ((flags & ~1u) != 0) post = GP_CORRUPT_PAYLOAD;
  else if (((flags & 1u) != 0) != (rl > 0)) post = GP_CORRUPT_PAYLOAD;
  else if (rl > 0 && value_id != GP_VALUE_FIT_POLY && value_id != GP_VALUE_FIT_DEXP) post = GP_CORRUPT_PAYLOAD;
  else if (r > d) post = GP_CORRUPT_PAYLOAD;
  else if (d < 1 || d > 0xffffffffULL) post = GP_CORRUPT_PAYLOAD;
  else if (use_hint && (index_id != hint.index_method || value_id != hint.value_method)) post = GP_UNSUPPORTED;
  else if (d > max_d) post = GP_CAPACITY;
  plan->post_crc_error = post;
}

__global__ void verify_container(Plan* plan, const uint32_t* crc, uint32_t* status) {
  if (failed(status)) return;
  if (static_cast<uint64_t>(*crc) != plan->crc_stored) return latch(status, GP_CHECKSUM);
  if (plan->post_crc_error) latch(status, plan->post_crc_error);
}

}  // namespace

void launch_crc_range(gp_ctx* ctx, const uint8_t* base, const uint64_t* off_dev, uint64_t off_host,
                      const uint64_t* la, const uint64_t* lb, const uint64_t* lc, uint64_t len_host,
                      uint64_t len_bound, uint32_t* out, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t span = static_cast<uint64_t>(kChunk) * kCrcBlock;
  const uint64_t nblocks = std::max<uint64_t>(1, (len_bound + span - 1) / span);
  const int grid = static_cast<int>(std::min<uint64_t>(nblocks, static_cast<uint64_t>(ctx->sm_count) * 8));
  GP_LAUNCH(ctx, crc_chunks, grid, kCrcBlock, 0, s, base, off_dev, off_host, la, lb, lc, len_host, w.crc_part,
            w.status);
  GP_LAUNCH(ctx, crc_merge, 1, 1024, 0, s, w.crc_part, la, lb, lc, len_host, out, w.status);
}

void launch_finish_container(gp_ctx* ctx, uint8_t* out, uint64_t cap, uint64_t* d_len, uint64_t len_bound,
                             cudaStream_t s) {
  Workspace& w = ctx->ws;
  uint32_t* crc = reinterpret_cast<uint32_t*>(&w.plan->crc_calc);
  launch_crc_range(ctx, out, &w.plan->off_index, 0, &w.plan->il, &w.plan->vl, &w.plan->rl, 0, len_bound, crc, s);
  GP_LAUNCH(ctx, finish_container, 1, 32, 0, s, out, cap, d_len, w.plan, crc, w.status);
}

void launch_parse_container(gp_ctx* ctx, const uint8_t* in, uint64_t len, const uint64_t* len_dev,
                            const gp_pipeline_config* hint, cudaStream_t s) {
  Workspace& w = ctx->ws;
  gp_pipeline_config h{};
  if (hint) h = *hint;
  GP_LAUNCH(ctx, parse_container, 1, 1, 0, s, in, len, len_dev, ctx->max_d, w.plan, h, hint ? 1 : 0, w.status);
  uint32_t* crc = reinterpret_cast<uint32_t*>(&w.plan->crc_calc);
  launch_crc_range(ctx, in, &w.plan->off_index, 0, &w.plan->il, &w.plan->vl, &w.plan->rl, 0, len, crc, s);
  GP_LAUNCH(ctx, verify_container, 1, 1, 0, s, w.plan, crc, w.status);
}

void launch_crc_host_range(gp_ctx* ctx, const uint8_t* data, uint64_t n, uint32_t* out, cudaStream_t s) {
  launch_crc_range(ctx, data, nullptr, 0, nullptr, nullptr, nullptr, n, n, out, s);
}

}  // namespace gp
