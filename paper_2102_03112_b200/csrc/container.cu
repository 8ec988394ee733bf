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
constexpr int kCrcBlock = 1024;
constexpr int kCrcBlocksPerSm = 1;  // the CRC grid is fixed: one 1024-lane block per SM (the lane stride is baked into M)
// slice-by-4 tables replicated per warp lane: entry e of table k for lane l at
// word (k * 256 + e) * 32 + l, so lane l only ever reads bank l — the random
// byte-indexed lookups of a warp are conflict-free (a shared 256-entry table
// serialises ~3.5-way on average).  128 KiB of dynamic shared memory.
constexpr int kCrcLaneTableWords = 4 * 256 * 32;
constexpr int kCrcSmallGrid = 24;  // blocks of the small-range CRC (1.5 MiB per row of 64-byte chunks)

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

// CRC-32C is linear over GF(2): with R(M) the raw register (init 0, no
// xorout) and S_L(c) = c * x^(8L) mod P,
//   crc(M) = XOR_q S_{after(q)}(R(C_q)) ^ S_{|M|}(0xFFFFFFFF) ^ 0xFFFFFFFF
// for any chunking M = C_0 ... C_{n-1}, after(q) = bytes following chunk q.
// Every thread folds one aligned 64-byte chunk (slice-by-4 tables), shifts it
// to the end of the range with x^(8L) = prod_i T_i[byte i of L] (byte-digit
// operator tables, 5 x 256 words, built on the host), and the chunks
// XOR-reduce — no combine tree, no sequential merge.
__device__ __forceinline__ uint64_t range_len(const uint64_t* len_a, const uint64_t* len_b, const uint64_t* len_c,
                                              uint64_t len_h) {
  return len_a ? (*len_a + (len_b ? *len_b : 0) + (len_c ? *len_c : 0)) : len_h;
}

__device__ __forceinline__ uint32_t shift_op(const uint32_t (*D)[256], uint64_t L) {
  uint32_t op = 1u << 31;  // x^0
  for (int i = 0; L; ++i, L >>= 8)
    if (L & 0xFF) op = multmodp(D[i][L & 0xFF], op);
  return op;
}

// Header (container.cpp:62-73) + CRC trailer (:77-80); lengths from the plan.
// Run by the CRC kernel's last block once the CRC is known (one thread).
__device__ void finish_body(uint8_t* out, uint64_t cap, uint64_t* d_len, Plan* plan, uint32_t crc,
                            uint32_t* status) {
  const uint64_t total = 49 + plan->il + plan->vl + plan->rl + 4;
  if (total > cap) return latch(status, GP_CAPACITY);
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
  st_u32_unaligned(out + total - 4, crc);
  plan->total_len = total;
  if (d_len) *d_len = total;
}

// the CRC verdict of unpack, then the post-CRC checks parse_container deferred
__device__ void verify_body(Plan* plan, uint32_t crc, uint32_t* status) {
  if (static_cast<uint64_t>(crc) != plan->crc_stored) return latch(status, GP_CHECKSUM);
  if (plan->post_crc_error) latch(status, plan->post_crc_error);
}

// what the CRC kernel's last block does with the result
struct CrcEpilogue {
  int mode = 0;  // 0 store only, 1 verify (unpack), 2 finish (pack)
  Plan* plan = nullptr;
  uint8_t* out = nullptr;
  uint64_t cap = 0;
  uint64_t* d_len = nullptr;
};

// Lane l of the fixed grid (kCrcLanes lanes) folds chunks l, l + kCrcLanes,
// ... in order, carrying its running value A across the kCrcLanes * 64-byte
// gap with one multiply by the constant x^(8 * 64 * kCrcLanes) mod P — a
// 4-lookup byte-table product (M) — instead of one bit-serial shift per
// chunk; a single variable shift per lane (digit tables D) carries A to the
// end of the range.  A chunk cut short by the range end is joined with a
// variable shift.  Tables: slice-by-4 T, constant multiply M, digits D.
__device__ __forceinline__ uint32_t mul_const(const uint32_t (*M)[256], uint32_t v) {
  return M[0][v & 0xFFu] ^ M[1][(v >> 8) & 0xFFu] ^ M[2][(v >> 16) & 0xFFu] ^ M[3][v >> 24];
}

__global__ void __launch_bounds__(kCrcBlock) crc_chunks(const uint8_t* __restrict__ base, const uint64_t* off_p,
                                                        uint64_t off_h, const uint64_t* len_a, const uint64_t* len_b,
                                                        const uint64_t* len_c, uint64_t len_h,
                                                        const uint32_t* __restrict__ digits,
                                                        const uint32_t* __restrict__ mtab, uint32_t* acc,
                                                        uint32_t* done, uint32_t* out, const CrcEpilogue ep,
                                                        uint32_t* status) {
  gp_pdl_wait();
  extern __shared__ uint32_t TL[];  // [4][256][32] per-lane slice-by-4 tables
  __shared__ uint32_t T0[256];
  __shared__ uint32_t D[5][256];
  __shared__ uint32_t M[4][256];
  __shared__ uint32_t red[kCrcBlock / 32];
  __shared__ bool last;
  if (failed(status)) return;
  const uint64_t off = off_p ? *off_p : off_h;
  const uint64_t len = range_len(len_a, len_b, len_c, len_h);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(base + off);
  const uintptr_t a1 = a0 + len;
  const uintptr_t c0 = a0 & ~static_cast<uintptr_t>(63);
  const uint64_t nchunks = len ? (a1 - c0 + 63) / 64 : 0;
  // blocks without chunks (most of the fixed grid for a small container) skip
  // the table setup and only join the reduction
  const bool active = static_cast<uint64_t>(blockIdx.x) * kCrcBlock < nchunks;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t* TLl = TL + lane;
  uint32_t A = 0;
  uintptr_t prev_end = 0;
  if (active) {
    for (int i = threadIdx.x; i < 256; i += kCrcBlock) {
      uint32_t c = static_cast<uint32_t>(i);
      for (int j = 0; j < 8; ++j) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
      T0[i] = c;
    }
    for (int i = threadIdx.x; i < 5 * 256; i += kCrcBlock) D[i / 256][i % 256] = digits[i];
    for (int i = threadIdx.x; i < 4 * 256; i += kCrcBlock) M[i / 256][i % 256] = mtab[i];  // this grid's lane stride
    __syncthreads();
    // T_k[e] = T_{k-1}[e] advanced by one zero byte; replicate into every lane's column
    for (int i = threadIdx.x; i < 4 * 256; i += kCrcBlock) {
      const int k = i >> 8, e = i & 255;
      uint32_t c = T0[e];
      for (int j = 0; j < k; ++j) c = (c >> 8) ^ T0[c & 0xFFu];
      uint32_t* dst = TL + static_cast<uint32_t>(i) * 32;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) dst[(l + threadIdx.x) & 31] = c;  // rotate the start: spread the banks
    }
    __syncthreads();
    const uint64_t lanes = static_cast<uint64_t>(gridDim.x) * kCrcBlock;  // == kCrcLanes (host)
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(kCrcBlock) + threadIdx.x; q < nchunks; q += lanes) {
      const uintptr_t cs = c0 + 64 * q;
      const uintptr_t lo = cs < a0 ? a0 : cs, hi = cs + 64 > a1 ? a1 : cs + 64;
      uint32_t c = 0;  // raw register of the chunk, init 0
      if (lo == cs && hi == cs + 64) {
        const uint4* p4 = reinterpret_cast<const uint4*>(cs);
        uint4 v4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v4[k] = p4[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t w[4] = {v4[k].x, v4[k].y, v4[k].z, v4[k].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            c ^= w[j];
            c = TLl[(3 * 256 + (c & 0xFFu)) * 32] ^ TLl[(2 * 256 + ((c >> 8) & 0xFFu)) * 32] ^
                TLl[(256 + ((c >> 16) & 0xFFu)) * 32] ^ TLl[(c >> 24) * 32];
          }
        }
      } else {
        const uint8_t* b = reinterpret_cast<const uint8_t*>(lo);
        for (uintptr_t i = 0; i < hi - lo; ++i) c = (c >> 8) ^ T0[(c ^ b[i]) & 0xFFu];
      }
      if (prev_end) A = (hi == cs + 64) ? mul_const(M, A) : multmodp(shift_op(D, hi - prev_end), A);
      A ^= c;
      prev_end = hi;
    }
  }  // active
  const uint64_t after = prev_end ? a1 - prev_end : 0;
  uint32_t x = after ? multmodp(shift_op(D, after), A) : A;
  // the init term x^(8 len) * 0xFFFFFFFF joins the XOR reduction from block 0
  // (active whenever len > 0, tables in shared memory), so the last block
  // — often one without tables — only applies the final inversion
  if (active && blockIdx.x == 0 && threadIdx.x == 0) x ^= multmodp(shift_op(D, len), 0xFFFFFFFFu);
  for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(kFull, x, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t y = 0;
    for (int w = 0; w < kCrcBlock / 32; ++w) y ^= red[w];
    if (y) atomicXor(acc, y);
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {  // the final block applies the final inversion
    __threadfence();
    const uint32_t raw = *reinterpret_cast<volatile uint32_t*>(acc);
    const uint32_t crc = len ? (raw ^ 0xFFFFFFFFu) : 0u;
    *out = crc;
    if (ep.mode == 1) verify_body(ep.plan, crc, status);
    if (ep.mode == 2) finish_body(ep.out, ep.cap, ep.d_len, ep.plan, crc, status);
    *acc = 0;   // ready for the next range
    *done = 0;
  }
}

// Small and medium ranges (container payloads up to a few MB: C1, C2, C4):
// `crc_tail` cuts the range into 64-byte chunks aligned to its END — chunk q
// = [E - 64(q+1), E - 64q), the first one front-padded with zeros, which a
// raw (init 0) CRC ignores — so chunk q's contribution is its raw CRC times
// x^(512 q) and no variable shift is ever needed: lane g of a G x 256 grid
// folds chunks g, g + T, g + 2T ... by Horner with the constant x^(512 T),
// then lanes combine in a tree (level j: v_L ^= x^(512 2^j) v_{L + 2^j}, in
// the warp by shuffles, across warps and then across blocks — the last
// block by ticket — through shared memory), every constant multiply one
// 8-lookup nibble-table product.  The CRC's init 0xFFFFFFFF is folded in by
// XORing the range's first four bytes with 0xFF (processing 4 zero bytes
// from register I equals processing I's bytes from register 0); the final
// XOR-out is one inversion.  Slice-by-4 tables are shared (not per lane): a
// chunk is 64 lookups, bank conflicts cost little at these sizes, and a
// block stages 12.5 KiB of tables instead of 138 KiB.
constexpr int kTailBlock = 256;
// crc_tail's largest grid (its partials buffer holds 256 blocks; x^(512 T) is built for it)
inline int tail_grid_max(const gp_ctx* ctx) { return ctx->sm_count < 256 ? ctx->sm_count : 256; }
__device__ __forceinline__ uint32_t mul_nib(const uint32_t* t, uint32_t v) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= t[i * 16 + ((v >> (4 * i)) & 15u)];
  return r;
}

__global__ void __launch_bounds__(kTailBlock) crc_tail(const uint8_t* __restrict__ base, const uint64_t* off_p,
                                                       uint64_t off_h, const uint64_t* len_a, const uint64_t* len_b,
                                                       const uint64_t* len_c, uint64_t len_h,
                                                       const uint32_t* __restrict__ tabs, uint32_t* partials,
                                                       uint32_t* ticket, uint32_t* out, const CrcEpilogue ep,
                                                       uint32_t* status) {
  gp_pdl_wait();
  constexpr int kTabWords = 4 * 256 + 17 * 128;  // T | K[0..17)
  __shared__ uint32_t T[4 * 256];
  __shared__ uint32_t K[17 * 128];  // K[j] = x^(512 * 2^j) for j < 16, K[16] = x^(512 T)
  __shared__ uint32_t red[kTailBlock / 32];
  __shared__ bool last;
  // every global read the block needs before its data — status, range, the
  // tables — is issued at once (one round trip instead of a chain)
  constexpr int kPer = (kTabWords + kTailBlock - 1) / kTailBlock;
  uint32_t tr[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * kTailBlock;
    tr[k] = i < 4 * 256 + 17 * 128 ? __ldg(tabs + i) : 0u;
  }
  const uint64_t off = off_p ? *off_p : off_h;
  const uint64_t len = range_len(len_a, len_b, len_c, len_h);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(base + off), E = a0 + len;
  const uint64_t nchunks = (len + 63) / 64;
  const uint64_t lanes = static_cast<uint64_t>(gridDim.x) * kTailBlock;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * kTailBlock;
    if (i < 4 * 256) T[i] = tr[k];
    else if (i < 4 * 256 + 17 * 128) K[i - 4 * 256] = tr[k];
  }
  // a latched error skips the work but not the ticket (block-uniform, and the
  // ticket always returns to 0)
  const bool skip = __syncthreads_or(failed(status));
  if (!skip && static_cast<uint64_t>(blockIdx.x) * kTailBlock < nchunks && len >= 4) {
    const uint32_t sh = 8 * static_cast<uint32_t>(E & 3);
    // the lane's chunks from the farthest (Horner: acc = x^(512 T) acc ^ crc(chunk))
    const uint64_t g = blockIdx.x * static_cast<uint64_t>(kTailBlock) + threadIdx.x;
    if (g < nchunks) {
      uint64_t q = g + ((nchunks - 1 - g) / lanes) * lanes;
      for (;;) {
        const uintptr_t cs = E - 64 * (q + 1);  // may precede a0 (then by < 64 bytes): zeros
        const uintptr_t wa = cs & ~static_cast<uintptr_t>(3);
        uint32_t W[17];
#pragma unroll
        for (int k = 0; k < 17; ++k) {
          const uintptr_t at = wa + 4 * k;
          W[k] = (at < E && at + 4 > a0) ? __ldg(reinterpret_cast<const uint32_t*>(at)) : 0u;
        }
        uint32_t c = 0;
        const bool head = cs < a0 + 4;  // the chunk holds the range's first bytes
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          uint32_t w = sh ? __funnelshift_r(W[k], W[k + 1], sh) : W[k];
          if (head) {
            const uintptr_t p0 = cs + 4 * k;  // bytes [p0, p0 + 4) of the range
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const uintptr_t p = p0 + b;
              if (p < a0) w &= ~(0xFFu << (8 * b));              // before the range: zero
              else if (p < a0 + 4) w ^= 0xFFu << (8 * b);      // the init term
            }
          }
          c ^= w;
          c = T[3 * 256 + (c & 0xFFu)] ^ T[2 * 256 + ((c >> 8) & 0xFFu)] ^ T[256 + ((c >> 16) & 0xFFu)] ^ T[c >> 24];
        }
        v ^= c;
        if (q < lanes) break;
        q -= lanes;
        v = mul_nib(K + 16 * 128, v);
      }
    }
    // tree over the block's lanes: lane L absorbs lane L + 2^j (farther from the end)
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const uint32_t o = __shfl_down_sync(kFull, v, 1u << j);
      if ((lane & ((2u << j) - 1)) == 0) v ^= mul_nib(K + j * 128, o);
    }
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
      v = lane < kTailBlock / 32 ? red[lane] : 0u;
#pragma unroll
      for (int j = 5; j < 8; ++j) {
        const uint32_t o = __shfl_down_sync(kFull, v, 1u << (j - 5));
        if ((lane & ((2u << (j - 5)) - 1)) == 0) v ^= mul_nib(K + j * 128, o);
      }
    }
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;  // block b's value, relative to chunk 256 b
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block: blocks b (chunk 256 b) combined with x^(512 * 256 * 2^j)
  uint32_t crc = 0;
  if (skip) {
  } else if (len >= 4) {
    const uint32_t nb = gridDim.x < 1024 ? gridDim.x : 1024;
    uint32_t x = threadIdx.x < nb ? __ldcg(partials + threadIdx.x) : 0u;
#pragma unroll
    for (int j = 0; j < 5; ++j) {  // blocks b, b + 2^j: x^(512 * 256 * 2^j) = K[j + 8]
      const uint32_t o = __shfl_down_sync(kFull, x, 1u << j);
      if ((lane & ((2u << j) - 1)) == 0) x ^= mul_nib(K + (j + 8) * 128, o);
    }
    if (lane == 0) red[warp] = x;
    __syncthreads();
    if (warp == 0) {
      x = lane < kTailBlock / 32 ? red[lane] : 0u;
#pragma unroll
      for (int j = 5; j < 8; ++j) {
        const uint32_t o = __shfl_down_sync(kFull, x, 1u << (j - 5));
        if ((lane & ((2u << (j - 5)) - 1)) == 0) x ^= mul_nib(K + (j + 8) * 128, o);
      }
    }
    crc = x ^ 0xFFFFFFFFu;
  } else if (threadIdx.x == 0) {  // 0-3 bytes: bytewise (table T0 = bit-serial here)
    uint32_t c = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < len; ++i) {
      c ^= reinterpret_cast<const uint8_t*>(a0)[i];
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
    }
    crc = len ? (c ^ 0xFFFFFFFFu) : 0u;
  }
  if (threadIdx.x == 0) {
    if (!skip) {
      *out = crc;
      if (ep.mode == 1) verify_body(ep.plan, crc, status);
      if (ep.mode == 2) finish_body(ep.out, ep.cap, ep.d_len, ep.plan, crc, status);
    }
    *ticket = 0;  // ready for the next range
  }
}

// unpack (container.cpp:84-127) up to, but not including, the CRC verdict.
//
// `pre` is the status word of the decode work that runs before the verdict,
// concurrently with the CRC (capi.cu decode_common): it starts as a copy of
// the main status, and every error found here — header errors and the
// post-CRC checks — goes to it at once, so that work never runs on a plan
// this kernel rejected; the main status gets the post-CRC checks only from
// the CRC kernel, after its verdict.
__global__ void parse_container(const uint8_t* __restrict__ in, uint64_t len_host, const uint64_t* len_dev,
                                uint64_t max_d, Plan* plan, const gp_pipeline_config hint, int use_hint,
                                uint32_t* status, uint32_t* pre) {
  gp_pdl_wait();
  *pre = *status;
  if (failed(status)) return;
  auto fail = [&](uint32_t code) {
    latch(status, code);
    latch(pre, code);
  };
  const uint64_t len = len_dev ? *len_dev : len_host;
  if (len_dev && len > len_host) return fail(GP_CAPACITY);  // len_host is the buffer capacity
  if (len < 4) return fail(GP_TRUNCATED);
  if (in[0] != 'D' || in[1] != 'R' || in[2] != 'C' || in[3] != '1') return fail(GP_CORRUPT_PAYLOAD);
  if (len < 6) return fail(GP_TRUNCATED);
  const uint32_t version = in[4] | (in[5] << 8);
  if (version != 1) return fail(GP_DECODE);
  if (len < 49) return fail(GP_TRUNCATED);
  const uint8_t index_id = in[6], value_id = in[7], flags = in[8];
  const uint64_t d = ld_u64_unaligned(in + 9), r = ld_u64_unaligned(in + 17);
  const uint64_t il = ld_u64_unaligned(in + 25), vl = ld_u64_unaligned(in + 33), rl = ld_u64_unaligned(in + 41);
  const uint64_t body = il + vl + rl + 4;  // u64 wrap-around, as in the reference
  const uint64_t rem = len - 49;
  if (rem < body) return fail(GP_TRUNCATED);
  if (rem > body) return fail(GP_CORRUPT_PAYLOAD);
  // bounds of the individual spans (guards against wrapped sums)
  if (il > rem || vl > rem || rl > rem) return fail(GP_TRUNCATED);
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
  plan->fused_bitmap = 0;
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
  if (post) latch(pre, post);
}

// After the join of the pre-verdict work: its first error, if the verdict and
// everything before it passed (the reference's order: header, CRC, post-CRC
// checks, then the method decoders in stream order).
__global__ void merge_status(uint32_t* status, const uint32_t* pre) {
  gp_pdl_wait();
  if (!failed(status) && *pre) latch(status, *pre);
}


}  // namespace

// Builds the CRC operator tables once per context (called from gp_ctx_create,
// which synchronizes and checks every error before the context is handed out,
// so no stream — captured or not — ever sees half-built tables).
int crc_tables_init(gp_ctx* ctx) {
  Workspace& w = ctx->ws;
  // byte-digit shift operators D[i][b] = x^(8 * b * 256^i) mod P
  auto mult = [](uint32_t a, uint32_t b) {
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
  };
  std::vector<uint32_t> tab(13 * 256 + kCrcSmallTabWords);
  uint32_t unit = 1u << 23;  // x^8: one byte
  for (int i = 0; i < 5; ++i) {
    uint32_t p = 1u << 31;
    for (int b = 0; b < 256; ++b) {
      tab[i * 256 + b] = p;
      p = mult(unit, p);
    }
    unit = p;  // x^(8 * 256^(i+1))
  }
  // M[j][b] = (b at byte j) * x^(8 * 64 * lanes) mod P: the lane stride of a
  // grid — the full one (one block per SM) and the small one (kCrcSmallGrid
  // blocks, for ranges of at most one of its rows: the launch and the
  // per-block table setup of ~120 idle blocks was most of a small CRC)
  for (int g = 0; g < 2; ++g) {
    uint64_t stride = 64ull * kCrcBlock *
                      static_cast<uint64_t>(g == 0 ? ctx->sm_count * kCrcBlocksPerSm : kCrcSmallGrid);
    uint32_t S = 1u << 31;
    for (int i = 0; stride; ++i, stride >>= 8)
      if (stride & 0xFF) S = mult(tab[i * 256 + (stride & 0xFF)], S);
    for (int j = 0; j < 4; ++j)
      for (int b = 0; b < 256; ++b)
        tab[(5 + 4 * g + j) * 256 + b] = b ? mult(static_cast<uint32_t>(b) << (8 * j), S) : 0u;
  }
  // crc_tail: slice-by-4 tables T_k (k zero bytes after the byte), nibble
  // tables of x^(512 * 2^j), j < 16, and of x^(512 T) for its full grid
  uint32_t* st = tab.data() + 13 * 256;
  for (int e = 0; e < 256; ++e) {
    uint32_t c = static_cast<uint32_t>(e);
    for (int j = 0; j < 8; ++j) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
    st[e] = c;
  }
  for (int k = 1; k < 4; ++k)
    for (int e = 0; e < 256; ++e) st[k * 256 + e] = (st[(k - 1) * 256 + e] >> 8) ^ st[st[(k - 1) * 256 + e] & 0xFFu];
  auto xpow = [&](uint64_t nbytes) {  // x^(8 nbytes) from the digit tables
    uint32_t S = 1u << 31;
    for (int i = 0; nbytes; ++i, nbytes >>= 8)
      if (nbytes & 0xFF) S = mult(tab[i * 256 + (nbytes & 0xFF)], S);
    return S;
  };
  for (int j = 0; j < 17; ++j) {
    const uint32_t S = xpow(j < 16 ? (64ull << j) : 64ull * kTailBlock * static_cast<uint64_t>(tail_grid_max(ctx)));
    for (int i = 0; i < 8; ++i)
      for (int n = 0; n < 16; ++n) st[4 * 256 + j * 128 + i * 16 + n] = n ? mult(static_cast<uint32_t>(n) << (4 * i), S) : 0u;
  }
  cudaError_t e = cudaFuncSetAttribute(crc_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kCrcLaneTableWords * static_cast<int>(sizeof(uint32_t)));
  if (e == cudaSuccess) e = cudaMemcpy(w.crc_digits, tab.data(), tab.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(w.crc_acc, 0, (64 + 256) * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  w.crc_ready = e == cudaSuccess;
  return e == cudaSuccess ? GP_OK : GP_CUDA;
}

namespace {
// len_bound: an upper bound of the range's length (host side)
void crc_range(gp_ctx* ctx, const uint8_t* base, const uint64_t* off_dev, uint64_t off_host, const uint64_t* la,
               const uint64_t* lb, const uint64_t* lc, uint64_t len_host, uint64_t len_bound, uint32_t* out,
               cudaStream_t s, const CrcEpilogue& ep) {
  Workspace& w = ctx->ws;
  static const uint64_t tail_max = getenv("GP_CRC_TAIL_MAX") ? strtoull(getenv("GP_CRC_TAIL_MAX"), nullptr, 10)
                                                              : (8ull << 20);
  if (len_bound <= tail_max) {  // crc_tail: one lane per 64-byte chunk (Horner rows above one grid)
    const uint64_t nch = (len_bound + 63) / 64;
    const uint64_t need = (nch + kTailBlock - 1) / kTailBlock;
    const int gmax = tail_grid_max(ctx);
    const int grid = static_cast<int>(need < static_cast<uint64_t>(gmax) ? (need ? need : 1) : gmax);
    // a grid below the full one never takes a second row (x^(512 T) is the full grid's)
    GP_LAUNCH(ctx, crc_tail, grid, kTailBlock, 0, s, base, off_dev, off_host, la, lb, lc, len_host,
              w.crc_digits + 13 * 256, w.crc_acc + 64, w.crc_acc + 2, out, ep, w.status);
    return;
  }
  const bool small = len_bound + 128 <= 64ull * kCrcBlock * kCrcSmallGrid;
  const int grid = small ? kCrcSmallGrid : ctx->sm_count * kCrcBlocksPerSm;
  const uint32_t* mtab = w.crc_digits + (small ? 9 : 5) * 256;
  GP_LAUNCH(ctx, crc_chunks, grid, kCrcBlock, kCrcLaneTableWords * sizeof(uint32_t), s, base, off_dev, off_host, la,
            lb, lc, len_host, w.crc_digits, mtab, w.crc_acc, w.crc_acc + 1, out, ep, w.status);
}
}  // namespace

void launch_crc_range(gp_ctx* ctx, const uint8_t* base, const uint64_t* off_dev, uint64_t off_host,
                      const uint64_t* la, const uint64_t* lb, const uint64_t* lc, uint64_t len_host,
                      uint64_t len_bound, uint32_t* out, cudaStream_t s) {
  crc_range(ctx, base, off_dev, off_host, la, lb, lc, len_host, len_bound, out, s, CrcEpilogue{});
}

void launch_finish_container(gp_ctx* ctx, uint8_t* out, uint64_t cap, uint64_t* d_len, uint64_t len_bound,
                             cudaStream_t s) {
  Workspace& w = ctx->ws;
  uint32_t* crc = reinterpret_cast<uint32_t*>(&w.plan->crc_calc);
  CrcEpilogue ep;
  ep.mode = 2;
  ep.plan = w.plan;
  ep.out = out;
  ep.cap = cap;
  ep.d_len = d_len;
  crc_range(ctx, out, &w.plan->off_index, 0, &w.plan->il, &w.plan->vl, &w.plan->rl, 0, len_bound, crc, s, ep);
}

void launch_parse_container(gp_ctx* ctx, const uint8_t* in, uint64_t len, const uint64_t* len_dev,
                            const gp_pipeline_config* hint, cudaStream_t s) {
  Workspace& w = ctx->ws;
  gp_pipeline_config h{};
  if (hint) h = *hint;
  GP_LAUNCH(ctx, parse_container, 1, 1, 0, s, in, len, len_dev, ctx->max_d, w.plan, h, hint ? 1 : 0, w.status,
            w.status_pre);
}

void launch_verify_crc(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  uint32_t* crc = reinterpret_cast<uint32_t*>(&w.plan->crc_calc);
  CrcEpilogue ep;
  ep.mode = 1;
  ep.plan = w.plan;
  crc_range(ctx, in, &w.plan->off_index, 0, &w.plan->il, &w.plan->vl, &w.plan->rl, 0, len_bound, crc, s, ep);
}

void launch_merge_status(gp_ctx* ctx, cudaStream_t s) {
  GP_LAUNCH(ctx, merge_status, 1, 1, 0, s, ctx->ws.status, ctx->ws.status_pre);
}

void launch_crc_host_range(gp_ctx* ctx, const uint8_t* data, uint64_t n, uint32_t* out, cudaStream_t s) {
  launch_crc_range(ctx, data, nullptr, 0, nullptr, nullptr, nullptr, n, n, out, s);
}

}  // namespace gp
