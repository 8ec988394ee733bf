// huffman.cu — index id 3: canonical Huffman over the 4 LE bytes of every
// support key (codecs.cpp:72-242, pipeline.cpp:179-184, :254-258), bit-exact.
//
// The table depends on d alone; one thread builds it on the device
// (huffman.cuh) so encode and decode need no host round trip.
// Encode: tiles of 1024 keys; every thread sums its 4 keys' code lengths, a
// decoupled look-back gives its bit offset, and it ORs its codes (MSB-first
// order = bit-reversed LSB-first words) into the zeroed payload.
// Decode (prefix codes have no random access): the stream is cut into
// 256-bit chunks and every chunk is decoded speculatively from its first bit;
// a chunk whose start differs from its predecessor's end is re-decoded from
// that end, a fixed number of rounds (Huffman codes resynchronise within a
// few codewords, so one round normally settles every chunk); a check latches
// any unsettled chunk to a sequential single-thread decode.  Then a scan of
// the per-chunk symbol counts and a final pass write the symbols straight into
// the support words (4 LE bytes per key), with decode errors reported in
// stream order exactly as decode() / decode_indices() raise them.
#include <cstdlib>

#include "gp_ctx.hpp"
#include "gp_device.cuh"
#include "huffman.cuh"

namespace gp {

namespace {

constexpr int kHBlock = 256;
constexpr int kHKeys = 4;  // keys per thread in encode
constexpr uint64_t kChunkBits = 256;
constexpr int kFixRounds = 24;

struct ChunkState {
  uint64_t start, end;
  uint32_t n, err_sym, err, pad;
};

__device__ __forceinline__ bool huff_active(const Plan* plan) { return plan->index_method == GP_INDEX_HUFFMAN; }

__global__ void huff_table(const Plan* plan, HuffTable* t, uint32_t* status) {
  gp_pdl_wait();
  __shared__ HuffScratch x;
  if (failed(status) || !huff_active(plan)) return;
  if (t->d == plan->d && t->nsym && !t->error) return;  // built for this d already (the table is a function of d)
  huff_build(plan->d, t, x);
  if (t->error) latch(status, GP_ERROR);  // from_frequencies throws Error (codecs.cpp:130)
}

__global__ void __launch_bounds__(kHBlock) huff_encode(const uint32_t* __restrict__ support, Plan* plan,
                                                       const HuffTable* __restrict__ gt, uint8_t* out,
                                                       uint64_t* tiles, uint32_t* ticket, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t rcode[256];  // codes bit-reversed: emission order LSB-first
  __shared__ uint8_t len[256];
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || !huff_active(plan)) return;
  for (int s = threadIdx.x; s < 256; s += kHBlock) {
    const uint32_t L = gt->len[s];
    len[s] = static_cast<uint8_t>(L);
    rcode[s] = L ? __brevll(gt->code[s]) >> (64 - L) : 0;
  }
  __syncthreads();
  const uint64_t r = plan->r;
  const uint64_t ntiles = (r + kHBlock * kHKeys - 1) / (kHBlock * kHKeys);
  const uintptr_t pa = reinterpret_cast<uintptr_t>(out + 49);
  uint32_t* words = reinterpret_cast<uint32_t*>(pa & ~static_cast<uintptr_t>(3));
  const uint64_t b0 = 8 * (pa & 3);
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t i0 = static_cast<uint64_t>(tile) * kHBlock * kHKeys + threadIdx.x * kHKeys;
    uint32_t key[kHKeys];
    uint64_t bits = 0;
#pragma unroll
    for (int q = 0; q < kHKeys; ++q) {
      key[q] = i0 + q < r ? support[i0 + q] : 0u;
      if (i0 + q < r)
        bits += len[key[q] & 255] + len[(key[q] >> 8) & 255] + len[(key[q] >> 16) & 255] + len[key[q] >> 24];
    }
    uint64_t total;
    uint64_t off = tile_exclusive_offset<kHBlock>(bits, tile, tiles, sh, total);
#pragma unroll
    for (int q = 0; q < kHKeys; ++q) {
      if (i0 + q >= r) break;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t s = (key[q] >> (8 * j)) & 255u;
        const uint32_t L = len[s];
        const uint64_t v = rcode[s];
        const uint64_t p = b0 + off;
        const uint64_t w = p >> 5;
        const uint32_t sft = static_cast<uint32_t>(p & 31);
        atomicOr(&words[w], static_cast<uint32_t>(v << sft));
        if (sft + L > 32) atomicOr(&words[w + 1], static_cast<uint32_t>(v >> (32 - sft)));
        if (sft + L > 64) atomicOr(&words[w + 2], static_cast<uint32_t>(v >> (64 - sft)));
        off += L;
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == kHBlock - 1) plan->il = (off + 7) / 8;
  }
}

// LSB-first 64-bit window of the stream at bit pos (zero past the end).
// Away from the end the 9 byte loads are unconditional, so they issue together.
__device__ __forceinline__ uint64_t peek64(const uint8_t* __restrict__ p, uint64_t nbytes, uint64_t pos) {
  const uint64_t b = pos >> 3;
  uint64_t lo = 0, hi = 0;
  if (b + 9 <= nbytes) {
    uint32_t v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(p + b + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) lo |= static_cast<uint64_t>(v[k]) << (8 * k);
    hi = v[8];
  } else {
    for (int k = 0; k < 8; ++k) lo |= (b + k < nbytes ? static_cast<uint64_t>(p[b + k]) : 0ull) << (8 * k);
    hi = b + 8 < nbytes ? p[b + 8] : 0u;
  }
  const uint32_t s = pos & 7;
  return s ? (lo >> s) | (hi << (64 - s)) : lo;
}

// Per-block decode tables in shared memory: a 2^kLut-entry direct table for
// codes of <= kLut bits ((len << 8) | symbol, 0 = longer or invalid) and the
// canonical per-length tables for the rest.
constexpr int kLut = 11;
struct HuffSmem {
  uint16_t lut[1 << kLut];
  uint64_t first_code[64];
  uint32_t first_index[64], count[64];
  uint64_t lim[64];   // per used length (ascending): (first_code + count) << (max_len - L)
  uint8_t lens[64];
  uint8_t sorted[256];
  uint32_t max_len, nl;
};

__device__ void load_smem_table(const HuffTable* __restrict__ g, HuffSmem& t) {
  for (int i = threadIdx.x; i < (1 << kLut); i += blockDim.x) t.lut[i] = 0;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    t.first_code[i] = g->first_code[i];
    t.first_index[i] = g->first_index[i];
    t.count[i] = g->count[i];
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) t.sorted[i] = g->sorted[i];
  if (threadIdx.x == 0) {
    const uint32_t ml = g->max_len;
    t.max_len = ml;
    uint32_t nl = 0;
    for (uint32_t L = 1; L <= ml; ++L)
      if (g->count[L]) {
        t.lens[nl] = static_cast<uint8_t>(L);
        t.lim[nl++] = (g->first_code[L] + g->count[L]) << (ml - L);
      }
    t.nl = nl;
  }
  __syncthreads();
  for (int sym = threadIdx.x; sym < 256; sym += blockDim.x) {
    const uint32_t L = g->len[sym];
    if (L == 0 || L > kLut) continue;
    const uint32_t base = static_cast<uint32_t>(g->code[sym]) << (kLut - L);
    for (uint32_t k = 0; k < (1u << (kLut - L)); ++k) t.lut[base + k] = static_cast<uint16_t>((L << 8) | sym);
  }
  __syncthreads();
}

// decode_symbol (codecs.cpp:181-190) from the LSB-first window: symbol >= 0
// and its length, -1 invalid code, -2 exhausted
__device__ __forceinline__ int decode_sym(const HuffSmem& t, uint64_t win, uint64_t avail, unsigned& len) {
  const uint32_t e = t.lut[__brev(static_cast<uint32_t>(win)) >> (32 - kLut)];
  if (e) {
    len = e >> 8;
    return len <= avail ? static_cast<int>(e & 255u) : -2;
  }
  // canonical codes left-justified to max_len bits are ordered by length:
  // the codeword's length is the first used length whose limit exceeds them
  const uint32_t ml = t.max_len;
  const uint64_t v = __brevll(win) >> (64 - ml);
  for (uint32_t i = 0; i < t.nl; ++i) {
    if (v < t.lim[i]) {
      const uint32_t L = t.lens[i];
      if (L > avail) return -2;  // the reference runs out of bits first
      len = L;
      const uint64_t code = v >> (ml - L);
      return t.sorted[t.first_index[L] + static_cast<uint32_t>(code - t.first_code[L])];
    }
  }
  return avail >= ml ? -1 : -2;  // no code: invalid, unless the stream ended first
}

// decode from `pos` until a codeword starts at or past `stop` (or an error)
__device__ void decode_run(const HuffSmem& t, const uint8_t* p, uint64_t nbytes, uint64_t pos, uint64_t stop,
                           ChunkState& cs, uint8_t* sym, uint64_t sym_off, uint64_t nsym_cap, uint64_t* end_bit) {
  const uint64_t nbits = 8 * nbytes;
  cs.start = pos;
  cs.n = 0;
  cs.err = 0;
  cs.err_sym = 0;
  while (pos < stop) {
    unsigned L = 0;
    const int s = decode_sym(t, peek64(p, nbytes, pos), nbits - pos, L);
    if (s < 0) {
      cs.err = s == -1 ? GP_CORRUPT_PAYLOAD : GP_TRUNCATED;
      cs.err_sym = cs.n;
      break;
    }
    pos += L;
    if (sym) {
      const uint64_t k = sym_off + cs.n;
      if (k < nsym_cap) sym[k] = static_cast<uint8_t>(s);
      if (k + 1 == nsym_cap) *end_bit = pos;  // bits consumed by the 4r-th symbol
    }
    ++cs.n;
  }
  cs.end = pos;
}

__device__ __forceinline__ uint64_t nchunks_of(const Plan* plan) { return (8 * plan->il + kChunkBits - 1) / kChunkBits; }

__global__ void huff_spec(const uint8_t* __restrict__ in, const Plan* plan, const HuffTable* __restrict__ gt,
                          ChunkState* cs, uint64_t cap, uint32_t* status) {
  gp_pdl_wait();
  __shared__ HuffSmem t;
  if (failed(status) || !huff_active(plan)) return;
  const uint64_t nch = nchunks_of(plan);
  if (nch > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_CAPACITY);
    return;
  }
  load_smem_table(gt, t);
  const uint8_t* p = in + plan->off_index;
  for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < nch;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    ChunkState s;
    decode_run(t, p, plan->il, c * kChunkBits, (c + 1) * kChunkBits, s, nullptr, 0, 0, nullptr);
    cs[c] = s;
  }
}

// one settling round: chunk c restarts at chunk c-1's end when they differ.
// A predecessor that stopped on an error leaves chunk c as it is: if that
// error is genuine the stream is invalid from there on, if it is an artefact
// of a misaligned start, a later round re-decodes the predecessor.
// changed[k] records whether round k moved any chunk; a round after a quiet
// one only copies (the rounds are a fixed launch sequence, graph-friendly).
__global__ void huff_fix(const uint8_t* __restrict__ in, const Plan* plan, const HuffTable* __restrict__ gt,
                         const ChunkState* __restrict__ a, ChunkState* b, uint32_t* changed, int k,
                         uint32_t* status) {
  gp_pdl_wait();
  __shared__ HuffSmem t;
  if (failed(status) || !huff_active(plan)) return;
  const uint64_t nch = nchunks_of(plan);
  const uint8_t* p = in + plan->off_index;
  const bool quiet = k > 0 && changed[k - 1] == 0;
  if (!quiet) load_smem_table(gt, t);
  bool moved = false;
  for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < nch;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    ChunkState s = a[c];
    if (c > 0 && !quiet) {
      const ChunkState prev = a[c - 1];
      if (!prev.err && prev.end != s.start) {
        decode_run(t, p, plan->il, prev.end, (c + 1) * kChunkBits, s, nullptr, 0, 0, nullptr);
        moved = true;
      }
    }
    b[c] = s;
  }
  if (__any_sync(kFull, moved) && (threadIdx.x & 31) == 0) changed[k] = 1u;
}

// Settled iff every chunk starts where its predecessor ended, up to the first
// chunk that stopped on an error (by induction from chunk 0 its start is a
// true codeword boundary, so that error is genuine and ends the stream).
__global__ void huff_check(const Plan* plan, const ChunkState* __restrict__ cs, uint32_t* flag, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !huff_active(plan)) return;
  const uint64_t nch = nchunks_of(plan);
  for (uint64_t c = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < nch;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (!cs[c - 1].err && cs[c].start != cs[c - 1].end) *flag = 1u;
}

// per-chunk symbol offsets (look-back scan), then the symbols; first error in
// stream order among the first 4r symbols
__global__ void __launch_bounds__(kHBlock) huff_emit(const uint8_t* __restrict__ in, Plan* plan,
                                                     const HuffTable* __restrict__ gt, const ChunkState* cs,
                                                     uint8_t* sym, uint64_t* res, uint64_t* tiles, uint32_t* ticket,
                                                     const uint32_t* flag, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  __shared__ HuffSmem t;
  if (failed(status) || !huff_active(plan) || *flag) return;
  load_smem_table(gt, t);
  const uint64_t nch = nchunks_of(plan);
  const uint64_t need = 4 * plan->r;
  const uint8_t* p = in + plan->off_index;
  const uint64_t ntiles = (nch + kHBlock - 1) / kHBlock;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t c = static_cast<uint64_t>(tile) * kHBlock + threadIdx.x;
    const ChunkState s = c < nch ? cs[c] : ChunkState{0, 0, 0, 0, 0, 0};
    uint64_t total;
    const uint64_t off = tile_exclusive_offset<kHBlock>(c < nch ? s.n : 0, tile, tiles, sh, total);
    if (c < nch) {
      if (off < need) {
        ChunkState t2;
        decode_run(t, p, plan->il, s.start, (c + 1) * kChunkBits, t2, sym, off, need, &res[1]);
      }
      if (s.err && off + s.err_sym < need) atomicMin(reinterpret_cast<unsigned long long*>(&res[0]),
                                                     ((off + s.err_sym) << 4) | s.err);
    }
    if (tile == ntiles - 1 && threadIdx.x == kHBlock - 1) res[2] = off + (c < nch ? s.n : 0);
  }
}

// the sequential decoder, for streams whose chunks did not settle
__global__ void huff_serial(const uint8_t* __restrict__ in, const Plan* plan, const HuffTable* __restrict__ gt,
                            uint8_t* sym, uint64_t* res, const uint32_t* flag, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ HuffSmem t;
  if (failed(status) || !huff_active(plan) || !*flag) return;
  load_smem_table(gt, t);
  ChunkState s;
  decode_run(t, in + plan->off_index, plan->il, 0, 8 * plan->il, s, sym, 0, 4 * plan->r, &res[1]);
  if (s.err && s.err_sym < 4 * plan->r) res[0] = (static_cast<uint64_t>(s.err_sym) << 4) | s.err;
  res[2] = s.n;
}

// decode(): first error, exhausted stream, trailing garbage (codecs.cpp:196-205)
__global__ void huff_verdict(Plan* plan, const uint64_t* res, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !huff_active(plan)) return;
  const uint64_t need = 4 * plan->r;
  if (res[0] != ~0ull) return latch(status, static_cast<uint32_t>(res[0] & 15));
  if (res[2] < need) return latch(status, GP_TRUNCATED);
  if (8 * plan->il - res[1] >= 8) return latch(status, GP_CORRUPT_PAYLOAD);
}

// decode_indices range check (codecs.cpp:232-241); the keys are already the
// LE words of the decoded bytes
__global__ void huff_keys(Plan* plan, const uint32_t* __restrict__ sel, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !huff_active(plan)) return;
  const uint64_t r = plan->r, d = plan->d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (sel[i] >= d) latch(status, GP_CORRUPT_PAYLOAD);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->n_sel = r;
    plan->n_values = r;
  }
}

__global__ void huff_reset(uint64_t* res, uint32_t* flag, uint32_t* changed) {
  gp_pdl_wait();
  res[0] = ~0ull;
  res[1] = 0;
  res[2] = 0;
  *flag = 0;
  for (int k = 0; k < kFixRounds; ++k) changed[k] = 0;
}

}  // namespace

void launch_index_huffman(gp_ctx* ctx, uint8_t* out, uint64_t r, uint64_t il_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  fill_async(ctx, out + 49, 0, il_bound, s);
  GP_LAUNCH(ctx, huff_table, 1, 1, 0, s, w.plan, w.huff, w.status);
  const uint64_t ntiles = (r + kHBlock * kHKeys - 1) / (kHBlock * kHKeys);
  reset_scan(ctx, s, ntiles + 1);
  GP_LAUNCH(ctx, huff_encode, static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL))),
            kHBlock, 0, s, w.support, w.plan, w.huff, out, w.tiles, w.ticket, w.status);
}

void launch_decode_index_huffman(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t cap = ctx->max_d / 4;  // chunk states per buffer (f64a / f64b are 8 D bytes each)
  const uint64_t nch_bound = std::min<uint64_t>((8 * len_bound + kChunkBits - 1) / kChunkBits, cap);
  ChunkState* a = reinterpret_cast<ChunkState*>(w.f64a);
  ChunkState* b = reinterpret_cast<ChunkState*>(w.f64b);
  uint64_t* res = w.huff_res;  // [first error, end bit, symbols]
  uint32_t* flag = reinterpret_cast<uint32_t*>(w.huff_res + 3);
  uint32_t* changed = reinterpret_cast<uint32_t*>(w.huff_res + 4);  // [kFixRounds]
  GP_LAUNCH(ctx, huff_reset, 1, 1, 0, s, res, flag, changed);
  GP_LAUNCH(ctx, huff_table, 1, 1, 0, s, w.plan, w.huff, w.status);
  const int g = grid_for(ctx, nch_bound, 128);
  GP_LAUNCH(ctx, huff_spec, g, 128, 0, s, in, w.plan, w.huff, a, cap, w.status);
  // GP_HUFF_FIX_ROUNDS (tests): fewer settling rounds force the sequential path
  const char* env = getenv("GP_HUFF_FIX_ROUNDS");
  const int rounds = env ? std::min(atoi(env), kFixRounds) : kFixRounds;
  for (int k = 0; k < rounds; ++k) {
    GP_LAUNCH(ctx, huff_fix, g, 128, 0, s, in, w.plan, w.huff, a, b, changed, k, w.status);
    std::swap(a, b);
  }
  GP_LAUNCH(ctx, huff_check, g, 128, 0, s, w.plan, a, flag, w.status);
  const uint64_t ntiles = (nch_bound + kHBlock - 1) / kHBlock;
  reset_scan(ctx, s, ntiles + 1);
  uint8_t* sym = reinterpret_cast<uint8_t*>(w.sel);
  GP_LAUNCH(ctx, huff_emit, static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL))),
            kHBlock, 0, s, in, w.plan, w.huff, a, sym, res, w.tiles, w.ticket, flag, w.status);
  GP_LAUNCH(ctx, huff_serial, 1, 1, 0, s, in, w.plan, w.huff, sym, res, flag, w.status);
  GP_LAUNCH(ctx, huff_verdict, 1, 1, 0, s, w.plan, res, w.status);
  GP_LAUNCH(ctx, huff_keys, grid_for(ctx, ctx->max_d, 256), 256, 0, s, w.plan, w.sel, w.status);
}

uint64_t huffman_il_bound(uint64_t d, uint64_t r) {
  HuffTable t;
  HuffScratch x;
  huff_build(d, &t, x);
  if (t.error) return 0;
  return (4 * r * static_cast<uint64_t>(t.max_len) + 7) / 8;
}

}  // namespace gp
