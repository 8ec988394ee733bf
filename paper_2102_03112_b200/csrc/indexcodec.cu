// indexcodec.cu — index payloads that carry the support explicitly:
//   id 0 raw u32 keys (pipeline.cpp:164-170, :230-238)
//   id 1 bitmap, ceil(d/8) bytes LSB-first (gradient.cpp:56-97, pipeline.cpp:171-173, :240-246)
// Encode reads the ascending support left by top-r in ws.support; decode
// writes the ascending support to ws.sel (count in plan->n_sel).
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kTileBlock = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileBlock * kTileItems;

__global__ void index_none_encode(const uint32_t* __restrict__ support, uint64_t r, uint8_t* out,
                                  const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  uint8_t* p = out + 49;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    st_u32_unaligned(p + 4 * i, support[i]);
}

// bitmap words (aligned scratch) from the ascending support; one atomicOr per
// distinct word per warp (consecutive keys usually share a word).
__global__ void bitmap_scatter(const uint32_t* __restrict__ support, uint64_t r, uint32_t* words,
                               const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i - threadIdx.x % 32 < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const bool ok = i < r;
    const uint32_t s = ok ? support[i] : 0xFFFFFFFFu;
    const uint32_t w = s >> 5;
    const unsigned peers = __match_any_sync(kFull, ok ? w : 0xFFFFFFFFu);
    const uint32_t bits = __reduce_or_sync(peers, ok ? (1u << (s & 31)) : 0u);
    const int leader = __ffs(peers) - 1;
    if (ok && (threadIdx.x & 31) == leader) atomicOr(&words[w], bits);
  }
}

// copy ceil(d/8) bitmap bytes to the (unaligned) payload position
__global__ void bitmap_emit(const uint32_t* __restrict__ words, uint64_t d, uint8_t* out, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t nbytes = (d + 7) / 8;
  uint8_t* p = out + 49;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(words);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nbytes;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = src[i];
}

// ------------------------------------------------------------ decode
__global__ void index_none_decode(const uint8_t* __restrict__ in, Plan* plan, uint32_t* sel, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_NONE) return;
  const uint64_t r = plan->r;
  if (plan->il != 4 * r) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_CORRUPT_PAYLOAD);
    return;
  }
  const uint8_t* p = in + plan->off_index;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    sel[i] = ld_u32_unaligned(p + 4 * i);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->n_sel = r;
    plan->n_values = r;
  }
}

// validate strictly increasing & < d (pipeline.cpp:299-305) — after the values
__global__ void support_validate(const Plan* plan, const uint32_t* __restrict__ sel, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || (plan->index_method != GP_INDEX_NONE && plan->index_method != GP_INDEX_HUFFMAN)) return;
  const uint64_t n = plan->n_sel, d = plan->d;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (static_cast<uint64_t>(sel[i]) >= d || (i > 0 && sel[i] <= sel[i - 1])) latch(status, GP_CORRUPT_PAYLOAD);
  }
}

// bitmap_from_bytes checks (gradient.cpp:88-97)
__global__ void bitmap_check(const uint8_t* __restrict__ in, Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_BITMAP) return;
  const uint64_t d = plan->d;
  if (plan->il != (d + 7) / 8) return latch(status, GP_CORRUPT_PAYLOAD);
  if (d % 8 != 0 && (in[plan->off_index + plan->il - 1] >> (d % 8)) != 0) return latch(status, GP_CORRUPT_PAYLOAD);
}

// ordered extraction of set bits, 4 KiB of bitmap per tile.  Warp w of a tile
// owns bytes [512w, 512w + 512) in four rounds of 128 bytes (4 per lane, so
// the byte loads are coalesced).  Emission is transposed: for each of the
// round's 32 words, the lanes whose bit is set store at their rank in the word,
// so every store instruction writes one contiguous run (a per-lane ffs loop
// stores 32 scattered runs per instruction and stalls on FLO/STS latency).
__global__ void __launch_bounds__(kTileBlock) bitmap_support(const uint8_t* __restrict__ in, Plan* plan,
                                                             uint32_t* sel, uint64_t* tiles, uint32_t* ticket,
                                                             uint64_t cap, uint32_t* status) {
  gp_pdl_wait();
  constexpr int kRounds = kTileItems / 4;
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->index_method != GP_INDEX_BITMAP) return;
  const uint64_t nbytes = plan->il;
  const uint8_t* p = in + plan->off_index;
  const uint64_t ntiles = (nbytes + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t wbase = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (kTileItems * 32);
    uint32_t x[kRounds];
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kRounds; ++q) {
      const uint64_t at = wbase + q * 128 + 4 * lane;
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (at + k < nbytes) v |= static_cast<uint32_t>(p[at + k]) << (8 * k);
      x[q] = v;
      c += __popc(v);
    }
    const uint32_t wc = __reduce_add_sync(kFull, c);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kTileBlock>(lane == 0 ? wc : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < kRounds; ++q) {
      const uint32_t n = __popc(x[q]);
      uint32_t incl = n;
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, k);
        if (lane >= k) incl += t;
      }
      const uint32_t total = __shfl_sync(kFull, incl, 31);
      const uint32_t excl = incl - n;
      // transposed emission: word k's set bits are written by the lanes whose
      // bit is set, each at its rank in the word -> one contiguous run per word
      const uint32_t bit0 = static_cast<uint32_t>(8 * (wbase + q * 128));
      if (__reduce_max_sync(kFull, n) <= 8) {  // sparse round: each lane stores its own few bits
        uint64_t at = o + excl;
        for (uint32_t v = x[q]; v; v &= v - 1, ++at)
          if (at < cap) sel[at] = bit0 + 32u * lane + static_cast<uint32_t>(__ffs(v) - 1);
        o += total;
        continue;
      }
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const uint32_t wk = __shfl_sync(kFull, x[q], k);
        if (wk == 0) continue;  // warp-uniform: sparse bitmaps skip their empty words
        const uint32_t ok = __shfl_sync(kFull, excl, k);
        if (wk >> lane & 1u) {
          const uint64_t at = o + ok + __popc(wk & lt);
          if (at < cap) sel[at] = bit0 + 32u * k + lane;
        }
      }
      o += total;
    }
    if (tile == ntiles - 1 && threadIdx.x == kTileBlock - 1) {
      // last tile, last warp: o is the grand total (popcount)
      plan->n_sel = o;
      plan->n_values = o;
    }
  }
}

__global__ void bitmap_popcount_check(Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_BITMAP) return;
  if (plan->il == 0) {
    plan->n_sel = 0;
    plan->n_values = 0;
  }
  if (plan->n_sel != plan->r) latch(status, GP_CORRUPT_PAYLOAD);  // pipeline.cpp:242-243
}

}  // namespace

void launch_index_none(gp_ctx* ctx, uint8_t* out, uint64_t r, cudaStream_t s) {
  GP_LAUNCH(ctx, index_none_encode, grid_for(ctx, r, 256), 256, 0, s, ctx->ws.support, r, out, ctx->ws.status);
}

void launch_index_bitmap(gp_ctx* ctx, uint8_t* out, uint64_t d, uint64_t r, cudaStream_t s) {
  Workspace& w = ctx->ws;
  fill_async(ctx, w.u32c, 0, ((d + 31) / 32) * 4, s);
  GP_LAUNCH(ctx, bitmap_scatter, grid_for(ctx, r, 256), 256, 0, s, w.support, r, w.u32c, w.status);
  GP_LAUNCH(ctx, bitmap_emit, grid_for(ctx, (d + 7) / 8, 256), 256, 0, s, w.u32c, d, out, w.status);
}

void launch_decode_index_none(gp_ctx* ctx, const uint8_t* in, uint64_t r_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, index_none_decode, grid_for(ctx, r_bound, 256), 256, 0, s, in, w.plan, w.sel, w.status);
}

void launch_validate_support(gp_ctx* ctx, uint64_t r_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, support_validate, grid_for(ctx, r_bound, 256), 256, 0, s, w.plan, w.sel, w.status);
}

void launch_decode_bitmap_check(gp_ctx* ctx, const uint8_t* in, cudaStream_t s) {
  GP_LAUNCH(ctx, bitmap_check, 1, 1, 0, s, in, ctx->ws.plan, ctx->ws.status);
}

void launch_decode_index_bitmap(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, bitmap_check, 1, 1, 0, s, in, w.plan, w.status);
  const uint64_t ntiles = ((d_bound + 7) / 8 + kTile - 1) / kTile;
  reset_scan(ctx, s, ntiles + 1);
  GP_LAUNCH(ctx, bitmap_support, grid_for(ctx, ntiles * kTileBlock, kTileBlock), kTileBlock, 0, s, in, w.plan,
            w.sel, w.tiles, w.ticket, static_cast<uint64_t>(ctx->max_d), w.status);
  GP_LAUNCH(ctx, bitmap_popcount_check, 1, 1, 0, s, w.plan, w.status);
}

// error feedback, own container: the decoded support of a none/bitmap/RLE
// container is the encoder's top-r support
namespace {
__global__ void own_support(Plan* plan, const uint32_t* __restrict__ support, uint32_t* sel, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t r = plan->r;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    sel[i] = support[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->n_sel = r;
    plan->n_values = r;
  }
}
}  // namespace

void launch_own_support(gp_ctx* ctx, uint64_t r_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, own_support, grid_for(ctx, r_bound, 256), 256, 0, s, w.plan, w.support, w.sel, w.status);
}

}  // namespace gp
