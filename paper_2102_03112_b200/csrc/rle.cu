// rle.cu — K3/K4: the run-length index payload (id 2; rle_encode/rle_decode,
// codecs.cpp:34-70; LEB128 groups inside the bit stream, bitio.hpp:79-99).
//
// Wire: 1 polarity bit (coordinate 0), then one varint per run, every group
// a full byte at bit offset 1 + 8t.  Byte t of the payload is therefore
// (group[t-1] >> 7) | (group[t] << 1) (byte 0: polarity | group[0] << 1), and
// the last byte is group[G-1] >> 7 = 0 since a varint's last group has a clear
// high bit.  Payload = G + 1 bytes.
//
// Encode from the ascending support: 1-runs are maximal chains of consecutive
// keys (ordered compaction of chain starts), each followed by its 0-gap; one
// thread per chain sizes its groups, a scan places them, the bytes are emitted
// with the one-bit shift.
//
// Decode reproduces the sequential reader's first failure exactly: groups are
// split into varints at their terminators, run lengths are scanned, and the
// first varint (in stream order) that is too long (> 10 groups), zero, or
// overruns d — or the absence of a completing run (truncation) — decides the
// error; a completed stream must end with < 8 zero slack bits.  The bitmap is
// the prefix-XOR of run-boundary toggles, and the support its set bits.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kBlock = 256;
constexpr int kItems = 16;
constexpr int kTile = kBlock * kItems;

__device__ __forceinline__ uint32_t vgroups(uint64_t x) {
  uint32_t g = 1;
  while (x >= 128) {
    x >>= 7;
    ++g;
  }
  return g;
}

__device__ __forceinline__ uint32_t put_varint(uint8_t* grp, uint64_t x) {
  uint32_t g = 0;
  do {
    uint8_t b = x & 0x7f;
    x >>= 7;
    if (x) b |= 0x80;
    grp[g++] = b;
  } while (x);
  return g;
}

// ---------------------------------------------------------------- encode
// chain starts of the ascending support: i == 0 or sup[i-1] + 1 != sup[i].
// Warp w of a tile owns entries [512w, 512w + 512) in 16 rounds of 32, lane l
// on entry 32q + l (coalesced; the predecessor comes from the lane below).
// Returns the round's start ballot.
__device__ __forceinline__ uint32_t start_ballot(const uint32_t* __restrict__ sup, uint64_t r, uint64_t i) {
  const int lane = threadIdx.x & 31;
  const uint32_t cur = i < r ? sup[i] : 0u;
  uint32_t prev = __shfl_up_sync(kFull, cur, 1);
  if (lane == 0 && i > 0 && i < r) prev = sup[i - 1];
  return __ballot_sync(kFull, i < r && (i == 0 || prev + 1 != cur));
}

// Starts are few (one per 1-run) and the support is long (r/4096 tiles):
// per-tile counts + one scan (scan_chunk_counts) place them.
__global__ void __launch_bounds__(kBlock) rle_starts_count(const uint32_t* __restrict__ sup, uint64_t r,
                                                           uint64_t* counts, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wc[kBlock / 32];
  if (failed(status)) return;
  const uint64_t ntiles = (r + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t wb = tile * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) c += __popc(start_ballot(sup, r, wb + 32 * q + lane));
    if (lane == 0) wc[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
#pragma unroll
      for (int w = 0; w < kBlock / 32; ++w) t += wc[w];
      counts[tile] = t;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) rle_starts(const uint32_t* __restrict__ sup, uint64_t r,
                                                     uint32_t* __restrict__ starts, Plan* plan,
                                                     const uint64_t* tile_offs, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  if (failed(status)) return;
  const uint64_t ntiles = (r + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t wb = tile * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t bal[kItems];
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      bal[q] = start_ballot(sup, r, wb + 32 * q + lane);
      c += __popc(bal[q]);
    }
    uint64_t tot;
    uint64_t o = tile_offs[tile] + block_exclusive_sum<uint64_t, kBlock>(lane == 0 ? c : 0, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      if (bal[q] >> lane & 1u) starts[o + __popc(bal[q] & lt)] = static_cast<uint32_t>(wb + 32 * q + lane);
      o += __popc(bal[q]);
    }
    if (tile == ntiles - 1 && threadIdx.x == kBlock - 1) plan->n_runs = o;
  }
}

// group count of chain k (its 1-run + the following 0-gap); exclusive scan
__global__ void __launch_bounds__(kBlock) rle_sizes(const uint32_t* __restrict__ sup, uint64_t r, uint64_t d,
                                                    const uint32_t* __restrict__ starts, Plan* plan,
                                                    uint32_t* __restrict__ goff, uint64_t* tiles, uint32_t* ticket,
                                                    const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint64_t R = plan->n_runs;
  const uint64_t lead = sup[0] > 0 ? vgroups(sup[0]) : 0;  // the leading 0-run
  const uint64_t ntiles = (R + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    // warp rounds: lane l on chain wb + 32q + l (coalesced loads of starts)
    const uint64_t wb = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t g[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t k = wb + 32 * q + lane;
      g[q] = 0;
      if (k < R) {
        const uint64_t i0 = starts[k], i1 = k + 1 < R ? starts[k + 1] : r;
        const uint64_t end = sup[i0] + (i1 - i0);
        const uint64_t gap = (k + 1 < R ? sup[i1] : d) - end;
        g[q] = vgroups(i1 - i0) + (gap ? vgroups(gap) : 0);
      }
      sum += g[q];
    }
    const uint32_t wsum = __reduce_add_sync(kFull, sum);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? wsum : 0, tile, tiles, sh, tot) + lead;
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint32_t incl = warp_inclusive_sum(g[q]);
      const uint64_t k = wb + 32 * q + lane;
      if (k < R) goff[k] = static_cast<uint32_t>(o + incl - g[q]);
      o += __shfl_sync(kFull, incl, 31);
    }
    if (tile == ntiles - 1 && threadIdx.x == kBlock - 1) {
      plan->n_groups = o;
      plan->il = o + 1;
    }
  }
}

__global__ void rle_groups(const uint32_t* __restrict__ sup, uint64_t r, uint64_t d,
                           const uint32_t* __restrict__ starts, const uint32_t* __restrict__ goff, const Plan* plan,
                           uint8_t* __restrict__ grp, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t R = plan->n_runs;
  if (blockIdx.x == 0 && threadIdx.x == 0 && sup[0] > 0) put_varint(grp, sup[0]);
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < R;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i0 = starts[k], i1 = k + 1 < R ? starts[k + 1] : r;
    const uint64_t end = sup[i0] + (i1 - i0);
    const uint64_t gap = (k + 1 < R ? sup[i1] : d) - end;
    uint8_t* g = grp + goff[k];
    g += put_varint(g, i1 - i0);
    if (gap) put_varint(g, gap);
  }
}

__global__ void rle_emit(const uint8_t* __restrict__ grp, const uint32_t* __restrict__ sup, const Plan* plan,
                         uint8_t* out, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t G = plan->n_groups;
  const uint8_t pol = sup[0] == 0 ? 1 : 0;
  uint8_t* p = out + 49;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t <= G;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t lo = t == 0 ? pol : (grp[t - 1] >> 7);
    const uint32_t hi = t < G ? static_cast<uint32_t>(grp[t]) << 1 : 0u;
    p[t] = static_cast<uint8_t>(lo | hi);
  }
}

// ---------------------------------------------------------------- decode
__device__ __forceinline__ uint32_t group_at(const uint8_t* p, uint64_t t) {
  return ((p[t] >> 1) | (p[t + 1] << 7)) & 0xFFu;
}

// terminator groups (high bit clear) in order: varint v ends at ends[v]
__global__ void __launch_bounds__(kBlock) rle_ends(const uint8_t* __restrict__ in, Plan* plan,
                                                   uint32_t* __restrict__ ends, uint64_t* tiles, uint32_t* ticket,
                                                   const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint8_t* p = in + plan->off_index;
  const uint64_t n = plan->il;
  const uint64_t gav = n >= 1 ? n - 1 : 0;  // complete groups in the stream
  const uint64_t ntiles = (gav + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    // warp rounds: lane l on group wb + 32q + l (coalesced byte loads)
    const uint64_t wb = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t bal[kItems];
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t t = wb + 32 * q + lane;
      bal[q] = __ballot_sync(kFull, t < gav && !(group_at(p, t) & 0x80u));
      c += __popc(bal[q]);
    }
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? c : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      if (bal[q] >> lane & 1u) ends[o + __popc(bal[q] & lt)] = static_cast<uint32_t>(wb + 32 * q + lane);
      o += __popc(bal[q]);
    }
    if (tile == ntiles - 1 && threadIdx.x == kBlock - 1) plan->n_runs = o;
  }
  if (gav == 0 && blockIdx.x == 0 && threadIdx.x == 0) plan->n_runs = 0;
}

// run length of varint v (a varint longer than 10 groups is flagged in rle_events)
__global__ void rle_values(const uint8_t* __restrict__ in, const Plan* plan, const uint32_t* __restrict__ ends,
                           uint64_t* __restrict__ runs, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint8_t* p = in + plan->off_index;
  const uint64_t V = plan->n_runs;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t start = v == 0 ? 0 : ends[v - 1] + 1ull;
    const uint64_t len = ends[v] - start + 1;
    uint64_t x = 0;
    for (uint64_t q = 0; q < len && q < 10; ++q) x |= static_cast<uint64_t>(group_at(p, start + q) & 0x7fu) << (7 * q);
    // saturate at d + 1 (any run > d overruns; keeps the u64 scan in range)
    runs[v] = x > plan->d ? plan->d + 1 : x;
  }
}

// inclusive scan of run lengths (u64), tiles of 4096 varints
__global__ void __launch_bounds__(kBlock) rle_scan(const Plan* plan, const uint64_t* __restrict__ runs,
                                                   uint64_t* __restrict__ cum, uint64_t* tiles, uint32_t* ticket,
                                                   const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint64_t V = plan->n_runs;
  const uint64_t ntiles = (V + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    // warp rounds (coalesced): lane l on varint wb + 32q + l
    const uint64_t wb = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint64_t x[kItems];
    uint64_t sum = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t v = wb + 32 * q + lane;
      x[q] = v < V ? runs[v] : 0;
      sum += x[q];
    }
    const uint64_t wsum = __shfl_sync(kFull, warp_inclusive_sum(sum), 31);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? wsum : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t incl = warp_inclusive_sum(x[q]);
      const uint64_t v = wb + 32 * q + lane;
      if (v < V) cum[v] = o + incl;
      o += __shfl_sync(kFull, incl, 31);
    }
  }
}

// first event in stream order: (v << 2) | type, type 0 long, 1 zero, 2 overrun, 3 done
__global__ void rle_events(const uint8_t* __restrict__ in, const Plan* plan, const uint32_t* __restrict__ ends,
                           const uint64_t* __restrict__ runs, const uint64_t* __restrict__ cum,
                           unsigned long long* first, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint64_t V = plan->n_runs, d = plan->d;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t start = v == 0 ? 0 : ends[v - 1] + 1ull;
    const uint64_t len = ends[v] - start + 1;
    const uint64_t before = v == 0 ? 0 : cum[v - 1];
    int type = -1;
    if (len > 10) type = 0;
    else if (runs[v] == 0) type = 1;
    else if (runs[v] > d - before) type = 2;
    else if (cum[v] == d) type = 3;
    if (type >= 0) atomicMin(first, (static_cast<unsigned long long>(v) << 2) | static_cast<unsigned>(type));
  }
}

// decide: error class, or the number of runs and the slack check
__global__ void rle_finish(const uint8_t* __restrict__ in, Plan* plan, const uint32_t* __restrict__ ends,
                           const unsigned long long* first, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint8_t* p = in + plan->off_index;
  const uint64_t n = plan->il, V = plan->n_runs;
  if (n == 0) return latch(status, GP_TRUNCATED);  // no polarity bit
  const unsigned long long f = *first;
  if (f == ~0ULL) {  // no terminating event among the complete varints
    const uint64_t gav = n - 1;
    const uint64_t tail = gav - (V ? ends[V - 1] + 1ull : 0);  // continuation groups after the last varint
    return latch(status, tail >= 10 ? GP_CORRUPT_PAYLOAD : GP_TRUNCATED);
  }
  const uint64_t v = f >> 2;
  const int type = static_cast<int>(f & 3);
  if (type != 3) return latch(status, GP_CORRUPT_PAYLOAD);
  const uint64_t e = ends[v];  // last group used
  if (n != e + 2) return latch(status, GP_CORRUPT_PAYLOAD);            // >= 8 slack bits
  if ((p[e + 1] >> 1) != 0) return latch(status, GP_CORRUPT_PAYLOAD);  // nonzero slack
  plan->n_runs = v + 1;
  plan->pd_variant = p[0] & 1u;  // polarity (scratch field on the decode path)
}

__global__ void rle_toggles(const Plan* plan, const uint64_t* __restrict__ cum, uint32_t* __restrict__ tog,
                            const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint64_t V = plan->n_runs, d = plan->d;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = cum[v];
    if (c < d) atomicOr(&tog[c >> 5], 1u << (c & 31));
  }
}

// bitmap = polarity XOR prefix-XOR(toggles); word parity carried by a scan
__global__ void __launch_bounds__(kBlock) rle_bitmap(const Plan* plan, uint32_t* __restrict__ words, uint64_t* tiles,
                                                     uint32_t* ticket, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint64_t d = plan->d, nw = (d + 31) / 32;
  const uint32_t pol = plan->pd_variant ? 0xFFFFFFFFu : 0u;
  const uint64_t ntiles = (nw + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    // warp rounds (coalesced): lane l on word wb + 32q + l; the inversion of a
    // word is the parity of the toggles in all earlier words
    const uint64_t wb = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t x[kItems];
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t w = wb + 32 * q + lane;
      x[q] = w < nw ? words[w] : 0u;
      c += __popc(x[q]);
    }
    const uint32_t wc = __reduce_add_sync(kFull, c);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? wc : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint32_t n = __popc(x[q]);
      const uint32_t incl = warp_inclusive_sum(n);
      uint32_t y = x[q];
      y ^= y << 1;
      y ^= y << 2;
      y ^= y << 4;
      y ^= y << 8;
      y ^= y << 16;
      uint32_t b = y ^ (((o + incl - n) & 1) ? 0xFFFFFFFFu : 0u) ^ pol;
      const uint64_t w = wb + 32 * q + lane;
      if (w < nw) {
        if (w == nw - 1 && (d & 31)) b &= (1u << (d & 31)) - 1u;
        words[w] = b;
      }
      o += __shfl_sync(kFull, incl, 31);
    }
  }
}

// set bits of the bitmap → ascending support (sel), n_sel; popcount must be r.
// Warp w of a tile owns words [512w, 512w + 512) in 16 rounds of 32 (lane l
// on word 32q + l: coalesced loads); emission is transposed as in
// bitmap_support (indexcodec.cu): for each word of a round the lanes whose
// bit is set store at their rank, one contiguous run per store instruction.
__global__ void __launch_bounds__(kBlock) rle_support(const uint32_t* __restrict__ words, Plan* plan,
                                                      uint32_t* __restrict__ sel, uint64_t cap, uint64_t* tiles,
                                                      uint32_t* ticket, const uint32_t* status) {
  gp_pdl_wait();
  constexpr int kRounds = kItems;
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  const uint64_t nw = (plan->d + 31) / 32;
  const uint64_t ntiles = (nw + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t wbase = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kRounds);
    uint32_t x[kRounds];
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kRounds; ++q) {
      const uint64_t w = wbase + 32 * q + lane;
      x[q] = w < nw ? words[w] : 0u;
      c += __popc(x[q]);
    }
    const uint32_t wc = __reduce_add_sync(kFull, c);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? wc : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
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
      const uint32_t bit0 = static_cast<uint32_t>(32 * (wbase + 32 * q));
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
        if (wk == 0) continue;
        const uint32_t ok = __shfl_sync(kFull, excl, k);
        if (wk >> lane & 1u) {
          const uint64_t at = o + ok + __popc(wk & lt);
          if (at < cap) sel[at] = bit0 + 32u * k + lane;
        }
      }
      o += total;
    }
    if (tile == ntiles - 1 && threadIdx.x == kBlock - 1) {
      plan->n_sel = o;
      plan->n_values = o;
    }
  }
}

__global__ void rle_check(Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_RLE) return;
  if (plan->n_sel != plan->r) latch(status, GP_CORRUPT_PAYLOAD);  // pipeline.cpp:249-250
}

__global__ void rle_reset(unsigned long long* first) {
  gp_pdl_wait(); *first = ~0ULL; }

}  // namespace

void launch_index_rle(gp_ctx* ctx, uint8_t* out, uint64_t d, uint64_t r, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t rt = (r + kTile - 1) / kTile;
  GP_LAUNCH(ctx, rle_starts_count, grid_for(ctx, rt * kBlock, kBlock), kBlock, 0, s, w.support, r, w.tiles,
            w.status);
  GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, w.tiles, nullptr, rt, w.status);
  GP_LAUNCH(ctx, rle_starts, grid_for(ctx, rt * kBlock, kBlock), kBlock, 0, s, w.support, r, w.u32a, w.plan, w.tiles,
            w.status);
  reset_scan(ctx, s, rt + 1);
  GP_LAUNCH(ctx, rle_sizes, grid_for(ctx, rt * kBlock, kBlock), kBlock, 0, s, w.support, r, d, w.u32a, w.plan, w.u32b,
            w.tiles, w.ticket, w.status);
  GP_LAUNCH(ctx, rle_groups, grid_for(ctx, r, 256), 256, 0, s, w.support, r, d, w.u32a, w.u32b, w.plan, w.scratch,
            w.status);
  GP_LAUNCH(ctx, rle_emit, grid_for(ctx, d + 1, 256), 256, 0, s, w.scratch, w.support, w.plan, out, w.status);
}

void launch_decode_index_rle(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, uint64_t d_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  unsigned long long* first = reinterpret_cast<unsigned long long*>(w.p2_alloc + 2);
  uint64_t* runs = reinterpret_cast<uint64_t*>(w.f64a);
  uint64_t* cum = reinterpret_cast<uint64_t*>(w.f64b);
  const uint64_t gt = (len_bound + kTile - 1) / kTile;
  GP_LAUNCH(ctx, rle_reset, 1, 1, 0, s, first);
  reset_scan(ctx, s, gt + 1);
  GP_LAUNCH(ctx, rle_ends, grid_for(ctx, gt * kBlock, kBlock), kBlock, 0, s, in, w.plan, w.u32a, w.tiles, w.ticket,
            w.status);
  GP_LAUNCH(ctx, rle_values, grid_for(ctx, len_bound, 256), 256, 0, s, in, w.plan, w.u32a, runs, w.status);
  reset_scan(ctx, s, gt + 1);
  GP_LAUNCH(ctx, rle_scan, grid_for(ctx, gt * kBlock, kBlock), kBlock, 0, s, w.plan, runs, cum, w.tiles, w.ticket,
            w.status);
  GP_LAUNCH(ctx, rle_events, grid_for(ctx, len_bound, 256), 256, 0, s, in, w.plan, w.u32a, runs, cum, first,
            w.status);
  GP_LAUNCH(ctx, rle_finish, 1, 1, 0, s, in, w.plan, w.u32a, first, w.status);
  const uint64_t nw = (d_bound + 31) / 32;
  fill_async(ctx, w.u32c, 0, nw * 4, s);
  GP_LAUNCH(ctx, rle_toggles, grid_for(ctx, len_bound, 256), 256, 0, s, w.plan, cum, w.u32c, w.status);
  const uint64_t wt = (nw + kTile - 1) / kTile;
  reset_scan(ctx, s, wt + 1);
  GP_LAUNCH(ctx, rle_bitmap, grid_for(ctx, wt * kBlock, kBlock), kBlock, 0, s, w.plan, w.u32c, w.tiles, w.ticket,
            w.status);
  reset_scan(ctx, s, wt + 1);
  GP_LAUNCH(ctx, rle_support, grid_for(ctx, wt * kBlock, kBlock), kBlock, 0, s, w.u32c, w.plan, w.sel,
            static_cast<uint64_t>(ctx->max_d), w.tiles, w.ticket, w.status);
  GP_LAUNCH(ctx, rle_check, 1, 1, 0, s, w.plan, w.status);
}

}  // namespace gp
