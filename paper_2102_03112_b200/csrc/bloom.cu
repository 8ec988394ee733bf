// bloom.cu — K5/K6: Bloom filter build and full-range membership scan
// (bloom.cpp:41-128, FORMAT.md:58-75), the filter payload, and the P0 / Pd /
// naive selections (pipeline.cpp:192-213, :261-293; bloom.cpp:130-138, :224-236).
//
// Probe positions: mix64(h_a(x) + i * h_b(x)) mod m, h_a = hash64(x, seed_a),
// h_b = hash64(x, seed_b).  The modulo is the exact 64-by-32 fast_mod
// (gp_device.cuh) since m < 2^32 on every configuration; h_b is computed
// lazily after the first probe hits (the reference computes it eagerly, the
// result is identical).
//
// The filter lives as u32 words in the workspace; their little-endian byte
// image IS the serialized LSB-first bit array, so the payload is a plain
// byte copy.  Build: one thread per key, k atomicOr's into the L2-resident
// words (r*k = 2.6M probes at C4).  Scan: ordered compaction over [0, d),
// 4096 keys per tile; the filter is staged in shared memory when it fits
// (<= 160 KiB: C1, C5 buckets), otherwise read through L1/L2 (C4: 459 KiB).
#include <cooperative_groups.h>

#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace cg = cooperative_groups;

namespace {

constexpr int kScanBlock = 256;
constexpr uint64_t kSmemFilterMax = 150 * 1024;

__global__ void bloom_insert(const uint32_t* __restrict__ keys, uint64_t r, const Plan* plan, uint32_t* words,
                             const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const FastMod fm{plan->m, plan->minv};
  const uint32_t k = plan->k;
  const uint64_t sa = plan->seed_a + kGamma, sb = plan->seed_b + kGamma;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = keys[i];
    const uint64_t a = mix64(x ^ sa), b = mix64(x ^ sb);
    uint64_t h = a;
    for (uint32_t j = 0; j < k; ++j, h += b) {
      const uint64_t pos = fast_mod(mix64(h), fm);
      atomicOr(&words[pos >> 5], 1u << (pos & 31));
    }
  }
}

// filter payload: m u64, k u16, seed_a u64, seed_b u64, ceil(m/8) bytes (+ Pd variant)
__global__ void bloom_emit(const uint32_t* __restrict__ words, const Plan* plan, uint8_t* out,
                           const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  uint8_t* p = out + 49;
  const uint64_t nb = (plan->m + 7) / 8;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st_u64_unaligned(p, plan->m);
    p[8] = static_cast<uint8_t>(plan->k);
    p[9] = static_cast<uint8_t>(plan->k >> 8);
    st_u64_unaligned(p + 10, plan->seed_a);
    st_u64_unaligned(p + 18, plan->seed_b);
    if (plan->index_method == GP_INDEX_BLOOM_PD) p[26 + nb] = plan->pd_variant;
  }
  const uint8_t* src = reinterpret_cast<const uint8_t*>(words);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nb;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[26 + i] = src[i];
}

// BloomFilter::deserialize (bloom.cpp:96-112) + pipeline.cpp:261-273 trailing checks.
__global__ void bloom_parse(const uint8_t* __restrict__ in, Plan* plan, uint64_t m_cap, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint8_t* p = in + plan->off_index;
  const uint64_t il = plan->il;
  if (il < 8) return latch(status, GP_TRUNCATED);
  const uint64_t m = ld_u64_unaligned(p);
  if (m < 1) return latch(status, GP_CORRUPT_PAYLOAD);
  if (il < 10) return latch(status, GP_TRUNCATED);
  const uint32_t k = p[8] | (p[9] << 8);
  if (k < 1) return latch(status, GP_CORRUPT_PAYLOAD);
  if (il < 26) return latch(status, GP_TRUNCATED);
  const uint64_t nb = (m + 7) / 8;
  if (il - 26 < nb) return latch(status, GP_TRUNCATED);
  const uint64_t tail = m % 64;  // bits past m within the last u64 word
  if (tail) {
    const uint64_t first_bad = m;                    // bit index
    const uint64_t last = 64 * ((m + 63) / 64);      // exclusive, in bits
    for (uint64_t b = first_bad; b < last && b < 8 * nb; ++b)
      if ((p[26 + b / 8] >> (b % 8)) & 1u) return latch(status, GP_CORRUPT_PAYLOAD);
  }
  uint64_t used = 26 + nb;
  if (im == GP_INDEX_BLOOM_PD) {
    if (il < used + 1) return latch(status, GP_TRUNCATED);
    const uint8_t v = p[used];
    if (v > 2) return latch(status, GP_CORRUPT_PAYLOAD);
    plan->pd_variant = v;
    used += 1;
  }
  if (il != used) return latch(status, GP_CORRUPT_PAYLOAD);
  if (m > m_cap || m >= (1ULL << 32)) return latch(status, GP_CAPACITY);
  plan->m = m;
  plan->k = k;
  plan->seed_a = ld_u64_unaligned(p + 10);
  plan->seed_b = ld_u64_unaligned(p + 18);
  plan->minv = ~0ULL / m;
}

// aligned filter words from the payload bytes
__global__ void bloom_load_words(const uint8_t* __restrict__ in, const Plan* plan, uint32_t* words,
                                 const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint8_t* p = in + plan->off_index + 26;
  const uint64_t nb = (plan->m + 7) / 8;
  const uint64_t nw = (plan->m + 31) / 32;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < nw;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t v = 0;
    for (int j = 0; j < 4; ++j)
      if (4 * w + j < nb) v |= static_cast<uint32_t>(p[4 * w + j]) << (8 * j);
    words[w] = v;
  }
}

// positive_scan (bloom.cpp:123-128) in two passes.
//
// (1) bloom_members: contains() exits at the first clear probe, so ~half the
// keys stop after one probe, a quarter after two, ...; a lane-per-key loop
// keeps a warp busy for its slowest lane.  Each warp instead keeps a shared
// work stack of pending probes (key, next probe j, h = h_a + j*h_b, h_b) and
// alternates two converged steps:
//   * first probes: kLaneKeys consecutive keys per lane (a chunk of
//     32*kLaneKeys keys); survivors are pushed with h_b computed once, in a
//     lane-strided pass over the new entries;
//   * a probe batch: pop 32*kLaneBatch entries (kLaneBatch independent probes
//     per lane in flight), test probe j, push survivors back with j+1 and
//     h += h_b; a key passing its k-th probe sets its bit in the d-bit
//     membership bitmap (zeroed beforehand; one atomicOr per member).
// A batch runs whenever the stack holds a full batch, so lanes stay busy
// across chunk boundaries instead of idling through each chunk's thin tail.
// (2) members_compact: ordered compaction of the set bits (look-back scan)
// — P ascending, |P| in the plan.
constexpr int kWarps = kScanBlock / 32;

template <bool kSmem, int kLaneKeys, int kLaneBatch>
struct ScanShape {
  static constexpr int kChunk = 32 * kLaneKeys;
  static constexpr int kBatch = 32 * kLaneBatch;
  static constexpr int kCap = kBatch + kChunk;  // stack < kBatch before a chunk pushes <= kChunk
  static constexpr size_t kStackBytes = static_cast<size_t>(kWarps) * kCap * (8 + 8 + 4 + 2);
};

// probe position of hash h (mix64(h) mod m): 32-bit tail when m <= 2^31
template <bool kSmallM>
__device__ __forceinline__ uint32_t probe_pos(uint64_t h, const FastMod& fm) {
  if (kSmallM) return fast_mod_small(mix64(h), fm.minv, static_cast<uint32_t>(fm.m));
  return static_cast<uint32_t>(fast_mod(mix64(h), fm));  // m < 2^32
}

template <bool kSmallM, int kLaneKeys, int kLaneBatch, int kCap>
__device__ __forceinline__ void members_body(const uint32_t* __restrict__ words, const Plan* plan,
                                             uint32_t* __restrict__ bitmap, uint8_t* dyn) {
  constexpr int kChunk = 32 * kLaneKeys, kBatch = 32 * kLaneBatch;
  // keys [lo, lo + d): the whole range, or a slice (gp_bloom_scan_range); the
  // stack holds global keys, the membership bitmap is slice-relative
  const uint32_t lo = static_cast<uint32_t>(plan->scan_lo);
  const uint32_t d = static_cast<uint32_t>(plan->scan_hi ? plan->scan_hi - plan->scan_lo : plan->d);
  const uint32_t k = plan->k;
  const FastMod fm{plan->m, plan->minv};
  const uint64_t sa = plan->seed_a + kGamma, sb = plan->seed_b + kGamma;
  // shared layout: [stack h | stack b | stack key | stack j]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* qh = reinterpret_cast<uint64_t*>(dyn) + warp * kCap;
  uint64_t* qb = reinterpret_cast<uint64_t*>(dyn) + (kWarps + warp) * kCap;
  uint32_t* qx = reinterpret_cast<uint32_t*>(dyn + 16 * kWarps * kCap) + warp * kCap;
  uint16_t* qj = reinterpret_cast<uint16_t*>(dyn + 20 * kWarps * kCap) + warp * kCap;  // k <= 65535
  const uint32_t nchunks = (d + kChunk - 1) / kChunk;
  const uint32_t nwarps = gridDim.x * kWarps;
  uint32_t c = blockIdx.x * kWarps + warp;
  uint32_t top = 0;  // warp-uniform stack height
  while (true) {
    if (top >= kBatch || (c >= nchunks && top > 0)) {
      // ---- probe batch: positions, then every word load, then the tests
      const uint32_t n = top < kBatch ? top : kBatch;
      const uint32_t base = top - n;
      uint32_t x[kLaneBatch], j[kLaneBatch], pos[kLaneBatch], wv[kLaneBatch];
      uint64_t h[kLaneBatch], hb[kLaneBatch];
#pragma unroll
      for (int u = 0; u < kLaneBatch; ++u) {
        const uint32_t e = min(base + 32 * u + lane, top - 1);  // clamped: duplicates are discarded
        x[u] = qx[e];
        j[u] = qj[e];
        h[u] = qh[e];
        hb[u] = qb[e];
        pos[u] = probe_pos<kSmallM>(h[u], fm);
      }
#pragma unroll
      for (int u = 0; u < kLaneBatch; ++u) wv[u] = words[pos[u] >> 5];
      __syncwarp();
      uint32_t wr = base;
#pragma unroll
      for (int u = 0; u < kLaneBatch; ++u) {
        const bool ok = base + 32 * u + lane < top && ((wv[u] >> (pos[u] & 31)) & 1u);
        const bool member = ok && j[u] + 1u == k;
        if (member) atomicOr(&bitmap[(x[u] - lo) >> 5], 1u << ((x[u] - lo) & 31));
        const bool keep = ok && !member;
        const unsigned bal = __ballot_sync(kFull, keep);
        if (keep) {
          const uint32_t e = wr + __popc(bal & ((1u << lane) - 1));
          qx[e] = x[u];
          qj[e] = static_cast<uint16_t>(j[u] + 1);
          qh[e] = h[u] + hb[u];
          qb[e] = hb[u];
        }
        wr += __popc(bal);
      }
      top = wr;
      __syncwarp();
    } else if (c < nchunks) {
      // ---- first probes of one chunk (positions, loads, tests)
      const uint32_t x0 = c * kChunk + kLaneKeys * lane;
      uint64_t av[kLaneKeys];
      uint32_t pos[kLaneKeys], wv[kLaneKeys];
#pragma unroll
      for (int q = 0; q < kLaneKeys; ++q) {
        av[q] = mix64(static_cast<uint64_t>(lo + x0 + q) ^ sa);
        pos[q] = probe_pos<kSmallM>(av[q], fm);
      }
#pragma unroll
      for (int q = 0; q < kLaneKeys; ++q) wv[q] = words[pos[q] >> 5];
      uint32_t pass = 0;
#pragma unroll
      for (int q = 0; q < kLaneKeys; ++q)
        pass |= ((wv[q] >> (pos[q] & 31)) & 1u) << q;
      if (x0 + kLaneKeys > d) pass &= x0 >= d ? 0u : (1u << (d - x0)) - 1u;
      c += nwarps;
      if (k == 1) {
        // kLaneKeys divides 32: a lane's keys share one bitmap word
        if (pass) atomicOr(&bitmap[x0 >> 5], pass << (x0 & 31));
        continue;
      }
      const uint32_t cnt = __popc(pass);
      const uint32_t inc = warp_inclusive_sum(cnt);
      uint32_t o = top + inc - cnt;
#pragma unroll
      for (int q = 0; q < kLaneKeys; ++q)
        if (pass >> q & 1u) {
          qx[o] = lo + x0 + q;
          qh[o] = av[q];
          ++o;
        }
      const uint32_t added = __shfl_sync(kFull, inc, 31);
      __syncwarp();
      for (uint32_t e = top + lane; e < top + added; e += 32) {  // h_b once per survivor
        const uint64_t b = mix64(static_cast<uint64_t>(qx[e]) ^ sb);
        qb[e] = b;
        qh[e] += b;
        qj[e] = 1;
      }
      top += added;
      __syncwarp();
    } else {
      break;
    }
  }
}

template <bool kSmem, int kLaneKeys, int kLaneBatch>
__global__ void __launch_bounds__(kScanBlock) bloom_members(const uint32_t* __restrict__ gwords, Plan* plan,
                                                            uint32_t* __restrict__ bitmap,
                                                            const uint32_t* status) {
  gp_pdl_wait();
  using S = ScanShape<kSmem, kLaneKeys, kLaneBatch>;
  extern __shared__ __align__(16) uint8_t dyn[];
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t m = plan->m;
  const uint32_t* words = gwords;
  if (kSmem) {
    uint32_t* sw = reinterpret_cast<uint32_t*>(dyn + (S::kStackBytes + 15) / 16 * 16);
    const uint64_t nw = (m + 31) / 32;
    for (uint64_t i = threadIdx.x; i < nw; i += kScanBlock) sw[i] = gwords[i];
    __syncthreads();
    words = sw;
  }
  if (m <= (1ull << 31))
    members_body<true, kLaneKeys, kLaneBatch, S::kCap>(words, plan, bitmap, dyn);
  else
    members_body<false, kLaneKeys, kLaneBatch, S::kCap>(words, plan, bitmap, dyn);
}

// ordered compaction of the membership bitmap: 16 words per thread, in warp
// rounds (lane l on word 32q + l of its warp's 512: coalesced loads); P is
// ~1% of d, so each lane stores its own few bits at its rank
__global__ void __launch_bounds__(kScanBlock) members_compact(const uint32_t* __restrict__ bitmap, Plan* plan,
                                                              uint32_t* __restrict__ pos_out, uint64_t cap,
                                                              uint64_t* tiles, uint32_t* ticket,
                                                              const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t lo = plan->scan_lo;
  const uint64_t nwd = ((plan->scan_hi ? plan->scan_hi - lo : plan->d) + 31) / 32;
  constexpr int kW = 16;
  const uint64_t ntiles = (nwd + kScanBlock * kW - 1) / (kScanBlock * kW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t wb = static_cast<uint64_t>(tile) * kScanBlock * kW + static_cast<uint64_t>(warp) * (32 * kW);
    uint32_t v[kW];
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      const uint64_t w = wb + 32 * i + lane;
      v[i] = w < nwd ? bitmap[w] : 0u;
      c += __popc(v[i]);
    }
    const uint32_t wc = __reduce_add_sync(kFull, c);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kScanBlock>(lane == 0 ? wc : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      const uint32_t n = __popc(v[i]);
      const uint32_t incl = warp_inclusive_sum(n);
      uint64_t at = o + incl - n;
      for (uint32_t x = v[i]; x; x &= x - 1, ++at)
        if (at < cap) pos_out[at] = static_cast<uint32_t>(lo + 32 * (wb + 32 * i + lane) + (__ffs(x) - 1));
      o += __shfl_sync(kFull, incl, 31);
    }
    if (tile == ntiles - 1 && threadIdx.x == kScanBlock - 1) plan->n_pos = o;
  }
}

// The same compaction as one cooperative launch of one block per tile (when
// the tiles fit one resident wave): every block keeps its 16 words per thread
// in registers, publishes its tile's member count, and after one grid
// barrier reads its offset — the sum of the earlier tiles' counts, one warp
// read — instead of spinning on a decoupled look-back chain (~200 tiles at
// C4: 19 us).
__device__ __forceinline__ void after_scan_body(Plan* plan, uint64_t n, uint64_t cap, int decoding,
                                                uint32_t* status);

// (the last tile's last thread also runs the post-scan bookkeeping of
// bloom_after_scan: one launch fewer per scan)
__global__ void __launch_bounds__(kScanBlock) members_compact_coop(const uint32_t* __restrict__ bitmap, Plan* plan,
                                                                   uint32_t* __restrict__ pos_out, uint64_t cap,
                                                                   uint64_t* tcnt, int decoding, uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  cg::grid_group grid = cg::this_grid();
  if (failed(status)) return;  // uniform: nothing latches this word while the kernel runs
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t lo = plan->scan_lo;
  const uint64_t nwd = ((plan->scan_hi ? plan->scan_hi - lo : plan->d) + 31) / 32;
  constexpr int kW = 16;
  const uint64_t ntiles = (nwd + kScanBlock * kW - 1) / (kScanBlock * kW);
  const uint64_t tile = blockIdx.x;
  const bool live = tile < ntiles;  // blocks past the last tile only join the barrier
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wb = tile * kScanBlock * kW + static_cast<uint64_t>(warp) * (32 * kW);
  uint32_t v[kW];
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kW; ++i) {
    const uint64_t w = wb + 32 * i + lane;
    v[i] = live && w < nwd ? bitmap[w] : 0u;
    c += __popc(v[i]);
  }
  const uint32_t wc = __reduce_add_sync(kFull, c);
  uint64_t tot;
  const uint64_t local = block_exclusive_sum<uint64_t, kScanBlock>(lane == 0 ? wc : 0, sh, tot);
  if (live && threadIdx.x == 0) tcnt[tile] = tot;
  grid.sync();
  if (!live) return;
  if (warp == 0) {
    uint64_t p = 0;
    for (uint64_t t = lane; t < tile; t += 32) p += __ldcg(tcnt + t);
    p = warp_sum(p);
    if (lane == 0) sh[34] = p;
  }
  __syncthreads();
  uint64_t o = __shfl_sync(kFull, sh[34] + local, 0);
#pragma unroll
  for (int i = 0; i < kW; ++i) {
    const uint32_t n = __popc(v[i]);
    const uint32_t incl = warp_inclusive_sum(n);
    uint64_t at = o + incl - n;
    for (uint32_t x = v[i]; x; x &= x - 1, ++at)
      if (at < cap) pos_out[at] = static_cast<uint32_t>(lo + 32 * (wb + 32 * i + lane) + (__ffs(x) - 1));
    o += __shfl_sync(kFull, incl, 31);
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanBlock - 1) {
    plan->n_pos = o;
    after_scan_body(plan, o, cap, decoding, status);
  }
}

// Post-scan bookkeeping: |P| >= r (pipeline.cpp:284-285), value counts, and
// the P0 / Pd / naive selections which are slices of P.
__device__ __forceinline__ void after_scan_body(Plan* plan, uint64_t n, uint64_t cap, int decoding,
                                                uint32_t* status) {
  const uint8_t im = plan->index_method;
  const uint64_t r = plan->r;
  if (n > cap) return latch(status, GP_CAPACITY);
  if (im == GP_INDEX_BLOOM_P0) {
    plan->n_sel = n;
    plan->n_values = n;
  } else if (im == GP_INDEX_BLOOM_NAIVE) {
    plan->n_sel = n;       // decode scatters over all of P
    plan->n_values = r;    // values carried for r entries (pipeline.cpp:275-277)
  } else {
    if (n < r) return latch(status, decoding ? GP_CORRUPT_PAYLOAD : GP_ERROR);
    plan->n_sel = r;
    plan->n_values = r;
  }
}

__global__ void bloom_after_scan(Plan* plan, uint64_t cap, int decoding, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  after_scan_body(plan, plan->n_pos, cap, decoding, status);
}

// sel <- P (P0, naive) or the Pd slice (bloom.cpp:224-236)
__global__ void select_slice(const uint32_t* __restrict__ P, const Plan* plan, uint32_t* sel,
                             const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  uint64_t begin = 0, count = 0;
  if (im == GP_INDEX_BLOOM_P0 || im == GP_INDEX_BLOOM_NAIVE) {
    count = plan->n_pos;
  } else if (im == GP_INDEX_BLOOM_PD) {
    const uint64_t n = plan->n_pos, r = plan->r;
    begin = plan->pd_variant == 0 ? 0 : plan->pd_variant == 1 ? (n - r) / 2 : n - r;
    count = r;
  } else {
    return;
  }
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    sel[i] = P[begin + i];
}

}  // namespace

void launch_bloom_build(gp_ctx* ctx, uint8_t* out, uint64_t m, uint64_t r, cudaStream_t s) {
  Workspace& w = ctx->ws;
  fill_async(ctx, w.filter, 0, ((m + 31) / 32) * 4, s);
  GP_LAUNCH(ctx, bloom_insert, grid_for(ctx, r, 128), 128, 0, s, w.support, r, w.plan, w.filter, w.status);
  GP_LAUNCH(ctx, bloom_emit, grid_for(ctx, (m + 7) / 8, 256), 256, 0, s, w.filter, w.plan, out, w.status);
}

void launch_bloom_parse(gp_ctx* ctx, const uint8_t* in, uint64_t m_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, bloom_parse, 1, 1, 0, s, in, w.plan, w.m_cap, w.status);
  GP_LAUNCH(ctx, bloom_load_words, grid_for(ctx, (m_bound + 31) / 32, 256), 256, 0, s, in, w.plan, w.filter,
            w.status);
}

template <int kLaneKeys, int kLaneBatch>
void launch_members_global(gp_ctx* ctx, uint64_t d_bound, uint32_t* bitmap, cudaStream_t s) {
  Workspace& w = ctx->ws;
  using S = ScanShape<false, kLaneKeys, kLaneBatch>;
  auto* kern = bloom_members<false, kLaneKeys, kLaneBatch>;
  const int per_sm = std::max<int>(1, std::min<int>(8, static_cast<int>((200 * 1024) / (S::kStackBytes + 1024))));
  const uint64_t nchunks = (d_bound + S::kChunk - 1) / S::kChunk;
  const int grid = static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>((nchunks + kWarps - 1) / kWarps, static_cast<uint64_t>(ctx->sm_count) * per_sm)));
  GP_LAUNCH(ctx, kern, grid, kScanBlock, S::kStackBytes, s, w.filter, w.plan, bitmap, w.status);
}

// m_host: the filter width when the host knows it (encode), else 0 (decode:
// the width is only on the device, so the global-memory variant is used).
void launch_bloom_scan(gp_ctx* ctx, uint64_t d_bound, uint64_t m_host, bool decoding, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t fbytes = ((m_host + 31) / 32) * 4;
  uint32_t* bitmap = w.u32c;  // d-bit membership bitmap
  const uint64_t nwd = (d_bound + 31) / 32;
  fill_async(ctx, bitmap, 0, nwd * 4, s);
  if (m_host && fbytes <= kSmemFilterMax) {
    using S = ScanShape<true, 4, 2>;
    auto* kern = bloom_members<true, 4, 2>;
    const size_t smem = (S::kStackBytes + 15) / 16 * 16 + fbytes;
    const int per_sm = std::max(1, static_cast<int>((220 * 1024) / (smem + 1024)));
    const uint64_t nchunks = (d_bound + S::kChunk - 1) / S::kChunk;
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((nchunks + kWarps - 1) / kWarps, static_cast<uint64_t>(ctx->sm_count) * per_sm)));
    GP_LAUNCH(ctx, kern, grid, kScanBlock, smem, s, w.filter, w.plan, bitmap, w.status);
  } else {
    launch_members_global<4, 4>(ctx, d_bound, bitmap, s);  // 4 first probes / 4 batch probes per lane in flight
  }
  const uint64_t ntiles = (nwd + kScanBlock * 16 - 1) / (kScanBlock * 16);
  static int coop_per_sm = -1;
  if (coop_per_sm < 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&coop_per_sm, members_compact_coop, kScanBlock, 0);
  if (ntiles <= static_cast<uint64_t>(coop_per_sm) * ctx->sm_count && ntiles <= w.tiles_cap) {
    int grid = static_cast<int>(std::max<uint64_t>(1, ntiles));
    uint32_t* bm = bitmap;
    Plan* plan = w.plan;
    uint32_t* pos = w.pos;
    uint64_t cap = ctx->max_d;
    uint64_t* tc = w.tiles;
    int dec = decoding ? 1 : 0;
    uint32_t* st = w.status;
    void* args[] = {&bm, &plan, &pos, &cap, &tc, &dec, &st};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(members_compact_coop), grid, kScanBlock, args, 0, s);
    ++ctx->launches;
  } else {
    reset_scan(ctx, s, ntiles + 1);
    GP_LAUNCH(ctx, members_compact,
              static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL))), kScanBlock, 0,
              s, bitmap, w.plan, w.pos, ctx->max_d, w.tiles, w.ticket, w.status);
    GP_LAUNCH(ctx, bloom_after_scan, 1, 1, 0, s, w.plan, ctx->max_d, decoding ? 1 : 0, w.status);
  }
}

void launch_bloom_after_scan(gp_ctx* ctx, bool decoding, cudaStream_t s) {
  GP_LAUNCH(ctx, bloom_after_scan, 1, 1, 0, s, ctx->ws.plan, ctx->max_d, decoding ? 1 : 0, ctx->ws.status);
}

void launch_select_slice(gp_ctx* ctx, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, select_slice, grid_for(ctx, n_bound, 256), 256, 0, s, w.pos, w.plan, w.sel, w.status);
}

// dynamic shared-memory opt-ins of this file's kernels, on the current device
// (gp_ctx_create runs it once per context)
void kernel_attrs_bloom() {
  using G = ScanShape<false, 4, 4>;
  using M = ScanShape<true, 4, 2>;
  cudaFuncSetAttribute(bloom_members<false, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(G::kStackBytes));
  cudaFuncSetAttribute(bloom_members<true, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>((M::kStackBytes + 15) / 16 * 16 + kSmemFilterMax));
}

}  // namespace gp
