// p2.cu — K9/K10: conflict sets and the P2 greedy selection
// (conflict_sets bloom.cpp:156-173, p2_select bloom.cpp:175-222), bit-exact.
//
// conflict_sets: every positive x (in P order) contributes its k probe
// positions; a bit's set is the ascending, de-duplicated list of positives
// probing it; sets are ordered by (size, bit).  Device form:
//   pairs    : one thread per positive, k positions de-duplicated in
//              registers, per-bit distinct counts = set sizes, each pair's
//              slot in its set from the count atomic
//   tiles    : per 4096-bit tile: bucket space for multi sets from a global
//              cursor, and the tile's histogram of set sizes
//   scatter  : per pair: a singleton's member is recorded and selected
//              (stage A); multi-set members go to their bucket
//   order    : one stable counting-sort pass by size over the bit domain,
//              which also compacts away empty bits → sets in (size, bit)
//              order (members stay unsorted; the engine ranks them)
//
// p2_select: pass 1 first visits every singleton (bit order) and selects its
// member.  Singleton members are always true keys (a false positive's probes
// all land on bits set by true keys, so they are shared), hence at most r
// distinct, and selection is a set: stage A is one parallel flag write.  When
// a crafted filter breaks that bound (decode only) the exact sequential engine
// below replays pass 1 from the first singleton instead.
// Stage B is inherently sequential (each visit depends on earlier selections
// and consumes the CounterRng stream): one warp walks the non-singleton sets
// in order, repeating passes until r are selected.  A set whose unselected
// member count is 0 retires, 1 selects it, >= 2 draws below(cnt) from the
// stream (rng.hpp:52-59, rejection exact) and selects that member.  Retired
// sets need no flag: revisiting them changes nothing and draws nothing.
#include <cooperative_groups.h>

#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace cg = cooperative_groups;

namespace {

constexpr int kTileBlock = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileBlock * kTileItems;
constexpr uint32_t kBigSet = 255;  // counting-sort digit of every set of >= 255 members (p2_sort_large orders them)
constexpr uint32_t kSingleton = 0x80000000u;  // slot flag of a size-1 set (bucket offsets < 2^31)

__device__ __forceinline__ bool p2_active(const Plan* plan) {
  return plan->index_method == GP_INDEX_BLOOM_P2;
}

// count[0, m] = 0 with m read on the device (decode only knows it there),
// the stage-A flags over P and the bucket-space cursor
__global__ void p2_zero_counts(Plan* plan, uint32_t* count, uint64_t m_cap, uint8_t* flags, uint64_t n_cap,
                               uint32_t* alloc, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p2_active(plan)) return;
  const uint64_t n = (plan->m < m_cap ? plan->m : m_cap) + 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->n_large = 0;
    plan->n_single_sel = 0;  // counted by p2_size_scatter's stage-A pass
    *alloc = 0;
  }
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t n4 = n / 4;
  uint4* c4 = reinterpret_cast<uint4*>(count);
  for (uint64_t i = t0; i < n4; i += stride) c4[i] = make_uint4(0, 0, 0, 0);
  for (uint64_t i = 4 * n4 + t0; i < n; i += stride) count[i] = 0;
  const uint64_t np = plan->n_pos < n_cap ? plan->n_pos : n_cap;
  for (uint64_t i = t0; i < (np + 15) / 16; i += stride) reinterpret_cast<uint4*>(flags)[i] = make_uint4(0, 0, 0, 0);
}

// One thread per positive p: h_a, h_b once, then its k probe positions
// mix64(h_a + j h_b) mod m (bloom.cpp:27-33), de-duplicated among themselves
// (one positive joins a set once, the consecutive-duplicate rule of
// bloom.cpp:159-164) — the first kReg in registers, beyond them (k > 16,
// eps < 2^-16) an earlier position recomputed per comparison.  count[bit]
// ends as the set's size; the count atomic hands each pair its slot in its
// set (all of a positive's atomics issued before any result is used).  Pair
// arrays are probe-major (j * n + p): each store instruction is coalesced.
template <bool kSmallM>
__device__ __forceinline__ void pairs_thread(const uint32_t* __restrict__ P, uint64_t n, uint32_t k,
                                             const FastMod& fm, uint64_t sa, uint64_t sb,
                                             uint32_t* __restrict__ pairs, uint32_t* __restrict__ rank,
                                             uint32_t* __restrict__ count) {
  constexpr int kReg = 16;
  auto probe = [&](uint64_t h) {
    return kSmallM ? fast_mod_small(mix64(h), fm.minv, static_cast<uint32_t>(fm.m))
                   : static_cast<uint32_t>(fast_mod(mix64(h), fm));
  };
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = P[p];
    const uint64_t a = mix64(x ^ sa), b = mix64(x ^ sb);
    uint32_t bit[kReg], rk[kReg];
    uint32_t keep = 0;  // bit j: probe j is the first occurrence of its position
#pragma unroll
    for (int j = 0; j < kReg; ++j) {
      bit[j] = j < static_cast<int>(k) ? probe(a + static_cast<uint64_t>(j) * b) : 0xFFFFFFFFu;
      bool dup = false;
#pragma unroll
      for (int i = 0; i < j; ++i) dup |= bit[i] == bit[j];
      if (j < static_cast<int>(k) && !dup) keep |= 1u << j;
    }
#pragma unroll
    for (int j = 0; j < kReg; ++j)
      if (keep >> j & 1u) rk[j] = atomicAdd(&count[bit[j]], 1u);
#pragma unroll
    for (int j = 0; j < kReg; ++j) {
      if (j < static_cast<int>(k)) {
        pairs[j * n + p] = (keep >> j & 1u) ? bit[j] : 0xFFFFFFFFu;
        if (keep >> j & 1u) rank[j * n + p] = rk[j];
      }
    }
    for (uint32_t j = kReg; j < k; ++j) {
      const uint32_t bj = probe(a + static_cast<uint64_t>(j) * b);
      bool dup = false;
#pragma unroll
      for (int i = 0; i < kReg; ++i) dup |= bit[i] == bj;
      for (uint32_t i = kReg; i < j && !dup; ++i) dup = probe(a + static_cast<uint64_t>(i) * b) == bj;
      pairs[j * n + p] = dup ? 0xFFFFFFFFu : bj;
      if (!dup) rank[j * n + p] = atomicAdd(&count[bj], 1u);
    }
  }
}

__global__ void __launch_bounds__(256) p2_pairs(const uint32_t* __restrict__ P, Plan* plan,
                                                uint32_t* __restrict__ pairs, uint32_t* __restrict__ rank,
                                                uint32_t* __restrict__ count, uint64_t pair_cap, uint64_t set_cap,
                                                uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p2_active(plan)) return;
  const uint64_t n = plan->n_pos, m = plan->m;
  const uint32_t k = plan->k;
  if (n * k > pair_cap || n * k >= kSingleton || m > set_cap || k > 64) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_CAPACITY);
    return;
  }
  const FastMod fm{m, plan->minv};
  const uint64_t sa = plan->seed_a + kGamma, sb = plan->seed_b + kGamma;
  if (m <= (1ull << 31))
    pairs_thread<true>(P, n, k, fm, sa, sb, pairs, rank, count);
  else
    pairs_thread<false>(P, n, k, fm, sa, sb, pairs, rank, count);
  if (blockIdx.x == 0 && threadIdx.x == 0) plan->n_pairs = n * k;
}

// One 4096-bit tile per block: bucket space for multi sets (count >= 2) from a
// global cursor (warp-aggregated; the CSR needs contiguity, not bit order),
// scatter cursors, and the tile's histogram of set sizes for the (size, bit)
// ordering (digit-major table[size * ntiles + tile]).
__global__ void __launch_bounds__(kTileBlock) p2_tiles(const uint32_t* __restrict__ count, Plan* plan,
                                                       uint32_t* __restrict__ slot, uint32_t* __restrict__ table,
                                                       uint32_t* alloc, uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t h[256];
  __shared__ uint32_t sh32[33];
  __shared__ uint32_t s_base;
  if (failed(status) || !p2_active(plan)) return;
  const uint64_t m = plan->m;
  const uint64_t ntiles = (m + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    uint32_t c[kTileItems];
    uint32_t need = 0;
    uint32_t small[4] = {0, 0, 0, 0};  // sizes 1..4 (almost every set) counted in registers
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      const uint64_t b = tile * kTile + static_cast<uint64_t>(q) * kTileBlock + threadIdx.x;
      c[q] = b < m ? count[b] : 0;
    }
    uint32_t big = 0;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
#pragma unroll
      for (int z = 0; z < 4; ++z) small[z] += c[q] == static_cast<uint32_t>(z + 1) ? 1u : 0u;
      if (c[q] > 4) atomicAdd(&h[c[q] < kBigSet ? c[q] : kBigSet], 1u);
      big += c[q] >= kBigSet ? 1u : 0u;
      need += c[q];
    }
    big = __reduce_add_sync(kFull, big);
    if ((threadIdx.x & 31) == 0 && big) atomicAdd(reinterpret_cast<unsigned long long*>(&plan->n_large), big);
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const uint32_t v = __reduce_add_sync(kFull, small[z]);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(&h[z + 1], v);
    }
    uint32_t tot;
    uint32_t o = block_exclusive_sum<uint32_t, kTileBlock>(need, sh32, tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(alloc, tot) : 0;  // one allocation per tile
    __syncthreads();
    o += s_base;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      if (c[q]) {
        const uint64_t b = tile * kTile + static_cast<uint64_t>(q) * kTileBlock + threadIdx.x;
        slot[b] = o | (c[q] == 1 ? kSingleton : 0u);  // bucket start; a pair's rank places it
        o += c[q];
      }
    }
    table[threadIdx.x * ntiles + tile] = h[threadIdx.x];
    __syncthreads();
  }
}

// One thread per pair: a size-1 set's member is selected in stage A (every
// singleton is visited first, p2_select pass 1; plain byte flags,
// idempotent); every member goes to bucket start + its rank (the slot
// p2_pairs' count atomic handed out) — no atomics here.  Buckets stay
// unsorted: the engine ranks members by value.
__global__ void p2_scatter(const uint32_t* __restrict__ pairs, const uint32_t* __restrict__ rank, const Plan* plan,
                           const uint32_t* __restrict__ slot, uint32_t* __restrict__ members,
                           uint8_t* __restrict__ flags, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p2_active(plan)) return;
  const uint64_t n = plan->n_pos;
  const uint32_t k = plan->k;
  const uint64_t np = n * k;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // kU pairs per thread per step, strided by the grid: kU independent chains in flight
  constexpr int kU = 8;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < np; i0 += kU * stride) {
    uint32_t bit[kU], v[kU], rk[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      bit[u] = i < np ? pairs[i] : 0xFFFFFFFFu;
      rk[u] = i < np ? rank[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = bit[u] != 0xFFFFFFFFu ? slot[bit[u]] : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (bit[u] == 0xFFFFFFFFu) continue;
      const uint64_t i = i0 + u * stride;
      const uint32_t p = static_cast<uint32_t>(np < (1ull << 32) ? static_cast<uint32_t>(i) % static_cast<uint32_t>(n)
                                                                 : i % n);  // probe-major: i = j * n + p
      members[(v[u] & ~kSingleton) + rk[u]] = p;
      if (v[u] & kSingleton) flags[p] = 1;  // flags were zeroed; every writer stores the same value
    }
  }
}

// Stable placement of the non-empty bits by size (counting sort over the
// digit table): sets[table[size][tile] + rank] = bit, one tile per block.
// Buckets stay unsorted: the engine ranks members by value instead.
//
// The same launch finishes the set bookkeeping: n_sets = the exclusive prefix
// at the first cell of digit 255 (every set below 255 members) + the large
// sets p2_tiles counted; n_cand = the number of singletons (the first multi
// set in the (size, bit) order); and stage A as a bitset over P (ballots of
// the byte flags p2_scatter wrote) with its population count.
__global__ void __launch_bounds__(kTileBlock) p2_size_scatter(Plan* plan, const uint32_t* __restrict__ size,
                                                              const uint32_t* __restrict__ table,
                                                              uint32_t* __restrict__ sets,
                                                              const uint8_t* __restrict__ flags,
                                                              uint32_t* __restrict__ selbits, const uint32_t* status) {
  gp_pdl_wait();
  constexpr int kW = kTileBlock / 32;
  __shared__ uint32_t wcnt[kW][256];
  __shared__ uint32_t bsum;
  if (failed(status) || !p2_active(plan)) return;
  const uint64_t m = plan->m;
  const uint64_t ntiles = (m + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->n_sets = table[kBigSet * ntiles] + plan->n_large;
    const uint64_t n1 = table[2 * ntiles] - table[1 * ntiles];  // sets of size 1
    plan->n_multi = plan->n_sets - n1;
    plan->n_cand = n1;
  }
  {  // stage A
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    const uint64_t n = plan->n_pos;
    const uint64_t nw = (n + 31) / 32;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * kW;
    uint32_t c = 0;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kW) + warp; w < nw; w += warps) {
      const uint64_t p = 32 * w + lane;
      const unsigned bits = __ballot_sync(kFull, p < n && flags[p]);
      if (lane == 0) selbits[w] = bits;
      c += __popc(bits);
    }
    if (lane == 0 && c) atomicAdd(&bsum, c);
    __syncthreads();  // one global atomic per block
    if (threadIdx.x == 0 && bsum) atomicAdd(reinterpret_cast<unsigned long long*>(&plan->n_single_sel), bsum);
  }
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int w = 0; w < kW; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    // warp w owns bits [seg, seg + 512): item j of lane l is bit seg + 32 j + l,
    // so processing order is bit order
    const uint64_t seg = tile * kTile + static_cast<uint64_t>(warp) * (32 * kTileItems);
    uint32_t sz[kTileItems];
    uint16_t rank[kTileItems];
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint64_t b = seg + 32 * j + lane;
      sz[j] = b < m ? min(size[b], kBigSet) : 0u;  // the digit
    }
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint32_t s = sz[j];
      const unsigned peers = __match_any_sync(kFull, s);
      const uint32_t lr = __popc(peers & ((1u << lane) - 1));
      const uint32_t cur = s ? wcnt[warp][s] : 0u;
      __syncwarp();
      if (s && lr == 0) wcnt[warp][s] = cur + __popc(peers);
      __syncwarp();
      rank[j] = static_cast<uint16_t>(cur + lr);
    }
    __syncthreads();
    {  // exclusive over warps, plus the tile's base for this size from the scanned table
      uint32_t run = table[threadIdx.x * ntiles + tile];
      for (int w = 0; w < kW; ++w) {
        const uint32_t c = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTileItems; ++j)
      if (sz[j]) sets[wcnt[warp][sz[j]] + rank[j]] = static_cast<uint32_t>(seg + 32 * j + lane);
    __syncthreads();
  }
}

// Sets of >= 255 members share digit 255 and leave p2_size_scatter in bit
// order; this orders them by (size, bit) as conflict_sets' stable sort does
// (bloom.cpp:166-172).  Nothing to do in practice (it takes 255 positives
// probing one bit); when there is, one block merge-sorts the composite keys
// size << 32 | bit (all distinct) with a binary-search merge per pass.
// Run by the engine's block before its first round (one block of 1024).
__device__ void p2_sort_large(const Plan* plan, const uint32_t* __restrict__ size, uint32_t* sets, uint64_t* ka,
                              uint64_t* kb) {
  const uint64_t n = plan->n_large;
  if (n < 2) return;
  uint32_t* big = sets + (plan->n_sets - n);
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
    ka[i] = static_cast<uint64_t>(size[big[i]]) << 32 | big[i];
  __syncthreads();
  uint64_t* src = ka;
  uint64_t* dst = kb;
  for (uint64_t w = 1; w < n; w *= 2) {  // merge runs [a, a+w) and [a+w, a+2w)
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t a = i / (2 * w) * (2 * w), mid = min(a + w, n), e = min(a + 2 * w, n);
      const uint64_t x = src[i];
      const bool left = i < mid;
      uint64_t lo = left ? mid : a, hi = left ? e : mid;  // count the other run's keys below x
      const uint64_t base = lo;
      while (lo < hi) {
        const uint64_t md = (lo + hi) / 2;
        if (src[md] < x) lo = md + 1; else hi = md;
      }
      dst[a + (left ? i - a : i - mid) + (lo - base)] = x;
    }
    __syncthreads();
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) big[i] = static_cast<uint32_t>(src[i]);
}

__device__ __forceinline__ bool bs_test(const uint32_t* bs, uint32_t p) { return (bs[p >> 5] >> (p & 31)) & 1u; }

// Stage B, windowed: 1024 consecutive visits per round, one thread each.
// Every visit counts its unselected members against the selection at the
// window start and registers them with atomicMin(first_touch[p], v).  A visit
// is dependent iff an earlier visit of the window shares an unselected member
// (only then can an earlier selection change its outcome).  Visits before the
// first dependent one are exact: their RNG positions are a prefix sum of the
// draw flags (a rejected draw ends the window right after its visit), their
// selections are committed together, and the r cut stops the commit at the
// selection that reaches r.  The next window starts at the first uncommitted
// visit, so every round commits >= 1 visit and the result equals the
// sequential loop of bloom.cpp:198-219 bit for bit.
// kSmem: the selection bitset lives in shared memory; kFt: so does the
// per-positive first-touch table (every visit's atomicMin and the dependency
// reads become shared-memory operations instead of L2 round trips — two of
// a round's dependent global chains; |P| up to ~48k, e.g. a C5 bucket)
template <bool kSmem, bool kFt>
__device__ __forceinline__ void p2_engine_body(Plan* plan, uint32_t* sets,
                                               const uint32_t* __restrict__ off, const uint32_t* __restrict__ size,
                                               const uint32_t* __restrict__ members,
                                               uint64_t* ka, uint64_t* kb, uint32_t* selbits,
                                               uint32_t* first_touch_g, uint32_t* status) {
  extern __shared__ uint32_t sbits[];
  __shared__ uint64_t sh[40];
  // per-round block results: one barrier each (shared atomicMin / the single
  // writer) instead of a three-barrier block reduction
  __shared__ uint32_t s_vstar, s_rejv, s_cut;
  __shared__ uint64_t s_cdraw, s_csel;
  if (failed(status) || !p2_active(plan)) return;
  p2_sort_large(plan, size, sets, ka, kb);  // ends with a barrier when it runs
  __syncthreads();
  constexpr uint32_t W = 1024;
  const uint32_t v = threadIdx.x;
  const uint64_t n = plan->n_pos, r = plan->r;
  const uint64_t nwords = (n + 31) / 32;
  uint32_t* bits = kSmem ? sbits : selbits;
  uint32_t* first_touch = kFt ? sbits + ((nwords + 3) & ~3ull) : first_touch_g;
  const bool fallback = plan->n_single_sel > r;
  if (kSmem || fallback)
    for (uint64_t w = v; w < nwords; w += W) bits[w] = fallback ? 0u : selbits[w];
  __syncthreads();
  uint64_t nsel = fallback ? 0 : plan->n_single_sel;
  const uint64_t nsets = plan->n_sets;
  const uint64_t start = fallback ? 0 : plan->n_cand;
  const uint64_t L = nsets - start;
  const uint64_t seed = hash64(plan->seed_a, plan->seed_b);  // derive_selection_seed (pipeline.cpp:23-25)
  uint64_t rpos = 0, cursor = 0, last_progress = 0;

  constexpr uint32_t kM = 8;  // members of a visit held in registers (larger sets re-read memory)
  while (nsel < r && L > 0) {
    if (v == 0) {  // the previous round read these before its closing barrier
      s_vstar = W;
      s_rejv = W;
      s_cut = W;
    }
    const uint64_t si = start + (cursor + v) % L;
    const uint32_t bit = sets[si];
    const uint32_t sz = size[bit];
    const uint32_t* mems = members + (off[bit] & ~kSingleton);  // slot = bucket start after the scatter
    uint32_t mr[kM];
#pragma unroll
    for (uint32_t j = 0; j < kM; ++j) mr[j] = j < sz ? mems[j] : 0u;
#pragma unroll
    for (uint32_t j = 0; j < kM; ++j)
      if (j < sz) first_touch[mr[j]] = 0xFFFFFFFFu;
    for (uint32_t j = kM; j < sz; ++j) first_touch[mems[j]] = 0xFFFFFFFFu;
    __syncthreads();
    uint32_t cnt = 0, unsel = 0;  // unsel: bitmask of unselected register members
#pragma unroll
    for (uint32_t j = 0; j < kM; ++j) {
      if (j < sz && !bs_test(bits, mr[j])) {
        ++cnt;
        unsel |= 1u << j;
        atomicMin(&first_touch[mr[j]], v);
      }
    }
    for (uint32_t j = kM; j < sz; ++j) {
      const uint32_t p = mems[j];
      if (!bs_test(bits, p)) {
        ++cnt;
        atomicMin(&first_touch[p], v);
      }
    }
    __syncthreads();
    bool dep = false;
    if (cnt) {
      uint32_t ft[kM];
#pragma unroll
      for (uint32_t j = 0; j < kM; ++j) ft[j] = (unsel >> j & 1u) ? first_touch[mr[j]] : 0xFFFFFFFFu;
#pragma unroll
      for (uint32_t j = 0; j < kM; ++j) dep |= ft[j] < v;
      for (uint32_t j = kM; j < sz && !dep; ++j) {
        const uint32_t p = mems[j];
        if (!bs_test(bits, p) && first_touch[p] < v) dep = true;
      }
    }
    if (dep) atomicMin(&s_vstar, v);
    __syncthreads();
    const uint32_t vstar = s_vstar;
    // RNG positions of the independent prefix
    const bool draw = v < vstar && cnt >= 2;
    // one scan for both prefixes: draws (low half) and visits with an
    // unselected member (high half) — below `limit` the latter are exactly
    // the selecting visits, so the selection prefix needs no second scan
    uint64_t tot2;
    const uint64_t pk = block_exclusive_sum<uint64_t, 1024>((draw ? 1ull : 0ull) | (cnt >= 1 ? 1ull << 32 : 0ull),
                                                            sh, tot2);
    const uint64_t dpos = pk & 0xFFFFFFFFull, spos = pk >> 32;
    uint32_t target = 0;
    bool rej = false;
    uint64_t bound = 0, val = 0;
    if (draw) {
      bound = below_bound(cnt);
      val = rng_at(seed, rpos + dpos);
      rej = val > bound;
    }
    if (rej) atomicMin(&s_rejv, v);
    __syncthreads();
    const uint32_t rejv = s_rejv;
    const uint32_t limit = min(vstar, rejv == W ? W : rejv + 1);
    uint64_t extra = 0;  // positions consumed beyond one by the rejecting visit
    if (draw && v < limit) {
      if (v == rejv) {
        uint64_t pos = rpos + dpos + 1;
        do {
          val = rng_at(seed, pos++);
        } while (val > bound);
        extra = pos - (rpos + dpos) - 1;
      }
      target = static_cast<uint32_t>(val % cnt);
    }
    // selections of the prefix and the r cut
    const bool sel = v < limit && cnt >= 1;
    const uint64_t need = r - nsel;
    if (sel && spos + 1 == need) s_cut = v + 1;  // at most one visit: spos rises along the selections
    __syncthreads();
    const uint32_t cut = s_cut;
    const uint32_t climit = min(limit, cut);
    // commit
    if (sel && v < climit) {  // the target-th smallest unselected member (buckets are unsorted)
      if (sz <= kM) {  // register members, unselected mask from the count above (no selection since)
#pragma unroll
        for (uint32_t j = 0; j < kM; ++j) {
          uint32_t rank = 0;
#pragma unroll
          for (uint32_t q = 0; q < kM; ++q) rank += ((unsel >> q & 1u) && mr[q] < mr[j]) ? 1u : 0u;
          if ((unsel >> j & 1u) && rank == target) atomicOr(&bits[mr[j] >> 5], 1u << (mr[j] & 31));
        }
      } else {
        for (uint32_t j = 0; j < sz; ++j) {
          const uint32_t p = mems[j];
          if (bs_test(bits, p)) continue;
          uint32_t rank = 0;
          for (uint32_t q = 0; q < sz; ++q) {
            const uint32_t o = mems[q];
            rank += (o < p && !bs_test(bits, o)) ? 1u : 0u;
          }
          if (rank == target) {
            atomicOr(&bits[p >> 5], 1u << (p & 31));
            break;
          }
        }
      }
    }
    // totals over the committed visits [0, climit), climit >= 1, from its
    // last visit: selections = its inclusive selection prefix, draws = its
    // inclusive draw prefix (it is the rejecting visit if one commits)
    if (v == climit - 1) {
      s_csel = spos + (cnt >= 1 ? 1 : 0);
      s_cdraw = dpos + (draw ? 1 + extra : 0);
    }
    __syncthreads();
    const uint64_t csel = s_csel;
    const uint64_t cdraw = s_cdraw;
    nsel += csel;
    rpos += cdraw;
    cursor += climit;
    if (csel) last_progress = cursor;
    if (cursor - last_progress > L + W) {  // a full cycle without a selection: |P| < r
      if (v == 0) latch(status, GP_ERROR);
      break;
    }
  }
  __syncthreads();
  if (kSmem)
    for (uint64_t w = v; w < nwords; w += W) selbits[w] = bits[w];
  if (v == 0) {
    plan->n_sel = nsel;
    plan->n_multi = cursor;  // visits replayed (diagnostic)
  }
}


constexpr int kSmemFtBytes = 200 * 1024;    // bitset + first-touch table
constexpr int kSmemBitsBytes = 160 * 1024;  // bitset alone (the rest stays L1 for the global chains)

__device__ __forceinline__ bool ft_fits(uint64_t n) {
  return (((n + 31) / 32 + 3) & ~3ull) * 4 + 4 * n <= static_cast<uint64_t>(kSmemFtBytes);
}

// |P| is only known on the device, so both engine launches are enqueued and
// exactly one runs: kFt (bitset and first-touch table in shared memory, when
// both fit) or the other (bitset in shared memory when it fits, else global).
// Separate launches keep the smaller shared-memory carveout — and the larger
// L1 for the global set / member chains — when the first-touch table does
// not fit (c4s: requesting 200 KiB there cost 40% on the engine).
template <bool kFt>
__global__ void __launch_bounds__(1024) p2_engine_dispatch(Plan* plan, uint32_t* sets,
                                                           const uint32_t* __restrict__ off,
                                                           const uint32_t* __restrict__ size,
                                                           const uint32_t* __restrict__ members,
                                                           uint64_t* ka, uint64_t* kb, uint32_t* selbits,
                                                           uint32_t* first_touch, bool alone, uint32_t* status) {
  gp_pdl_wait();
  const uint64_t n = plan->n_pos;
  if (!alone && ft_fits(n) != kFt) return;  // alone: the other kernel was not launched
  if (kFt)
    p2_engine_body<true, true>(plan, sets, off, size, members, ka, kb, selbits, first_touch, status);
  else if (((n + 31) / 32) * 4 <= static_cast<uint64_t>(kSmemBitsBytes))
    p2_engine_body<true, false>(plan, sets, off, size, members, ka, kb, selbits, first_touch, status);
  else
    p2_engine_body<false, false>(plan, sets, off, size, members, ka, kb, selbits, first_touch, status);
}

// sel = ascending P[p] for flagged p (bloom.cpp:221 sort), count must be r.
// One cooperative launch: every block counts the selected positives of its
// tiles (strided by the grid), publishes the counts, and after one grid
// barrier writes each tile from the sum of the earlier tiles' counts (one
// warp read) — no decoupled look-back chain, no ticket reset.
__global__ void __launch_bounds__(kTileBlock) flags_compact(const uint32_t* __restrict__ P,
                                                            const uint32_t* __restrict__ selbits, Plan* plan,
                                                            int method, uint32_t* __restrict__ sel, uint64_t* tcnt,
                                                            uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  cg::grid_group grid = cg::this_grid();
  if (failed(status) || plan->index_method != method) return;  // uniform over the grid
  const uint64_t n = plan->n_pos;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  // warp rounds: round q of warp w covers positions wb + 32q + lane, one
  // selection word (wb is a multiple of 32), so P loads and sel stores are
  // coalesced (~90% of P is selected at C4)
  auto load = [&](uint64_t tile, uint32_t (&word)[kTileItems]) {
    const uint64_t wb = tile * kTile + static_cast<uint64_t>(warp) * (32 * kTileItems);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      const uint64_t p0 = wb + 32 * q;
      uint32_t x = p0 < n ? selbits[p0 >> 5] : 0u;
      if (p0 + 32 > n) x &= p0 >= n ? 0u : (1u << (n - p0)) - 1u;
      word[q] = x;
      c += __popc(x);
    }
    return c;
  };
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t word[kTileItems];
    const uint32_t c = load(tile, word);  // every lane: the warp's count (one word per round)
    uint64_t tot;
    (void)block_exclusive_sum<uint64_t, kTileBlock>(lane == 0 ? c : 0, sh, tot);
    if (threadIdx.x == 0) tcnt[tile] = tot;
  }
  grid.sync();
  const uint64_t r = plan->r;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (warp == 0) {
      uint64_t p = 0;
      for (uint64_t t = lane; t < tile; t += 32) p += __ldcg(tcnt + t);
      p = warp_sum(p);
      if (lane == 0) sh[34] = p;
    }
    uint32_t word[kTileItems];
    const uint32_t c = load(tile, word);  // every lane: the warp's count (one word per round)
    uint64_t tot;
    const uint64_t local = block_exclusive_sum<uint64_t, kTileBlock>(lane == 0 ? c : 0, sh, tot);  // barrier
    uint64_t o = __shfl_sync(kFull, sh[34] + local, 0);
    const uint64_t wb = tile * kTile + static_cast<uint64_t>(warp) * (32 * kTileItems);
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      if (word[q] >> lane & 1u) {
        const uint64_t at = o + __popc(word[q] & lt);
        if (at < r) sel[at] = P[wb + 32 * q + lane];
      }
      o += __popc(word[q]);
    }
    if (tile == ntiles - 1 && threadIdx.x == kTileBlock - 1 && o != plan->r) latch(status, GP_ERROR);
    __syncthreads();  // sh[34] is rewritten by the next tile
  }
}

}  // namespace

void launch_flags_compact(gp_ctx* ctx, int method, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  // cooperative: every block resident (48 registers x 256 threads: 5 per SM)
  const uint64_t ptiles = (n_bound + kTile - 1) / kTile;
  int grid = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(ptiles, 1), 2ull * ctx->sm_count));
  const uint32_t* P = w.pos;
  const uint32_t* sb = w.selbits;
  Plan* plan = w.plan;
  uint32_t* sel = w.sel;
  uint64_t* tc = w.tiles;
  uint32_t* st = w.status;
  void* args[] = {&P, &sb, &plan, &method, &sel, &tc, &st};
  cudaLaunchCooperativeKernel(reinterpret_cast<void*>(flags_compact), grid, kTileBlock, args, 0, s);
  ++ctx->launches;
}

void launch_select_p2(gp_ctx* ctx, uint64_t n_bound, uint64_t m_bound, uint32_t k_bound, bool decoding,
                      cudaStream_t s, uint64_t n_expect) {
  Workspace& w = ctx->ws;
  stage_begin(ctx, decoding ? ST_DEC_P2_SETS : ST_P2_SETS, s);
  const uint64_t m_cap = std::min<uint64_t>(m_bound, w.set_cap);
  GP_LAUNCH(ctx, p2_zero_counts, ctx->sm_count * 4, 256, 0, s, w.plan, w.p2_count, m_cap, w.flags, n_bound, w.p2_alloc,
            w.status);
  GP_LAUNCH(ctx, p2_pairs, grid_for(ctx, n_bound, 256), 256, 0, s, w.pos, w.plan, w.pairs, w.p2_rank, w.p2_count,
            w.pair_cap, w.set_cap, w.status);
  const uint64_t mtiles = (m_cap + kTile - 1) / kTile;
  const int tgrid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(mtiles, ctx->sm_count * 8ULL)));
  GP_LAUNCH(ctx, p2_tiles, tgrid, kTileBlock, 0, s, w.p2_count, w.plan, w.p2_off, w.p2_table, w.p2_alloc, w.status);
  GP_LAUNCH(ctx, p2_scatter, grid_for(ctx, n_bound * k_bound, 256), 256, 0, s, w.pairs, w.p2_rank, w.plan, w.p2_off,
            w.p2_members, w.flags, w.status);
  launch_table_scan(ctx, w.p2_table, &w.plan->m, m_cap, 12, s);
  GP_LAUNCH(ctx, p2_size_scatter, tgrid, kTileBlock, 0, s, w.plan, w.p2_count, w.p2_table, w.p2_sets, w.flags,
            w.selbits, w.status);
  stage_end(ctx, s);
  stage_begin(ctx, decoding ? ST_DEC_P2_ENGINE : ST_P2_ENGINE, s);
  {
    const uint64_t bits_b = (((n_bound + 31) / 32 + 3) & ~3ull) * 4;  // for |P| <= n_bound
    uint64_t* ka = reinterpret_cast<uint64_t*>(w.f64a);
    uint64_t* kb = reinterpret_cast<uint64_t*>(w.f64b);
    // n_expect (the encode's r + eps d, 0 when unknown): far above what the
    // first-touch table holds, the shared-memory engine is not even launched
    const bool ft_possible = n_expect == 0 || (((n_expect + 31) / 32 + 4) * 4 + 4 * n_expect) * 10 <=
                                                  9ull * kSmemFtBytes;
    if (ft_possible)
      GP_LAUNCH(ctx, p2_engine_dispatch<true>, 1, 1024, std::min<uint64_t>(bits_b + 4 * n_bound, kSmemFtBytes), s,
                w.plan, w.p2_sets, w.p2_off, w.p2_count, w.p2_members, ka, kb, w.selbits, w.first_touch, false,
                w.status);
    if (!ft_possible) {  // the other kernel must take every |P| (ft_fits is never consulted)
      GP_LAUNCH(ctx, p2_engine_dispatch<false>, 1, 1024, std::min<uint64_t>(bits_b, kSmemBitsBytes), s, w.plan,
                w.p2_sets, w.p2_off, w.p2_count, w.p2_members, ka, kb, w.selbits, w.first_touch, true, w.status);
    } else if (bits_b + 4 * n_bound > static_cast<uint64_t>(kSmemFtBytes))  // else |P| <= n_bound always fits
      GP_LAUNCH(ctx, p2_engine_dispatch<false>, 1, 1024, std::min<uint64_t>(bits_b, kSmemBitsBytes), s, w.plan,
                w.p2_sets, w.p2_off, w.p2_count, w.p2_members, ka, kb, w.selbits, w.first_touch, false, w.status);
  }
  stage_end(ctx, s);
  launch_flags_compact(ctx, GP_INDEX_BLOOM_P2, n_bound, s);
}

void kernel_attrs_p2() {
  cudaFuncSetAttribute(p2_engine_dispatch<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFtBytes);
  cudaFuncSetAttribute(p2_engine_dispatch<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBitsBytes);
}

}  // namespace gp
