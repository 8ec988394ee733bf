// gp_device.cuh — device-side building blocks shared by every kernel.
//
//  * SplitMix64 hashing and the CounterRng stream (rng.hpp:25-73) as
//    __host__ __device__ functions, plus an exact 64-by-32 modular reduction
//    for Bloom probe positions (bloom.cpp:54-56 computes mix64(.) % m).
//  * The per-context device status word: the first failing check latches its
//    gp_status code; every kernel returns early once it is set, so a failed
//    decode never touches the caller's dense gradient.
//  * Warp/block scans and the decoupled look-back tile scan used for every
//    order-preserving compaction (support lists, positive sets, selections).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gradpack_b200.h"

namespace gp {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash64(uint64_t x, uint64_t seed) {
  return mix64(x ^ (seed + kGamma));
}

// CounterRng draw number `pos` (0-based) of a stream seeded with `seed`:
// state after pos+1 increments (rng.hpp:46-49).
__host__ __device__ __forceinline__ uint64_t rng_at(uint64_t seed, uint64_t pos) {
  return mix64(seed + (pos + 1) * kGamma);
}

// below(n) rejection bound (rng.hpp:52-59): draws r > bound are rejected.
__host__ __device__ __forceinline__ uint64_t below_bound(uint64_t n) {
  const uint64_t rem = (~0ULL % n + 1) % n;
  return ~0ULL - rem;
}

// Exact x mod m for 1 <= m < 2^32, with minv = floor((2^64-1)/m) = (2^64-e)/m,
// 0 < e <= m: x*minv/2^64 = x/m - x*e/(m*2^64) > x/m - 1, so the quotient
// estimate umulhi(x, minv) is floor(x/m) or one below it — one correction.
struct FastMod {
  uint64_t m;
  uint64_t minv;
};
inline FastMod make_fastmod(uint64_t m) { return FastMod{m, m ? ~0ULL / m : 0}; }

__device__ __forceinline__ uint64_t fast_mod(uint64_t x, const FastMod& f) {
  const uint64_t q = __umul64hi(x, f.minv);
  const uint64_t r = x - q * f.m;
  return r >= f.m ? r - f.m : r;
}

// The same for m <= 2^31: the pre-correction remainder is < 2m <= 2^32, so
// it is exact in 32-bit arithmetic.
__device__ __forceinline__ uint32_t fast_mod_small(uint64_t x, uint64_t minv, uint32_t m) {
  const uint32_t q = static_cast<uint32_t>(__umul64hi(x, minv));
  const uint32_t r = static_cast<uint32_t>(x) - q * m;
  return r >= m ? r - m : r;
}

// ---------------------------------------------------------------- status
__device__ __forceinline__ void latch(uint32_t* status, uint32_t code) {
  atomicCAS(status, 0u, code);
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// GPU-scope relaxed load: a volatile read is a system-scope strong load,
// which every block of every kernel paid at entry (ncu: ~40% of a small-
// container CRC's samples); writers are kernels on the same device
__device__ __forceinline__ bool failed(const uint32_t* status) {
  return ld_relaxed_u32(status) != 0u;
}

// ---------------------------------------------------------------- warp/block scans
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block-wide exclusive sum; `total` receives the block total.  `scratch`
// needs 33 entries of T in shared memory.  All threads must call.
template <typename T, int BLOCK>
__device__ __forceinline__ T block_exclusive_sum(T v, T* scratch, T& total) {
  constexpr int W = BLOCK / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_inclusive_sum(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < W ? scratch[lane] : T(0);
    const T winc = warp_inclusive_sum(w);
    if (lane < W) scratch[lane] = winc - w;
    if (lane == W - 1) scratch[32] = winc;
  }
  __syncthreads();
  const T out = scratch[warp] + inc - v;
  total = scratch[32];
  __syncthreads();
  return out;
}

// ---------------------------------------------------------------- decoupled look-back
// Tile descriptors: bits 62-63 = flag (0 invalid, 1 aggregate, 2 inclusive),
// bits 0-61 = value.  Tiles are claimed in order through an atomic ticket so
// that every predecessor of a waiting tile is already running.
constexpr uint64_t kFlagAgg = 1ULL << 62;
constexpr uint64_t kFlagInc = 2ULL << 62;
constexpr uint64_t kValMask = (1ULL << 62) - 1;

struct ScanState {
  uint64_t* tiles;   // >= number of tiles, zeroed before the scan
  uint32_t* ticket;  // zeroed before the scan
};

// GPU-scope relaxed accesses (a volatile access compiles to a system-scope
// strong one, which the descriptors never need: producers and consumers are
// CTAs of the same grid)
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Called by warp 0 of the block after the block aggregate is known.
// Returns the exclusive prefix of the tile (valid in every lane of warp 0).
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* tiles, uint32_t tile, uint64_t aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_volatile(&tiles[0], kFlagInc | aggregate);
    return 0;
  }
  if (lane == 0) st_volatile(&tiles[tile], kFlagAgg | aggregate);
  uint64_t exclusive = 0;
  int64_t base = static_cast<int64_t>(tile) - 1;
  while (true) {
    const int64_t idx = base - lane;
    uint64_t s = idx >= 0 ? ld_volatile(&tiles[idx]) : kFlagInc;
    while (__any_sync(kFull, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_volatile(&tiles[idx]);
    }
    const unsigned inc_mask = __ballot_sync(kFull, (s >> 62) == 2);
    const int first = inc_mask ? __ffs(inc_mask) - 1 : 32;
    uint64_t v = lane <= first ? (s & kValMask) : 0;
    v = warp_sum(v);
    exclusive += v;
    if (inc_mask) break;
    base -= 32;
  }
  // flag and value travel in one 64-bit word and readers use nothing else the
  // tile wrote, so no fence (it would wait for this thread's payload stores of
  // the previous tile to drain)
  if (lane == 0) st_volatile(&tiles[tile], kFlagInc | (exclusive + aggregate));
  return exclusive;
}

// The same with kW descriptors per lane per round (32 kW predecessors per L2
// round trip), for passes whose tiles all run in one wave: every tile then
// looks back at once and the nearest inclusive prefix trails by up to the
// whole grid, so the walk length, not the work, sets the pass time.
template <int kW>
__device__ __forceinline__ uint64_t lookback_warp_wide(uint64_t* tiles, uint32_t tile, uint64_t aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_volatile(&tiles[0], kFlagInc | aggregate);
    return 0;
  }
  if (lane == 0) st_volatile(&tiles[tile], kFlagAgg | aggregate);
  uint64_t exclusive = 0;
  int64_t base = static_cast<int64_t>(tile) - 1;
  while (true) {
    uint64_t s[kW];  // lane l, slot k: predecessor base - (kW l + k), nearest first
#pragma unroll
    for (int k = 0; k < kW; ++k) {
      const int64_t idx = base - (kW * lane + k);
      s[k] = idx >= 0 ? ld_volatile(&tiles[idx]) : kFlagInc;
    }
    bool pending = false;
#pragma unroll
    for (int k = 0; k < kW; ++k) pending |= (s[k] >> 62) == 0;
    while (__any_sync(kFull, pending)) {
      pending = false;
#pragma unroll
      for (int k = 0; k < kW; ++k)
        if ((s[k] >> 62) == 0) {
          s[k] = ld_volatile(&tiles[base - (kW * lane + k)]);
          pending |= (s[k] >> 62) == 0;
        }
    }
    int kin = kW;
#pragma unroll
    for (int k = kW - 1; k >= 0; --k)
      if ((s[k] >> 62) == 2) kin = k;
    const unsigned inc_mask = __ballot_sync(kFull, kin < kW);
    const int first = inc_mask ? __ffs(inc_mask) - 1 : 32;
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < kW; ++k)
      if (lane < first || (lane == first && k <= kin)) v += s[k] & kValMask;
    exclusive += warp_sum(v);
    if (inc_mask) break;
    base -= 32 * kW;
  }
  if (lane == 0) st_volatile(&tiles[tile], kFlagInc | (exclusive + aggregate));
  return exclusive;
}

// Claim the next tile (thread 0) and broadcast it through shared memory.
__device__ __forceinline__ uint32_t claim_tile(uint32_t* ticket, uint32_t* smem_slot) {
  __syncthreads();
  if (threadIdx.x == 0) *smem_slot = atomicAdd(ticket, 1u);
  __syncthreads();
  return *smem_slot;
}

// Full tile-scan step: every thread contributes `count`; returns the global
// exclusive offset of this thread's first element.  `sh` = 33 + 2 u64 slots.
template <int BLOCK>
__device__ __forceinline__ uint64_t tile_exclusive_offset(uint64_t count, uint32_t tile, uint64_t* tiles,
                                                          uint64_t* sh, uint64_t& tile_total) {
  uint64_t total;
  const uint64_t local = block_exclusive_sum<uint64_t, BLOCK>(count, sh, total);
  if (threadIdx.x < 32) {
    const uint64_t prefix = lookback_warp(tiles, tile, total);
    if (threadIdx.x == 0) sh[34] = prefix;
  }
  __syncthreads();
  const uint64_t prefix = sh[34];
  tile_total = total;
  __syncthreads();
  return prefix + local;
}

// One block: in-place exclusive scan of per-chunk counts (`b` may be null).
// For passes with thousands of small chunks a separate count pass + this scan
// replaces the decoupled look-back, whose chain of L2 round trips dominates
// when every chunk carries little work.  Counts and prefixes are < 2^32 (they
// count u32-indexed keys), so 8192 of them are staged as u32 in shared memory:
// coalesced loads, one block scan over per-thread runs of kPer, coalesced stores.
template <int kPer>
__global__ void __launch_bounds__(1024) scan_chunk_counts(uint64_t* a, uint64_t* b, uint64_t n,
                                                          const uint32_t* status) {
  __shared__ uint64_t sh[40];
  __shared__ uint32_t st[1024 * kPer];
  if (failed(status)) return;
  for (int k = 0; k < 2; ++k) {
    uint64_t* x = k == 0 ? a : b;
    if (x == nullptr) continue;
    uint64_t carry = 0;
    for (uint64_t base = 0; base < n; base += 1024 * kPer) {
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const uint64_t i = base + q * 1024 + threadIdx.x;
        st[q * 1024 + threadIdx.x] = i < n ? static_cast<uint32_t>(x[i]) : 0u;
      }
      __syncthreads();
      uint32_t v[kPer];
      uint64_t sum = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        v[q] = st[threadIdx.x * kPer + q];
        sum += v[q];
      }
      uint64_t tot;
      uint64_t e = block_exclusive_sum<uint64_t, 1024>(sum, sh, tot);  // ends with a barrier
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        st[threadIdx.x * kPer + q] = static_cast<uint32_t>(e);
        e += v[q];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const uint64_t i = base + q * 1024 + threadIdx.x;
        if (i < n) x[i] = carry + st[q * 1024 + threadIdx.x];
      }
      carry += tot;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- misc
__device__ __forceinline__ uint32_t ld_u32_unaligned(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
         (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
}
__device__ __forceinline__ uint64_t ld_u64_unaligned(const uint8_t* p) {
  return static_cast<uint64_t>(ld_u32_unaligned(p)) | (static_cast<uint64_t>(ld_u32_unaligned(p + 4)) << 32);
}
__device__ __forceinline__ void st_u32_unaligned(uint8_t* p, uint32_t v) {
  p[0] = static_cast<uint8_t>(v);
  p[1] = static_cast<uint8_t>(v >> 8);
  p[2] = static_cast<uint8_t>(v >> 16);
  p[3] = static_cast<uint8_t>(v >> 24);
}
__device__ __forceinline__ void st_u64_unaligned(uint8_t* p, uint64_t v) {
  st_u32_unaligned(p, static_cast<uint32_t>(v));
  st_u32_unaligned(p + 4, static_cast<uint32_t>(v >> 32));
}

// 16-byte loads with an L2 eviction-priority hint: evict_last for data a later
// pass of the same step reads again (kept in the 126 MB L2), evict_first for
// its last use.
__device__ __forceinline__ float4 ld_f4_keep(const float4* p) {
  float4 v;
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_f4_last(const float4* p) {
  float4 v;
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
      "ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}

// The value sequence an encode hands to the value codec: f32 (top-r of an f32
// gradient, exact as doubles) or f64 (compress_gradient's own Vector values,
// pipeline.cpp:146-221, and the f64 error-feedback input).  Read as double.
struct ValSrc {
  const float* f32;
  const double* f64;
  __device__ __forceinline__ double operator[](uint64_t i) const {
    return f64 ? f64[i] : static_cast<double>(f32[i]);
  }
};

}  // namespace gp
