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
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kScanBlock = 256;
constexpr uint64_t kSmemFilterMax = 150 * 1024;

__device__ __forceinline__ bool test_bit(const uint32_t* w, uint64_t pos) {
  return (w[pos >> 5] >> (pos & 31)) & 1u;
}

__global__ void bloom_insert(const uint32_t* __restrict__ keys, uint64_t r, const Plan* plan, uint32_t* words,
                             const uint32_t* status) {
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
// keeps a warp busy for its slowest lane.  Each warp instead owns 2048-key
// super-tiles and runs probe ROUNDS: round 1 probes every key (h_a, probe 0,
// 16 independent keys per lane in flight), the survivors' key offsets
// (u16, compacted in place in a per-warp shared queue) are the only work of
// round j+1 (h_a, h_b recomputed, probe j, 4 entries per lane in flight).
// Rounds stay converged; membership bits land in a per-warp mask that is
// stored to a d-bit membership bitmap.  No cross-warp ordering is needed.
// (2) members_compact: ordered compaction of the set bits (look-back scan,
// 131072 keys per tile) — P ascending, |P| in the plan.
constexpr int kLaneKeys = 16;
constexpr int kChunkKeys = 32 * kLaneKeys;   // 512 keys per round-1 chunk
constexpr int kChunks = 2;
constexpr int kSuperKeys = kChunks * kChunkKeys;   // 1024 keys per warp super-tile
constexpr int kWarps = kScanBlock / 32;

template <bool kSmem>
__global__ void __launch_bounds__(kScanBlock) bloom_members(const uint32_t* __restrict__ gwords, Plan* plan,
                                                            uint32_t* __restrict__ bitmap,
                                                            const uint32_t* status) {
  extern __shared__ uint32_t sw[];
  __shared__ uint16_t queue[kWarps][kSuperKeys];
  __shared__ uint32_t member[kWarps][kSuperKeys / 32];
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t d = plan->d, m = plan->m;
  const uint32_t k = plan->k;
  const FastMod fm{m, plan->minv};
  const uint64_t sa = plan->seed_a + kGamma, sb = plan->seed_b + kGamma;
  const uint32_t* words = gwords;
  if (kSmem) {
    const uint64_t nw = (m + 31) / 32;
    for (uint64_t i = threadIdx.x; i < nw; i += kScanBlock) sw[i] = gwords[i];
    __syncthreads();
    words = sw;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* q = queue[warp];
  uint32_t* wm = member[warp];
  const uint64_t nsuper = (d + kSuperKeys - 1) / kSuperKeys;
  const uint64_t gw = static_cast<uint64_t>(gridDim.x) * kWarps;
  for (uint64_t st = static_cast<uint64_t>(blockIdx.x) * kWarps + warp; st < nsuper; st += gw) {
    const uint64_t sbase = st * kSuperKeys;
    for (int i = lane; i < kSuperKeys / 32; i += 32) wm[i] = 0;
    __syncwarp();
    uint32_t nq = 0;
    // ---- round 1
    for (int c = 0; c < kChunks; ++c) {
      const uint32_t off0 = c * kChunkKeys + kLaneKeys * lane;
      uint32_t pass = 0;
#pragma unroll
      for (int j = 0; j < kLaneKeys; ++j) {
        const uint64_t x = sbase + off0 + j;
        const uint64_t a = mix64(x ^ sa);
        if (x < d && test_bit(words, fast_mod(mix64(a), fm))) pass |= 1u << j;
      }
      if (k == 1) {
        if (pass) atomicOr(&wm[off0 >> 5], pass << (off0 & 31));
        continue;
      }
      const uint32_t cnt = __popc(pass);
      const uint32_t inc = warp_inclusive_sum(cnt);
      uint32_t o = nq + inc - cnt;
      while (pass) {
        const int j = __ffs(pass) - 1;
        q[o++] = static_cast<uint16_t>(off0 + j);
        pass &= pass - 1;
      }
      nq += __shfl_sync(kFull, inc, 31);
    }
    __syncwarp();
    // ---- rounds 2..k
    for (uint32_t j = 1; j < k && nq; ++j) {
      uint32_t wr = 0;
      const bool last = j + 1 == k;
      // 4 entries per lane in flight while the queue is long, 1 in the thin tail
      const int per = nq > 64 ? 4 : 1;
      for (uint32_t base = 0; base < nq; base += 32 * per) {
        uint16_t kk[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (u >= per) {
            ok[u] = false;
            kk[u] = 0;
            continue;
          }
          const uint32_t e = base + 32 * u + lane;
          ok[u] = false;
          kk[u] = 0;
          if (e < nq) {
            kk[u] = q[e];
            const uint64_t x = sbase + kk[u];
            const uint64_t a = mix64(x ^ sa), b = mix64(x ^ sb);
            ok[u] = test_bit(words, fast_mod(mix64(a + static_cast<uint64_t>(j) * b), fm));
          }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (last) {
            if (ok[u]) atomicOr(&wm[kk[u] >> 5], 1u << (kk[u] & 31));
          } else {
            const unsigned bal = __ballot_sync(kFull, ok[u]);
            if (ok[u]) q[wr + __popc(bal & ((1u << lane) - 1))] = kk[u];
            wr += __popc(bal);
          }
        }
        __syncwarp();
      }
      nq = last ? 0 : wr;
    }
    __syncwarp();
    // ---- membership words (the super-tile is word aligned: 2048 keys = 64 words)
    const uint64_t nwd = (d + 31) / 32;
    for (int i = lane; i < kSuperKeys / 32; i += 32)
      if (sbase / 32 + i < nwd) bitmap[sbase / 32 + i] = wm[i];
    __syncwarp();
  }
}

// ordered compaction of the membership bitmap: 16 words per thread
__global__ void __launch_bounds__(kScanBlock) members_compact(const uint32_t* __restrict__ bitmap, Plan* plan,
                                                              uint32_t* __restrict__ pos_out, uint64_t cap,
                                                              uint64_t* tiles, uint32_t* ticket,
                                                              const uint32_t* status) {
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t nwd = (plan->d + 31) / 32;
  constexpr int kW = 16;
  const uint64_t ntiles = (nwd + kScanBlock * kW - 1) / (kScanBlock * kW);
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t w0 = static_cast<uint64_t>(tile) * kScanBlock * kW + static_cast<uint64_t>(threadIdx.x) * kW;
    uint32_t v[kW];
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      v[i] = w0 + i < nwd ? bitmap[w0 + i] : 0u;
      c += __popc(v[i]);
    }
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kScanBlock>(c, tile, tiles, sh, tot);
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      uint32_t x = v[i];
      while (x) {
        const int b = __ffs(x) - 1;
        if (o < cap) pos_out[o] = static_cast<uint32_t>(32 * (w0 + i) + b);
        ++o;
        x &= x - 1;
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == kScanBlock - 1) plan->n_pos = o;
  }
}

// Post-scan bookkeeping: |P| >= r (pipeline.cpp:284-285), value counts, and
// the P0 / Pd / naive selections which are slices of P.
__global__ void bloom_after_scan(Plan* plan, uint64_t cap, int decoding, uint32_t* status) {
  if (failed(status)) return;
  const uint8_t im = plan->index_method;
  if (im < GP_INDEX_BLOOM_P0 || im > GP_INDEX_BLOOM_NAIVE) return;
  const uint64_t n = plan->n_pos, r = plan->r;
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

// sel <- P (P0, naive) or the Pd slice (bloom.cpp:224-236)
__global__ void select_slice(const uint32_t* __restrict__ P, const Plan* plan, uint32_t* sel,
                             const uint32_t* status) {
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
  cudaMemsetAsync(w.filter, 0, ((m + 31) / 32) * 4, s);
  GP_LAUNCH(ctx, bloom_insert, grid_for(ctx, r, 128), 128, 0, s, w.support, r, w.plan, w.filter, w.status);
  GP_LAUNCH(ctx, bloom_emit, grid_for(ctx, (m + 7) / 8, 256), 256, 0, s, w.filter, w.plan, out, w.status);
}

void launch_bloom_parse(gp_ctx* ctx, const uint8_t* in, uint64_t m_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, bloom_parse, 1, 1, 0, s, in, w.plan, w.m_cap, w.status);
  GP_LAUNCH(ctx, bloom_load_words, grid_for(ctx, (m_bound + 31) / 32, 256), 256, 0, s, in, w.plan, w.filter,
            w.status);
}

// m_host: the filter width when the host knows it (encode), else 0 (decode:
// the width is only on the device, so the global-memory variant is used).
void launch_bloom_scan(gp_ctx* ctx, uint64_t d_bound, uint64_t m_host, bool decoding, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t fbytes = ((m_host + 31) / 32) * 4;
  const uint64_t nsuper = (d_bound + kSuperKeys - 1) / kSuperKeys;
  uint32_t* bitmap = w.u32c;  // d-bit membership bitmap
  if (m_host && fbytes <= kSmemFilterMax) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(bloom_members<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kSmemFilterMax));
      attr = true;
    }
    const int per_sm = std::max(1, static_cast<int>((200 * 1024) / (fbytes + 40 * 1024)));
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((nsuper + kWarps - 1) / kWarps, static_cast<uint64_t>(ctx->sm_count) * per_sm)));
    GP_LAUNCH(ctx, bloom_members<true>, grid, kScanBlock, fbytes, s, w.filter, w.plan, bitmap, w.status);
  } else {
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((nsuper + kWarps - 1) / kWarps, static_cast<uint64_t>(ctx->sm_count) * 6)));
    GP_LAUNCH(ctx, bloom_members<false>, grid, kScanBlock, 0, s, w.filter, w.plan, bitmap, w.status);
  }
  const uint64_t nwd = (d_bound + 31) / 32;
  const uint64_t ntiles = (nwd + kScanBlock * 16 - 1) / (kScanBlock * 16);
  reset_scan(ctx, s, ntiles + 1);
  GP_LAUNCH(ctx, members_compact, static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL))),
            kScanBlock, 0, s, bitmap, w.plan, w.pos, ctx->max_d, w.tiles, w.ticket, w.status);
  GP_LAUNCH(ctx, bloom_after_scan, 1, 1, 0, s, w.plan, ctx->max_d, decoding ? 1 : 0, w.status);
}

void launch_select_slice(gp_ctx* ctx, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, select_slice, grid_for(ctx, n_bound, 256), 256, 0, s, w.pos, w.plan, w.sel, w.status);
}

}  // namespace gp
