// topr.cu — K1/K2: top-r selection (sparsify.cpp:32-46) as a radix threshold
// select with order-preserving compaction.
//
// Reference semantics: nth_element over indices with the comparator
// (|g_a| > |g_b|) || (|g_a| == |g_b| && a < b), then sort ascending.  For f32
// data |g| orders exactly like the u32 key (bits & 0x7FFFFFFF), so the kept
// set is {key > T} plus the lowest-index {key == T} until r are kept, where
// T is the r-th largest key.
//
// Passes over the d-element gradient (HBM-bound, 4 B/element each):
//   1. topr_hist      : 8192-bin histogram of key >> 18 (shared-memory bins)
//   2. topr_pick_bin  : one block finds the threshold bin b* and the quota
//   3. topr_candidates: one ordered pass emitting every key in bins >= b*
//                       (the final support when b* is kept whole) and, via a
//                       second look-back, the keys of bin b* alone
// then on the small tie-bin list (~0.2% of d for normal data):
//   4. topr_refine    : exact T, quota q and the index of the q-th tie
//   5. topr_final     : order-preserving filter of the candidate list.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kShift = 18;
constexpr int kBins = 1 << (31 - kShift);  // 8192
constexpr int kHistBlock = 512;
constexpr int kTileBlock = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileBlock * kTileItems;

__device__ __forceinline__ uint32_t key_of(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__global__ void __launch_bounds__(kHistBlock) topr_hist(const float* __restrict__ g, uint64_t d,
                                                        uint32_t* __restrict__ ghist,
                                                        const uint32_t* status) {
  __shared__ uint32_t h[kBins];
  if (failed(status)) return;
  for (int i = threadIdx.x; i < kBins; i += kHistBlock) h[i] = 0;
  __syncthreads();
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t n4 = aligned ? d / 4 : 0;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHistBlock;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(&g4[i]);
    atomicAdd(&h[key_of(v.x) >> kShift], 1u);
    atomicAdd(&h[key_of(v.y) >> kShift], 1u);
    atomicAdd(&h[key_of(v.z) >> kShift], 1u);
    atomicAdd(&h[key_of(v.w) >> kShift], 1u);
  }
  for (uint64_t i = n4 * 4 + static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i < d; i += stride)
    atomicAdd(&h[key_of(g[i]) >> kShift], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kHistBlock)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// One block of 1024 threads; thread t owns bins [8t, 8t+8).
__global__ void __launch_bounds__(1024) topr_pick_bin(const uint32_t* __restrict__ ghist, uint64_t r,
                                                      Plan* plan, const uint32_t* status) {
  __shared__ uint64_t sh[40];
  if (failed(status)) return;
  const int t = threadIdx.x;
  uint32_t b[8];
  uint64_t mine = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    b[j] = ghist[8 * t + j];
    mine += b[j];
  }
  // suffix sums: scan in reversed thread order
  const int rt = 1023 - t;
  (void)rt;
  uint64_t total;
  // exclusive sum over threads with larger t == sum of bins above this thread's range
  // computed as total - inclusive prefix
  const uint64_t excl = block_exclusive_sum<uint64_t, 1024>(mine, sh, total);
  const uint64_t above_mine = total - excl - mine;  // keys in bins >= 8t+8
  if (above_mine < r && r <= above_mine + mine) {
    uint64_t acc = above_mine;
    for (int j = 7; j >= 0; --j) {
      if (acc + b[j] >= r) {
        plan->bin_star = 8 * t + j;
        plan->above = acc;
        plan->full_bin = (acc + b[j] == r) ? 1u : 0u;
        plan->n_cand = acc + b[j];
        plan->thresh = static_cast<uint32_t>(8 * t + j) << kShift;  // refined later unless full
        plan->tie_cut = 0xFFFFFFFFu;
        break;
      }
      acc += b[j];
    }
  }
}

// Order-preserving pass over the gradient.  Writes candidates (bin >= b*) to
// (cidx, cval) — or straight to (sidx, sval) when b* is kept whole — and the
// keys of bin b* to (tidx, tval).
__global__ void __launch_bounds__(kTileBlock) topr_candidates(
    const float* __restrict__ g, uint64_t d, const Plan* __restrict__ plan, uint32_t* cidx, float* cval,
    uint32_t* sidx, float* sval, uint32_t* tidx, float* tval, uint64_t* tiles_c, uint64_t* tiles_t,
    uint32_t* ticket, const uint32_t* status) {
  __shared__ uint64_t sh_c[36];
  __shared__ uint64_t sh_t[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint32_t bstar = plan->bin_star;
  const bool full = plan->full_bin != 0;
  uint32_t* oidx = full ? sidx : cidx;
  float* oval = full ? sval : cval;
  const uint64_t ntiles = (d + kTile - 1) / kTile;
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t base = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(threadIdx.x) * kTileItems;
    float v[kTileItems];
    if (aligned && base + kTileItems <= d) {
      const float4* p = reinterpret_cast<const float4*>(g + base);
#pragma unroll
      for (int q = 0; q < kTileItems / 4; ++q) {
        const float4 x = __ldg(p + q);
        v[4 * q] = x.x;
        v[4 * q + 1] = x.y;
        v[4 * q + 2] = x.z;
        v[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < kTileItems; ++q) v[q] = base + q < d ? g[base + q] : 0.0f;
    }
    uint32_t mc = 0, mt = 0;
    uint64_t cc = 0, ct = 0;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      const bool ok = base + q < d;
      const uint32_t bin = key_of(v[q]) >> kShift;
      if (ok && bin >= bstar) {
        mc |= 1u << q;
        ++cc;
      }
      if (ok && bin == bstar && !full) {
        mt |= 1u << q;
        ++ct;
      }
    }
    // two independent scans: warp 0 looks back on the candidate tiles, warp 1 on the tie tiles
    uint64_t tot_c, tot_t;
    const uint64_t loc_c = block_exclusive_sum<uint64_t, kTileBlock>(cc, sh_c, tot_c);
    const uint64_t loc_t = block_exclusive_sum<uint64_t, kTileBlock>(ct, sh_t, tot_t);
    if (threadIdx.x < 32) {
      const uint64_t p = lookback_warp(tiles_c, tile, tot_c);
      if (threadIdx.x == 0) sh_c[34] = p;
    } else if (threadIdx.x < 64 && !full) {
      const uint64_t p = lookback_warp(tiles_t, tile, tot_t);
      if (threadIdx.x == 32) sh_t[34] = p;
    }
    __syncthreads();
    uint64_t oc = sh_c[34] + loc_c;
    uint64_t ot = full ? 0 : sh_t[34] + loc_t;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      if (mc >> q & 1u) {
        oidx[oc] = static_cast<uint32_t>(base + q);
        oval[oc] = v[q];
        ++oc;
      }
      if (mt >> q & 1u) {
        tidx[ot] = static_cast<uint32_t>(base + q);
        tval[ot] = v[q];
        ++ot;
      }
    }
  }
}

// One block: exact threshold key within bin b*, quota, and the tie cut.
__global__ void __launch_bounds__(1024) topr_refine(const uint32_t* __restrict__ tidx,
                                                    const float* __restrict__ tval, const uint32_t* ghist,
                                                    uint64_t r, Plan* plan, const uint32_t* status) {
  __shared__ uint32_t h[512];
  __shared__ uint64_t sh[40];
  __shared__ uint32_t s_digit, s_found;
  __shared__ uint64_t s_rem;
  if (failed(status) || plan->full_bin) return;
  const uint32_t bstar = plan->bin_star;
  const uint64_t nt = ghist[bstar];
  uint64_t remaining = r - plan->above;  // how many of bin b* to keep, by (key desc, idx asc)
  uint32_t prefix = bstar << kShift, mask = 0xFFFFFFFFu << kShift;
  // two 9-bit digit rounds: bits 17..9 then 8..0
  for (int round = 0; round < 2; ++round) {
    const int sh_bits = round == 0 ? 9 : 0;
    for (int i = threadIdx.x; i < 512; i += 1024) h[i] = 0;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < nt; i += 1024) {
      const uint32_t key = key_of(tval[i]);
      if ((key & mask) == prefix) atomicAdd(&h[(key >> sh_bits) & 511], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t rem = remaining;
      int dig = 511;
      for (; dig > 0; --dig) {
        if (rem <= h[dig]) break;
        rem -= h[dig];
      }
      s_digit = static_cast<uint32_t>(dig);
      s_rem = rem;
    }
    __syncthreads();
    prefix |= s_digit << sh_bits;
    mask |= 511u << sh_bits;
    remaining = s_rem;
    __syncthreads();
  }
  const uint32_t T = prefix;
  const uint64_t q = remaining;  // keep the first q keys == T in index order
  // count ties == T; find the q-th in list (index) order
  if (threadIdx.x == 0) s_found = 0xFFFFFFFFu;
  uint64_t seen = 0;
  for (uint64_t base = 0; base < nt; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t is_t = (i < nt && key_of(tval[i]) == T) ? 1 : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum<uint64_t, 1024>(is_t, sh, tot);
    if (is_t && seen + ex + 1 == q) s_found = tidx[i];
    seen += tot;
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    plan->thresh = T;
    // all ties kept → no cut needed; otherwise the index of the q-th tie
    plan->tie_cut = (seen == q) ? 0xFFFFFFFFu : s_found;
  }
}

// Ordered filter of the candidate list into the final support.
__global__ void __launch_bounds__(kTileBlock) topr_final(const uint32_t* __restrict__ cidx,
                                                         const float* __restrict__ cval, const Plan* plan,
                                                         uint32_t* sidx, float* sval, uint64_t* tiles,
                                                         uint32_t* ticket, const uint32_t* status) {
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status) || plan->full_bin) return;
  const uint64_t n = plan->n_cand;
  const uint32_t T = plan->thresh, cut = plan->tie_cut;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t base = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(threadIdx.x) * kTileItems;
    uint32_t m = 0;
    uint64_t c = 0;
#pragma unroll
    for (int q = 0; q < kTileItems; ++q) {
      if (base + q < n) {
        const uint32_t key = key_of(cval[base + q]);
        if (key > T || (key == T && cidx[base + q] <= cut)) {
          m |= 1u << q;
          ++c;
        }
      }
    }
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kTileBlock>(c, tile, tiles, sh, tot);
#pragma unroll
    for (int q = 0; q < kTileItems; ++q)
      if (m >> q & 1u) {
        sidx[o] = cidx[base + q];
        sval[o] = cval[base + q];
        ++o;
      }
  }
}

}  // namespace

void launch_top_r(gp_ctx* ctx, const float* grad, uint64_t d, uint64_t r, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = (d + kTile - 1) / kTile;
  cudaMemsetAsync(w.hist, 0, kBins * sizeof(uint32_t), s);
  reset_scan(ctx, s, 3 * (ntiles + 1));
  uint64_t* tiles_c = w.tiles;
  uint64_t* tiles_t = w.tiles + ntiles + 1;
  const int hist_grid = static_cast<int>(std::min<uint64_t>((d / 4 + kHistBlock - 1) / kHistBlock + 1,
                                                            static_cast<uint64_t>(ctx->sm_count) * 4));
  GP_LAUNCH(ctx, topr_hist, hist_grid, kHistBlock, 0, s, grad, d, w.hist, w.status);
  GP_LAUNCH(ctx, topr_pick_bin, 1, 1024, 0, s, w.hist, r, w.plan, w.status);
  const int grid = static_cast<int>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(ctx->sm_count) * 8));
  GP_LAUNCH(ctx, topr_candidates, std::max(grid, 1), kTileBlock, 0, s, grad, d, w.plan, w.cand_idx,
            w.cand_val, w.support, w.values, w.u32a, reinterpret_cast<float*>(w.u32b), tiles_c, tiles_t,
            w.ticket, w.status);
  GP_LAUNCH(ctx, topr_refine, 1, 1024, 0, s, w.u32a, reinterpret_cast<const float*>(w.u32b), w.hist, r,
            w.plan, w.status);
  // final filter: its own scan state (tiles after both previous arrays)
  uint64_t* tiles_f = w.tiles + 2 * (ntiles + 1);
  const int fgrid = static_cast<int>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(ctx->sm_count) * 4));
  GP_LAUNCH(ctx, topr_final, std::max(fgrid, 1), kTileBlock, 0, s, w.cand_idx, w.cand_val, w.plan, w.support,
            w.values, tiles_f, w.ticket + 2, w.status);
}

}  // namespace gp
