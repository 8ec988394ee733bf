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
//   1. topr_hist      : 32768-bin histogram of key >> 16 (shared-memory bins)
//   2. topr_pick_bin  : one block finds the threshold bin b* and the quota
//   3. topr_candidates: one ordered pass (a contiguous chunk per block,
//                       shared-memory staging, one look-back per block)
//                       emitting every key in bins >= b* (the final support
//                       when b* is kept whole) and the keys of bin b* alone
// then on the small tie-bin list (~0.2% of d for normal data):
//   4. topr_refine    : exact T, quota q and the index of the q-th tie
//   5. topr_final     : order-preserving filter of the candidate list.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kShift = 16;
constexpr int kBins = 1 << (31 - kShift);  // 32768 (128 KiB of shared counters)
constexpr int kHistBlock = 1024;
constexpr int kTileBlock = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileBlock * kTileItems;

__device__ __forceinline__ uint32_t key_of(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__global__ void __launch_bounds__(kHistBlock) topr_hist(const float* __restrict__ g, uint64_t d,
                                                        uint32_t* __restrict__ ghist,
                                                        const uint32_t* status) {
  extern __shared__ uint32_t h[];  // kBins counters
  if (failed(status)) return;
  for (int i = threadIdx.x; i < kBins; i += kHistBlock) h[i] = 0;
  __syncthreads();
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t n4 = aligned ? d / 4 : 0;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHistBlock;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    float4 v[4];  // four independent 16-byte loads in flight per thread
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * stride < n4 ? __ldcs(&g4[i0 + u * stride]) : make_float4(-1, -1, -1, -1);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u * stride < n4) {
        atomicAdd(&h[key_of(v[u].x) >> kShift], 1u);
        atomicAdd(&h[key_of(v[u].y) >> kShift], 1u);
        atomicAdd(&h[key_of(v[u].z) >> kShift], 1u);
        atomicAdd(&h[key_of(v[u].w) >> kShift], 1u);
      }
    }
  }
  for (uint64_t i = n4 * 4 + static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i < d; i += stride)
    atomicAdd(&h[key_of(g[i]) >> kShift], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kHistBlock)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// One block of 1024 threads; thread t owns bins [kPer*t, kPer*t + kPer).
constexpr int kPer = kBins / 1024;
__global__ void __launch_bounds__(1024) topr_pick_bin(const uint32_t* __restrict__ ghist, uint64_t r,
                                                      Plan* plan, const uint32_t* status) {
  __shared__ uint64_t sh[40];
  if (failed(status)) return;
  const int t = threadIdx.x;
  uint64_t mine = 0;
  const uint4* gh4 = reinterpret_cast<const uint4*>(ghist + kPer * t);
#pragma unroll
  for (int j = 0; j < kPer / 4; ++j) {
    const uint4 x = gh4[j];
    mine += static_cast<uint64_t>(x.x) + x.y + x.z + x.w;
  }
  uint64_t total;
  // exclusive sum over threads with larger t == sum of bins above this thread's range
  // computed as total - inclusive prefix
  const uint64_t excl = block_exclusive_sum<uint64_t, 1024>(mine, sh, total);
  const uint64_t above_mine = total - excl - mine;  // keys in bins above this thread's range
  if (above_mine < r && r <= above_mine + mine) {
    uint64_t acc = above_mine;
    for (int j = kPer - 1; j >= 0; --j) {
      const uint32_t b = ghist[kPer * t + j];
      if (acc + b >= r) {
        plan->bin_star = kPer * t + j;
        plan->above = acc;
        plan->full_bin = (acc + b == r) ? 1u : 0u;
        plan->n_cand = acc + b;
        plan->thresh = static_cast<uint32_t>(kPer * t + j) << kShift;  // refined later unless full
        plan->tie_cut = 0xFFFFFFFFu;
        break;
      }
      acc += b;
    }
  }
}

// One contiguous chunk of the gradient per block (claimed in order): stream it
// once with float4 loads, buffering in shared memory, in index order, the
// candidates (bin >= b*) and the keys of bin b* alone; one look-back per block
// (candidates on warp 0, ties on warp 1) places them.  A chunk whose
// candidates overflow the buffer (e.g. natural sparsity, r ~ 0.6 d) streams
// its slice a second time and writes directly.
constexpr int kCandBlock = 256;
constexpr int kCandCap = 3072;
constexpr int kTieCap = 1536;

__device__ __forceinline__ void load4(const float* __restrict__ g, uint64_t i, uint64_t hi, bool aligned, float v[4]) {
  if (aligned && i + 3 < hi) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(g + i));
    v[0] = x.x;
    v[1] = x.y;
    v[2] = x.z;
    v[3] = x.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = i + q < hi ? g[i + q] : 0.0f;
  }
}

__global__ void __launch_bounds__(kCandBlock) topr_candidates(
    const float* __restrict__ g, uint64_t d, uint64_t chunk, const Plan* __restrict__ plan, uint32_t* cidx,
    float* cval, uint32_t* sidx, float* sval, uint32_t* tidx, float* tval, uint64_t* tiles_c, uint64_t* tiles_t,
    uint32_t* ticket, const uint32_t* status) {
  __shared__ uint32_t bidx[kCandCap];
  __shared__ float bval[kCandCap];
  __shared__ uint32_t tbidx[kTieCap];
  __shared__ float tbval[kTieCap];
  __shared__ uint64_t sh_c[36];
  __shared__ uint64_t sh_t[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint32_t bstar = plan->bin_star;
  const bool full = plan->full_bin != 0;
  uint32_t* oidx = full ? sidx : cidx;
  float* oval = full ? sval : cval;
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t nchunks = (d + chunk - 1) / chunk;
  while (true) {
    const uint32_t c = claim_tile(ticket, &slot);
    if (c >= nchunks) break;
    const uint64_t lo = static_cast<uint64_t>(c) * chunk, hi = lo + chunk < d ? lo + chunk : d;
    uint64_t nc = 0, nt = 0;  // block-uniform running counts
    for (uint64_t base = lo; base < hi; base += 16 * kCandBlock) {
      const uint64_t i = base + 16 * threadIdx.x;  // 16 consecutive keys per thread, 4 loads in flight
      float v[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) load4(g, i + 4 * u, hi, aligned, v + 4 * u);
      uint32_t mc = 0, mt = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const uint32_t bin = key_of(v[q]) >> kShift;
        if (i + q < hi && bin >= bstar) mc |= 1u << q;
        if (i + q < hi && bin == bstar && !full) mt |= 1u << q;
      }
      uint64_t tc, tt;
      uint64_t oc = nc + block_exclusive_sum<uint64_t, kCandBlock>(__popc(mc), sh_c, tc);
      uint64_t ot = nt + block_exclusive_sum<uint64_t, kCandBlock>(__popc(mt), sh_t, tt);
      while (mc) {
        const int q = __ffs(mc) - 1;
        if (oc < kCandCap) {
          bidx[oc] = static_cast<uint32_t>(i + q);
          bval[oc] = v[q];
        }
        ++oc;
        mc &= mc - 1;
      }
      while (mt) {
        const int q = __ffs(mt) - 1;
        if (ot < kTieCap) {
          tbidx[ot] = static_cast<uint32_t>(i + q);
          tbval[ot] = v[q];
        }
        ++ot;
        mt &= mt - 1;
      }
      nc += tc;
      nt += tt;
    }
    if (threadIdx.x < 32) {
      const uint64_t p = lookback_warp(tiles_c, c, nc);
      if (threadIdx.x == 0) sh_c[34] = p;
    } else if (threadIdx.x < 64 && !full) {
      const uint64_t p = lookback_warp(tiles_t, c, nt);
      if (threadIdx.x == 32) sh_t[34] = p;
    }
    __syncthreads();
    const uint64_t pc = sh_c[34], pt = full ? 0 : sh_t[34];
    if (nc <= kCandCap && nt <= kTieCap) {
      for (uint64_t k = threadIdx.x; k < nc; k += kCandBlock) {
        oidx[pc + k] = bidx[k];
        oval[pc + k] = bval[k];
      }
      for (uint64_t k = threadIdx.x; k < nt; k += kCandBlock) {
        tidx[pt + k] = tbidx[k];
        tval[pt + k] = tbval[k];
      }
    } else {  // overflow: second pass over this chunk, writing directly
      uint64_t rc = pc, rt = pt;
      for (uint64_t base = lo; base < hi; base += 16 * kCandBlock) {
        const uint64_t i = base + 16 * threadIdx.x;
        float v[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) load4(g, i + 4 * u, hi, aligned, v + 4 * u);
        uint32_t mc = 0, mt = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t bin = key_of(v[q]) >> kShift;
          if (i + q < hi && bin >= bstar) mc |= 1u << q;
          if (i + q < hi && bin == bstar && !full) mt |= 1u << q;
        }
        uint64_t tc, tt;
        uint64_t oc = rc + block_exclusive_sum<uint64_t, kCandBlock>(__popc(mc), sh_c, tc);
        uint64_t ot = rt + block_exclusive_sum<uint64_t, kCandBlock>(__popc(mt), sh_t, tt);
        while (mc) {
          const int q = __ffs(mc) - 1;
          oidx[oc] = static_cast<uint32_t>(i + q);
          oval[oc] = v[q];
          ++oc;
          mc &= mc - 1;
        }
        while (mt) {
          const int q = __ffs(mt) - 1;
          tidx[ot] = static_cast<uint32_t>(i + q);
          tval[ot] = v[q];
          ++ot;
          mt &= mt - 1;
        }
        rc += tc;
        rt += tt;
      }
    }
  }
}

// One block: exact threshold key within bin b*, quota, and the tie cut.
__global__ void __launch_bounds__(1024) topr_refine(const uint32_t* __restrict__ tidx,
                                                    const float* __restrict__ tval, const uint32_t* ghist,
                                                    uint64_t r, Plan* plan, const uint32_t* status) {
  __shared__ uint32_t h[256];
  __shared__ uint64_t sh[40];
  __shared__ uint32_t s_digit, s_found;
  __shared__ uint64_t s_rem;
  if (failed(status) || plan->full_bin) return;
  const uint32_t bstar = plan->bin_star;
  const uint64_t nt = ghist[bstar];
  uint64_t remaining = r - plan->above;  // how many of bin b* to keep, by (key desc, idx asc)
  uint32_t prefix = bstar << kShift, mask = 0xFFFFFFFFu << kShift;
  // two 8-bit digit rounds below the bin: bits 15..8 then 7..0
  static_assert(kShift == 16, "digit rounds assume 16 bits below the bin");
  for (int round = 0; round < 2; ++round) {
    const int sh_bits = round == 0 ? 8 : 0;
    for (int i = threadIdx.x; i < 256; i += 1024) h[i] = 0;
    __syncthreads();
    for (uint64_t base = 0; base < nt; base += 4096) {  // 4 independent loads per thread in flight
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t i = base + u * 1024 + threadIdx.x;
        v[u] = i < nt ? tval[i] : -1.0f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t i = base + u * 1024 + threadIdx.x;
        const uint32_t key = key_of(v[u]);
        if (i < nt && (key & mask) == prefix) atomicAdd(&h[(key >> sh_bits) & 255], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t rem = remaining;
      int dig = 255;
      for (; dig > 0; --dig) {
        if (rem <= h[dig]) break;
        rem -= h[dig];
      }
      s_digit = static_cast<uint32_t>(dig);
      s_rem = rem;
    }
    __syncthreads();
    prefix |= s_digit << sh_bits;
    mask |= 255u << sh_bits;
    remaining = s_rem;
    __syncthreads();
  }
  const uint32_t T = prefix;
  const uint64_t q = remaining;  // keep the first q keys == T in index order
  // the q-th key == T in list (index) order: each thread counts one contiguous
  // slice, one block scan places the slices, the owning thread walks its slice
  if (threadIdx.x == 0) s_found = 0xFFFFFFFFu;
  const uint64_t per = (nt + 1023) / 1024;
  const uint64_t lo = threadIdx.x * per, hi = lo + per < nt ? lo + per : nt;
  uint64_t mine = 0;
#pragma unroll 8
  for (uint64_t i = lo; i < hi; ++i) mine += key_of(tval[i]) == T ? 1 : 0;
  uint64_t seen;
  const uint64_t before = block_exclusive_sum<uint64_t, 1024>(mine, sh, seen);
  if (before < q && q <= before + mine) {
    uint64_t c = before;
    for (uint64_t i = lo; i < hi; ++i)
      if (key_of(tval[i]) == T && ++c == q) {
        s_found = tidx[i];
        break;
      }
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
                                                            static_cast<uint64_t>(ctx->sm_count)));
  static bool attr = false;  // opt in to the 128 KiB shared histogram once per process
  if (!attr) {
    cudaFuncSetAttribute(topr_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
    attr = true;
  }
  GP_LAUNCH(ctx, topr_hist, hist_grid, kHistBlock, kBins * 4, s, grad, d, w.hist, w.status);
  GP_LAUNCH(ctx, topr_pick_bin, 1, 1024, 0, s, w.hist, r, w.plan, w.status);
  const uint64_t nblk = static_cast<uint64_t>(ctx->sm_count) * 4;
  const uint64_t chunk = std::max<uint64_t>(4096, ((d + nblk - 1) / nblk + 4095) / 4096 * 4096);  // multiple of 16*256
  const int grid = static_cast<int>(std::max<uint64_t>(1, (d + chunk - 1) / chunk));
  GP_LAUNCH(ctx, topr_candidates, grid, kCandBlock, 0, s, grad, d, chunk, w.plan, w.cand_idx, w.cand_val, w.support,
            w.values, w.u32a, reinterpret_cast<float*>(w.u32b), tiles_c, tiles_t, w.ticket, w.status);
  GP_LAUNCH(ctx, topr_refine, 1, 1024, 0, s, w.u32a, reinterpret_cast<const float*>(w.u32b), w.hist, r,
            w.plan, w.status);
  // final filter: its own scan state (tiles after both previous arrays)
  uint64_t* tiles_f = w.tiles + 2 * (ntiles + 1);
  const int fgrid = static_cast<int>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(ctx->sm_count) * 4));
  GP_LAUNCH(ctx, topr_final, std::max(fgrid, 1), kTileBlock, 0, s, w.cand_idx, w.cand_val, w.plan, w.support,
            w.values, tiles_f, w.ticket + 2, w.status);
}

}  // namespace gp
