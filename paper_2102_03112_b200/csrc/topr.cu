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

// kEF: error feedback fused into the first pass (harness.cpp:230): the pass
// reads g and the residual e, writes input = g + e over e (every later pass
// and the value gather read e as the dense input) and histograms the input.
template <bool kEF>
__global__ void __launch_bounds__(kHistBlock) topr_hist(const float* __restrict__ g, float* __restrict__ e,
                                                        uint64_t d, uint32_t* __restrict__ ghist,
                                                        const uint32_t* status) {
  extern __shared__ uint32_t h[];  // kBins counters
  if (failed(status)) return;
  for (int i = threadIdx.x; i < kBins; i += kHistBlock) h[i] = 0;
  __syncthreads();
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (!kEF || (reinterpret_cast<uintptr_t>(e) & 15) == 0);
  const uint64_t n4 = aligned ? d / 4 : 0;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* e4 = reinterpret_cast<float4*>(e);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHistBlock;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    float4 v[4];  // four independent 16-byte loads in flight per thread
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * stride < n4 ? __ldcs(&g4[i0 + u * stride]) : make_float4(-1, -1, -1, -1);
    if (kEF) {
      float4 r4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r4[u] = i0 + u * stride < n4 ? e4[i0 + u * stride] : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = make_float4(__fadd_rn(v[u].x, r4[u].x), __fadd_rn(v[u].y, r4[u].y), __fadd_rn(v[u].z, r4[u].z),
                           __fadd_rn(v[u].w, r4[u].w));
        if (i0 + u * stride < n4) e4[i0 + u * stride] = v[u];
      }
    }
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
  for (uint64_t i = n4 * 4 + static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i < d; i += stride) {
    float v = g[i];
    if (kEF) {
      v = __fadd_rn(v, e[i]);
      e[i] = v;
    }
    atomicAdd(&h[key_of(v) >> kShift], 1u);
  }
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

// One contiguous chunk of the gradient per block (claimed in order), split
// into one contiguous segment per warp.  Each warp streams its segment with
// float4 loads (16 keys per lane in flight) and buffers, in index order, its
// candidates (bin >= b*) and the keys of bin b* alone in its own shared-memory
// buffers — ballot ranks only, no block barriers in the stream.  Then one block
// combine: per-warp offsets, one look-back per block (candidates on warp 0,
// ties on warp 1), and every warp copies its buffers out.  A warp whose buffer
// overflowed (e.g. natural sparsity, r ~ 0.6 d) streams its segment again and
// writes directly.
constexpr int kCandBlock = 256;
constexpr int kCandWarps = kCandBlock / 32;
constexpr int kWarpCandCap = 512;  // = one 512-key warp segment: dense segments never overflow
constexpr int kWarpTieCap = 192;

// One 128-key row of a warp: lane l holds keys 4l..4l+3 (one float4).  Ballots
// per component give, for every kept key, its rank in index order within the
// row: keys of lower lanes, then this lane's lower components.
struct RowRank {
  uint32_t own;    // this lane's 4-bit mask
  uint32_t before; // kept keys of the row before this lane's first key
  uint32_t total;  // kept keys in the row
};
__device__ __forceinline__ RowRank row_rank(bool k0, bool k1, bool k2, bool k3, unsigned lt) {
  const unsigned b0 = __ballot_sync(kFull, k0), b1 = __ballot_sync(kFull, k1);
  const unsigned b2 = __ballot_sync(kFull, k2), b3 = __ballot_sync(kFull, k3);
  RowRank r;
  r.own = (k0 ? 1u : 0u) | (k1 ? 2u : 0u) | (k2 ? 4u : 0u) | (k3 ? 8u : 0u);
  r.before = __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
  r.total = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
  return r;
}

__device__ __forceinline__ float4 load_row(const float* __restrict__ g, uint64_t i, uint64_t hi, bool aligned) {
  if (aligned && i + 3 < hi) return __ldg(reinterpret_cast<const float4*>(g + i));
  float4 x;
  x.x = i < hi ? g[i] : 0.0f;
  x.y = i + 1 < hi ? g[i + 1] : 0.0f;
  x.z = i + 2 < hi ? g[i + 2] : 0.0f;
  x.w = i + 3 < hi ? g[i + 3] : 0.0f;
  return x;
}

// Streams [lo, hi) of one warp in 128-key rows (4 rows in flight), calling
// emit_c(rank, index, value) for candidates and emit_t(...) for tie-bin keys
// with their warp-local ranks; returns the warp's (candidate, tie) counts.
template <typename EC, typename ET>
__device__ __forceinline__ void stream_segment(const float* __restrict__ g, uint64_t lo, uint64_t hi, bool aligned,
                                               uint32_t klo, uint32_t khi, bool ties, uint32_t& nc, uint32_t& nt,
                                               EC emit_c, ET emit_t) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  nc = 0;
  nt = 0;
  for (uint64_t base = lo; base < hi; base += 512) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = load_row(g, base + 128 * u + 4 * lane, hi, aligned);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = base + 128 * u + 4 * lane;
      const float v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
      bool kc[4], kt[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t key = key_of(v[q]);
        kc[q] = key >= klo && i + q < hi;
        kt[q] = ties && kc[q] && key < khi;
      }
      const RowRank rc = row_rank(kc[0], kc[1], kc[2], kc[3], lt);
      if (rc.total) {
        uint32_t o = nc + rc.before;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rc.own >> q & 1u) emit_c(o++, static_cast<uint32_t>(i + q), v[q]);
        nc += rc.total;
        if (ties) {
          const RowRank rt = row_rank(kt[0], kt[1], kt[2], kt[3], lt);
          uint32_t ot = nt + rt.before;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (rt.own >> q & 1u) emit_t(ot++, static_cast<uint32_t>(i + q), v[q]);
          nt += rt.total;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kCandBlock) topr_candidates(
    const float* __restrict__ g, uint64_t d, uint64_t chunk, const Plan* __restrict__ plan, uint32_t* cidx,
    float* cval, uint32_t* sidx, float* sval, uint32_t* tidx, float* tval, uint64_t* tiles_c, uint64_t* tiles_t,
    uint32_t* ticket, bool counted, const uint32_t* status) {
  __shared__ uint32_t bidx[kCandWarps][kWarpCandCap];
  __shared__ float bval[kCandWarps][kWarpCandCap];
  __shared__ uint32_t tbidx[kCandWarps][kWarpTieCap];
  __shared__ float tbval[kCandWarps][kWarpTieCap];
  __shared__ uint32_t wc[kCandWarps], wt[kCandWarps];
  __shared__ uint64_t s_pc, s_pt;
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint32_t bstar = plan->bin_star;
  const uint32_t klo = bstar << kShift, khi = (bstar + 1) << kShift;
  const bool full = plan->full_bin != 0;
  uint32_t* oidx = full ? sidx : cidx;
  float* oval = full ? sval : cval;
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t nchunks = (d + chunk - 1) / chunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wseg = chunk / kCandWarps;  // chunk is a multiple of 8 * 512
  while (true) {
    const uint32_t c = claim_tile(ticket, &slot);
    if (c >= nchunks) break;
    const uint64_t clo = static_cast<uint64_t>(c) * chunk, chi = clo + chunk < d ? clo + chunk : d;
    const uint64_t lo = clo + warp * wseg < chi ? clo + warp * wseg : chi;
    const uint64_t hi = lo + wseg < chi ? lo + wseg : chi;
    uint32_t nc, nt;
    stream_segment(
        g, lo, hi, aligned, klo, khi, !full, nc, nt,
        [&](uint32_t o, uint32_t idx, float v) {
          if (o < kWarpCandCap) {
            bidx[warp][o] = idx;
            bval[warp][o] = v;
          }
        },
        [&](uint32_t o, uint32_t idx, float v) {
          if (o < kWarpTieCap) {
            tbidx[warp][o] = idx;
            tbval[warp][o] = v;
          }
        });
    if (lane == 0) {
      wc[warp] = nc;
      wt[warp] = nt;
    }
    __syncthreads();
    uint32_t bc = 0, bt = 0, pc_w = 0, pt_w = 0;  // block totals, this warp's offsets in the block
#pragma unroll
    for (int w = 0; w < kCandWarps; ++w) {
      if (w == warp) {
        pc_w = bc;
        pt_w = bt;
      }
      bc += wc[w];
      bt += wt[w];
    }
    if (counted) {  // dense selections: exclusive chunk offsets from topr_count_chunks + scan_chunk_counts
      if (threadIdx.x == 0) {
        s_pc = tiles_c[c];
        s_pt = full ? 0 : tiles_t[c];
      }
    } else if (warp == 0) {
      const uint64_t p = lookback_warp(tiles_c, c, bc);
      if (lane == 0) s_pc = p;
    } else if (warp == 1 && !full) {
      const uint64_t p = lookback_warp(tiles_t, c, bt);
      if (lane == 0) s_pt = p;
    }
    __syncthreads();
    const uint64_t pc = s_pc + pc_w, pt = (full ? 0 : s_pt) + pt_w;
    if (nc <= kWarpCandCap && nt <= kWarpTieCap) {
      for (uint32_t k = lane; k < nc; k += 32) {
        oidx[pc + k] = bidx[warp][k];
        oval[pc + k] = bval[warp][k];
      }
      for (uint32_t k = lane; k < nt; k += 32) {
        tidx[pt + k] = tbidx[warp][k];
        tval[pt + k] = tbval[warp][k];
      }
    } else {  // overflow: this warp streams its segment again, writing directly
      uint32_t c2, t2;
      stream_segment(
          g, lo, hi, aligned, klo, khi, !full, c2, t2,
          [&](uint32_t o, uint32_t idx, float v) {
            oidx[pc + o] = idx;
            oval[pc + o] = v;
          },
          [&](uint32_t o, uint32_t idx, float v) {
            tidx[pt + o] = idx;
            tval[pt + o] = v;
          });
    }
  }
}

// Dense selections (r > d/16): the candidates pass over 4096-key chunks would
// spend most of its time in the look-back chain (thousands of chunks, each
// walking back over aggregates at L2 latency), so the chunk counts come from
// their own streaming pass and one scan instead.
__global__ void __launch_bounds__(kCandBlock) topr_count_chunks(const float* __restrict__ g, uint64_t d,
                                                                const Plan* __restrict__ plan, uint64_t* cnt_c,
                                                                uint64_t* cnt_t, const uint32_t* status) {
  __shared__ uint32_t wc[kCandWarps], wt[kCandWarps];
  if (failed(status)) return;
  const uint32_t bstar = plan->bin_star;
  const uint32_t klo = bstar << kShift, khi = (bstar + 1) << kShift;
  const bool full = plan->full_bin != 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t nchunks = (d + 4095) / 4096;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t lo = c * 4096 + warp * 512 < d ? c * 4096 + warp * 512 : d;
    const uint64_t hi = lo + 512 < d ? lo + 512 : d;
    uint32_t nc, nt;
    stream_segment(g, lo, hi, aligned, klo, khi, !full, nc, nt, [](uint32_t, uint32_t, float) {},
                   [](uint32_t, uint32_t, float) {});
    if (lane == 0) {
      wc[warp] = nc;
      wt[warp] = nt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0, b = 0;
#pragma unroll
      for (int w = 0; w < kCandWarps; ++w) {
        a += wc[w];
        b += wt[w];
      }
      cnt_c[c] = a;
      cnt_t[c] = b;
    }
    __syncthreads();
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
    // digit of the remaining-th key from the top: dig = the largest digit
    // with rem <= h[dig] after subtracting the digits above it (digit 0 if none
    // above it qualifies).  Warp 0, lane l owning digits 255-8l .. 248-8l: a
    // warp scan of the lane sums from the top finds the crossing lane, which
    // walks its eight digits — the same result as the sequential walk down
    // from 255, without 255 dependent shared-memory steps.
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t cnt[8];
      uint64_t sum = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        cnt[u] = h[255 - 8 * lane - u];
        sum += cnt[u];
      }
      const uint64_t incl = warp_inclusive_sum(sum);
      const unsigned cross = __ballot_sync(kFull, incl >= remaining);
      const int owner = cross ? __ffs(cross) - 1 : 31;
      if (lane == owner) {
        uint64_t rem = remaining - (incl - sum);
        int dig = 255 - 8 * lane;
#pragma unroll
        for (int u = 0; u < 8; ++u, --dig) {
          if (dig == 0 || rem <= cnt[u]) break;
          rem -= cnt[u];
        }
        s_digit = static_cast<uint32_t>(dig);
        s_rem = rem;
      }
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

// Ordered filter of the candidate list into the final support: one chunk of
// the list per claimed ticket, one segment per warp, 128-entry rows ranked by
// ballots; a counting pass, one look-back per block, then a writing pass over
// the (L2-resident) segment.
template <bool kWrite>
__device__ __forceinline__ uint32_t final_segment(const uint32_t* __restrict__ cidx, const float* __restrict__ cval,
                                                  uint64_t lo, uint64_t hi, uint32_t T, uint32_t cut,
                                                  uint32_t* sidx, float* sval, uint64_t o) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t n = 0;
  for (uint64_t base = lo; base < hi; base += 128) {
    const uint64_t i = base + 4 * lane;
    float v[4];
    uint32_t x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = i + q < hi ? cval[i + q] : 0.0f;
      x[q] = i + q < hi ? cidx[i + q] : 0u;
    }
    bool k[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = key_of(v[q]);
      k[q] = i + q < hi && (key > T || (key == T && x[q] <= cut));
    }
    const RowRank r = row_rank(k[0], k[1], k[2], k[3], lt);
    if (kWrite) {
      uint64_t oo = o + n + r.before;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (k[q]) {
          sidx[oo] = x[q];
          sval[oo] = v[q];
          ++oo;
        }
    }
    n += r.total;
  }
  return n;
}

__global__ void __launch_bounds__(kCandBlock) topr_final(const uint32_t* __restrict__ cidx,
                                                         const float* __restrict__ cval, const Plan* plan,
                                                         uint32_t* sidx, float* sval, uint64_t* tiles,
                                                         uint32_t* ticket, const uint32_t* status) {
  __shared__ uint32_t wk[kCandWarps];
  __shared__ uint64_t s_p;
  __shared__ uint32_t slot;
  if (failed(status) || plan->full_bin) return;
  const uint64_t n = plan->n_cand;
  const uint32_t T = plan->thresh, cut = plan->tie_cut;
  const uint64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 1023) / 1024 * 1024;
  const uint64_t nchunks = (n + chunk - 1) / chunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wseg = chunk / kCandWarps;  // multiple of 128
  while (true) {
    const uint32_t c = claim_tile(ticket, &slot);
    if (c >= nchunks) break;
    const uint64_t clo = static_cast<uint64_t>(c) * chunk, chi = clo + chunk < n ? clo + chunk : n;
    const uint64_t lo = clo + warp * wseg < chi ? clo + warp * wseg : chi;
    const uint64_t hi = lo + wseg < chi ? lo + wseg : chi;
    const uint32_t nk = final_segment<false>(cidx, cval, lo, hi, T, cut, sidx, sval, 0);
    if (lane == 0) wk[warp] = nk;
    __syncthreads();
    uint32_t bk = 0, pw = 0;
#pragma unroll
    for (int w = 0; w < kCandWarps; ++w) {
      if (w == warp) pw = bk;
      bk += wk[w];
    }
    if (warp == 0) {
      const uint64_t p = lookback_warp(tiles, c, bk);
      if (lane == 0) s_p = p;
    }
    __syncthreads();
    final_segment<true>(cidx, cval, lo, hi, T, cut, sidx, sval, s_p + pw);
  }
}

}  // namespace

// residual != nullptr: error feedback — the first pass writes grad + residual
// over residual, and the selection runs on that input.
void launch_top_r(gp_ctx* ctx, const float* grad, uint64_t d, uint64_t r, cudaStream_t s, float* residual) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = (d + kTile - 1) / kTile;
  cudaMemsetAsync(w.hist, 0, kBins * sizeof(uint32_t), s);
  const int fgrid = ctx->sm_count * 2;  // topr_final blocks = its chunk count bound
  reset_scan(ctx, s, 2 * (ntiles + 1) + fgrid + 1);
  uint64_t* tiles_c = w.tiles;
  uint64_t* tiles_t = w.tiles + ntiles + 1;
  const int hist_grid = static_cast<int>(std::min<uint64_t>((d / 4 + kHistBlock - 1) / kHistBlock + 1,
                                                            static_cast<uint64_t>(ctx->sm_count)));
  if (residual) {
    GP_LAUNCH(ctx, topr_hist<true>, hist_grid, kHistBlock, kBins * 4, s, grad, residual, d, w.hist, w.status);
    grad = residual;
  } else {
    GP_LAUNCH(ctx, topr_hist<false>, hist_grid, kHistBlock, kBins * 4, s, grad, nullptr, d, w.hist, w.status);
  }
  GP_LAUNCH(ctx, topr_pick_bin, 1, 1024, 0, s, w.hist, r, w.plan, w.status);
  const uint64_t nblk = static_cast<uint64_t>(ctx->sm_count) * 4;
  // multiple of 8 warps * 512.  Dense selections (r > d/16, e.g. natural
  // sparsity with r = nnz) take 4096-key chunks: one 512-key segment per warp
  // fits the staging buffers, so no segment is streamed twice.
  const uint64_t chunk = r > d / 16 ? 4096 : std::max<uint64_t>(4096, ((d + nblk - 1) / nblk + 4095) / 4096 * 4096);
  // chunks are claimed through a ticket, so the grid only needs to fill the
  // machine (5 x 44 KiB blocks per SM); a gated-off launch (dense.cu fast
  // path) then costs one wave of empty blocks instead of d / 4096
  const uint64_t nchunks = std::max<uint64_t>(1, (d + chunk - 1) / chunk);
  const int grid = static_cast<int>(std::min<uint64_t>(nchunks, static_cast<uint64_t>(ctx->sm_count) * 5));
  const bool counted = r > d / 16;
  if (counted) {
    GP_LAUNCH(ctx, topr_count_chunks, ctx->sm_count * 8, kCandBlock, 0, s, grad, d, w.plan, tiles_c, tiles_t,
              w.status);
    GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, tiles_c, tiles_t, nchunks, w.status);
  }
  GP_LAUNCH(ctx, topr_candidates, grid, kCandBlock, 0, s, grad, d, chunk, w.plan, w.cand_idx, w.cand_val, w.support,
            w.values, w.u32a, reinterpret_cast<float*>(w.u32b), tiles_c, tiles_t, w.ticket, counted, w.status);
  GP_LAUNCH(ctx, topr_refine, 1, 1024, 0, s, w.u32a, reinterpret_cast<const float*>(w.u32b), w.hist, r,
            w.plan, w.status);
  // final filter: its own scan state (tiles after both previous arrays)
  uint64_t* tiles_f = w.tiles + 2 * (ntiles + 1);
  GP_LAUNCH(ctx, topr_final, fgrid, kCandBlock, 0, s, w.cand_idx, w.cand_val, w.plan, w.support,
            w.values, tiles_f, w.ticket + 2, w.status);
}

void launch_topr_pick_bin(gp_ctx* ctx, uint64_t r, cudaStream_t s) {
  GP_LAUNCH(ctx, topr_pick_bin, 1, 1024, 0, s, ctx->ws.hist, r, ctx->ws.plan, ctx->ws.status);
}

void kernel_attrs_topr() {  // the 128 KiB shared histogram
  cudaFuncSetAttribute(topr_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
  cudaFuncSetAttribute(topr_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
}

}  // namespace gp
