// topr.cu — K1/K2: top-r selection (sparsify.cpp:32-46) as a radix threshold
// select with order-preserving compaction.
//
// Reference semantics: nth_element over indices with the comparator
// (|g_a| > |g_b|) || (|g_a| == |g_b| && a < b), then sort ascending.  For f32
// data |g| orders exactly like the u32 key (bits & 0x7FFFFFFF), so the kept
// set is {key > T} plus the lowest-index {key == T} until r are kept, where
// T is the r-th largest key.
//
// Three kernels, one full pass over the d-element gradient:
//   1. topr_hist      : 32768-bin histogram of key >> 16 (shared bins) plus a
//                       256-bin coarse one (key >> 23); and a skip index: the
//                       largest bin of every 8-key group (u16 per group,
//                       d/4 bytes)
//   2. topr_select    : (cooperative) every block picks the threshold bin b*
//                       from the two-level histogram, then one ordered pass over the skip index (contiguous
//                       chunks, shared-memory staging, one look-back per
//                       chunk): only groups whose largest bin is >= b* are
//                       loaded — for a top-1% selection ~9% of the gradient's
//                       32-byte sectors — emitting every key in bins >= b*
//                       (the final support when b* is kept whole) and a
//                       two-level histogram of the low 16 key bits of bin
//                       b*'s keys; its last block reads the exact threshold T
//                       and the tie quota q off that histogram
//   3. topr_final     : order-preserving filter of the (L2-resident)
//                       candidate list: key > T, or key == T among the first
//                       q such keys — one look-back over (kept, ties) pairs
#include <cooperative_groups.h>

#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace cg = cooperative_groups;

namespace gp {

namespace {

constexpr int kShift = 16;
constexpr int kBins = 1 << (31 - kShift);  // 32768 (128 KiB of shared counters)
constexpr int kHistBlock = 1024;
constexpr int kCoarse = 256;            // key >> 23 (the exponent): 128 fine bins each
constexpr int kGroup = 8;               // keys per skip-index entry (one 32-byte sector)
constexpr uint16_t kGroupAll = 0xFFFF;  // skip-index entry that always loads

__device__ __forceinline__ uint32_t key_of(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// pick_bin: the threshold bin b* — the bin holding the r-th largest key —
// and the keys above it, from the coarse histogram (256 exponent bins), then
// the 128 fine bins of that exponent.  Block-wide (BLOCK >= 256 threads); the
// results come back in every thread.
struct BinPick {
  uint32_t bstar, full;
  uint64_t above, n_cand;
};
template <int BLOCK>
__device__ BinPick pick_bin(const uint32_t* ghist, const uint32_t* gcoarse, uint64_t r, uint64_t* sh) {
  __shared__ uint32_t s_e;
  __shared__ uint64_t s_above;
  __shared__ BinPick s_pick;
  const int t = threadIdx.x;
  // coarse: thread t owns exponent 255 - t (so the exclusive prefix counts higher exponents)
  const uint64_t mine = t < kCoarse ? __ldcg(gcoarse + (kCoarse - 1 - t)) : 0;
  uint64_t total;
  const uint64_t above = block_exclusive_sum<uint64_t, BLOCK>(mine, sh, total);
  if (t < kCoarse && above < r && r <= above + mine) {
    s_e = kCoarse - 1 - t;
    s_above = above;
  }
  __syncthreads();
  const uint32_t e = s_e;
  // fine: thread t < 128 owns bin e*128 + 127 - t
  constexpr int kSub = kBins / kCoarse;  // 128
  const uint64_t f = t < kSub ? __ldcg(ghist + e * kSub + (kSub - 1 - t)) : 0;
  const uint64_t fa = s_above + block_exclusive_sum<uint64_t, BLOCK>(f, sh, total);
  if (t < kSub && fa < r && r <= fa + f) s_pick = BinPick{e * kSub + (kSub - 1 - t), fa + f == r ? 1u : 0u, fa, fa + f};
  __syncthreads();
  return s_pick;
}

// kEF: error feedback fused into the first pass (harness.cpp:230): the pass
// reads g and the residual e, writes input = g + e over e (every later pass
// and the value gather read e as the dense input) and histograms the input.
template <bool kEF>
__global__ void __launch_bounds__(kHistBlock) topr_hist(const float* __restrict__ g, float* __restrict__ e,
                                                        uint64_t d, uint32_t* __restrict__ ghist,
                                                        uint32_t* __restrict__ gcoarse, uint16_t* __restrict__ gmax,
                                                        const uint32_t* status) {
  gp_pdl_wait();
  extern __shared__ uint32_t h[];  // kBins counters
  if (failed(status)) return;
  for (int i = threadIdx.x; i < kBins; i += kHistBlock) h[i] = 0;
  __syncthreads();
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (!kEF || (reinterpret_cast<uintptr_t>(e) & 15) == 0);
  const uint64_t n4 = aligned ? d / 4 : 0;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* e4 = reinterpret_cast<float4*>(e);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHistBlock;
  const uint32_t lane = threadIdx.x & 31;
  // warp-uniform trip count (the skip-index shuffle below needs whole warps)
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i0 - lane < n4;
       i0 += 4 * stride) {
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
      const bool ok = i0 + u * stride < n4;
      uint32_t b[4] = {key_of(v[u].x) >> kShift, key_of(v[u].y) >> kShift, key_of(v[u].z) >> kShift,
                       key_of(v[u].w) >> kShift};
      if (ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicAdd(&h[b[q]], 1u);
      }
      // skip index: the float4 pair (2j, 2j+1) is 8-key group j, held by lanes l, l^1
      uint32_t mx = ok ? max(max(b[0], b[1]), max(b[2], b[3])) : 0u;
      mx = max(mx, __shfl_xor_sync(kFull, mx, 1));
      const uint64_t f = i0 + u * stride;
      if (ok && !(f & 1) && (f >> 1) < n4 / 2) gmax[f >> 1] = static_cast<uint16_t>(mx);  // tail groups: below
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
  // groups reaching into the scalar tail (and every group of an unaligned
  // gradient) always load
  if (blockIdx.x == 0)
    for (uint64_t j = (4 * n4) / kGroup + threadIdx.x; j < (d + kGroup - 1) / kGroup; j += kHistBlock)
      gmax[j] = kGroupAll;
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kHistBlock)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
  if (threadIdx.x < kCoarse) {  // coarse bin = the 128 fine bins of one exponent
    uint32_t c = 0;
    for (int j = 0; j < kBins / kCoarse; ++j) c += h[threadIdx.x * (kBins / kCoarse) + j];
    if (c) atomicAdd(&gcoarse[threadIdx.x], c);
  }
}

// standalone pick (topr64.cu's histogram of key >> 48): the coarse level is
// summed here from the fine one
__global__ void __launch_bounds__(1024) topr_pick_bin(const uint32_t* __restrict__ ghist, uint32_t* gcoarse,
                                                      uint64_t r, Plan* plan, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[40];
  if (failed(status)) return;
  if (threadIdx.x < kCoarse) {
    uint32_t c = 0;
    for (int j = 0; j < kBins / kCoarse; ++j) c += ghist[threadIdx.x * (kBins / kCoarse) + j];
    gcoarse[threadIdx.x] = c;
  }
  __threadfence_block();
  __syncthreads();
  const BinPick p = pick_bin<1024>(ghist, gcoarse, r, sh);
  if (threadIdx.x == 0) {
    plan->bin_star = p.bstar;
    plan->above = p.above;
    plan->full_bin = p.full;
    plan->n_cand = p.n_cand;
  }
}

// One contiguous chunk of the gradient per block (claimed in order), split
// into one contiguous segment per warp.  Each warp streams its segment with
// float4 loads (16 keys per lane in flight) and buffers, in index order, its
// candidates (bin >= b*) in its own shared-memory buffer — ballot ranks only,
// no block barriers in the stream; keys of bin b* itself also count into the
// 65536-bin histogram of their low 16 bits.  Then one block combine:
// per-warp offsets, one look-back per chunk, and every warp copies its buffer
// out.  A warp whose buffer overflowed (e.g. natural sparsity, r ~ 0.6 d)
// streams its segment again and writes directly.
constexpr int kCandBlock = 256;
constexpr int kCandWarps = kCandBlock / 32;
constexpr int kWarpCandCap = 512;  // = one 512-key warp segment: dense segments never overflow
constexpr int kFine = 1 << kShift; // low-bit histogram of the threshold bin

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

// the exact threshold T within bin b* and the tie quota q (keep the first q
// keys == T in index order), read off the two-level low-bit histogram of bin
// b*: 256 coarse bins of low >> 8, then the 256 fine bins of the one found.
// Every block of topr_select computes it (2 x 1 KiB of L2 reads) instead of
// one block plus a grid barrier.
__device__ void fine_threshold(const uint32_t* fine, const uint32_t* fcoarse, uint64_t need, uint32_t bstar,
                               uint64_t* sh, uint32_t& T, uint64_t& q, uint32_t& all) {
  __shared__ uint32_t s_c, s_T, s_all;
  __shared__ uint64_t s_before, s_q;
  const int t = threadIdx.x;  // kCandBlock = 256 threads
  const uint64_t mc = __ldcg(fcoarse + (255 - t));
  uint64_t total;
  const uint64_t bc = block_exclusive_sum<uint64_t, kCandBlock>(mc, sh, total);
  if (bc < need && need <= bc + mc) {
    s_c = 255 - t;
    s_before = bc;
  }
  __syncthreads();
  const uint32_t c = s_c;
  const uint64_t mf = __ldcg(fine + c * 256 + (255 - t));
  const uint64_t bf = s_before + block_exclusive_sum<uint64_t, kCandBlock>(mf, sh, total);
  if (bf < need && need <= bf + mf) {
    s_T = (bstar << kShift) | (c * 256 + (255 - t));
    s_q = need - bf;
    s_all = (bf + mf == need) ? 1u : 0u;
  }
  __syncthreads();
  T = s_T;
  q = s_q;
  all = s_all;
}

// The skip-index stream of one warp over groups [glo, ghi) of 8 keys, in
// windows of kWin groups: (1) the window's skip-index entries, lane = group,
// ballots compact the live groups (largest bin >= b*) into the warp's list in
// shared memory — index order kept; (2) the live groups, lane = group again,
// 4 rows of 32 in flight: two 16-byte loads (one 32-byte sector) each, the
// candidates ranked by a warp scan.  Work follows the live groups (~9% of
// them at a top-1% selection), not the gradient.  emit_c(rank, index, value)
// for candidates, tie(key) for threshold-bin keys; returns the candidate count.
constexpr int kWin = 256;
template <typename EC, typename ET>
__device__ __forceinline__ uint32_t stream_groups(const float* __restrict__ g, const uint16_t* __restrict__ gmax,
                                                  uint64_t glo, uint64_t ghi, uint64_t d, bool aligned,
                                                  uint32_t bstar, uint32_t klo, uint32_t khi, uint32_t* list,
                                                  EC emit_c, ET tie) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t nc = 0;
  for (uint64_t w0 = glo; w0 < ghi; w0 += kWin) {
    const uint64_t w1 = w0 + kWin < ghi ? w0 + kWin : ghi;
    uint32_t nl = 0;
#pragma unroll 4
    for (uint64_t j0 = w0; j0 < w1; j0 += 32) {
      const uint64_t j = j0 + lane;
      const bool live = j < w1 && __ldcs(gmax + j) >= bstar;
      const unsigned bal = __ballot_sync(kFull, live);
      if (live) list[nl + __popc(bal & lt)] = static_cast<uint32_t>(j - w0);
      nl += __popc(bal);
    }
    __syncwarp();
    for (uint32_t l0 = 0; l0 < nl; l0 += 128) {
      float v[4][kGroup];
      uint64_t k0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t l = l0 + 32 * u + lane;
        k0[u] = l < nl ? (w0 + list[l]) * kGroup : d;  // d: no group
        if (k0[u] >= d) {
#pragma unroll
          for (int q = 0; q < kGroup; ++q) v[u][q] = 0.0f;
        } else if (aligned && k0[u] + kGroup <= d) {
          const float4 a = ld_f4_last(reinterpret_cast<const float4*>(g + k0[u]));
          const float4 b = ld_f4_last(reinterpret_cast<const float4*>(g + k0[u]) + 1);
          v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
          v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
        } else {
#pragma unroll
          for (int q = 0; q < kGroup; ++q) v[u][q] = k0[u] + q < d ? g[k0[u] + q] : 0.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (l0 + 32 * u >= nl) break;  // warp-uniform
        uint32_t mask = 0;
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
          const uint32_t key = key_of(v[u][q]);
          if (k0[u] + q < d && key >= klo) {
            mask |= 1u << q;
            if (key < khi) tie(key);
          }
        }
        const uint32_t cnt = __popc(mask);
        const uint32_t incl = warp_inclusive_sum(cnt);
        uint32_t o = nc + incl - cnt;
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          if (mask >> q & 1u) emit_c(o++, static_cast<uint32_t>(k0[u] + q), v[u][q]);
        nc += __shfl_sync(kFull, incl, 31);
      }
    }
    __syncwarp();
  }
  return nc;
}

// Dense selections (r > d/16, e.g. natural sparsity with r = nnz): every
// group is live, so the skip index and the live lists only cost; lane =
// group, two 16-byte loads per lane per row of 32 groups, ranks by a warp
// scan.  Same contract as stream_groups.
template <typename EC, typename ET>
__device__ __forceinline__ uint32_t stream_dense(const float* __restrict__ g, uint64_t glo, uint64_t ghi, uint64_t d,
                                                 bool aligned, uint32_t klo, uint32_t khi, EC emit_c, ET tie) {
  const int lane = threadIdx.x & 31;
  uint32_t nc = 0;
  for (uint64_t base = glo; base < ghi; base += 64) {
    float v[2][kGroup];
    uint64_t k0[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t j = base + 32 * u + lane;
      k0[u] = j < ghi ? j * kGroup : d;
      if (k0[u] >= d) {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) v[u][q] = 0.0f;
      } else if (aligned && k0[u] + kGroup <= d) {
        const float4 a = ld_f4_last(reinterpret_cast<const float4*>(g + k0[u]));
        const float4 b = ld_f4_last(reinterpret_cast<const float4*>(g + k0[u]) + 1);
        v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
        v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
      } else {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) v[u][q] = k0[u] + q < d ? g[k0[u] + q] : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      uint32_t mask = 0;
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        const uint32_t key = key_of(v[u][q]);
        if (k0[u] + q < d && key >= klo) {
          mask |= 1u << q;
          if (key < khi) tie(key);
        }
      }
      const uint32_t cnt = __popc(mask);
      const uint32_t incl = warp_inclusive_sum(cnt);
      uint32_t o = nc + incl - cnt;
#pragma unroll
      for (int q = 0; q < kGroup; ++q)
        if (mask >> q & 1u) emit_c(o++, static_cast<uint32_t>(k0[u] + q), v[u][q]);
      nc += __shfl_sync(kFull, incl, 31);
    }
  }
  return nc;
}

// Ordered filter of the candidate list into the final support: one chunk of
// the list per claimed ticket, one segment per warp, 128-entry rows ranked by
// ballots.  Keys == T are kept while their rank among the list's T-ties is
// below q, so the look-back carries (greater-than-T count, T-tie count) as
// one packed word; a tile's output offset is A + min(q, B) for the exclusive
// pair (A, B).  A counting pass, the look-back, then a writing pass over the
// (L2-resident) segment.
constexpr int kPairShift = 31;
constexpr uint64_t kPairMask = (1ull << kPairShift) - 1;
__device__ __forceinline__ uint64_t final_counts(const uint32_t* __restrict__ cidx, const float* __restrict__ cval,
                                                 uint64_t lo, uint64_t hi, uint32_t T) {
  const int lane = threadIdx.x & 31;
  uint32_t gt = 0, eq = 0;
  for (uint64_t base = lo; base < hi; base += 128) {
    const uint64_t i = base + 4 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = i + q < hi ? key_of(cval[i + q]) : 0u;
      gt += key > T ? 1u : 0u;
      eq += i + q < hi && key == T ? 1u : 0u;
    }
  }
  gt = __reduce_add_sync(kFull, gt);
  eq = __reduce_add_sync(kFull, eq);
  return static_cast<uint64_t>(gt) | (static_cast<uint64_t>(eq) << kPairShift);
}

// writes the warp's kept entries; A = kept output offset, B = T-ties before the segment
// The dense selection's two passes over a warp segment of 8-key groups
// [glo, ghi): kCount counts the keys >= klo (per-lane popcounts, one warp sum
// at the end); otherwise the kept (index, value) pairs of each 512-key round
// are staged in the warp's shared buffers at their in-round rank and copied
// out by consecutive lanes to consecutive addresses (a per-lane run of
// direct stores scattered 32 partial sectors per store instruction; at r =
// 60% of d that was most of the select's time).
template <bool kCount>
__device__ __forceinline__ uint32_t dense_pass(const float* __restrict__ g, uint64_t glo, uint64_t ghi, uint64_t d,
                                               bool aligned, uint32_t klo, uint32_t* sbi, float* sbv,
                                               uint32_t* __restrict__ oi, float* __restrict__ ov, uint64_t at) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t nc = 0;
  for (uint64_t base = glo; base < ghi; base += 64) {
    float v[2][kGroup];
    uint64_t k0[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t j = base + 32 * u + lane;
      k0[u] = j < ghi ? j * kGroup : d;
      if (k0[u] >= d) {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) v[u][q] = 0.0f;
      } else if (aligned && k0[u] + kGroup <= d) {
        const float4 a = __ldcg(reinterpret_cast<const float4*>(g + k0[u]));
        const float4 b = __ldcg(reinterpret_cast<const float4*>(g + k0[u]) + 1);
        v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
        v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
      } else {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) v[u][q] = k0[u] + q < d ? g[k0[u] + q] : 0.0f;
      }
    }
    uint32_t mask[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      mask[u] = 0;
#pragma unroll
      for (int q = 0; q < kGroup; ++q)
        if (k0[u] + q < d && key_of(v[u][q]) >= klo) mask[u] |= 1u << q;
    }
    if (kCount) {
      nc += __popc(mask[0]) + __popc(mask[1]);
      continue;
    }
    uint32_t o = 0;  // in-round rank: group (u, lane) order is index order
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t c = __popc(mask[u]);
      const uint32_t incl = warp_inclusive_sum(c);
      uint32_t p = o + incl - c;
#pragma unroll
      for (int q = 0; q < kGroup; ++q)
        if (mask[u] >> q & 1u) {
          sbi[p] = static_cast<uint32_t>(k0[u] + q);
          sbv[p] = v[u][q];
          ++p;
        }
      o += __shfl_sync(kFull, incl, 31);
    }
    __syncwarp();
    for (uint32_t k = lane; k < o; k += 32) {
      oi[at + nc + k] = sbi[k];
      ov[at + nc + k] = sbv[k];
    }
    __syncwarp();
    nc += o;
    (void)lt;
  }
  return kCount ? warp_sum(nc) : nc;
}

__device__ __forceinline__ void final_write(const uint32_t* __restrict__ cidx, const float* __restrict__ cval,
                                            uint64_t lo, uint64_t hi, uint32_t T, uint64_t q, uint64_t out,
                                            uint64_t ties, uint32_t* sidx, float* sval) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t base = lo; base < hi; base += 128) {
    const uint64_t i = base + 4 * lane;
    float v[4];
    uint32_t x[4];
    bool g4[4], e4[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      v[qq] = i + qq < hi ? cval[i + qq] : 0.0f;
      x[qq] = i + qq < hi ? cidx[i + qq] : 0u;
      const uint32_t key = key_of(v[qq]);
      g4[qq] = i + qq < hi && key > T;
      e4[qq] = i + qq < hi && key == T;
    }
    // rank of each tie among the row's ties (row order = index order)
    const RowRank re = row_rank(e4[0], e4[1], e4[2], e4[3], lt);
    bool k[4];
    uint32_t er = re.before;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      k[qq] = g4[qq] || (e4[qq] && ties + er < q);
      if (e4[qq]) ++er;
    }
    const RowRank rk = row_rank(k[0], k[1], k[2], k[3], lt);
    uint64_t oo = out + rk.before;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
      if (k[qq]) {
        sidx[oo] = x[qq];
        sval[oo] = v[qq];
        ++oo;
      }
    out += rk.total;
    ties += re.total;
  }
}

// Everything after the histogram pass, as one cooperative kernel over
// one chunk per block (about d / grid keys, grid-stride if more; no tickets,
// no look-back spins):
//   A  stream the skip index of each chunk; candidates (bins >= b*) go, in
//      index order, to the chunk's own slot [c*chunk, ...) of the
//      candidate buffer (a chunk never holds more than its keys), their count
//      to cnt[c]; threshold-bin keys feed the two-level low-bit histogram
//   B  every block reads T and q off that histogram
//   C  per chunk, the (greater than T, equal to T) counts of its candidates
//   D  per chunk, its output offset A + min(q, B) from the exclusive sum of
//      the earlier chunks' pairs (one warp reads them all), and the ordered
//      write of the kept candidates into the support
// Two grid.sync()s separate the phases; the histogram pass is the only other
// top-r kernel.
constexpr uint64_t kSelAlign = 2048;  // chunk sizes: whole 8-key groups for each of the 8 warps
__device__ void chunk_pairs(const uint32_t* __restrict__ cidx, const float* __restrict__ cval, uint64_t lo,
                            uint64_t n, uint32_t T, uint64_t* wp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t per = ((n + kCandWarps - 1) / kCandWarps + 127) / 128 * 128;
  const uint64_t a = lo + (warp * per < n ? warp * per : n), b = lo + ((warp + 1) * per < n ? (warp + 1) * per : n);
  const uint64_t pr = final_counts(cidx, cval, a, b, T);
  if (lane == 0) wp[warp] = pr;
}

__global__ void __launch_bounds__(kCandBlock) topr_select(
    const float* __restrict__ g, const uint16_t* __restrict__ gmax, const uint32_t* __restrict__ ghist,
    const uint32_t* __restrict__ gcoarse, uint64_t d, uint64_t r, Plan* plan, uint32_t* cidx, float* cval,
    uint32_t* sidx, float* sval, uint32_t* fine, uint32_t* fcoarse, uint64_t* cnt, uint64_t* pair, uint32_t* wcnt,
    uint64_t chunk, bool dense, const uint32_t* status) {
  gp_pdl_wait();
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t bidx[kCandWarps][kWarpCandCap];
  __shared__ float bval[kCandWarps][kWarpCandCap];
  __shared__ uint32_t wc[kCandWarps];
  __shared__ uint64_t wp[kCandWarps];
  __shared__ uint64_t sh[40];
  __shared__ uint64_t s_pre;
  __shared__ uint32_t live_list[kCandWarps][kWin];
  if (failed(status)) return;  // uniform: every block returns before the first grid.sync
  // the threshold bin, in every block (a few hundred L2 words; no serial
  // tail in the histogram pass, no barrier here)
  const BinPick pk = pick_bin<kCandBlock>(ghist, gcoarse, r, sh);
  const uint32_t bstar = pk.bstar;
  const uint32_t klo = bstar << kShift, khi = (bstar + 1) << kShift;
  const bool full = pk.full != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->bin_star = bstar;
    plan->above = pk.above;
    plan->full_bin = pk.full;
    plan->n_cand = pk.n_cand;
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t nchunks = (d + chunk - 1) / chunk;
  const uint64_t wseg = chunk / kCandWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto tie = [&](uint32_t key) {
    if (!full) {
      atomicAdd(&fine[key & (kFine - 1)], 1u);
      atomicAdd(&fcoarse[(key >> 8) & 255], 1u);
    }
  };
  // ---- A: candidates into per-chunk slots
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t slot = c * chunk;
    const uint64_t lo = slot + warp * wseg < d ? slot + warp * wseg : d;
    const uint64_t hi = lo + wseg < d ? lo + wseg : d;
    if (dense) {  // count now; the write pass follows (below, or straight to the support when b* is kept whole)
      uint32_t nd;
      if (full) {  // no tie histogram needed: count only
        nd = dense_pass<true>(g, lo / kGroup, (hi + kGroup - 1) / kGroup, d, aligned, klo, nullptr, nullptr,
                              nullptr, nullptr, 0);
      } else {
        nd = stream_dense(g, lo / kGroup, (hi + kGroup - 1) / kGroup, d, aligned, klo, khi,
                          [](uint32_t, uint32_t, float) {}, tie);
      }
      if (lane == 0) wcnt[c * kCandWarps + warp] = nd;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint64_t tot = 0;
        for (int w = 0; w < kCandWarps; ++w) tot += wcnt[c * kCandWarps + w];
        cnt[c] = tot;
      }
      __syncthreads();
      continue;
    }
    const uint32_t nc = stream_groups(
        g, gmax, lo / kGroup, (hi + kGroup - 1) / kGroup, d, aligned, bstar, klo, khi, live_list[warp],
        [&](uint32_t o, uint32_t idx, float v) {
          if (o < kWarpCandCap) {
            bidx[warp][o] = idx;
            bval[warp][o] = v;
          }
        },
        tie);
    if (lane == 0) wc[warp] = nc;
    __syncthreads();
    uint32_t pw = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kCandWarps; ++w) {
      if (w == warp) pw = tot;
      tot += wc[w];
    }
    const uint64_t at = slot + pw;
    if (nc <= kWarpCandCap) {
      for (uint32_t k = lane; k < nc; k += 32) {
        cidx[at + k] = bidx[warp][k];
        cval[at + k] = bval[warp][k];
      }
    } else {  // overflow (dense selections): stream the segment again, writing directly
      stream_groups(
          g, gmax, lo / kGroup, (hi + kGroup - 1) / kGroup, d, aligned, bstar, klo, khi, live_list[warp],
          [&](uint32_t o, uint32_t idx, float v) {
            cidx[at + o] = idx;
            cval[at + o] = v;
          },
          [](uint32_t) {});
    }
    if (threadIdx.x == 0) cnt[c] = tot;
    __syncthreads();
  }
  grid.sync();
  if (dense) {  // the write pass of the dense selection (the re-read of g comes largely from L2)
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const uint64_t lo = c * chunk + warp * wseg < d ? c * chunk + warp * wseg : d;
      const uint64_t hi = lo + wseg < d ? lo + wseg : d;
      uint64_t at = c * chunk;  // the chunk's slot ...
      if (full) {               // ... or, b* kept whole, its final place in the support
        if (warp == 0) {
          uint64_t v = 0;
          for (uint64_t k = lane; k < c; k += 32) v += __ldcg(cnt + k);
          v = warp_sum(v);
          if (lane == 0) s_pre = v;
        }
        __syncthreads();
        at = s_pre;
      }
      for (int w = 0; w < warp; ++w) at += __ldcg(wcnt + c * kCandWarps + w);
      uint32_t* oi = full ? sidx : cidx;
      float* ov = full ? sval : cval;
      dense_pass<false>(g, lo / kGroup, (hi + kGroup - 1) / kGroup, d, aligned, klo, bidx[warp], bval[warp], oi, ov,
                        at);
      __syncthreads();
    }
    if (full) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        plan->thresh = klo;
        plan->tie_all = 1;
      }
      return;  // uniform: every block leaves before the next grid.sync
    }
    grid.sync();
  }
  // ---- B: the exact threshold, in every block
  uint32_t T = klo, tall = 1;
  uint64_t q = 0;
  if (!full) fine_threshold(fine, fcoarse, r - pk.above, bstar, sh, T, q, tall);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan->thresh = T;
    plan->tie_q = q;
    plan->tie_all = tall;
  }
  if (tall) q = ~0ull;
  // ---- C: per-chunk (greater, equal) pairs
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    chunk_pairs(cidx, cval, c * chunk, __ldcg(cnt + c), T, wp);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
      for (int w = 0; w < kCandWarps; ++w) t += wp[w];
      pair[c] = t;
    }
    __syncthreads();
  }
  grid.sync();
  // ---- D: offsets and the ordered write
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    if (warp == 0) {
      uint64_t v = 0;
      for (uint64_t k = lane; k < c; k += 32) v += __ldcg(pair + k);
      v = warp_sum(v);
      if (lane == 0) s_pre = v;
    }
    const uint64_t n = __ldcg(cnt + c);
    chunk_pairs(cidx, cval, c * chunk, n, T, wp);
    __syncthreads();
    uint64_t pre = s_pre;
    for (int w = 0; w < warp; ++w) pre += wp[w];
    const uint64_t A = pre & kPairMask, B = pre >> kPairShift;
    const uint64_t per = ((n + kCandWarps - 1) / kCandWarps + 127) / 128 * 128;
    const uint64_t lo = c * chunk + (warp * per < n ? warp * per : n);
    const uint64_t hi = c * chunk + ((warp + 1) * per < n ? (warp + 1) * per : n);
    final_write(cidx, cval, lo, hi, T, q, A + (B < q ? B : q), B, sidx, sval);
    __syncthreads();
  }
}

}  // namespace

// residual != nullptr: error feedback — the first pass writes grad + residual
// over residual, and the selection runs on that input.
void launch_top_r(gp_ctx* ctx, const float* grad, uint64_t d, uint64_t r, cudaStream_t s, float* residual) {
  Workspace& w = ctx->ws;
  // [kBins fine | kCoarse coarse | kFine low-bit | 256 low-bit coarse] counters
  uint32_t* coarse = w.hist + kBins;
  uint32_t* fine = coarse + kCoarse;
  uint32_t* fcoarse = fine + kFine;
  fill_async(ctx, w.hist, 0, (kBins + kCoarse + kFine + 256) * sizeof(uint32_t), s);
  uint16_t* gmax = reinterpret_cast<uint16_t*>(w.u32d);  // skip index, d/8 entries
  const int hist_grid = static_cast<int>(std::min<uint64_t>((d / 4 + kHistBlock - 1) / kHistBlock + 1,
                                                            static_cast<uint64_t>(ctx->sm_count)));
  if (residual) {
    GP_LAUNCH(ctx, topr_hist<true>, hist_grid, kHistBlock, kBins * 4, s, grad, residual, d, w.hist, coarse, gmax,
              w.status);
    grad = residual;
  } else {
    GP_LAUNCH(ctx, topr_hist<false>, hist_grid, kHistBlock, kBins * 4, s, grad, nullptr, d, w.hist, coarse, gmax,
              w.status);
  }
  {  // cooperative: every block of the grid resident
    static int per_sm = 0;
    if (!per_sm) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, topr_select, kCandBlock, 0);
      per_sm = std::max(1, per_sm);
    }
    const uint64_t blocks = static_cast<uint64_t>(per_sm) * ctx->sm_count;
    uint64_t chunk = ((d + blocks - 1) / blocks + kSelAlign - 1) / kSelAlign * kSelAlign;
    chunk = std::max<uint64_t>(chunk, kSelAlign);
    const uint64_t nchunks = (d + chunk - 1) / chunk;
    const int grid = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(1, nchunks), blocks));
    uint64_t* cnt = w.tiles;
    uint64_t* pair = w.tiles + nchunks + 1;
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(w.tiles + 2 * (nchunks + 1));  // per-warp counts (dense)
    const float* gp = grad;
    const uint32_t* gh = w.hist;
    const uint32_t* gc = coarse;
    Plan* plan = w.plan;
    uint32_t* ci = w.cand_idx;
    float* cv = w.cand_val;
    uint32_t* si = w.support;
    float* sv = w.values;
    const uint32_t* st = w.status;
    bool dense = r > d / 16;
    void* args[] = {&gp, &gmax, &gh, &gc, &d, &r, &plan, &ci, &cv, &si, &sv, &fine, &fcoarse, &cnt, &pair, &wcnt, &chunk,
                    &dense, &st};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(topr_select), grid, kCandBlock, args, 0, s);
    ++ctx->launches;
  }
}

void launch_topr_pick_bin(gp_ctx* ctx, uint64_t r, cudaStream_t s) {
  GP_LAUNCH(ctx, topr_pick_bin, 1, 1024, 0, s, ctx->ws.hist, ctx->ws.hist + kBins, r, ctx->ws.plan, ctx->ws.status);
}

void kernel_attrs_topr() {  // the 128 KiB shared histogram
  cudaFuncSetAttribute(topr_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
  cudaFuncSetAttribute(topr_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
}

}  // namespace gp
