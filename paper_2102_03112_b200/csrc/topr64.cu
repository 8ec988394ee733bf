// topr64.cu — top_r (sparsify.cpp:32-46) over an f64 input: the compensated
// worker input input = g + residual that the reference keeps in f64
// (harness.cpp:230, gradient.hpp:29), for gp_encode_topr_ef64.
//
// Same threshold select as topr.cu on the 63-bit key bits & 0x7FFF...FFFF
// (orders exactly like |x|, lower index first on ties):
//   1. topr64_hist   : input = double(g) + e written over e, 32768-bin shared
//                      histogram of key >> 48
//   2. pick_bin      : threshold bin b* and the keys above it (topr.cu)
//   3. topr64_count  : per 4096-key chunk, keys in bins >= b* and in b* alone
//      scan          : exclusive chunk offsets (scan_chunk_counts)
//      topr64_write  : candidate and tie-bin lists in index order (the tie
//                      keys compacted too) and a two-level histogram of bits
//                      47..32 of the tie keys
//   4. topr64_refine : the 32-bit key prefix off that histogram, the few keys
//                      under it from the compact tie keys, four 8-bit digit
//                      rounds for the exact T, the index of the q-th tie
//                      (topr64_refine_slow: six digit rounds over the whole
//                      tie list when one prefix holds > 4096 keys)
//   5. topr64_final  : order-preserving filter key > T or (key == T and
//                      idx <= cut) of the candidate list (count, scan, write)
//                      → support + f64 values (the gathered input)
// Lists hold indices only; keys are re-read from the (L2-resident) input.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kShift = 48;
constexpr int kBins = 1 << (63 - kShift);  // 32768
constexpr int kHistBlock = 1024;
constexpr int kChunk = 4096;
constexpr int kBlock = 256;  // 8 warps x 512 keys per chunk

__device__ __forceinline__ uint64_t key_of(double v) {
  return static_cast<uint64_t>(__double_as_longlong(v)) & 0x7FFFFFFFFFFFFFFFull;
}

__global__ void __launch_bounds__(kHistBlock) topr64_hist(const float* __restrict__ g, double* __restrict__ e,
                                                          uint64_t d, uint32_t* __restrict__ ghist,
                                                          const uint32_t* status) {
  gp_pdl_wait();
  extern __shared__ uint32_t h[];
  if (failed(status)) return;
  for (int i = threadIdx.x; i < kBins; i += kHistBlock) h[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHistBlock;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kHistBlock + threadIdx.x; i0 < d; i0 += 4 * stride) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = i0 + u * stride;
      v[u] = i < d ? __dadd_rn(static_cast<double>(g[i]), e[i]) : 0.0;  // harness.cpp:230 in f64
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < d) {
        e[i] = v[u];
        atomicAdd(&h[key_of(v[u]) >> kShift], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kHistBlock)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// per warp of a chunk: ballot masks of "bin >= b*" and "bin == b*" for row k
__device__ __forceinline__ void row_masks(const double* __restrict__ x, uint64_t i, uint64_t d, uint32_t bstar,
                                          unsigned& mc, unsigned& mt) {
  bool c = false, t = false;
  if (i < d) {
    const uint32_t bin = static_cast<uint32_t>(key_of(x[i]) >> kShift);
    c = bin >= bstar;
    t = bin == bstar;
  }
  mc = __ballot_sync(kFull, c);
  mt = __ballot_sync(kFull, t);
}

__global__ void __launch_bounds__(kBlock) topr64_count(const double* __restrict__ x, uint64_t d,
                                                       const Plan* __restrict__ plan, uint64_t* cnt_c,
                                                       uint64_t* cnt_t, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wc[kBlock / 32], wt[kBlock / 32];
  if (failed(status)) return;
  const uint32_t bstar = plan->bin_star;
  const uint64_t nchunks = (d + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t base = c * kChunk + static_cast<uint64_t>(warp) * 512;
    uint32_t nc = 0, nt = 0;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      unsigned mc, mt;
      row_masks(x, base + 32 * k + lane, d, bstar, mc, mt);
      nc += __popc(mc);
      nt += __popc(mt);
    }
    if (lane == 0) {
      wc[warp] = nc;
      wt[warp] = nt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0, b = 0;
      for (int w = 0; w < kBlock / 32; ++w) {
        a += wc[w];
        b += wt[w];
      }
      cnt_c[c] = a;
      cnt_t[c] = b;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) topr64_write(const double* __restrict__ x, uint64_t d,
                                                       const Plan* __restrict__ plan, const uint64_t* off_c,
                                                       const uint64_t* off_t, uint32_t* __restrict__ cidx,
                                                       uint32_t* __restrict__ tidx, uint64_t* __restrict__ tkey,
                                                       uint32_t* fine, uint32_t* fcoarse, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wc[kBlock / 32], wt[kBlock / 32];
  __shared__ uint32_t sc[256];  // the coarse level: few distinct values, so counted per block first
  if (failed(status)) return;
  sc[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t bstar = plan->bin_star;
  const uint64_t nchunks = (d + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t base = c * kChunk + static_cast<uint64_t>(warp) * 512;
    uint32_t nc = 0, nt = 0;
    for (int k = 0; k < 16; ++k) {
      unsigned mc, mt;
      row_masks(x, base + 32 * k + lane, d, bstar, mc, mt);
      nc += __popc(mc);
      nt += __popc(mt);
    }
    if (lane == 0) {
      wc[warp] = nc;
      wt[warp] = nt;
    }
    __syncthreads();
    uint64_t oc = off_c[c], ot = off_t[c];
    for (int w = 0; w < warp; ++w) {
      oc += wc[w];
      ot += wt[w];
    }
    for (int k = 0; k < 16; ++k) {  // the chunk is L1/L2-resident from the count above
      const uint64_t i = base + 32 * k + lane;
      unsigned mc, mt;
      row_masks(x, i, d, bstar, mc, mt);
      if (mc >> lane & 1u) cidx[oc + __popc(mc & lt)] = static_cast<uint32_t>(i);
      if (mt >> lane & 1u) {
        const uint64_t key = key_of(x[i]);
        tidx[ot + __popc(mt & lt)] = static_cast<uint32_t>(i);
        tkey[ot + __popc(mt & lt)] = key;
        atomicAdd(&fine[(key >> 32) & 0xFFFF], 1u);
        atomicAdd(&sc[(key >> 40) & 0xFF], 1u);
      }
      oc += __popc(mc);
      ot += __popc(mt);
    }
    __syncthreads();
  }
  if (sc[threadIdx.x]) atomicAdd(&fcoarse[threadIdx.x], sc[threadIdx.x]);
}

// One block: the exact threshold key T within bin b*, the tie quota and the
// tie cut, from (1) the two-level histogram of bits 47..32 of bin b*'s keys
// (built by topr64_write): the 32-bit key prefix holding the need-th key
// and its rank among the keys with that prefix — for smooth data a handful;
// (2) those keys (low 32 bits, tie-list position) collected from the compact
// tie-key list (sequential reads) into shared memory; four 8-bit digit
// rounds there give T; (3) the q-th of the keys == T in index order (tie
// list order) by a block-parallel rank.  More than kFew keys under one 32-bit
// prefix (quantised data) falls back to topr64_refine_slow.
constexpr int kFew = 4096;
// (1): the 32-bit prefix and the rank under it; one block
__global__ void __launch_bounds__(1024) topr64_refine_a(const uint32_t* ghist, const uint32_t* fine,
                                                        const uint32_t* fcoarse, uint64_t r, Plan* plan,
                                                        uint32_t* slow, uint32_t* nlist, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[40];
  __shared__ uint32_t s_c;
  __shared__ uint64_t s_before;
  if (failed(status)) return;
  const int t = threadIdx.x;
  const uint32_t bstar = plan->bin_star;
  const uint64_t need = r - plan->above;  // keys of bin b* to keep, from the top
  const uint64_t mc = t < 256 ? __ldcg(fcoarse + (255 - t)) : 0;
  uint64_t total;
  const uint64_t bc = block_exclusive_sum<uint64_t, 1024>(mc, sh, total);
  if (t < 256 && bc < need && need <= bc + mc) {
    s_c = 255 - t;
    s_before = bc;
  }
  __syncthreads();
  const uint32_t c = s_c;
  const uint64_t mf = t < 256 ? __ldcg(fine + c * 256 + (255 - t)) : 0;
  const uint64_t bf = s_before + block_exclusive_sum<uint64_t, 1024>(mf, sh, total);
  if (t < 256 && bf < need && need <= bf + mf) {
    plan->r64_prefix = (static_cast<uint64_t>(bstar) << 48) | (static_cast<uint64_t>(c * 256 + (255 - t)) << 32);
    plan->r64_need = need - bf;
    plan->r64_n = static_cast<uint32_t>(mf);
    *slow = mf > static_cast<uint64_t>(kFew) ? 1u : 0u;
    *nlist = 0;
  }
}

// (2): the tie keys under the prefix — low 32 bits and tie-list position — into
// a short global list (warp-aggregated appends; order does not matter below)
__global__ void topr64_collect(const uint64_t* __restrict__ tkey, const uint32_t* ghist, const Plan* plan,
                               const uint32_t* slow, uint32_t* lo32, uint32_t* lpos, uint32_t* nlist,
                               const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || *slow) return;
  const uint64_t nt = ghist[plan->bin_star];
  const uint64_t prefix = plan->r64_prefix;
  const int lane = threadIdx.x & 31;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x - lane; i0 < nt; i0 += stride) {
    const uint64_t i = i0 + lane;
    const bool m = i < nt && (tkey[i] & 0xFFFFFFFF00000000ull) == prefix;
    const unsigned bal = __ballot_sync(kFull, m);
    if (!bal) continue;
    uint32_t wbase = 0;
    if (lane == 0) wbase = atomicAdd(nlist, static_cast<uint32_t>(__popc(bal)));
    wbase = __shfl_sync(kFull, wbase, 0);
    if (m) {
      const uint32_t at = wbase + __popc(bal & ((1u << lane) - 1u));
      lo32[at] = static_cast<uint32_t>(tkey[i]);
      lpos[at] = static_cast<uint32_t>(i);
    }
  }
}

// (3): four 8-bit digit rounds over the list for the exact T, then the q-th of
// the keys == T in index (tie-list) order; one block
__global__ void __launch_bounds__(1024) topr64_refine_b(const uint32_t* __restrict__ tidx, const uint32_t* lo32g,
                                                        const uint32_t* lposg, Plan* plan, const uint32_t* slow,
                                                        const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t lo32[kFew], lpos[kFew];
  __shared__ uint32_t h[256];
  __shared__ uint64_t sh[40];
  __shared__ uint32_t s_digit, s_found;
  __shared__ uint64_t s_rem;
  if (failed(status) || *slow) return;
  const int t = threadIdx.x;
  const uint32_t n2 = plan->r64_n;
  const uint64_t prefix = plan->r64_prefix;
  for (uint32_t i = t; i < n2; i += 1024) {
    lo32[i] = lo32g[i];
    lpos[i] = lposg[i];
  }
  __syncthreads();
  uint64_t remaining = plan->r64_need;
  uint32_t pre = 0, mask = 0;
  for (int sh_bits = 24; sh_bits >= 0; sh_bits -= 8) {
    if (t < 256) h[t] = 0;
    __syncthreads();
    for (uint32_t i = t; i < n2; i += 1024)
      if ((lo32[i] & mask) == pre) atomicAdd(&h[(lo32[i] >> sh_bits) & 255], 1u);
    __syncthreads();
    if (t < 32) {  // the largest digit whose cumulative count from the top reaches `remaining`
      uint32_t cnt[8];
      uint64_t sum = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        cnt[u] = h[255 - 8 * t - u];
        sum += cnt[u];
      }
      const uint64_t incl = warp_inclusive_sum(sum);
      const unsigned cross = __ballot_sync(kFull, incl >= remaining);
      const int owner = cross ? __ffs(cross) - 1 : 31;
      if (t == owner) {
        uint64_t rem = remaining - (incl - sum);
        int dig = 255 - 8 * t;
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
    pre |= s_digit << sh_bits;
    mask |= 255u << sh_bits;
    remaining = s_rem;
    __syncthreads();
  }
  const uint64_t T = prefix | pre;
  const uint64_t q = remaining;  // keep the first q keys == T in index order
  // (3) the q-th of the keys == T by tie-list position; all kept -> no cut
  uint32_t eq = 0;
  for (uint32_t i = t; i < n2; i += 1024) eq += lo32[i] == pre ? 1u : 0u;
  uint64_t eqs;
  block_exclusive_sum<uint64_t, 1024>(eq, sh, eqs);
  if (t == 0) s_found = 0xFFFFFFFFu;
  __syncthreads();
  if (eqs > q) {
    for (uint32_t i = t; i < n2; i += 1024) {
      if (lo32[i] != pre) continue;
      uint32_t rank = 0;  // keys == T at earlier positions
      for (uint32_t k = 0; k < n2; ++k) rank += (lo32[k] == pre && lpos[k] < lpos[i]) ? 1u : 0u;
      if (rank + 1 == q) s_found = tidx[lpos[i]];
    }
  }
  __syncthreads();
  if (t == 0) {
    plan->thresh64 = T;
    plan->tie_cut = (eqs == q) ? 0xFFFFFFFFu : s_found;
  }
}

// The fallback of topr64_refine (> kFew keys under one 32-bit prefix): six
// 8-bit digit rounds over the whole tie list, one block.
__global__ void __launch_bounds__(1024) topr64_refine_slow(const double* __restrict__ x, const uint32_t* __restrict__ tidx,
                                                      const uint32_t* ghist, uint64_t r, Plan* plan,
                                                      const uint32_t* slow, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t h[256];
  __shared__ uint64_t sh[40];
  __shared__ uint32_t s_digit, s_found;
  __shared__ uint64_t s_rem;
  if (failed(status) || !*slow) return;
  const uint32_t bstar = plan->bin_star;
  const uint64_t nt = ghist[bstar];
  uint64_t remaining = r - plan->above;  // how many of bin b* to keep, by (key desc, idx asc)
  uint64_t prefix = static_cast<uint64_t>(bstar) << kShift, mask = ~0ull << kShift;
  for (int sh_bits = kShift - 8; sh_bits >= 0; sh_bits -= 8) {
    for (int i = threadIdx.x; i < 256; i += 1024) h[i] = 0;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < nt; i += 1024) {
      const uint64_t key = key_of(x[tidx[i]]);
      if ((key & mask) == prefix) atomicAdd(&h[(key >> sh_bits) & 255], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // the largest digit whose cumulative count from the top reaches `remaining`
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
    prefix |= static_cast<uint64_t>(s_digit) << sh_bits;
    mask |= 255ull << sh_bits;
    remaining = s_rem;
    __syncthreads();
  }
  const uint64_t T = prefix;
  const uint64_t q = remaining;  // keep the first q keys == T in index order
  if (threadIdx.x == 0) s_found = 0xFFFFFFFFu;
  const uint64_t per = (nt + 1023) / 1024;
  const uint64_t lo = threadIdx.x * per, hi = lo + per < nt ? lo + per : nt;
  uint64_t mine = 0;
  for (uint64_t i = lo; i < hi; ++i) mine += key_of(x[tidx[i]]) == T ? 1 : 0;
  uint64_t seen;
  const uint64_t before = block_exclusive_sum<uint64_t, 1024>(mine, sh, seen);
  if (before < q && q <= before + mine) {
    uint64_t c = before;
    for (uint64_t i = lo; i < hi; ++i)
      if (key_of(x[tidx[i]]) == T && ++c == q) {
        s_found = tidx[i];
        break;
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    plan->thresh64 = T;
    plan->tie_cut = (seen == q) ? 0xFFFFFFFFu : s_found;
  }
}

__device__ __forceinline__ bool keep64(const double* __restrict__ x, const uint32_t* __restrict__ cidx, uint64_t i,
                                       uint64_t n, uint64_t T, uint32_t cut) {
  if (i >= n) return false;
  const uint32_t id = cidx[i];
  const uint64_t key = key_of(x[id]);
  return key > T || (key == T && id <= cut);
}

__global__ void __launch_bounds__(kBlock) topr64_final_count(const double* __restrict__ x,
                                                             const uint32_t* __restrict__ cidx, const Plan* plan,
                                                             uint64_t* cnt, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wk[kBlock / 32];
  if (failed(status)) return;
  const uint64_t n = plan->n_cand, T = plan->thresh64;
  const uint32_t cut = plan->tie_cut;
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t base = c * kChunk + static_cast<uint64_t>(warp) * 512;
    uint32_t k = 0;
    for (int j = 0; j < 16; ++j) k += __popc(__ballot_sync(kFull, keep64(x, cidx, base + 32 * j + lane, n, T, cut)));
    if (lane == 0) wk[warp] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0;
      for (int w = 0; w < kBlock / 32; ++w) a += wk[w];
      cnt[c] = a;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) topr64_final_write(const double* __restrict__ x,
                                                             const uint32_t* __restrict__ cidx, Plan* plan,
                                                             const uint64_t* off, uint32_t* __restrict__ sidx,
                                                             double* __restrict__ sval, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wk[kBlock / 32];
  if (failed(status)) return;
  const uint64_t n = plan->n_cand, T = plan->thresh64;
  const uint32_t cut = plan->tie_cut;
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t base = c * kChunk + static_cast<uint64_t>(warp) * 512;
    uint32_t k = 0;
    for (int j = 0; j < 16; ++j) k += __popc(__ballot_sync(kFull, keep64(x, cidx, base + 32 * j + lane, n, T, cut)));
    if (lane == 0) wk[warp] = k;
    __syncthreads();
    uint64_t o = off[c];
    for (int w = 0; w < warp; ++w) o += wk[w];
    for (int j = 0; j < 16; ++j) {
      const uint64_t i = base + 32 * j + lane;
      const bool kp = keep64(x, cidx, i, n, T, cut);
      const unsigned m = __ballot_sync(kFull, kp);
      if (kp) {
        const uint32_t id = cidx[i];
        sidx[o + __popc(m & lt)] = id;
        sval[o + __popc(m & lt)] = x[id];
      }
      o += __popc(m);
    }
    __syncthreads();
  }
}

}  // namespace

void launch_topr_pick_bin(gp_ctx* ctx, uint64_t r, cudaStream_t s);  // topr.cu

// support -> ws.support, values -> ws.f64a; `residual` becomes the input g + residual
void launch_top_r64(gp_ctx* ctx, const float* grad, double* residual, uint64_t d, uint64_t r, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t nchunks = (d + kChunk - 1) / kChunk;
  fill_async(ctx, w.hist, 0, (kBins + 256 + 65536 + 256) * sizeof(uint32_t), s);
  const int hist_grid = static_cast<int>(std::min<uint64_t>((d + 4 * kHistBlock - 1) / (4 * kHistBlock),
                                                            static_cast<uint64_t>(ctx->sm_count)));
  GP_LAUNCH(ctx, topr64_hist, std::max(1, hist_grid), kHistBlock, kBins * 4, s, grad, residual, d, w.hist, w.status);
  launch_topr_pick_bin(ctx, r, s);
  uint64_t* off_c = w.tiles;
  uint64_t* off_t = w.tiles + nchunks + 1;
  uint64_t* off_f = w.tiles + 2 * (nchunks + 1);
  const int grid = static_cast<int>(std::min<uint64_t>(nchunks, static_cast<uint64_t>(ctx->sm_count) * 8));
  GP_LAUNCH(ctx, topr64_count, grid, kBlock, 0, s, residual, d, w.plan, off_c, off_t, w.status);
  GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, off_c, off_t, nchunks, w.status);
  uint32_t* fine = w.hist + kBins + 256;  // [kBins | 256 | 65536 fine | 256 coarse] (cleared above)
  uint32_t* fcoarse = fine + 65536;
  uint64_t* tkey = reinterpret_cast<uint64_t*>(w.f64b);  // compact tie keys (free during top-r)
  uint32_t* slow = w.ticket + 12;                        // zeroed below
  fill_async(ctx, slow, 0, sizeof(uint32_t), s);
  GP_LAUNCH(ctx, topr64_write, grid, kBlock, 0, s, residual, d, w.plan, off_c, off_t, w.cand_idx, w.u32a, tkey, fine,
            fcoarse, w.status);
  uint32_t* nlist = w.ticket + 13;
  GP_LAUNCH(ctx, topr64_refine_a, 1, 1024, 0, s, w.hist, fine, fcoarse, r, w.plan, slow, nlist, w.status);
  GP_LAUNCH(ctx, topr64_collect, ctx->sm_count * 4, 256, 0, s, tkey, w.hist, w.plan, slow, w.u32c, w.u32b, nlist,
            w.status);
  GP_LAUNCH(ctx, topr64_refine_b, 1, 1024, 0, s, w.u32a, w.u32c, w.u32b, w.plan, slow, w.status);
  GP_LAUNCH(ctx, topr64_refine_slow, 1, 1024, 0, s, residual, w.u32a, w.hist, r, w.plan, slow, w.status);
  GP_LAUNCH(ctx, topr64_final_count, grid, kBlock, 0, s, residual, w.cand_idx, w.plan, off_f, w.status);
  GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, off_f, nullptr, nchunks, w.status);
  GP_LAUNCH(ctx, topr64_final_write, grid, kBlock, 0, s, residual, w.cand_idx, w.plan, off_f, w.support, w.f64a,
            w.status);
}

void kernel_attrs_topr64() {
  cudaFuncSetAttribute(topr64_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins * 4);
}

}  // namespace gp
