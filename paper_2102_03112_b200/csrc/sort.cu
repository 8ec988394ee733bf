// sort.cu — stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits.
//
// Used by the value codec's sort_view (curvefit.cpp:26-39: std::stable_sort
// descending) with keys mapped so that ascending key order is descending
// value order and equal values keep their input order, and by the P1 replay
// (stable sort of draws).  The element count is read from a device word, so
// the sort runs without a host round trip.
//
// One histogram kernel computes the global digit counts of every pass in one
// read; then one "onesweep" kernel per pass: each block claims a 4096-key
// tile in order, ranks its keys stably (warp match_any + per-warp digit
// counters, warp-striped so that processing order is index order), publishes
// its 256 digit counts, resolves its per-digit prefix over earlier tiles with
// a decoupled look-back done one 32-tile window at a time by warp 0, and
// scatters.  Tile flags carry the pass number, so they are zeroed once per sort.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kBlock = 256;
constexpr int kItems = 8;
constexpr int kTile = kBlock * kItems;
static_assert(kTile == kSortTileKeys, "the workspace sizes the per-tile tables for kSortTileKeys");
constexpr int kSortWarps = kBlock / 32;

// digit histograms of passes [0, npass) over the keys (shared bins, warp-aggregated)
__global__ void __launch_bounds__(kBlock) radix_hist(const uint32_t* __restrict__ keys, const uint64_t* n_dev,
                                                     int npass, uint32_t* __restrict__ ghist,
                                                     const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t h[4][256];
  if (failed(status)) return;
  const uint64_t n = *n_dev;
  for (int i = threadIdx.x; i < 4 * 256; i += kBlock) h[i >> 8][i & 255] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * kBlock; i0 < n; i0 += stride) {  // warp-uniform trip count
    const uint64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    const uint32_t key = ok ? keys[i] : 0u;
    for (int p = 0; p < npass; ++p) {
      const uint32_t dig = ok ? (key >> (8 * p)) & 255u : 256u;
      const unsigned peers = __match_any_sync(kFull, dig);
      if (ok && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&h[p][dig], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += kBlock)
    if (h[i >> 8][i & 255]) atomicAdd(&ghist[i], h[i >> 8][i & 255]);
}

// FitOut (the value codec's last pass, f32 values): besides the sorted
// (key, index) pairs, write the folded fp64 sequence t of fit_prepare —
// t[s] = v[map[s]] below the sign split l, -v[map[n-1-(s-l)]] above it
// (curvefit.cpp:26-39) — and clear the identity flag if any index moved.
struct FitOut {
  const float* v = nullptr;
  double* t = nullptr;
  Plan* plan = nullptr;
};

__global__ void __launch_bounds__(kBlock) radix_onesweep(const uint32_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, const uint64_t* n_dev,
                                                         int pass, const uint32_t* __restrict__ ghist,
                                                         uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                         uint32_t* flags, uint32_t* agg, uint32_t* inc,
                                                         uint32_t* ticket, const FitOut fo, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t wcnt[kSortWarps][256];
  __shared__ uint32_t base[256];
  __shared__ __align__(16) uint32_t red_sh[kSortWarps][256];
  __shared__ uint64_t sh[40];
  __shared__ uint32_t slot;
  __shared__ int s_inc, s_lo;
  if (failed(status)) return;
  const uint64_t n = *n_dev;
  const uint32_t ntiles = static_cast<uint32_t>((n + kTile - 1) / kTile);
  const int shift = 8 * pass;
  const uint32_t kAgg = 2 * pass + 1, kInc = 2 * pass + 2;
  const uint32_t tile = claim_tile(ticket + pass, &slot);
  if (tile >= ntiles) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, d = threadIdx.x;
  for (int w = 0; w < kSortWarps; ++w) wcnt[w][d] = 0;
  // global digit base of this pass: exclusive scan of the histogram
  {
    uint64_t tot;
    base[d] = static_cast<uint32_t>(block_exclusive_sum<uint64_t, kBlock>(ghist[256 * pass + d], sh, tot));
  }
  __syncthreads();
  // ---- stable in-tile ranks (warp-striped: item j of lane l is seg[32 j + l])
  const uint64_t seg = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
  uint32_t key[kItems], val[kItems];
  uint16_t rank[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t i = seg + 32 * j + lane;
    key[j] = i < n ? kin[i] : 0u;
    val[j] = i < n ? vin[i] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const bool ok = seg + 32 * j + lane < n;
    const uint32_t dig = ok ? (key[j] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(kFull, dig);
    const uint32_t lr = __popc(peers & ((1u << lane) - 1));
    const uint32_t cur = ok ? wcnt[warp][dig] : 0u;
    __syncwarp();
    if (ok && lr == 0) wcnt[warp][dig] = cur + __popc(peers);
    __syncwarp();
    rank[j] = static_cast<uint16_t>(cur + lr);
  }
  __syncthreads();
  uint32_t total = 0;  // this tile's count of digit d; wcnt becomes the exclusive prefix over warps
  for (int w = 0; w < kSortWarps; ++w) {
    const uint32_t c = wcnt[w][d];
    wcnt[w][d] = total;
    total += c;
  }
  // ---- publish the aggregate, then look back
  agg[static_cast<uint64_t>(tile) * 256 + d] = total;
  if (tile == 0) inc[d] = total;
  __threadfence();
  __syncthreads();
  if (d == 0) atomicExch(&flags[tile], tile == 0 ? kInc : kAgg);
  uint32_t prefix = 0;
  if (tile > 0) {
    if (warp == 0) {
      // nearest predecessor with an inclusive prefix; everything after it adds its aggregate
      int start = static_cast<int>(tile);
      int found = -1;
      while (true) {
        const int p = start - 1 - lane;
        uint32_t f = kInc;
        if (p >= 0) {
          do {
            f = ld_relaxed_u32(&flags[p]);
          } while (f < kAgg);
        }
        const unsigned im = __ballot_sync(kFull, p < 0 || f == kInc);
        if (im) {
          const int q = __ffs(im) - 1;
          found = start - 1 - q;  // -1: no predecessor published an inclusive prefix
          break;
        }
        start -= 32;
      }
      if (lane == 0) {
        s_inc = found;
        s_lo = found + 1;
      }
    }
    __syncthreads();
    __threadfence();
    // inclusive prefix of tile q (if any) + aggregates of tiles (q, tile): warp w
    // sums rows lo + w, lo + w + 8, ... (lane owns 8 digits), then a cross-warp sum
    {
      const int q = s_inc, lo = s_lo;
      uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      auto add_row = [&](const uint32_t* row) {
        const uint4 x0 = __ldcg(reinterpret_cast<const uint4*>(row) + 2 * lane);
        const uint4 x1 = __ldcg(reinterpret_cast<const uint4*>(row) + 2 * lane + 1);
        acc[0] += x0.x; acc[1] += x0.y; acc[2] += x0.z; acc[3] += x0.w;
        acc[4] += x1.x; acc[5] += x1.y; acc[6] += x1.z; acc[7] += x1.w;
      };
      if (warp == 0 && q >= 0) add_row(inc + static_cast<uint64_t>(q) * 256);
      int p = lo + warp;
      for (; p + 3 * kSortWarps < static_cast<int>(tile); p += 4 * kSortWarps) {
#pragma unroll
        for (int u = 0; u < 4; ++u) add_row(agg + static_cast<uint64_t>(p + u * kSortWarps) * 256);
      }
      for (; p < static_cast<int>(tile); p += kSortWarps) add_row(agg + static_cast<uint64_t>(p) * 256);
      uint32_t* red = &red_sh[warp][0];
#pragma unroll
      for (int u = 0; u < 8; ++u) red[8 * lane + u] = acc[u];
      __syncthreads();
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) prefix += red_sh[w][d];
    }
    inc[static_cast<uint64_t>(tile) * 256 + d] = prefix + total;
    __threadfence();
    __syncthreads();
    if (d == 0) atomicExch(&flags[tile], kInc);
  }
  base[d] += prefix;
  __syncthreads();
  // ---- scatter
  const uint64_t l = fo.t ? fo.plan->sign_split : 0;
  bool moved = false;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (seg + 32 * j + lane < n) {
      const uint32_t dig = (key[j] >> shift) & 255u;
      const uint32_t dst = base[dig] + wcnt[warp][dig] + rank[j];
      kout[dst] = key[j];
      vout[dst] = val[j];
      if (fo.t) {
        const double x = static_cast<double>(fo.v[val[j]]);
        if (dst < l) fo.t[dst] = x;
        else fo.t[n - 1 - (dst - l)] = -x;
        moved |= val[j] != dst;
      }
    }
  }
  if (fo.t && __syncthreads_or(moved) && threadIdx.x == 0) fo.plan->identity = 0;
}

// In-place exclusive scan of a u32 array whose length is n_mul * tiles(*n_dev)
// entries (n_mul = 256 for digit tables), decoupled look-back, kTile per tile.
__global__ void __launch_bounds__(kBlock) scan_u32(uint32_t* data, const uint64_t* n_dev, uint64_t n_mul,
                                                   int tile_shift, uint64_t* tiles, uint32_t* ticket,
                                                   const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint64_t n = n_mul * ((*n_dev + (1ull << tile_shift) - 1) >> tile_shift);
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    // warp rounds: lane l on entry wb + 32q + l (coalesced); index order is
    // round-major within the warp, warp-major within the tile
    const uint64_t wb = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(warp) * (32 * kItems);
    uint32_t v[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint64_t i = wb + 32 * q + lane;
      v[q] = i < n ? data[i] : 0;
      sum += v[q];
    }
    const uint32_t wsum = __reduce_add_sync(kFull, sum);
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(lane == 0 ? wsum : 0, tile, tiles, sh, tot);
    o = __shfl_sync(kFull, o, 0);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      const uint32_t incl = warp_inclusive_sum(v[q]);
      const uint64_t i = wb + 32 * q + lane;
      if (i < n) data[i] = static_cast<uint32_t>(o + incl - v[q]);
      o += __shfl_sync(kFull, incl, 31);
    }
  }
}

}  // namespace

// Exclusive scan of the digit-major table of 256 * tiles(n) entries (tiles of
// 1 << tile_shift elements) with n read from a device word.
void launch_table_scan(gp_ctx* ctx, uint32_t* table, const uint64_t* n_dev, uint64_t n_bound, int tile_shift,
                       cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t entries = 256 * ((n_bound + (1ull << tile_shift) - 1) >> tile_shift);
  const uint64_t ntiles = (entries + kTile - 1) / kTile;
  reset_scan(ctx, s, ntiles + 1);
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL)));
  GP_LAUNCH(ctx, scan_u32, grid, kBlock, 0, s, table, n_dev, 256, tile_shift, w.tiles, w.ticket, w.status);
}

// Sorts (keys, vals) of length *n_dev in place over `bits` low key bits
// (multiple of 8, <= 32), ping-ponging through (ktmp, vtmp).  n_bound sizes grids.
// hist_ready: the caller already accumulated the digit histograms of every
// pass into sort_hist (the value codec's key kernel does).
void launch_radix_sort(gp_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* ktmp, uint32_t* vtmp,
                       const uint64_t* n_dev, uint64_t n_bound, int bits, cudaStream_t s, bool hist_ready,
                       const float* fit_v, double* fit_t) {
  Workspace& w = ctx->ws;
  const int npass = bits / 8;
  const uint64_t ntiles = (n_bound + kTile - 1) / kTile;
  fill_async(ctx, w.sort_flags, 0, (64 + ntiles) * sizeof(uint32_t), s);
  if (!hist_ready) {
    fill_async(ctx, w.sort_hist, 0, 4 * 256 * sizeof(uint32_t), s);
    const int hgrid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n_bound + kBlock - 1) / kBlock,
                                                                                 ctx->sm_count * 2ULL)));
    GP_LAUNCH(ctx, radix_hist, hgrid, kBlock, 0, s, keys, n_dev, npass, w.sort_hist, w.status);
  }
  uint32_t *ki = keys, *vi = vals, *ko = ktmp, *vo = vtmp;
  uint32_t* agg = w.sort_table;
  uint32_t* inc = w.sort_table + 256 * (ntiles + 1);
  for (int p = 0; p < npass; ++p) {
    FitOut fo;
    if (fit_t && p == npass - 1) {
      fo.v = fit_v;
      fo.t = fit_t;
      fo.plan = w.plan;
    }
    GP_LAUNCH(ctx, radix_onesweep, static_cast<int>(std::max<uint64_t>(1, ntiles)), kBlock, 0, s, ki, vi, n_dev, p,
              w.sort_hist, ko, vo, w.sort_flags + 64, agg, inc, w.sort_flags, fo, w.status);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  if (ki != keys) {  // odd number of passes: copy back
    cudaMemcpyAsync(keys, ki, n_bound * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(vals, vi, n_bound * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  }
}

}  // namespace gp
