// sort.cu — stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits.
//
// Used by the value codec's sort_view (curvefit.cpp:26-39: std::stable_sort
// descending) with keys mapped so that ascending key order is descending
// value order and equal values keep their input order.  The element count is
// read from a device word, so the sort runs without a host round trip.
//
// Per pass: upsweep (per-tile digit histograms, digit-major table), a
// decoupled look-back scan of the table, downsweep (stable in-tile ranks from warp
// match_any + cross-warp digit counts, 256 elements per round).
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kBlock = 256;
constexpr int kItems = 16;
constexpr int kTile = kBlock * kItems;

__global__ void __launch_bounds__(kBlock) radix_upsweep(const uint32_t* __restrict__ keys, const uint64_t* n_dev,
                                                        int shift, uint32_t* __restrict__ table,
                                                        const uint32_t* status) {
  __shared__ uint32_t h[256];
  if (failed(status)) return;
  const uint64_t n = *n_dev;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = tile * kTile;
    for (int q = threadIdx.x; q < kTile; q += kBlock)
      if (base + q < n) atomicAdd(&h[(keys[base + q] >> shift) & 255u], 1u);
    __syncthreads();
    table[threadIdx.x * ntiles + tile] = h[threadIdx.x];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) radix_downsweep(const uint32_t* __restrict__ kin,
                                                          const uint32_t* __restrict__ vin, const uint64_t* n_dev,
                                                          int shift, const uint32_t* __restrict__ table,
                                                          uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                          const uint32_t* status) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kBlock / 32][256];
  if (failed(status)) return;
  const uint64_t n = *n_dev;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    run[threadIdx.x] = table[threadIdx.x * ntiles + tile];
    __syncthreads();
    const uint64_t base = tile * kTile;
    for (int round = 0; round < kItems; ++round) {
      const uint64_t i = base + static_cast<uint64_t>(round) * kBlock + threadIdx.x;
      const bool ok = i < n;
      const uint32_t key = ok ? kin[i] : 0xFFFFFFFFu;
      const uint32_t val = ok ? vin[i] : 0u;
      const uint32_t dig = ok ? (key >> shift) & 255u : 256u;  // 256: padding, never emitted
      const unsigned peers = __match_any_sync(kFull, dig);
      const uint32_t lrank = __popc(peers & ((1u << lane) - 1));
      for (int j = lane; j < 256; j += 32) wcnt[warp][j] = 0;
      __syncwarp();
      if (ok && lrank == 0) wcnt[warp][dig] = __popc(peers);
      __syncthreads();
      if (ok) {
        uint32_t before = 0;
        for (int w2 = 0; w2 < warp; ++w2) before += wcnt[w2][dig];
        const uint32_t dst = run[dig] + before + lrank;
        kout[dst] = key;
        vout[dst] = val;
      }
      __syncthreads();
      uint32_t tot = 0;
      for (int w2 = 0; w2 < kBlock / 32; ++w2) tot += wcnt[w2][threadIdx.x];
      run[threadIdx.x] += tot;
      __syncthreads();
    }
  }
}

// In-place exclusive scan of a u32 array whose length is n_mul * tiles(*n_dev)
// entries (n_mul = 256 for digit tables), decoupled look-back, 4096 per tile.
__global__ void __launch_bounds__(kBlock) scan_u32(uint32_t* data, const uint64_t* n_dev, uint64_t n_mul,
                                                   int tile_shift, uint64_t* tiles, uint32_t* ticket,
                                                   const uint32_t* status) {
  __shared__ uint64_t sh[36];
  __shared__ uint32_t slot;
  if (failed(status)) return;
  const uint64_t n = n_mul * ((*n_dev + (1ull << tile_shift) - 1) >> tile_shift);
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  while (true) {
    const uint32_t tile = claim_tile(ticket, &slot);
    if (tile >= ntiles) break;
    const uint64_t base = static_cast<uint64_t>(tile) * kTile + static_cast<uint64_t>(threadIdx.x) * kItems;
    uint32_t v[kItems];
    uint64_t sum = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      v[q] = base + q < n ? data[base + q] : 0;
      sum += v[q];
    }
    uint64_t tot;
    uint64_t o = tile_exclusive_offset<kBlock>(sum, tile, tiles, sh, tot);
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
      if (base + q < n) data[base + q] = static_cast<uint32_t>(o);
      o += v[q];
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
// (multiple of 8), ping-ponging through (ktmp, vtmp).  n_bound sizes grids.
void launch_radix_sort(gp_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* ktmp, uint32_t* vtmp,
                       const uint64_t* n_dev, uint64_t n_bound, int bits, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = (n_bound + kTile - 1) / kTile;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, ctx->sm_count * 4ULL)));
  uint32_t *ki = keys, *vi = vals, *ko = ktmp, *vo = vtmp;
  for (int shift = 0; shift < bits; shift += 8) {
    GP_LAUNCH(ctx, radix_upsweep, grid, kBlock, 0, s, ki, n_dev, shift, w.sort_table, w.status);
    launch_table_scan(ctx, w.sort_table, n_dev, n_bound, 12, s);
    GP_LAUNCH(ctx, radix_downsweep, grid, kBlock, 0, s, ki, vi, n_dev, shift, w.sort_table, ko, vo, w.status);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  if (ki != keys) {  // odd number of passes: copy back
    cudaMemcpyAsync(keys, ki, n_bound * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(vals, vi, n_bound * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  }
}

}  // namespace gp
