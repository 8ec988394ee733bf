// dense.cu — the dense-selection fast path: bitmap index + raw f32 values in
// one pass each way (C3, NCF-style natural sparsity, where the support is the
// nonzeros: top_r(g, nnz)).
//
// Encode (`nz_count` → `nz_write`, two reads of g, the second partly from
// L2): every 8192-element tile ballots its nonzeros into the bitmap words
// (gradient.cpp:56-65, :81-86: bit i of byte i/8, LSB-first), compacts the
// nonzero values in shared memory and stores both straight into the container
// at the tile's value offset (index payload at 49, value payload at 49 +
// ceil(d/8); pipeline.cpp:171-173, :56-93 raw f32) with 16-byte stores; the
// offsets come from a counting pass over g, not a look-back chain.  The
// selection is SPECULATIVE: top_r(g, r) is the nonzero set exactly when r
// equals the nonzero count (the r largest |g| are then all nonzero keys and
// ties cannot straddle the cut, sparsify.cpp:32-46), which the counting pass
// knows.  It opens a gate word: SKIP when the count matched (the general
// top-r + bitmap + raw kernels that follow on the stream, launched against the
// gate as their status word, return at once), 0 otherwise (they run and
// overwrite every byte).  gate_merge then moves any error the general path
// latched into the context status.
//
// Decode (`bm_counts` → one-block scan → `bm_total` → `bm_scatter`): per-tile
// popcounts of the bitmap, their prefix, the popcount == r check
// (pipeline.cpp:242-243) BEFORE any write, then one pass that reads each
// tile's bitmap words and contiguous value run and writes the tile's dense
// slice: dense = fmaf(scale, v, dense) on the support (accumulate), or, in
// overwrite mode, the whole slice (scale·v on the support, 0 elsewhere —
// identical to accumulating into a zeroed vector) without reading it.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kNzBlock = 256;                  // 8 warps
constexpr int kNzTile = kNzBlock * 32;         // elements per tile: 32 per lane, 1024 per warp
constexpr uint32_t kGateSkip = 0xFFFFu;        // gate value: the fast path produced the payloads

// Copies n bytes from 4-byte-aligned shared memory to an arbitrary global
// address: single bytes up to the first 16-byte boundary and after the last,
// 16-byte stores in between (each assembled from five shared words with funnel
// shifts).  Neighbouring tiles write the other bytes of the boundary words.
// `src` must be readable 16 bytes past n.
__device__ __forceinline__ void block_store_bytes(uint8_t* dst, const uint32_t* src, uint64_t n) {
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(src);
  const uint32_t head = static_cast<uint32_t>((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
  if (n <= head + 16) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = sb[i];
    return;
  }
  for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) dst[i] = sb[i];
  const uint64_t nvec = (n - head) / 16;
  const uint32_t sh = 8 * (head & 3);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (uint64_t v = threadIdx.x; v < nvec; v += blockDim.x) {
    const uint32_t* s = src + ((head + 16 * v) >> 2);
    const uint32_t w0 = s[0], w1 = s[1], w2 = s[2], w3 = s[3], w4 = s[4];
    uint4 o;
    o.x = __funnelshift_r(w0, w1, sh);
    o.y = __funnelshift_r(w1, w2, sh);
    o.z = __funnelshift_r(w2, w3, sh);
    o.w = __funnelshift_r(w3, w4, sh);
    d4[v] = o;
  }
  for (uint64_t i = head + 16 * nvec + threadIdx.x; i < n; i += blockDim.x) dst[i] = sb[i];
}

// Loads n bytes from an arbitrary global address into 4-byte-aligned shared
// memory (the mirror of block_store_bytes): 16-byte loads from the enclosing
// aligned blocks, each output word assembled with one funnel shift (plus one
// 4-byte load of the following word); no byte-granular shared stores.  Only
// aligned blocks holding at least one wanted byte are read, so nothing past
// the source's last page is touched.  `dst` must hold ceil(n/4) + 4 words.
__device__ __forceinline__ void block_load_bytes(uint32_t* dst, const uint8_t* src, uint64_t n) {
  if (n == 0) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~static_cast<uintptr_t>(15);
  const uint32_t delta = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src) - a);
  const uint32_t q = delta >> 2, sh = 8 * (delta & 3);
  const uintptr_t end = reinterpret_cast<uintptr_t>(src) + n;
  const uint64_t nwords = (n + 3) / 4;
  const uint64_t nblk = (end - a + 15) / 16;
  for (uint64_t v = threadIdx.x; v < nblk; v += blockDim.x) {
    const uintptr_t at = a + 16 * v;
    const uint4 x = __ldcs(reinterpret_cast<const uint4*>(at));  // streamed once
    const uint32_t nx = at + 16 < end ? __ldg(reinterpret_cast<const uint32_t*>(at + 16)) : 0u;
    const uint32_t w[5] = {x.x, x.y, x.z, x.w, nx};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t j = static_cast<int64_t>(4 * v + t) - q;
      if (j >= 0 && static_cast<uint64_t>(j) < nwords) dst[j] = __funnelshift_r(w[t], w[t + 1], sh);
    }
  }
}

__device__ __forceinline__ void nz_load(const float* __restrict__ g, uint64_t d, uint64_t base, uint32_t (&x)[32]) {
  const int lane = threadIdx.x & 31;
  if (base + 1024 <= d) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = __float_as_uint(__ldcs(g + base + 32 * k + lane));
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint64_t i = base + 32 * k + lane;
      x[k] = i < d ? __float_as_uint(__ldcs(g + i)) : 0u;
    }
  }
}

// `nz_count` streams g once in warp items of 1024 keys (no block barrier; each
// warp adds its count into its tile's zeroed counter); the last block to
// finish (ticket) turns the tile counts into exclusive prefixes in place,
// checks nnz == r and opens the gate.  `nz_write` then walks the tiles in
// DESCENDING order — the tail of g that nz_count read last may still be in
// the 126 MB L2 — and stores each tile at its known offset.  Measured
// against the one-pass form with a decoupled look-back (round 2): that kernel
// spent ~2/3 of its warp samples parked at the barrier behind warp 0's
// look-back walk (ncu: 4367 of ~7000 samples "barrier"); C3 index stage
// 0.109 -> 0.077 ms, step 0.290 -> 0.251 ms (with the later PDL launches).
__global__ void __launch_bounds__(kNzBlock) nz_count(const float* __restrict__ g, uint64_t d, uint64_t r, Plan* plan,
                                                     uint64_t* tiles, uint32_t* ticket, uint32_t* gate,
                                                     const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint64_t scratch[33];
  __shared__ bool s_last;
  if (failed(status)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *gate = ld_relaxed_u32(status);  // the general path stays shut
    return;
  }
  const int lane = threadIdx.x & 31;
  const uint64_t ntiles = (d + kNzTile - 1) / kNzTile;
  const uint64_t nitems = (d + 1023) / 1024;  // warp items of 1024 keys, 8 per tile
  const bool vec = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (kNzBlock / 32);
  // no block barrier per tile: each warp adds its item's count into the
  // tile's (zeroed) counter, two items' loads in flight per iteration
  for (uint64_t it = blockIdx.x * static_cast<uint64_t>(kNzBlock / 32) + (threadIdx.x >> 5); it < nitems;
       it += 2 * nwarps) {
    const uint64_t it2 = it + nwarps;
    const uint64_t base = it * 1024, base2 = it2 * 1024;
    uint32_t c = 0, c2 = 0;
    // each item on the vector path unless it is the ragged last one (a second
    // item past the end is simply absent: no scalar fallback for it)
    const bool v1 = vec && base + 1024 <= d, v2 = vec && base2 + 1024 <= d;
    float4 v[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = v1 ? __ldg(reinterpret_cast<const float4*>(g + base + 4 * (lane + 32 * j))) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[8 + j] = v2 ? __ldg(reinterpret_cast<const float4*>(g + base2 + 4 * (lane + 32 * j)))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t n = ((__float_as_uint(v[j].x) & 0x7FFFFFFFu) != 0u) + ((__float_as_uint(v[j].y) & 0x7FFFFFFFu) != 0u) +
                         ((__float_as_uint(v[j].z) & 0x7FFFFFFFu) != 0u) + ((__float_as_uint(v[j].w) & 0x7FFFFFFFu) != 0u);
      if (j < 8) c += n; else c2 += n;
    }
    if (!v1)
      for (int k = 0; k < 32; ++k) {
        const uint64_t i = base + 32 * k + lane;
        if (i < d) c += (__float_as_uint(g[i]) & 0x7FFFFFFFu) != 0u;
      }
    if (!v2 && it2 < nitems)
      for (int k = 0; k < 32; ++k) {
        const uint64_t i = base2 + 32 * k + lane;
        if (i < d) c2 += (__float_as_uint(g[i]) & 0x7FFFFFFFu) != 0u;
      }
    c = __reduce_add_sync(kFull, c);
    c2 = __reduce_add_sync(kFull, c2);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&tiles[it >> 3]), static_cast<unsigned long long>(c));
      if (it2 < nitems)
        atomicAdd(reinterpret_cast<unsigned long long*>(&tiles[it2 >> 3]), static_cast<unsigned long long>(c2));
    }
  }
  __threadfence();  // this thread's counter adds, before the block's ticket (one fence per thread, not per item)
  __syncthreads();
  // last block done: exclusive prefixes of the tile counts, the nnz == r gate
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // thread i owns tiles [i per, (i + 1) per): its counts are read once, all
  // loads in flight together (16 per batch), summed, scanned, written back
  const uint64_t per = (ntiles + kNzBlock - 1) / kNzBlock;
  const uint64_t t0 = threadIdx.x * per;
  const uint64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
  constexpr int kBatch = 16;
  uint64_t cnt[kBatch];
  uint64_t mine = 0;
  for (uint64_t b = t0; b < t1; b += kBatch) {
#pragma unroll
    for (int k = 0; k < kBatch; ++k) cnt[k] = b + k < t1 ? __ldcg(&tiles[b + k]) : 0;
#pragma unroll
    for (int k = 0; k < kBatch; ++k) mine += cnt[k];
  }
  uint64_t nnz = 0;
  uint64_t run = block_exclusive_sum<uint64_t, kNzBlock>(mine, scratch, nnz);
  for (uint64_t b = t0; b < t1; b += kBatch) {
    if (per > kBatch) {  // more than one batch: reload this one (the registers hold the last)
#pragma unroll
      for (int k = 0; k < kBatch; ++k) cnt[k] = b + k < t1 ? __ldcg(&tiles[b + k]) : 0;
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k)
      if (b + k < t1) {
        tiles[b + k] = run;
        run += cnt[k];
      }
  }
  if (threadIdx.x == 0) {
    if (nnz == r) {
      plan->vl = 4 * r;
      plan->n_values = r;
      plan->n_sel = r;
      *gate = kGateSkip;
    } else {
      *gate = 0u;
    }
  }
}

__global__ void __launch_bounds__(kNzBlock, 4) nz_write(const float* __restrict__ g, uint64_t d, uint64_t r,
                                                     uint8_t* out, const uint64_t* tiles, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t vals[kNzTile + 8];
  __shared__ uint32_t words[kNzBlock + 8];
  __shared__ uint32_t wcnt[kNzBlock / 32];
  if (failed(status)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t ntiles = (d + kNzTile - 1) / kNzTile;
  const uint64_t bm_bytes = (d + 7) / 8;
  uint8_t* bm_out = out + 49;
  uint8_t* val_out = out + 49 + bm_bytes;
  uint32_t x[32];
  uint64_t i = blockIdx.x;
  if (i < ntiles) nz_load(g, d, (ntiles - 1 - i) * kNzTile + static_cast<uint64_t>(warp) * 1024, x);
  for (; i < ntiles; i += gridDim.x) {
    const uint64_t tile = ntiles - 1 - i;
    uint32_t cnt = 0, myword = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const unsigned bal = __ballot_sync(kFull, (x[k] & 0x7FFFFFFFu) != 0u);
      if (lane == k) myword = bal;
      cnt += __popc(bal);
    }
    words[threadIdx.x] = myword;
    if (lane == 0) wcnt[warp] = cnt;
    const uint64_t tile_prefix = __ldg(&tiles[tile]);
    __syncthreads();
    uint32_t at = 0, tile_total = 0;
#pragma unroll
    for (int w = 0; w < kNzBlock / 32; ++w) {
      const uint32_t c = wcnt[w];
      at += w < warp ? c : 0u;
      tile_total += c;
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const bool nz = (x[k] & 0x7FFFFFFFu) != 0u;
      const unsigned bal = __ballot_sync(kFull, nz);
      if (nz) vals[at + __popc(bal & lt)] = x[k];
      at += __popc(bal);
    }
    __syncthreads();
    const uint64_t nx = i + gridDim.x;
    if (nx < ntiles) nz_load(g, d, (ntiles - 1 - nx) * kNzTile + static_cast<uint64_t>(warp) * 1024, x);
    const uint64_t b0 = tile * (kNzTile / 8);
    const uint64_t nb = b0 + kNzTile / 8 <= bm_bytes ? kNzTile / 8 : bm_bytes - b0;
    block_store_bytes(bm_out + b0, words, nb);
    const uint64_t keep = tile_prefix >= r ? 0 : (r - tile_prefix < tile_total ? r - tile_prefix : tile_total);
    block_store_bytes(val_out + 4 * tile_prefix, vals, 4ull * keep);
    __syncthreads();
  }
}

__global__ void gate_merge(const uint32_t* gate, uint32_t* status) {
  gp_pdl_wait();
  const uint32_t gv = *gate;
  if (gv != 0u && gv != kGateSkip) latch(status, gv);
}

// ------------------------------------------------------------ decode
constexpr int kBmTileBytes = kNzTile / 8;  // 1 KiB of bitmap = 8192 coordinates per tile

// per-tile popcounts of the bitmap payload (tiles[t], u64)
__global__ void bm_counts(const uint8_t* __restrict__ in, const Plan* plan, uint64_t* counts,
                          const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_BITMAP) return;
  const uint64_t nbytes = plan->il;
  const uint8_t* p = in + plan->off_index;
  const uint64_t ntiles = (nbytes + kBmTileBytes - 1) / kBmTileBytes;
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles;
       t += warps) {
    uint32_t c = 0;
    const uint64_t b0 = t * kBmTileBytes;
#pragma unroll
    for (int q = 0; q < kBmTileBytes / 128; ++q) {
      const uint64_t at = b0 + q * 128 + 4 * lane;
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (at + k < nbytes) v |= static_cast<uint32_t>(p[at + k]) << (8 * k);
      c += __popc(v);
    }
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) counts[t] = c;
  }
}

// after the scan: total popcount, the decode's support size, the r check
__global__ void bm_total(Plan* plan, const uint64_t* counts_excl, const uint64_t* counts, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->index_method != GP_INDEX_BITMAP) return;
  const uint64_t ntiles = (plan->il + kBmTileBytes - 1) / kBmTileBytes;
  const uint64_t n = ntiles ? counts_excl[ntiles - 1] + counts[ntiles - 1] : 0;
  plan->n_sel = n;
  plan->n_values = n;
  plan->fused_bitmap = 1;
  if (n != plan->r) latch(status, GP_CORRUPT_PAYLOAD);  // pipeline.cpp:242-243
}

// One tile (8192 coordinates) per block iteration: the tile's value run is
// staged in shared memory, then warp w writes coordinates [1024w, 1024w+1024)
// of the tile, lane l coordinate 32k + l of word k (coalesced).
__global__ void __launch_bounds__(kNzBlock) bm_scatter(const uint8_t* __restrict__ in, const Plan* plan,
                                                       const uint64_t* offs, float* dense, uint64_t dense_d,
                                                       float scale, int overwrite, uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t vals[kNzTile + 8];
  __shared__ uint32_t words[kNzBlock + 8];
  __shared__ uint32_t woff[kNzBlock / 32];
  if (failed(status) || !plan->fused_bitmap) return;
  const uint64_t d = plan->d;
  if (d != dense_d) {  // to_dense builds a d-vector (gradient.cpp:38-42): a mismatch is caller misuse
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_ERROR);
    return;
  }
  const uint64_t nbytes = plan->il;
  const uint8_t* bm = in + plan->off_index;
  const uint8_t* vp = in + plan->off_value;
  const bool f64 = plan->value_method == GP_VALUE_RAW_F64;
  const uint64_t ntiles = (nbytes + kBmTileBytes - 1) / kBmTileBytes;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t b0 = t * kBmTileBytes;
    const uint64_t nb = b0 + kBmTileBytes <= nbytes ? kBmTileBytes : nbytes - b0;
    if (threadIdx.x < kNzBlock) {
      const uint64_t at = b0 + 4 * static_cast<uint64_t>(threadIdx.x);
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (at + k < b0 + nb) v |= static_cast<uint32_t>(bm[at + k]) << (8 * k);
      words[threadIdx.x] = v;
    }
    const uint64_t off = offs[t];
    __syncthreads();
    const uint32_t cnt_w = __reduce_add_sync(kFull, __popc(words[threadIdx.x]));
    if (lane == 0) woff[warp] = cnt_w;
    __syncthreads();
    uint32_t tile_n = 0, my_off = 0;
    for (int w = 0; w < kNzBlock / 32; ++w) {
      if (w == warp) my_off = tile_n;
      tile_n += woff[w];
    }
    if (!f64) {
      block_load_bytes(vals, vp + 4 * off, 4ull * tile_n);
    }
    __syncthreads();
    const uint64_t base = t * kNzTile + static_cast<uint64_t>(warp) * 1024;
    uint32_t at = my_off;
    if (!f64 && base + 1024 <= d && (reinterpret_cast<uintptr_t>(dense) & 15) == 0) {
      // 16-byte stores: row u = coordinates [128u, 128u + 128) of the warp's
      // 1024 = words 4u .. 4u + 3; lane l owns coordinates 4l .. 4l + 3 of the
      // row = bits 4(l % 8) .. +3 of word 4u + l / 8
      const uint32_t* ww = words + warp * 32;
      const int sub = lane >> 3, sh = 4 * (lane & 7);
#pragma unroll 2
      for (int u = 0; u < 8; ++u) {
        const uint32_t w0 = ww[4 * u], w1 = ww[4 * u + 1], w2 = ww[4 * u + 2], w3 = ww[4 * u + 3];
        const uint32_t wk = sub == 0 ? w0 : sub == 1 ? w1 : sub == 2 ? w2 : w3;
        const uint32_t before = (sub > 0 ? __popc(w0) : 0) + (sub > 1 ? __popc(w1) : 0) + (sub > 2 ? __popc(w2) : 0);
        const uint32_t nib = (wk >> sh) & 0xFu;
        uint32_t j = at + before + __popc(wk & ((1u << sh) - 1u));
        float4* p = reinterpret_cast<float4*>(dense + base + 128 * u + 4 * lane);
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (nib >> q & 1u) ? __uint_as_float(vals[j++]) : 0.0f;
        if (overwrite) {
          *p = make_float4((nib & 1u) ? fmaf(scale, v[0], 0.0f) : 0.0f, (nib & 2u) ? fmaf(scale, v[1], 0.0f) : 0.0f,
                           (nib & 4u) ? fmaf(scale, v[2], 0.0f) : 0.0f, (nib & 8u) ? fmaf(scale, v[3], 0.0f) : 0.0f);
        } else if (nib) {
          float4 o = *p;
          if (nib & 1u) o.x = fmaf(scale, v[0], o.x);
          if (nib & 2u) o.y = fmaf(scale, v[1], o.y);
          if (nib & 4u) o.z = fmaf(scale, v[2], o.z);
          if (nib & 8u) o.w = fmaf(scale, v[3], o.w);
          *p = o;
        }
        at += __popc(w0) + __popc(w1) + __popc(w2) + __popc(w3);
      }
    } else {
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const uint32_t wk = words[warp * 32 + k];
      const uint64_t i = base + 32 * k + lane;
      const bool on = (wk >> lane) & 1u;
      if (i < d) {
        float v = 0.0f;
        if (on) {
          const uint32_t j = at + __popc(wk & lt);
          v = f64 ? static_cast<float>(__longlong_as_double(static_cast<long long>(
                        ld_u64_unaligned(vp + 8 * (off + j)))))
                  : __uint_as_float(vals[j]);
        }
        if (overwrite) {
          dense[i] = on ? fmaf(scale, v, 0.0f) : 0.0f;
        } else if (on) {
          dense[i] = fmaf(scale, v, dense[i]);
        }
      }
      at += __popc(wk);
    }
    }
    __syncthreads();
  }
}

// overwrite mode on the general scatter path: zero the dense buffer first
// (skipped when the fused bitmap scatter writes every coordinate itself)
__global__ void dense_zero(float* dense, uint64_t n, const Plan* plan, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->fused_bitmap) return;
  float4* d4 = reinterpret_cast<float4*>(dense);
  const uint64_t n4 = (reinterpret_cast<uintptr_t>(dense) & 15) ? 0 : n / 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride)
    d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint64_t i = 4 * n4 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    dense[i] = 0.f;
}

}  // namespace

void launch_dense_zero(gp_ctx* ctx, float* dense, uint64_t n, cudaStream_t s) {
  GP_LAUNCH(ctx, dense_zero, grid_for(ctx, (n + 3) / 4, 256), 256, 0, s, dense, n, ctx->ws.plan, ctx->ws.status);
}

bool nz_fast_path_eligible(uint64_t d, uint64_t r, int index_method, int value_method) {
  // nonzero-selection workloads keep most coordinates; a top-1% selection
  // would always miss the speculation and pay an extra pass over g
  return index_method == GP_INDEX_BITMAP && value_method == GP_VALUE_NONE && 4 * r >= d && d >= kNzTile;
}

void kernel_attrs_dense() {
}

uint32_t* gate_word(gp_ctx* ctx) { return ctx->ws.status + 32; }

void launch_nz_encode(gp_ctx* ctx, const float* g, uint64_t d, uint64_t r, uint8_t* out, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = (d + kNzTile - 1) / kNzTile;
  reset_scan(ctx, s, ntiles);  // the ticket and the per-tile counters
  const uint64_t ccap = static_cast<uint64_t>(ctx->sm_count) * 8;
  const int cgrid = static_cast<int>(ntiles < ccap ? ntiles : ccap);
  const uint64_t wcap = static_cast<uint64_t>(ctx->sm_count) * 4;  // 4 resident blocks per SM (64 registers)
  const int wgrid = static_cast<int>(ntiles < wcap ? ntiles : wcap);
  GP_LAUNCH(ctx, nz_count, cgrid, kNzBlock, 0, s, g, d, r, w.plan, w.tiles, w.ticket, gate_word(ctx), w.status);
  GP_LAUNCH(ctx, nz_write, wgrid, kNzBlock, 0, s, g, d, r, out, w.tiles, w.status);
}

void launch_gate_merge(gp_ctx* ctx, cudaStream_t s) {
  GP_LAUNCH(ctx, gate_merge, 1, 1, 0, s, gate_word(ctx), ctx->ws.status);
}

// decode: counts → scan → total/check (the scatter is launch_bm_scatter)
void launch_bm_prepare(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = ((d_bound + 7) / 8 + kBmTileBytes - 1) / kBmTileBytes;
  uint64_t* counts = w.tiles;
  uint64_t* excl = w.tiles + ntiles + 1;
  GP_LAUNCH(ctx, bm_counts, grid_for(ctx, ntiles * 32, 256), 256, 0, s, in, w.plan, counts, w.status);
  cudaMemcpyAsync(excl, counts, ntiles * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
  GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, excl, nullptr, ntiles, w.status);
  GP_LAUNCH(ctx, bm_total, 1, 1, 0, s, w.plan, excl, counts, w.status);
}

void launch_bm_scatter(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, float* dense, uint64_t dense_d, float scale,
                       bool overwrite, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const uint64_t ntiles = ((d_bound + 7) / 8 + kBmTileBytes - 1) / kBmTileBytes;
  const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 6;
  const int grid = static_cast<int>(ntiles < cap ? (ntiles ? ntiles : 1) : cap);
  GP_LAUNCH(ctx, bm_scatter, grid, kNzBlock, 0, s, in, w.plan, w.tiles + ntiles + 1, dense, dense_d, scale,
            overwrite ? 1 : 0, w.status);
}

}  // namespace gp
