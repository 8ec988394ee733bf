// deflate.cu — encode side of the Deflate byte-codec slot (value id 4, byte
// codec 1; byte_compress, codecs.cpp:244-266): the slot body is a zlib stream
// (RFC 1950: 0x78 0x9C header, RFC 1951 blocks, big-endian Adler-32) of the
// 4·n little-endian f32 value bytes, framed as [codec u8][raw_len u64][body].
//
// The reference calls zlib's compress2 (level 6).  Its exact output is a
// property of zlib's sequential match finder and block heuristics; the format
// only requires a zlib stream that inflates to the bytes, which is what every
// decoder (zlib's uncompress in the reference, inflate.cu here) checks.  This
// encoder is chunk-parallel, pigz-style: the raw bytes are cut into 32 KiB
// chunks, one CTA per chunk, each coded independently as
//   * one dynamic-Huffman block of literals (f32 gradient bytes carry their
//     redundancy in the byte distribution — sign/exponent bytes — not in
//     repeated strings, so no LZ77 search), codes length-limited to 15 bits by
//     package-merge (complete codes, as inflate_table requires), or
//   * a stored block when that is not smaller,
// ending byte-aligned (an empty stored block after a Huffman block, the sync
// flush of RFC 1951 §3.2.4) so the chunks concatenate as byte strings: pass 1
// sizes every chunk, one scan places them, pass 2 writes each chunk's bits
// straight into the container.  Adler-32 is combined from per-chunk sums.
// Containers are therefore valid and round-trip exactly, but their Deflate
// slot bytes differ from zlib's.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kChunk = 32768;    // bytes per chunk (a stored block holds it whole)
constexpr int kThreads = 256;
constexpr int kPer = kChunk / kThreads;  // 128 bytes per thread
constexpr int kLit = 257;        // literals 0-255 + end of block
constexpr int kMaxBits = 15;
constexpr int kClMaxBits = 7;
constexpr int kBufWords = (kChunk + 1024) / 4;  // Huffman chunks are < kChunk + 5 bytes; + header

// package-merge work arrays (shared memory: one thread uses them)
constexpr int kMaxList = 2 * kLit;
struct PmScratch {
  uint64_t w[kLit];
  uint64_t prev[kMaxList], cur[kMaxList];
  int idx[kLit];
  int cnt[kMaxBits + 1];
  uint8_t pk[kMaxBits + 1][kMaxList];
};

// Optimal length-limited code lengths by package-merge (one thread).  freq[0..n),
// out len[0..n); symbols with freq 0 get 0.  A single used symbol is given a
// partner (zlib's trees.c does the same: a code needs two codes of length 1).
__device__ void package_merge(const uint32_t* freq, int n, int limit, uint8_t* len, PmScratch& S) {
  int* idx = S.idx;
  uint64_t* w = S.w;
  int m = 0;
  for (int i = 0; i < n; ++i) {
    len[i] = 0;
    if (freq[i]) {
      idx[m] = i;
      w[m] = freq[i];
      ++m;
    }
  }
  if (m == 0) return;
  if (m == 1) {
    len[idx[0]] = 1;
    len[idx[0] == 0 ? 1 : 0] = 1;
    return;
  }
  for (int i = 1; i < m; ++i) {  // insertion sort by weight (stable)
    const uint64_t x = w[i];
    const int y = idx[i];
    int j = i;
    while (j > 0 && w[j - 1] > x) {
      w[j] = w[j - 1];
      idx[j] = idx[j - 1];
      --j;
    }
    w[j] = x;
    idx[j] = y;
  }
  // level lists from the deepest (limit) to 1: merge of the leaves with the
  // packages (pairs) of the previous list; flags record package positions
  uint8_t(*pk)[kMaxList] = S.pk;
  int* cnt = S.cnt;
  uint64_t* prev = S.prev;
  uint64_t* cur = S.cur;
  int np = m;
  for (int i = 0; i < m; ++i) {
    prev[i] = w[i];
    pk[limit][i] = 0;
  }
  cnt[limit] = m;
  for (int lev = limit - 1; lev >= 1; --lev) {
    const int npk = np / 2;
    int a = 0, b = 0, k = 0;
    while (a < m || b < npk) {
      const uint64_t pw = b < npk ? prev[2 * b] + prev[2 * b + 1] : ~0ull;
      if (a < m && (b >= npk || w[a] <= pw)) {
        cur[k] = w[a++];
        pk[lev][k++] = 0;
      } else {
        cur[k] = pw;
        pk[lev][k++] = 1;
        ++b;
      }
    }
    cnt[lev] = k;
    for (int i = 0; i < k; ++i) prev[i] = cur[i];
    np = k;
  }
  int take = 2 * m - 2;
  for (int lev = 1; lev <= limit && take > 0; ++lev) {
    int leaves = 0, packs = 0;
    for (int i = 0; i < take && i < cnt[lev]; ++i) {
      if (pk[lev][i]) ++packs;
      else ++leaves;
    }
    for (int i = 0; i < leaves; ++i) ++len[idx[i]];
    take = 2 * packs;
  }
}

// canonical codes (RFC 1951 §3.2.2), bit-reversed for the LSB-first stream
__device__ void canonical(const uint8_t* len, int n, uint16_t* code) {
  uint16_t bl_count[kMaxBits + 1] = {0};
  for (int i = 0; i < n; ++i) bl_count[len[i]]++;
  bl_count[0] = 0;
  uint16_t next[kMaxBits + 2];
  uint32_t c = 0;
  for (int b = 1; b <= kMaxBits; ++b) {
    c = (c + bl_count[b - 1]) << 1;
    next[b] = static_cast<uint16_t>(c);
  }
  for (int i = 0; i < n; ++i) {
    const int l = len[i];
    if (!l) {
      code[i] = 0;
      continue;
    }
    uint32_t v = next[l]++, r = 0;
    for (int b = 0; b < l; ++b) r |= ((v >> b) & 1u) << (l - 1 - b);
    code[i] = static_cast<uint16_t>(r);
  }
}

// Per-chunk code tables (shared memory) and the dynamic-block header as a bit string.
struct ChunkCode {
  uint32_t freq[kLit];
  uint8_t len[kLit];
  uint16_t code[kLit];
  uint32_t hdr[96];      // header bits, LSB-first
  uint32_t hdr_bits;
  uint64_t huff_bits;    // header + data + EOB
  uint32_t stored;       // 1: this chunk goes out as a stored block
  uint32_t out_bytes;    // the chunk's bytes in the stream
};

__device__ __forceinline__ void put_bits(uint32_t* buf, uint32_t& at, uint32_t v, uint32_t n) {
  for (uint32_t b = 0; b < n; ++b, ++at)
    if ((v >> b) & 1u) buf[at >> 5] |= 1u << (at & 31);
}

// histogram + code lengths + header of chunk c (all threads; thread 0 builds)
__device__ void chunk_code(const uint8_t* __restrict__ raw, uint64_t L, uint64_t c, bool final_chunk,
                           ChunkCode& cc, PmScratch& pm) {
  for (int i = threadIdx.x; i < kLit; i += kThreads) cc.freq[i] = 0;
  __syncthreads();
  const uint64_t b0 = c * kChunk;
  const uint32_t nb = static_cast<uint32_t>(L - b0 < kChunk ? L - b0 : kChunk);
  for (uint32_t i = threadIdx.x; i < nb; i += kThreads) atomicAdd(&cc.freq[raw[b0 + i]], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    cc.freq[256] = 1;  // end of block
    package_merge(cc.freq, kLit, kMaxBits, cc.len, pm);
    canonical(cc.len, kLit, cc.code);
    // code-length sequence: 257 literal/length lengths, then 2 distance codes of
    // length 1 (no distances are used; inflate needs a valid distance code set)
    uint8_t seq[kLit + 2];
    for (int i = 0; i < kLit; ++i) seq[i] = cc.len[i];
    seq[kLit] = 1;
    seq[kLit + 1] = 1;
    // RLE into code-length symbols (16: repeat previous 3-6, 17: zeros 3-10, 18: zeros 11-138)
    uint8_t sym[kLit + 2], extra[kLit + 2];
    int ns = 0;
    for (int i = 0; i < kLit + 2;) {
      int run = 1;
      while (i + run < kLit + 2 && seq[i + run] == seq[i]) ++run;
      if (seq[i] == 0 && run >= 3) {
        const int r = run > 138 ? 138 : run;
        if (r >= 11) { sym[ns] = 18; extra[ns++] = static_cast<uint8_t>(r - 11); }
        else { sym[ns] = 17; extra[ns++] = static_cast<uint8_t>(r - 3); }
        i += r;
      } else if (seq[i] != 0 && run >= 4) {
        sym[ns] = seq[i];
        extra[ns++] = 0;
        const int r = run - 1 > 6 ? 6 : run - 1;
        sym[ns] = 16;
        extra[ns++] = static_cast<uint8_t>(r - 3);
        i += 1 + r;
      } else {
        sym[ns] = seq[i];
        extra[ns++] = 0;
        i += 1;
      }
    }
    uint32_t clf[19] = {0};
    for (int i = 0; i < ns; ++i) clf[sym[i]]++;
    uint8_t cll[19];
    uint16_t clc[19];
    package_merge(clf, 19, kClMaxBits, cll, pm);
    canonical(cll, 19, clc);
    static const uint8_t kOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int nclen = 19;
    while (nclen > 4 && cll[kOrder[nclen - 1]] == 0) --nclen;
    for (int i = 0; i < 96; ++i) cc.hdr[i] = 0;
    uint32_t at = 0;
    put_bits(cc.hdr, at, final_chunk ? 1u : 0u, 1);
    put_bits(cc.hdr, at, 2u, 2);  // BTYPE 10: dynamic
    put_bits(cc.hdr, at, 0u, 5);  // HLIT = 257 - 257
    put_bits(cc.hdr, at, 1u, 5);  // HDIST = 2 - 1
    put_bits(cc.hdr, at, static_cast<uint32_t>(nclen - 4), 4);
    for (int i = 0; i < nclen; ++i) put_bits(cc.hdr, at, cll[kOrder[i]], 3);
    for (int i = 0; i < ns; ++i) {
      put_bits(cc.hdr, at, clc[sym[i]], cll[sym[i]]);
      if (sym[i] == 16) put_bits(cc.hdr, at, extra[i], 2);
      if (sym[i] == 17) put_bits(cc.hdr, at, extra[i], 3);
      if (sym[i] == 18) put_bits(cc.hdr, at, extra[i], 7);
    }
    cc.hdr_bits = at;
    uint64_t bits = at;
    for (int i = 0; i < 256; ++i) bits += static_cast<uint64_t>(cc.freq[i]) * cc.len[i];
    bits += cc.len[256];
    cc.huff_bits = bits;
    // byte-aligned end: the final chunk pads; others add an empty stored block
    const uint64_t huff_bytes = final_chunk ? (bits + 7) / 8 : ((bits + 3 + 7) / 8 + 4);
    const uint64_t stored_bytes = 5 + static_cast<uint64_t>(nb);
    cc.stored = huff_bytes >= stored_bytes ? 1u : 0u;
    cc.out_bytes = static_cast<uint32_t>(cc.stored ? stored_bytes : huff_bytes);
  }
  __syncthreads();
}

// pass 1: per-chunk output sizes (sizes[c]) and Adler-32 partials
__global__ void __launch_bounds__(kThreads) deflate_size(const float* __restrict__ v32, const Plan* plan,
                                                         uint64_t* sizes, uint64_t* adler, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ ChunkCode cc;
  __shared__ PmScratch pm;
  __shared__ uint64_t red[2][kThreads / 32];
  if (failed(status) || plan->value_method != GP_VALUE_DEFLATE_SLOT) return;
  const uint64_t L = 4 * plan->n_values;
  const uint64_t nch = (L + kChunk - 1) / kChunk;
  const uint8_t* raw = reinterpret_cast<const uint8_t*>(v32);
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    chunk_code(raw, L, c, c + 1 == nch, cc, pm);
    // Adler-32 of the chunk: s1 = sum of bytes, s2 = sum (nb - i) * byte_i (exact, reduced at the combine)
    const uint64_t b0 = c * kChunk;
    const uint32_t nb = static_cast<uint32_t>(L - b0 < kChunk ? L - b0 : kChunk);
    uint64_t s1 = 0, s2 = 0;
    for (uint32_t i = threadIdx.x; i < nb; i += kThreads) {
      const uint64_t x = raw[b0 + i];
      s1 += x;
      s2 += x * (nb - i);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = s1;
      red[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0, b = 0;
      for (int w = 0; w < kThreads / 32; ++w) {
        a += red[0][w];
        b += red[1][w];
      }
      sizes[c] = cc.out_bytes;
      adler[2 * c] = a;
      adler[2 * c + 1] = b;
    }
    __syncthreads();
  }
}

// pass 2: every chunk's bytes at its offset (offs = exclusive scan of sizes)
__global__ void __launch_bounds__(kThreads) deflate_emit(const float* __restrict__ v32, const Plan* plan,
                                                         const uint64_t* offs, uint8_t* out, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ ChunkCode cc;
  __shared__ uint32_t buf[kBufWords];
  __shared__ uint64_t sh[40];
  if (failed(status) || plan->value_method != GP_VALUE_DEFLATE_SLOT) return;
  const uint64_t L = 4 * plan->n_values;
  const uint64_t nch = (L + kChunk - 1) / kChunk;
  const uint8_t* raw = reinterpret_cast<const uint8_t*>(v32);
  uint8_t* body = out + 49 + plan->il + 9 + 2;  // after the slot framing and the zlib header
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const bool fin = c + 1 == nch;
    static_assert(sizeof(PmScratch) <= sizeof(buf), "package-merge scratch lives in the bit buffer");
    chunk_code(raw, L, c, fin, cc, *reinterpret_cast<PmScratch*>(buf));
    const uint64_t b0 = c * kChunk;
    const uint32_t nb = static_cast<uint32_t>(L - b0 < kChunk ? L - b0 : kChunk);
    uint8_t* dst = body + offs[c];
    if (cc.stored) {  // BFINAL, BTYPE 00, pad, LEN, NLEN, the bytes
      if (threadIdx.x == 0) {
        dst[0] = fin ? 1 : 0;
        dst[1] = static_cast<uint8_t>(nb);
        dst[2] = static_cast<uint8_t>(nb >> 8);
        dst[3] = static_cast<uint8_t>(~nb);
        dst[4] = static_cast<uint8_t>(~nb >> 8);
      }
      for (uint32_t i = threadIdx.x; i < nb; i += kThreads) dst[5 + i] = raw[b0 + i];
      __syncthreads();
      continue;
    }
    for (int i = threadIdx.x; i < kBufWords; i += kThreads) buf[i] = 0;
    __syncthreads();
    // bits of this thread's 128-byte run, its offset after the header
    const uint32_t lo = threadIdx.x * kPer, hi = lo + kPer < nb ? lo + kPer : nb;
    uint64_t mine = 0;
    for (uint32_t i = lo; i < hi; ++i) mine += cc.len[raw[b0 + i]];
    uint64_t tot;
    uint64_t at64 = cc.hdr_bits + block_exclusive_sum<uint64_t, kThreads>(mine, sh, tot);
    if (threadIdx.x == 0)
      for (uint32_t i = 0; i < (cc.hdr_bits + 31) / 32; ++i) atomicOr(&buf[i], cc.hdr[i]);
    // pack codes into 64-bit accumulators, OR whole 32-bit words into the buffer
    uint64_t acc = 0;
    uint32_t fill = static_cast<uint32_t>(at64 & 31);
    uint32_t word = static_cast<uint32_t>(at64 >> 5);
    for (uint32_t i = lo; i < hi; ++i) {
      const uint8_t s = raw[b0 + i];
      acc |= static_cast<uint64_t>(cc.code[s]) << fill;
      fill += cc.len[s];
      if (fill >= 32) {
        atomicOr(&buf[word++], static_cast<uint32_t>(acc));
        acc >>= 32;
        fill -= 32;
      }
    }
    if (fill) atomicOr(&buf[word], static_cast<uint32_t>(acc));
    __syncthreads();
    uint32_t bytes = 0;
    if (threadIdx.x == 0) {  // end of block, then the byte alignment
      uint32_t at = static_cast<uint32_t>(cc.hdr_bits + tot);
      put_bits(buf, at, cc.code[256], cc.len[256]);
      if (!fin) {
        put_bits(buf, at, 0u, 3);  // BFINAL 0, BTYPE 00: empty stored block
        at = (at + 7) & ~7u;
        put_bits(buf, at, 0x0000u, 16);
        put_bits(buf, at, 0xFFFFu, 16);
      }
      bytes = (at + 7) / 8;
      sh[36] = bytes;
    }
    __syncthreads();
    bytes = static_cast<uint32_t>(sh[36]);
    const uint8_t* bb = reinterpret_cast<const uint8_t*>(buf);
    for (uint32_t i = threadIdx.x; i < bytes; i += kThreads) dst[i] = bb[i];
    __syncthreads();
  }
}

// framing, zlib header, the empty stream's block, Adler-32, vl
__global__ void deflate_finish(Plan* plan, uint8_t* out, const uint64_t* offs, const uint64_t* sizes,
                               const uint64_t* adler, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->value_method != GP_VALUE_DEFLATE_SLOT || threadIdx.x != 0) return;
  const uint64_t L = 4 * plan->n_values;
  const uint64_t nch = (L + kChunk - 1) / kChunk;
  uint8_t* p = out + 49 + plan->il;
  p[0] = 1;  // ByteCodec::Deflate
  st_u64_unaligned(p + 1, L);
  p[9] = 0x78;  // CM 8, CINFO 7 (32 KiB window)
  p[10] = 0x9C; // FLEVEL 2 (default), FCHECK: 0x789C % 31 == 0
  uint64_t body = nch ? offs[nch - 1] + sizes[nch - 1] : 0;
  if (nch == 0) {  // empty input: one final empty stored block
    uint8_t* q = p + 11;
    q[0] = 1;
    q[1] = 0;
    q[2] = 0;
    q[3] = 0xFF;
    q[4] = 0xFF;
    body = 5;
  }
  constexpr uint64_t kMod = 65521;
  uint64_t a = 1, b = 0;
  for (uint64_t c = 0; c < nch; ++c) {  // adler32_combine, chunk by chunk
    const uint64_t nb = L - c * kChunk < kChunk ? L - c * kChunk : kChunk;
    b = (b + adler[2 * c + 1] + (nb % kMod) * a) % kMod;
    a = (a + adler[2 * c]) % kMod;
  }
  const uint32_t ad = static_cast<uint32_t>((b << 16) | a);
  uint8_t* t = p + 11 + body;
  t[0] = static_cast<uint8_t>(ad >> 24);
  t[1] = static_cast<uint8_t>(ad >> 16);
  t[2] = static_cast<uint8_t>(ad >> 8);
  t[3] = static_cast<uint8_t>(ad);
  plan->vl = 9 + 2 + body + 4;
  plan->rl = 0;
}

// f64 value sequences: their f32 bytes first (pipeline.cpp:77-80 put_f32)
__global__ void deflate_raw32(const double* __restrict__ v64, const Plan* plan, float* raw, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->value_method != GP_VALUE_DEFLATE_SLOT) return;
  const uint64_t n = plan->n_values;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    raw[i] = __double2float_rn(v64[i]);
}

}  // namespace

uint64_t deflate_slot_bound(uint64_t n) {
  const uint64_t L = 4 * n;
  return 9 + 2 + L + 5 * ((L + kChunk - 1) / kChunk) + 5 + 4;
}

void launch_values_deflate(gp_ctx* ctx, uint8_t* out, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  const float* raw = w.values;
  if (ctx->vals64) {
    float* r32 = reinterpret_cast<float*>(w.f64b);  // free during an encode's value stage
    GP_LAUNCH(ctx, deflate_raw32, grid_for(ctx, n_bound, 256), 256, 0, s, ctx->vals64, w.plan, r32, w.status);
    raw = r32;
  }
  const uint64_t nch = (4 * n_bound + kChunk - 1) / kChunk;
  uint64_t* sizes = w.tiles;
  uint64_t* offs = w.tiles + nch + 1;
  uint64_t* adler = reinterpret_cast<uint64_t*>(w.u32c);  // 2 per chunk
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(nch, ctx->sm_count * 4ull)));
  GP_LAUNCH(ctx, deflate_size, grid, kThreads, 0, s, raw, w.plan, sizes, adler, w.status);
  cudaMemcpyAsync(offs, sizes, nch * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
  GP_LAUNCH(ctx, scan_chunk_counts<8>, 1, 1024, 0, s, offs, nullptr, nch, w.status);
  GP_LAUNCH(ctx, deflate_emit, grid, kThreads, 0, s, raw, w.plan, offs, out, w.status);
  GP_LAUNCH(ctx, deflate_finish, 1, 32, 0, s, w.plan, out, offs, sizes, adler, w.status);
}

}  // namespace gp
