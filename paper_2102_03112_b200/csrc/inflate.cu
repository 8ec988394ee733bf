// inflate.cu — decode side of the Deflate byte-codec slot (value id 4, byte codec 1).
//   byte_decompress (codecs.cpp:268-290): the slot body is a zlib stream
//   (RFC 1950 header + RFC 1951 blocks + big-endian Adler-32) that must
//   inflate to exactly raw_len = 4·count bytes; pipeline.cpp:130-139 then reads
//   count little-endian f32 values from it.
//
// The reference calls zlib's uncompress (zlib 1.3 in this image), so a stream
// is accepted here exactly when uncompress returns Z_OK with out_len == raw_len;
// every other outcome is CorruptPayloadError on both sides.  The checks mirror
// zlib's inflate: header (FCHECK, CM = 8, CINFO <= 7, no preset dictionary),
// block type 3, stored LEN/NLEN, HLIT <= 286 and HDIST <= 30, code sets that are
// over-subscribed or incomplete (incomplete allowed only for a single length-1
// code of a literal/length or distance set — inflate_table's rule), repeat code
// 16 with no previous length, repeats past HLIT + HDIST, a missing end-of-block
// code, literal/length symbols 286-287 and distance symbols 30-31, distances
// reaching before the start of the output, output beyond raw_len, input that
// ends early, and the Adler-32 trailer.  Bytes after the trailer are ignored,
// as uncompress ignores them.
//
// A DEFLATE stream is one serial dependency chain (every symbol's bit offset
// depends on every earlier symbol), so one thread inflates it: a 10-bit lookup
// table per code with a canonical bit-serial decode for longer codes, the
// 32 KiB history window in shared memory for back-references, the output
// streamed to global memory.  This is a correctness path for containers the
// reference's default CLI writes (codecs.cpp:252-259), not a bench config; the
// widen kernel then spreads the f32 bytes to the f64 value array the decode
// scatter reads.  The encode side (byte-identical zlib level-6 output) is not
// on the device path: GP_UNSUPPORTED.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

constexpr int kLutBits = 10;
constexpr int kCodes = 0, kLens = 1, kDists = 2;  // inflate_table's codetype

// canonical code over up to 288 symbols (RFC 1951 §3.2.2)
struct Code {
  uint16_t count[16];
  uint16_t sym[288];
  uint16_t lut[1 << kLutBits];  // next kLutBits stream bits -> sym << 4 | len; 0: longer (or no) code
};

struct Bits {
  const uint8_t* p;
  uint64_t pos, end;
  uint64_t buf;
  int cnt;
  __device__ __forceinline__ void fill() {
    if (cnt > 56) return;
    if (pos + 16 <= end) {  // two aligned 8-byte loads + funnel shift: whole bytes up to 57+ bits
      const uintptr_t a = reinterpret_cast<uintptr_t>(p + pos);
      const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t{7});
      const uint32_t sh = static_cast<uint32_t>(a & 7) * 8;
      const uint64_t w0 = __ldg(w), w1 = __ldg(w + 1);
      const uint64_t v = sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
      const int k = (64 - cnt) >> 3;  // bytes that fit
      buf |= (k >= 8 ? v : v & ((1ull << (8 * k)) - 1)) << cnt;
      pos += k;
      cnt += 8 * k;
      return;
    }
    while (cnt <= 56 && pos < end) {
      buf |= static_cast<uint64_t>(p[pos++]) << cnt;
      cnt += 8;
    }
  }
  __device__ __forceinline__ bool need(int n) {
    if (cnt < n) fill();
    return cnt >= n;
  }
  __device__ __forceinline__ uint32_t take(int n) {
    const uint32_t v = static_cast<uint32_t>(buf & ((1ull << n) - 1));
    buf >>= n;
    cnt -= n;
    return v;
  }
};

__constant__ uint16_t kLenBase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                      31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t kLenExtra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t kDistBase[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                       33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                       1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t kDistExtra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// inflate_table's acceptance rule plus the decode structures; false = invalid set
__device__ bool build(Code& c, const uint8_t* len, int n, int kind) {
  for (int l = 0; l < 16; ++l) c.count[l] = 0;
  for (int s = 0; s < n; ++s) ++c.count[len[s]];
  for (int e = 0; e < (1 << kLutBits); ++e) c.lut[e] = 0;
  int max = 15;
  while (max >= 1 && c.count[max] == 0) --max;
  if (max == 0) return true;  // no symbols: accepted, every decode from it fails
  int left = 1;
  for (int l = 1; l < 16; ++l) {
    left = (left << 1) - c.count[l];
    if (left < 0) return false;  // over-subscribed
  }
  if (left > 0 && (kind == kCodes || max != 1)) return false;  // incomplete
  uint16_t offs[16], next[16];
  offs[1] = 0;
  for (int l = 1; l < 15; ++l) offs[l + 1] = offs[l] + c.count[l];
  uint32_t code = 0;
  next[0] = 0;
  for (int l = 1; l < 16; ++l) {
    code = (code + (l > 1 ? c.count[l - 1] : 0)) << 1;
    next[l] = static_cast<uint16_t>(code);
  }
  for (int s = 0; s < n; ++s) {
    const int l = len[s];
    if (l == 0) continue;
    c.sym[offs[l]++] = static_cast<uint16_t>(s);
    const uint32_t cde = next[l]++;
    if (l <= kLutBits) {
      const uint32_t rev = __brev(cde) >> (32 - l);  // codes are sent MSB first into an LSB-first stream
      for (uint32_t e = rev; e < (1u << kLutBits); e += 1u << l) c.lut[e] = static_cast<uint16_t>(s << 4 | l);
    }
  }
  return true;
}

// one symbol, or -1 (invalid code / input ended)
// the kernel's tables and window live at namespace scope so every access is a
// direct LDS/STS (through a reference the compiler re-derives the shared
// window base from the CTA id on every symbol)
__shared__ uint8_t s_win[32768];
__shared__ Code s_lit, s_dist;

template <bool kDist>
__device__ __forceinline__ int decode(Bits& b) {
  const Code& c = kDist ? s_dist : s_lit;
  if (b.cnt < 15) b.fill();  // a refill (a global load) every few symbols, not on every symbol's chain
  const uint32_t e = c.lut[b.buf & ((1u << kLutBits) - 1)];
  if (e) {
    const int l = e & 15;
    if (l > b.cnt) return -1;
    b.take(l);
    return static_cast<int>(e >> 4);
  }
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    if (!b.need(1)) return -1;
    code |= static_cast<int>(b.take(1));
    const int count = c.count[l];
    if (code - count < first) return c.sym[index + (code - first)];
    index += count;
    first = (first + count) << 1;
    code <<= 1;
  }
  return -1;
}

struct Out {
  uint8_t* dst;
  uint64_t o, cap;
  uint32_t s1, s2, run;
  __device__ __forceinline__ void put(uint8_t v) {
    dst[o] = v;
    s_win[o & 32767] = v;
    ++o;
    s1 += v;
    s2 += s1;
    if (++run == 5552) {  // zlib's NMAX: no 32-bit overflow before the reduction
      s1 %= 65521u;
      s2 %= 65521u;
      run = 0;
    }
  }
};

__global__ void slot_inflate(const uint8_t* __restrict__ in, const Plan* plan, uint8_t* __restrict__ out,
                             uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  if (plan->value_method != GP_VALUE_DEFLATE_SLOT || plan->slot_id != 1) return;
  __shared__ uint8_t lens[320];
  __shared__ uint8_t cl[19];
#define GP_INFLATE_FAIL()                   \
  do {                                      \
    latch(status, GP_CORRUPT_PAYLOAD);      \
    return;                                 \
  } while (0)
  Bits b{in + plan->off_value + 9, 0, plan->vl - 9, 0, 0};
  Out w{out, 0, 4 * plan->n_values, 1, 0, 0};
  // RFC 1950 header (inflate.c HEAD)
  if (!b.need(16)) GP_INFLATE_FAIL();
  const uint32_t cmf = b.take(8), flg = b.take(8);
  if (((cmf << 8) | flg) % 31u != 0) GP_INFLATE_FAIL();
  if ((cmf & 15) != 8) GP_INFLATE_FAIL();
  if ((cmf >> 4) + 8 > 15) GP_INFLATE_FAIL();
  if (flg & 0x20) GP_INFLATE_FAIL();  // preset dictionary: uncompress reports Z_DATA_ERROR
  bool last = false;
  while (!last) {
    if (!b.need(3)) GP_INFLATE_FAIL();
    last = b.take(1) != 0;
    const uint32_t type = b.take(2);
    if (type == 0) {  // stored
      b.take(b.cnt & 7);
      if (!b.need(32)) GP_INFLATE_FAIL();
      const uint32_t n = b.take(16), nn = b.take(16);
      if (n != (~nn & 0xFFFFu)) GP_INFLATE_FAIL();
      for (uint32_t k = 0; k < n; ++k) {
        if (!b.need(8)) GP_INFLATE_FAIL();
        if (w.o >= w.cap) GP_INFLATE_FAIL();
        w.put(static_cast<uint8_t>(b.take(8)));
      }
      continue;
    }
    if (type == 3) GP_INFLATE_FAIL();
    if (type == 1) {  // fixed codes (RFC 1951 §3.2.6)
      for (int s = 0; s < 288; ++s) lens[s] = s < 144 ? 8 : s < 256 ? 9 : s < 280 ? 7 : 8;
      build(s_lit, lens, 288, kLens);
      for (int s = 0; s < 32; ++s) lens[s] = 5;
      build(s_dist, lens, 32, kDists);
    } else {  // dynamic codes (inflate.c TABLE / LENLENS / CODELENS)
      if (!b.need(14)) GP_INFLATE_FAIL();
      const int nlen = static_cast<int>(b.take(5)) + 257, ndist = static_cast<int>(b.take(5)) + 1;
      const int ncode = static_cast<int>(b.take(4)) + 4;
      if (nlen > 286 || ndist > 30) GP_INFLATE_FAIL();
      for (int k = 0; k < 19; ++k) cl[k] = 0;
      for (int k = 0; k < ncode; ++k) {
        if (!b.need(3)) GP_INFLATE_FAIL();
        cl[kClOrder[k]] = static_cast<uint8_t>(b.take(3));
      }
      if (!build(s_lit, cl, 19, kCodes)) GP_INFLATE_FAIL();
      int have = 0;
      while (have < nlen + ndist) {
        const int sym = decode<false>(b);
        if (sym < 0) GP_INFLATE_FAIL();
        if (sym < 16) {
          lens[have++] = static_cast<uint8_t>(sym);
          continue;
        }
        uint8_t l = 0;
        int copy;
        if (sym == 16) {
          if (have == 0) GP_INFLATE_FAIL();
          l = lens[have - 1];
          if (!b.need(2)) GP_INFLATE_FAIL();
          copy = 3 + static_cast<int>(b.take(2));
        } else if (sym == 17) {
          if (!b.need(3)) GP_INFLATE_FAIL();
          copy = 3 + static_cast<int>(b.take(3));
        } else {
          if (!b.need(7)) GP_INFLATE_FAIL();
          copy = 11 + static_cast<int>(b.take(7));
        }
        if (have + copy > nlen + ndist) GP_INFLATE_FAIL();
        while (copy--) lens[have++] = l;
      }
      if (lens[256] == 0) GP_INFLATE_FAIL();  // missing end-of-block code
      if (!build(s_lit, lens, nlen, kLens)) GP_INFLATE_FAIL();
      if (!build(s_dist, lens + nlen, ndist, kDists)) GP_INFLATE_FAIL();
    }
    for (;;) {
      int sym = decode<false>(b);
      if (sym < 0) GP_INFLATE_FAIL();
      if (sym < 256) {
        if (w.o >= w.cap) GP_INFLATE_FAIL();
        w.put(static_cast<uint8_t>(sym));
        continue;
      }
      if (sym == 256) break;
      sym -= 257;
      if (sym >= 29) GP_INFLATE_FAIL();  // symbols 286, 287
      if (!b.need(kLenExtra[sym])) GP_INFLATE_FAIL();
      const uint32_t len = kLenBase[sym] + b.take(kLenExtra[sym]);
      const int ds = decode<true>(b);
      if (ds < 0 || ds >= 30) GP_INFLATE_FAIL();
      if (!b.need(kDistExtra[ds])) GP_INFLATE_FAIL();
      const uint32_t dd = kDistBase[ds] + b.take(kDistExtra[ds]);
      if (dd > w.o) GP_INFLATE_FAIL();  // too far back (no dictionary)
      if (w.o + len > w.cap) GP_INFLATE_FAIL();
      uint32_t k = 0;
      if (dd >= 8) {  // source bytes all precede the destination run: batch the window loads
        for (; k + 8 <= len; k += 8) {
          uint8_t t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = s_win[(w.o - dd + j) & 32767];
#pragma unroll
          for (int j = 0; j < 8; ++j) w.put(t[j]);
        }
      }
      for (; k < len; ++k) w.put(s_win[(w.o - dd) & 32767]);
    }
  }
  // RFC 1950 trailer: Adler-32 of the output, big-endian, at the next byte
  b.take(b.cnt & 7);
  if (!b.need(32)) GP_INFLATE_FAIL();
  uint32_t adler = 0;
  for (int k = 0; k < 4; ++k) adler = adler << 8 | b.take(8);
  if (adler != ((w.s2 % 65521u) << 16 | (w.s1 % 65521u))) GP_INFLATE_FAIL();
  if (w.o != w.cap) GP_INFLATE_FAIL();  // out_len != raw_len
#undef GP_INFLATE_FAIL
}

// inflated little-endian f32 bytes -> the f64 value array decode_scatter reads
__global__ void slot_widen(const uint8_t* __restrict__ raw, const Plan* plan, double* __restrict__ values,
                           const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  if (plan->value_method != GP_VALUE_DEFLATE_SLOT || plan->slot_id != 1) return;
  const uint64_t n = plan->n_values;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    values[i] = static_cast<double>(__uint_as_float(ld_u32_unaligned(raw + 4 * i)));
}

}  // namespace

void launch_decode_inflate(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  uint8_t* raw = reinterpret_cast<uint8_t*>(w.values);  // 4·max_d bytes, unused by the decode otherwise
  GP_LAUNCH(ctx, slot_inflate, 1, 1, 0, s, in, w.plan, raw, w.status);
  GP_LAUNCH(ctx, slot_widen, grid_for(ctx, n_bound, 256), 256, 0, s, raw, w.plan, w.f64a, w.status);
}

}  // namespace gp
