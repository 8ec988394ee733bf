// volume.cpp — host-side container accounting (volume(), container.cpp:148-243).
//
// "Bits per nonzero" = total_bits / r, with the exact decomposition into
// index / value / reorder / metadata bits.  This is O(header) host work over a
// HOST copy of the container (the benchmark reads the 49-byte header plus the
// fit header it needs), so it stays on the CPU like the reference's own
// reporting; nothing of the encode → decode path runs here.
#include <cstdint>
#include <cstring>

#include "../../include/gradpack_b200.h"
#include "huffman.cuh"

namespace {

uint64_t rd64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}
uint32_t rd32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

}  // namespace

extern "C" GP_API int gp_volume(const uint8_t* h, uint64_t len, gp_volume_report* out) {
  if (!h || !out) return GP_ERROR;
  std::memset(out, 0, sizeof(*out));
  if (len < 49 + 4 || std::memcmp(h, "DRC1", 4) != 0) return GP_CORRUPT_PAYLOAD;
  const uint8_t im = h[6], vm = h[7];
  const uint64_t d = rd64(h + 9), r = rd64(h + 17), il = rd64(h + 25), vl = rd64(h + 33), rl = rd64(h + 41);
  if (49 + il + vl + rl + 4 != len) return GP_CORRUPT_PAYLOAD;
  const uint8_t* ip = h + 49;
  const uint8_t* vp = ip + il;
  out->total_bits = 8 * len;
  switch (im) {
    case GP_INDEX_NONE:
      if (il != 4 * r) return GP_CORRUPT_PAYLOAD;
      out->index_bits = 32 * r;
      break;
    case GP_INDEX_BITMAP:
      if (il != (d + 7) / 8) return GP_CORRUPT_PAYLOAD;
      out->index_bits = d;
      break;
    case GP_INDEX_RLE:
      if (il == 0) return GP_CORRUPT_PAYLOAD;
      out->index_bits = 8 * il - 7;  // 1 lead bit plus whole groups (the writer pads < 8 bits)
      break;
    case GP_INDEX_HUFFMAN: {  // container.cpp:171-178: the bits of the 4r decoded codes
      gp::HuffTable t;
      gp::HuffScratch x;
      gp::huff_build(d, &t, x);
      if (t.error) return GP_ERROR;
      const uint64_t nbits = 8 * il;
      uint64_t pos = 0;
      for (uint64_t i = 0; i < 4 * r; ++i) {
        uint64_t win = 0;
        for (int k = 0; k < 9; ++k) {
          const uint64_t b = pos / 8 + k;
          const uint64_t byte = b < il ? ip[b] : 0;
          const int sh = 8 * k - static_cast<int>(pos % 8);
          if (sh >= 64) break;
          win |= sh >= 0 ? byte << sh : byte >> -sh;
        }
        unsigned L = 0;
        const int sym = gp::huff_decode_one(t, win, nbits - pos, L);
        if (sym < 0) return sym == -1 ? GP_CORRUPT_PAYLOAD : GP_TRUNCATED;
        pos += L;
      }
      if (nbits - pos >= 8) return GP_CORRUPT_PAYLOAD;
      out->index_bits = pos;
      break;
    }
    default:
      if (im > GP_INDEX_BLOOM_NAIVE) return GP_UNKNOWN_METHOD;
      if (il < 8) return GP_TRUNCATED;
      out->index_bits = rd64(ip);  // m, the filter width
  }
  uint64_t count = r;
  switch (vm) {
    case GP_VALUE_NONE:
      if (vl % 4) return GP_CORRUPT_PAYLOAD;
      count = vl / 4;
      out->value_bits = 8 * vl;
      break;
    case GP_VALUE_RAW_F64:
      if (vl % 8) return GP_CORRUPT_PAYLOAD;
      count = vl / 8;
      out->value_bits = 8 * vl;
      break;
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP: {  // fit_shape, container.cpp:131-145
      if (vl < 3) return GP_TRUNCATED;
      const uint8_t kind = vp[0];
      if (kind > 1) return GP_UNKNOWN_METHOD;
      const uint32_t segs = vp[1] | (vp[2] << 8);
      if (segs < 1) return GP_CORRUPT_PAYLOAD;
      if (vl < 3 + 4ull * segs + 1) return GP_TRUNCATED;
      const uint32_t last = rd32(vp + 3 + 4ull * (segs - 1));
      const uint8_t degree = vp[3 + 4 * segs];
      out->value_bits = 32ull * segs * (kind == 1 ? 4u : degree + 1u);
      count = last;
      break;
    }
    case GP_VALUE_QUANT: {  // container.cpp:213-225
      // with Bloom-P0 indices the value count is |P|, which needs the full
      // positive scan: out of this host-side header accounting
      if (im == GP_INDEX_BLOOM_P0) return GP_UNSUPPORTED;
      if (vl < 1) return GP_TRUNCATED;
      const uint8_t bits = vp[0];
      if (vl < 5) return GP_TRUNCATED;
      const uint32_t bucket = rd32(vp + 1);
      if (bits < 1 || bucket < 1) return GP_CORRUPT_PAYLOAD;
      out->value_bits = 32 * ((count + bucket - 1) / bucket) + static_cast<uint64_t>(bits) * count;
      break;
    }
    case GP_VALUE_DEFLATE_SLOT:
      if (vl < 9) return GP_CORRUPT_PAYLOAD;
      out->value_bits = 8 * (vl - 9);
      break;
    default:
      return vm > GP_VALUE_RAW_F64 ? GP_UNKNOWN_METHOD : GP_UNSUPPORTED;
  }
  if (rl) {
    uint32_t w = 0;
    for (uint64_t x = d - 1; x; x >>= 1) ++w;
    out->reorder_bits = count * w;
    if (rl != (out->reorder_bits + 7) / 8) return GP_CORRUPT_PAYLOAD;
  }
  out->metadata_bits = out->total_bits - out->index_bits - out->value_bits - out->reorder_bits;
  if (d) out->ratio_dense = static_cast<double>(out->total_bits) / (32.0 * static_cast<double>(d));
  if (r) out->ratio_sparse = static_cast<double>(out->total_bits) / (64.0 * static_cast<double>(r));
  return GP_OK;
}
