// huffman.cuh — the canonical Huffman table of the index-byte codec
// (codecs.cpp:72-170), built identically on the host (capacity bounds,
// volume()) and on the device (one thread, from the container's d).
//   frequencies: the byte distribution of 0..d-1 as 4 LE bytes (:72-91)
//   tree: min-heap on (weight, creation order), pairs merged smallest-first;
//         code length = leaf depth, > 57 is an Error (:93-135)
//   codes: canonical by (length, symbol) (:137-155); decode tables
//         first_code / first_index / count per length (:156-168)
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define GP_HD __host__ __device__
#else
#define GP_HD
#endif

namespace gp {

struct HuffTable {
  uint64_t code[256];
  uint64_t first_code[64];
  uint32_t first_index[64];
  uint32_t count[64];
  uint8_t len[256];
  uint8_t sorted[256];
  uint32_t nsym, max_len;
  int32_t error;  // 1: d out of range, 2: empty alphabet, 3: a code longer than 57 bits
  uint64_t d;     // the d this table was built for (device cache key)
};

GP_HD inline void huff_freqs(uint64_t d, uint64_t* freq) {
  for (int b = 0; b < 256; ++b) freq[b] = 0;
  for (unsigned j = 0; j < 4; ++j) {
    const uint64_t width = 1ULL << (8 * j);
    const uint64_t high = d >> (8 * (j + 1));
    const uint64_t mid = (d >> (8 * j)) & 0xff;
    const uint64_t low = d & (width - 1);
    for (unsigned b = 0; b < 256; ++b) freq[b] += high * width + (b < mid ? width : (b == mid ? low : 0));
  }
}

GP_HD inline bool huff_less(const uint64_t* w, int a, int b) { return w[a] < w[b] || (w[a] == w[b] && a < b); }

GP_HD inline void huff_push(int* heap, int& hn, const uint64_t* w, int id) {
  int i = hn++;
  heap[i] = id;
  while (i > 0 && huff_less(w, heap[i], heap[(i - 1) / 2])) {
    const int t = heap[i];
    heap[i] = heap[(i - 1) / 2];
    heap[(i - 1) / 2] = t;
    i = (i - 1) / 2;
  }
}

GP_HD inline int huff_pop(int* heap, int& hn, const uint64_t* w) {
  const int top = heap[0];
  heap[0] = heap[--hn];
  int i = 0;
  for (;;) {
    const int l = 2 * i + 1, r = l + 1;
    int m = i;
    if (l < hn && huff_less(w, heap[l], heap[m])) m = l;
    if (r < hn && huff_less(w, heap[r], heap[m])) m = r;
    if (m == i) break;
    const int t = heap[i];
    heap[i] = heap[m];
    heap[m] = t;
    i = m;
  }
  return top;
}

struct HuffScratch {
  uint64_t w[511];
  uint64_t freq[256];
  int16_t left[511], right[511], sym[511], st[511];
  uint8_t dp[511];
  int heap[256];
  uint32_t cnt[64], at[64];
};

// Builds the table for index streams over [0, d).  The ~12 KB of scratch is
// the caller's: a host local, or shared memory of the one-thread device build.
GP_HD inline void huff_build(uint64_t d, HuffTable* t, HuffScratch& x) {
  for (int s = 0; s < 256; ++s) {
    t->len[s] = 0;
    t->code[s] = 0;
  }
  for (int l = 0; l < 64; ++l) {
    t->first_code[l] = 0;
    t->first_index[l] = 0;
    t->count[l] = 0;
  }
  t->nsym = 0;
  t->max_len = 0;
  t->error = 0;
  t->d = d;
  if (d < 1 || d > 0x100000000ULL) {
    t->error = 1;
    return;
  }
  uint64_t* w = x.w;
  int16_t *left = x.left, *right = x.right, *sym = x.sym;
  int* heap = x.heap;
  int hn = 0, nn = 0;
  uint64_t* freq = x.freq;
  huff_freqs(d, freq);
  for (int s = 0; s < 256; ++s) {
    if (!freq[s]) continue;
    w[nn] = freq[s];
    left[nn] = right[nn] = -1;
    sym[nn] = static_cast<int16_t>(s);
    huff_push(heap, hn, w, nn++);
  }
  if (nn == 0) {
    t->error = 2;
    return;
  }
  if (nn == 1) {
    t->len[sym[0]] = 1;
  } else {
    while (hn > 1) {
      const int a = huff_pop(heap, hn, w);
      const int b = huff_pop(heap, hn, w);
      w[nn] = w[a] + w[b];
      left[nn] = static_cast<int16_t>(a);
      right[nn] = static_cast<int16_t>(b);
      sym[nn] = -1;
      huff_push(heap, hn, w, nn++);
    }
    int16_t* st = x.st;
    uint8_t* dp = x.dp;
    int sn = 0;
    st[sn] = static_cast<int16_t>(nn - 1);
    dp[sn++] = 0;
    while (sn) {
      --sn;
      const int id = st[sn], dep = dp[sn];
      if (sym[id] >= 0) {
        if (dep > 57) {
          t->error = 3;
          return;
        }
        t->len[sym[id]] = static_cast<uint8_t>(dep);
      } else {
        st[sn] = left[id];
        dp[sn++] = static_cast<uint8_t>(dep + 1);
        st[sn] = right[id];
        dp[sn++] = static_cast<uint8_t>(dep + 1);
      }
    }
  }
  // canonical order by (length, symbol): counting sort over the lengths
  uint32_t* cnt = x.cnt;
  for (int l = 0; l < 64; ++l) cnt[l] = 0;
  for (int s = 0; s < 256; ++s)
    if (t->len[s]) ++cnt[t->len[s]];
  uint32_t* at = x.at;
  uint32_t run = 0;
  for (int l = 0; l < 64; ++l) {
    at[l] = run;
    run += cnt[l];
  }
  for (int s = 0; s < 256; ++s)
    if (t->len[s]) t->sorted[at[t->len[s]]++] = static_cast<uint8_t>(s);
  t->nsym = run;
  t->max_len = t->len[t->sorted[run - 1]];
  uint64_t code = 0;
  unsigned prev = t->len[t->sorted[0]];
  for (uint32_t i = 0; i < run; ++i) {
    const unsigned L = t->len[t->sorted[i]];
    code = i ? (code + 1) << (L - prev) : 0;
    t->code[t->sorted[i]] = code;
    prev = L;
    if (t->count[L] == 0) {
      t->first_index[L] = i;
      t->first_code[L] = code;
    }
    ++t->count[L];
  }
}

// One canonical decode (decode_symbol, codecs.cpp:181-190) from a 64-bit
// LSB-first window `win` of the stream at bit `pos` (avail bits valid):
// returns the symbol (>= 0) and its length, -1 invalid code, -2 exhausted.
GP_HD inline int huff_decode_one(const HuffTable& t, uint64_t win, uint64_t avail, unsigned& len) {
  uint64_t code = 0;
  for (unsigned L = 1; L <= t.max_len; ++L) {
    if (L > avail) return -2;
    code = (code << 1) | ((win >> (L - 1)) & 1u);
    if (t.count[L] && code >= t.first_code[L] && code - t.first_code[L] < t.count[L]) {
      len = L;
      return t.sorted[t.first_index[L] + static_cast<uint32_t>(code - t.first_code[L])];
    }
  }
  return -1;
}

}  // namespace gp
