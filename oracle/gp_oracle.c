/*
 * gp_oracle.c — CPU restatement of gradpack's sparse-gradient encode → decode
 * path (TEST INFRASTRUCTURE; see gp_oracle.h for who may load it).
 *
 * Each function cites the reference function it restates, as file:line under
 * /root/reference/proj.  Single-threaded per call; thread-safe across threads
 * (all scratch state is thread-local).  Compile with -ffp-contract=off: the
 * reference build has no -march flag (CMakeLists.txt:8-10), so the x86-64
 * baseline never fuses multiply-adds, and the curve-fit segmentation compares
 * fp64 chord deviations exactly (curvefit.cpp:50-67).
 */
#include "gp_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ==================================================================== errors
 * errors.hpp:21-53 → gp_status codes; a failing check longjmps to the API
 * entry, which releases every scratch allocation of the call. */
static _Thread_local jmp_buf* g_jb;
static _Thread_local int g_code;
static _Thread_local char g_msg[256];

static void fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof g_msg, fmt, ap);
  va_end(ap);
  g_code = code;
  longjmp(*g_jb, 1);
}

const char* gpo_last_error(void) { return g_msg; }
void gpo_free(void* p) { free(p); }

/* scratch arena: every xalloc of an API call is freed when it returns */
static _Thread_local void** g_arena;
static _Thread_local size_t g_arena_n, g_arena_cap;

static size_t arena_push(void* p) {
  if (g_arena_n == g_arena_cap) {
    size_t cap = g_arena_cap ? 2 * g_arena_cap : 256;
    void** a = (void**)realloc(g_arena, cap * sizeof(void*));
    if (!a) {
      free(p);
      fail(GP_ERROR, "oracle: out of memory");
    }
    g_arena = a;
    g_arena_cap = cap;
  }
  g_arena[g_arena_n] = p;
  return g_arena_n++;
}
static void arena_release(size_t mark) {
  while (g_arena_n > mark) free(g_arena[--g_arena_n]);
}
static void* xalloc(size_t n) {
  void* p = calloc(n ? n : 1, 1);
  if (!p) fail(GP_ERROR, "oracle: out of memory");
  arena_push(p);
  return p;
}
/* moves an arena allocation out to the caller (it survives the API return) */
static void* detach(const void* p, size_t n) {
  void* out = malloc(n ? n : 1);
  if (!out) fail(GP_ERROR, "oracle: out of memory");
  if (n) memcpy(out, p, n);
  return out;
}

#define API_BEGIN                       \
  jmp_buf jb_;                          \
  jmp_buf* prev_jb_ = g_jb;             \
  size_t mark_ = g_arena_n;             \
  g_jb = &jb_;                          \
  if (setjmp(jb_)) {                    \
    arena_release(mark_);               \
    g_jb = prev_jb_;                    \
    return g_code;                      \
  }                                     \
  g_msg[0] = 0
#define API_END                         \
  arena_release(mark_);                 \
  g_jb = prev_jb_;                      \
  return GP_OK

/* growable byte buffer (std::vector<uint8_t>) in the arena */
typedef struct {
  uint8_t* p;
  size_t n, cap, slot;
} bytes_t;

static void bytes_init(bytes_t* b, size_t cap) {
  b->cap = cap ? cap : 16;
  b->p = (uint8_t*)calloc(b->cap, 1);
  if (!b->p) fail(GP_ERROR, "oracle: out of memory");
  b->slot = arena_push(b->p);
  b->n = 0;
}
static void bytes_reserve(bytes_t* b, size_t need) {
  if (need <= b->cap) return;
  size_t cap = b->cap;
  while (cap < need) cap *= 2;
  uint8_t* p = (uint8_t*)realloc(b->p, cap);
  if (!p) fail(GP_ERROR, "oracle: out of memory");
  memset(p + b->cap, 0, cap - b->cap);
  b->p = p;
  b->cap = cap;
  g_arena[b->slot] = p;
}
static void put_u8(bytes_t* b, uint8_t v) {
  bytes_reserve(b, b->n + 1);
  b->p[b->n++] = v;
}
static void put_le(bytes_t* b, uint64_t v, unsigned n) { /* bitio.hpp:137-139 */
  for (unsigned i = 0; i < n; ++i) put_u8(b, (uint8_t)(v >> (8 * i)));
}
static void put_f32(bytes_t* b, float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  put_le(b, u, 4);
}
static void put_f64(bytes_t* b, double v) {
  uint64_t u;
  memcpy(&u, &v, 8);
  put_le(b, u, 8);
}
static void put_bytes(bytes_t* b, const uint8_t* s, size_t n) {
  bytes_reserve(b, b->n + n);
  if (n) memcpy(b->p + b->n, s, n);
  b->n += n;
}

/* byte reader (bitio.hpp:142-167): short reads raise TruncatedError */
typedef struct {
  const uint8_t* p;
  size_t n, pos;
} breader_t;

static uint64_t get_le(breader_t* r, unsigned n) {
  if (r->n - r->pos < n) fail(GP_TRUNCATED, "byte stream exhausted");
  uint64_t v = 0;
  for (unsigned i = 0; i < n; ++i) v |= (uint64_t)r->p[r->pos + i] << (8 * i);
  r->pos += n;
  return v;
}
static const uint8_t* get_bytes(breader_t* r, size_t n) {
  if (r->n - r->pos < n) fail(GP_TRUNCATED, "byte stream exhausted");
  const uint8_t* s = r->p + r->pos;
  r->pos += n;
  return s;
}
static float get_f32(breader_t* r) {
  uint32_t u = (uint32_t)get_le(r, 4);
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static double get_f64(breader_t* r) {
  uint64_t u = get_le(r, 8);
  double f;
  memcpy(&f, &u, 8);
  return f;
}

/* bit writer/reader, LSB-first (bitio.hpp:26-76) */
typedef struct {
  bytes_t b;
  uint64_t nbits;
} bitw_t;
static void bw_init(bitw_t* w, size_t cap) {
  bytes_init(&w->b, cap);
  w->nbits = 0;
}
static void bw_bit(bitw_t* w, int bit) { /* bitio.hpp:28-32 */
  if (w->nbits % 8 == 0) put_u8(&w->b, 0);
  if (bit) w->b.p[w->b.n - 1] |= (uint8_t)(1u << (w->nbits % 8));
  ++w->nbits;
}
static void bw_bits(bitw_t* w, uint64_t v, unsigned width) { /* bitio.hpp:35-37 */
  for (unsigned i = 0; i < width; ++i) bw_bit(w, (int)((v >> i) & 1u));
}
static unsigned bw_varint(bitw_t* w, uint64_t v) { /* bitio.hpp:79-89 */
  unsigned groups = 0;
  do {
    uint8_t g = v & 0x7f;
    v >>= 7;
    if (v != 0) g |= 0x80;
    bw_bits(w, g, 8);
    ++groups;
  } while (v != 0);
  return groups;
}

typedef struct {
  const uint8_t* p;
  size_t n;
  uint64_t pos;
} bitr_t;
static int br_bit(bitr_t* r) { /* bitio.hpp:55-60 */
  if (r->pos >= 8 * (uint64_t)r->n) fail(GP_TRUNCATED, "bit stream exhausted");
  int b = (r->p[r->pos / 8] >> (r->pos % 8)) & 1;
  ++r->pos;
  return b;
}
static uint64_t br_bits(bitr_t* r, unsigned width) {
  uint64_t v = 0;
  for (unsigned i = 0; i < width; ++i) v |= (uint64_t)br_bit(r) << i;
  return v;
}
static uint64_t br_remaining(const bitr_t* r) { return 8 * (uint64_t)r->n - r->pos; }
static uint64_t br_varint(bitr_t* r) { /* bitio.hpp:91-99 */
  uint64_t v = 0;
  for (unsigned shift = 0; shift < 64; shift += 7) {
    uint8_t g = (uint8_t)br_bits(r, 8);
    v |= (uint64_t)(g & 0x7f) << shift;
    if ((g & 0x80) == 0) return v;
  }
  fail(GP_CORRUPT_PAYLOAD, "varint exceeds 64 bits");
  return 0;
}

/* ==================================================================== rng.hpp */
uint64_t gpo_mix64(uint64_t z) { /* rng.hpp:25-31 */
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t gpo_hash64(uint64_t x, uint64_t seed) { /* rng.hpp:35-37 */
  return gpo_mix64(x ^ (seed + 0x9E3779B97F4A7C15ULL));
}

typedef struct {
  uint64_t state;
} rng_t;
static uint64_t rng_next(rng_t* g) { /* rng.hpp:46-49 */
  g->state += 0x9E3779B97F4A7C15ULL;
  return gpo_mix64(g->state);
}
static uint64_t rng_below(rng_t* g, uint64_t n) { /* rng.hpp:52-59 */
  if (n == 0) fail(GP_ERROR, "CounterRng::below: n must be positive");
  const uint64_t rem = (UINT64_MAX % n + 1) % n;
  const uint64_t bound = UINT64_MAX - rem;
  uint64_t r = rng_next(g);
  while (r > bound) r = rng_next(g);
  return r % n;
}
static double rng_unit(rng_t* g) { /* rng.hpp:62 */
  return (double)(rng_next(g) >> 11) * 0x1.0p-53;
}
static double rng_normal(rng_t* g) { /* rng.hpp:65-69 */
  const double u1 = 1.0 - rng_unit(g);
  const double u2 = rng_unit(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

int gpo_rng_below_seq(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out) {
  API_BEGIN;
  rng_t g = {seed};
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_below(&g, bound);
  API_END;
}

void gpo_fill_normal_f32(uint64_t seed, float* out, uint64_t n) {
  /* gradpack_main.cpp:279-281 generator (rank-extended seeds are the caller's) */
  rng_t g = {seed};
  for (uint64_t i = 0; i < n; ++i) out[i] = (float)rng_normal(&g);
}

uint64_t gpo_pipeline_seed(uint64_t seed, int worker, int step) {
  /* Problem::batch_seed harness.cpp:47-51, Simulation::pipeline_seed :201-203 */
  const uint64_t key = ((uint64_t)(uint32_t)worker << 32) | (uint32_t)step;
  const uint64_t batch = gpo_hash64(key, gpo_hash64(0xDA7A, seed));
  return gpo_hash64(0xC0DEC, batch);
}

/* seeds, pipeline.cpp:21-26 */
static uint64_t seed_a_of(uint64_t seed) { return gpo_hash64(0xA, seed); }
static uint64_t seed_b_of(uint64_t seed) { return gpo_hash64(0xB, seed); }
static uint64_t selection_seed(uint64_t a, uint64_t b) { return gpo_hash64(a, b); }

/* ==================================================================== crc32c
 * container.cpp:30-48: reflected Castagnoli, init/xorout 0xFFFFFFFF */
static uint32_t crc_table[256];
static int crc_ready;
static void crc_init(void) {
  if (crc_ready) return;
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int j = 0; j < 8; ++j) c = (c >> 1) ^ ((c & 1u) ? 0x82F63B78u : 0u);
    crc_table[i] = c;
  }
  crc_ready = 1;
}
static uint32_t crc_update(uint32_t crc, const uint8_t* p, size_t n) {
  for (size_t i = 0; i < n; ++i) crc = (crc >> 8) ^ crc_table[(crc ^ p[i]) & 0xFFu];
  return crc;
}
uint32_t gpo_crc32c(const uint8_t* data, size_t n) {
  crc_init();
  return crc_update(0xFFFFFFFFu, data, n) ^ 0xFFFFFFFFu;
}

/* ==================================================================== sparse gradient */
typedef struct {
  uint64_t d;
  uint32_t* support;
  double* values;
  uint64_t count;
} sparse_t;

static void validate_sparse(const sparse_t* g) { /* gradient.cpp:19-30 */
  if (g->d < 1) fail(GP_ERROR, "sparse gradient: dim must be >= 1");
  for (uint64_t i = 0; i < g->count; ++i) {
    if (i > 0 && g->support[i] <= g->support[i - 1])
      fail(GP_ERROR, "sparse gradient: support not strictly increasing");
    if ((uint64_t)g->support[i] >= g->d) fail(GP_ERROR, "sparse gradient: index out of range");
  }
}

/* top_r, sparsify.cpp:32-46.  nth_element under the comparator
 * (|g_a| > |g_b|) || (|g_a| == |g_b| && a < b), then sort ascending.  For f32
 * inputs |g| orders exactly like the u32 key bits & 0x7FFFFFFF, so the kept set
 * is: every key above the r-th largest key T, plus the lowest-index keys equal
 * to T until r are kept.  T is found by an MSB-first byte radix select. */
int gpo_top_r(const float* g, uint64_t d, uint64_t r, uint32_t* support) {
  API_BEGIN;
  if (d < 1) fail(GP_ERROR, "sparsifier: dim must be >= 1");          /* sparsify.cpp:25 */
  if (d > 0xFFFFFFFFULL) fail(GP_ERROR, "sparsifier: dim exceeds 32-bit index space");
  if (r < 1 || r > d) fail(GP_ERROR, "sparsifier: r out of range [1, d]");
  uint32_t prefix = 0, mask = 0;
  uint64_t remaining = r;
  for (int shift = 24; shift >= 0; shift -= 8) {
    uint64_t hist[256] = {0};
    for (uint64_t i = 0; i < d; ++i) {
      uint32_t key;
      memcpy(&key, &g[i], 4);
      key &= 0x7FFFFFFFu;
      if ((key & mask) == prefix) ++hist[(key >> shift) & 0xFF];
    }
    int digit = 255;
    for (; digit > 0; --digit) {
      if (remaining <= hist[digit]) break;
      remaining -= hist[digit];
    }
    prefix |= (uint32_t)digit << shift;
    mask |= 0xFFu << shift;
  }
  uint64_t kept = 0;
  for (uint64_t i = 0; i < d; ++i) {
    uint32_t key;
    memcpy(&key, &g[i], 4);
    key &= 0x7FFFFFFFu;
    if (key > prefix || (key == prefix && remaining > 0)) {
      if (key == prefix) --remaining;
      support[kept++] = (uint32_t)i;
    }
  }
  if (kept != r) fail(GP_ERROR, "top_r: internal selection mismatch");
  API_END;
}

/* ==================================================================== bitmap / RLE */
static uint64_t* to_bitmap(const uint32_t* support, uint64_t r, uint64_t d) {
  /* support_to_bitmap, gradient.cpp:56-63 */
  uint64_t* w = (uint64_t*)xalloc(((d + 63) / 64) * 8);
  for (uint64_t i = 0; i < r; ++i) {
    if ((uint64_t)support[i] >= d) fail(GP_ERROR, "bitmap: index out of range");
    w[support[i] / 64] |= 1ULL << (support[i] % 64);
  }
  return w;
}
static int bm_test(const uint64_t* w, uint64_t i) { return (int)((w[i / 64] >> (i % 64)) & 1u); }

static void bitmap_to_bytes(const uint64_t* w, uint64_t d, uint8_t* out) { /* gradient.cpp:81-86 */
  for (uint64_t i = 0; i < (d + 7) / 8; ++i) out[i] = (uint8_t)(w[i / 8] >> (8 * (i % 8)));
}
static uint64_t* bitmap_from_bytes(const uint8_t* b, size_t n, uint64_t d) { /* gradient.cpp:88-97 */
  if (n != (d + 7) / 8) fail(GP_CORRUPT_PAYLOAD, "bitmap: payload length mismatch");
  uint64_t* w = (uint64_t*)xalloc(((d + 63) / 64) * 8);
  for (size_t i = 0; i < n; ++i) w[i / 8] |= (uint64_t)b[i] << (8 * (i % 8));
  if (d % 8 != 0 && (b[n - 1] >> (d % 8)) != 0) fail(GP_CORRUPT_PAYLOAD, "bitmap: bits set past dim");
  return w;
}
static uint64_t bitmap_popcount(const uint64_t* w, uint64_t d) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < (d + 63) / 64; ++i) c += (uint64_t)__builtin_popcountll(w[i]);
  return c;
}
static uint32_t* bitmap_support(const uint64_t* w, uint64_t d, uint64_t count) { /* gradient.cpp:67-79 */
  uint32_t* out = (uint32_t*)xalloc(count * 4);
  uint64_t k = 0;
  for (uint64_t i = 0; i < (d + 63) / 64; ++i) {
    uint64_t word = w[i];
    while (word) {
      out[k++] = (uint32_t)(64 * i + (uint64_t)__builtin_ctzll(word));
      word &= word - 1;
    }
  }
  return out;
}

static void rle_encode(const uint64_t* w, uint64_t d, bitw_t* out) { /* codecs.cpp:34-50 */
  if (d < 1) fail(GP_ERROR, "rle_encode: empty bitmap");
  bw_bit(out, bm_test(w, 0));
  uint64_t i = 0;
  while (i < d) {
    const int cur = bm_test(w, i);
    uint64_t j = i;
    while (j < d && bm_test(w, j) == cur) ++j;
    bw_varint(out, j - i);
    i = j;
  }
}
static uint64_t* rle_decode(const uint8_t* p, size_t n, uint64_t d) { /* codecs.cpp:52-70 */
  if (d < 1) fail(GP_ERROR, "rle_decode: d must be >= 1");
  bitr_t r = {p, n, 0};
  int cur = br_bit(&r);
  uint64_t* w = (uint64_t*)xalloc(((d + 63) / 64) * 8);
  uint64_t pos = 0;
  while (pos < d) {
    const uint64_t run = br_varint(&r);
    if (run == 0) fail(GP_CORRUPT_PAYLOAD, "rle: zero-length run");
    if (run > d - pos) fail(GP_CORRUPT_PAYLOAD, "rle: runs exceed d");
    if (cur)
      for (uint64_t i = pos; i < pos + run; ++i) w[i / 64] |= 1ULL << (i % 64);
    pos += run;
    cur = !cur;
  }
  if (br_remaining(&r) >= 8 || br_bits(&r, (unsigned)br_remaining(&r)) != 0)
    fail(GP_CORRUPT_PAYLOAD, "rle: trailing garbage");
  return w;
}

int gpo_bitmap_bytes(const uint32_t* support, uint64_t r, uint64_t d, uint8_t* out) {
  API_BEGIN;
  bitmap_to_bytes(to_bitmap(support, r, d), d, out);
  API_END;
}
int gpo_rle_encode(const uint32_t* support, uint64_t r, uint64_t d, uint8_t** out, size_t* len) {
  API_BEGIN;
  bitw_t w;
  bw_init(&w, 64);
  rle_encode(to_bitmap(support, r, d), d, &w);
  *len = w.b.n;
  *out = (uint8_t*)detach(w.b.p, w.b.n);
  API_END;
}

/* ==================================================================== bloom.cpp */
int gpo_bloom_params(double eps, uint64_t r, uint64_t* m, uint32_t* k) { /* bloom.cpp:22-31 */
  API_BEGIN;
  if (!(eps > 0.0 && eps < 1.0)) fail(GP_ERROR, "bloom_params: epsilon must be in (0, 1)");
  if (r < 1) fail(GP_ERROR, "bloom_params: r must be >= 1");
  const double ln2 = 0.693147180559945309417232121458176568; /* std::numbers::ln2 */
  const double lninv = log(1.0 / eps);
  *m = (uint64_t)ceil((double)r * lninv / (ln2 * ln2));
  *k = (uint32_t)ceil(lninv / ln2);
  API_END;
}

typedef struct {
  uint64_t m;
  unsigned k;
  uint64_t sa, sb;
  uint64_t* words;
} bloom_t;

static void bloom_new(bloom_t* f, uint64_t m, unsigned k, uint64_t sa, uint64_t sb) { /* bloom.cpp:41-45 */
  if (m < 1) fail(GP_ERROR, "bloom filter: m must be >= 1");
  if (k < 1) fail(GP_ERROR, "bloom filter: k must be >= 1");
  f->m = m;
  f->k = k;
  f->sa = sa;
  f->sb = sb;
  f->words = (uint64_t*)xalloc(((m + 63) / 64) * 8);
}
static int bloom_bit(const bloom_t* f, uint64_t i) { return (int)((f->words[i / 64] >> (i % 64)) & 1u); }
static void bloom_insert(bloom_t* f, uint64_t key) { /* bloom.cpp:58-66 */
  const uint64_t a = gpo_hash64(key, f->sa), b = gpo_hash64(key, f->sb);
  uint64_t x = a;
  for (unsigned i = 0; i < f->k; ++i, x += b) {
    const uint64_t pos = gpo_mix64(x) % f->m;
    f->words[pos / 64] |= 1ULL << (pos % 64);
  }
}
static int bloom_contains(const bloom_t* f, uint64_t key) { /* bloom.cpp:68-76 */
  const uint64_t a = gpo_hash64(key, f->sa), b = gpo_hash64(key, f->sb);
  uint64_t x = a;
  for (unsigned i = 0; i < f->k; ++i, x += b)
    if (!bloom_bit(f, gpo_mix64(x) % f->m)) return 0;
  return 1;
}
static void bloom_serialize(const bloom_t* f, bytes_t* out) { /* bloom.cpp:84-94 */
  put_le(out, f->m, 8);
  put_le(out, (uint16_t)f->k, 2);
  put_le(out, f->sa, 8);
  put_le(out, f->sb, 8);
  const uint64_t nbytes = (f->m + 7) / 8;
  bytes_reserve(out, out->n + nbytes);
  for (uint64_t i = 0; i < nbytes; ++i) out->p[out->n + i] = (uint8_t)(f->words[i / 8] >> (8 * (i % 8)));
  out->n += nbytes;
}
static void bloom_deserialize(breader_t* r, bloom_t* f) { /* bloom.cpp:96-112 */
  const uint64_t m = get_le(r, 8);
  if (m < 1) fail(GP_CORRUPT_PAYLOAD, "bloom payload: m must be >= 1");
  const unsigned k = (unsigned)get_le(r, 2);
  if (k < 1) fail(GP_CORRUPT_PAYLOAD, "bloom payload: k must be >= 1");
  const uint64_t sa = get_le(r, 8), sb = get_le(r, 8);
  bloom_new(f, m, k, sa, sb);
  const uint64_t nbytes = (m + 7) / 8;
  const uint8_t* bits = get_bytes(r, nbytes);
  for (uint64_t i = 0; i < nbytes; ++i) f->words[i / 8] |= (uint64_t)bits[i] << (8 * (i % 8));
  const uint64_t tail = m % 64;
  if (tail != 0 && (f->words[(m + 63) / 64 - 1] >> tail) != 0)
    fail(GP_CORRUPT_PAYLOAD, "bloom payload: bits set past m");
}
static void build_filter(bloom_t* f, const uint32_t* support, uint64_t r, double eps, uint64_t sa,
                         uint64_t sb) { /* bloom.cpp:114-121 */
  if (r == 0) fail(GP_ERROR, "build_filter: empty support");
  uint64_t m;
  uint32_t k;
  int rc = gpo_bloom_params(eps, r, &m, &k);
  if (rc != GP_OK) fail(rc, "%s", g_msg);
  bloom_new(f, m, k, sa, sb);
  for (uint64_t i = 0; i < r; ++i) bloom_insert(f, support[i]);
}
static uint32_t* positive_scan(const bloom_t* f, uint64_t d, uint64_t* n) { /* bloom.cpp:123-128 */
  uint64_t cap = 1024, cnt = 0;
  bytes_t buf;
  bytes_init(&buf, cap * 4);
  for (uint64_t i = 0; i < d; ++i)
    if (bloom_contains(f, i)) {
      bytes_reserve(&buf, (cnt + 1) * 4);
      ((uint32_t*)buf.p)[cnt++] = (uint32_t)i;
    }
  *n = cnt;
  return (uint32_t*)buf.p;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static uint32_t* p1_select(const uint32_t* P, uint64_t n, uint64_t r, rng_t* g) { /* bloom.cpp:140-154 */
  if (r > n) fail(GP_ERROR, "p1_select: r exceeds |P|");
  uint32_t* pool = (uint32_t*)xalloc((n ? n : 1) * 4);
  memcpy(pool, P, n * 4);
  for (uint64_t i = 0; i < r; ++i) {
    const uint64_t j = i + rng_below(g, n - i);
    uint32_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  qsort(pool, r, 4, cmp_u32);
  return pool;
}

/* conflict_sets, bloom.cpp:156-173.  std::map<bit, members> with consecutive
 * dedup, then stable_sort by (size, bit).  Members are kept as positions in P
 * (P is ascending and unique, so lower_bound(P, x) is that position). */
typedef struct {
  uint64_t bit;
  uint32_t member; /* position in P */
  uint64_t order;  /* generation order: keeps the sort stable */
} pair_t;
static int cmp_pair(const void* a, const void* b) {
  const pair_t *x = (const pair_t*)a, *y = (const pair_t*)b;
  if (x->bit != y->bit) return x->bit < y->bit ? -1 : 1;
  return (x->order > y->order) - (x->order < y->order);
}
typedef struct {
  uint64_t bit;
  uint64_t off, size;
} cset_t;
static int cmp_cset(const void* a, const void* b) {
  const cset_t *x = (const cset_t*)a, *y = (const cset_t*)b;
  if (x->size != y->size) return x->size < y->size ? -1 : 1;
  return (x->bit > y->bit) - (x->bit < y->bit);
}
static cset_t* conflict_sets(const uint32_t* P, uint64_t n, const bloom_t* f, uint32_t** members_out,
                             uint64_t* nsets_out) {
  const uint64_t np = n * f->k;
  pair_t* pairs = (pair_t*)xalloc((np ? np : 1) * sizeof(pair_t));
  for (uint64_t j = 0; j < n; ++j) { /* positions(x), bloom.cpp:78-82 */
    const uint64_t a = gpo_hash64(P[j], f->sa), b = gpo_hash64(P[j], f->sb);
    for (unsigned i = 0; i < f->k; ++i) {
      pair_t* p = &pairs[j * f->k + i];
      p->bit = gpo_mix64(a + (uint64_t)i * b) % f->m;
      p->member = (uint32_t)j;
      p->order = j * f->k + i;
    }
  }
  qsort(pairs, np, sizeof(pair_t), cmp_pair);
  uint32_t* members = (uint32_t*)xalloc((np ? np : 1) * 4);
  cset_t* sets = (cset_t*)xalloc((np ? np : 1) * sizeof(cset_t));
  uint64_t nm = 0, ns = 0;
  for (uint64_t i = 0; i < np; ++i) {
    if (i == 0 || pairs[i].bit != pairs[i - 1].bit) {
      sets[ns].bit = pairs[i].bit;
      sets[ns].off = nm;
      sets[ns].size = 0;
      ++ns;
    }
    cset_t* s = &sets[ns - 1];
    if (s->size == 0 || members[s->off + s->size - 1] != pairs[i].member) {
      members[nm++] = pairs[i].member;
      ++s->size;
    }
  }
  qsort(sets, ns, sizeof(cset_t), cmp_cset); /* (size, bit) keys are unique: stable */
  *members_out = members;
  *nsets_out = ns;
  return sets;
}

static uint32_t* p2_select(const uint32_t* P, uint64_t n, const bloom_t* f, uint64_t r,
                           rng_t* g) { /* bloom.cpp:175-222 */
  if (r > n) fail(GP_ERROR, "p2_select: r exceeds |P|");
  uint32_t* members;
  uint64_t ns;
  cset_t* sets = conflict_sets(P, n, f, &members, &ns);
  uint8_t* retired = (uint8_t*)xalloc(ns ? ns : 1);
  uint8_t* in_sel = (uint8_t*)xalloc(n ? n : 1);
  uint32_t* selected = (uint32_t*)xalloc((r ? r : 1) * 4);
  uint64_t nsel = 0;
#define SELECT(pos)                           \
  do {                                        \
    const uint32_t p_ = (pos);                \
    if (!in_sel[p_]) {                        \
      in_sel[p_] = 1;                         \
      selected[nsel++] = P[p_];               \
    }                                         \
  } while (0)
  while (nsel < r) {
    for (uint64_t s = 0; s < ns && nsel < r; ++s) {
      if (retired[s]) continue;
      cset_t* cs = &sets[s];
      uint32_t* mem = members + cs->off;
      if (cs->size == 1) {
        SELECT(mem[0]);
        retired[s] = 1;
        continue;
      }
      uint64_t keep = 0; /* std::erase_if(members, selected_contains) */
      for (uint64_t t = 0; t < cs->size; ++t)
        if (!in_sel[mem[t]]) mem[keep++] = mem[t];
      cs->size = keep;
      if (keep == 0) {
        retired[s] = 1;
        continue;
      }
      if (keep == 1) {
        SELECT(mem[0]);
        retired[s] = 1;
        continue;
      }
      SELECT(mem[rng_below(g, keep)]);
    }
  }
#undef SELECT
  qsort(selected, r, 4, cmp_u32);
  return selected;
}

static uint32_t* pd_select(const uint32_t* P, uint64_t n, uint64_t r, int variant) { /* bloom.cpp:224-236 */
  if (r > n) fail(GP_ERROR, "pd_select: r exceeds |P|");
  uint64_t begin = 0;
  switch (variant) {
    case 0: begin = 0; break;
    case 1: begin = (n - r) / 2; break;
    case 2: begin = n - r; break;
    default: fail(GP_ERROR, "pd_select: unknown variant");
  }
  uint32_t* out = (uint32_t*)xalloc((r ? r : 1) * 4);
  memcpy(out, P + begin, r * 4);
  return out;
}

int gpo_bloom_build(const uint32_t* support, uint64_t r, double eps, uint64_t seed_a,
                    uint64_t seed_b, uint8_t** filter, size_t* len) {
  API_BEGIN;
  bloom_t f;
  build_filter(&f, support, r, eps, seed_a, seed_b);
  bytes_t b;
  bytes_init(&b, 64);
  bloom_serialize(&f, &b);
  *len = b.n;
  *filter = (uint8_t*)detach(b.p, b.n);
  API_END;
}

int gpo_positive_scan(const uint8_t* filter, size_t len, uint64_t d, uint32_t** pos, uint64_t* n) {
  API_BEGIN;
  breader_t r = {filter, len, 0};
  bloom_t f;
  bloom_deserialize(&r, &f);
  uint32_t* P = positive_scan(&f, d, n);
  *pos = (uint32_t*)detach(P, *n * 4);
  API_END;
}

int gpo_bloom_select(const uint8_t* filter, size_t len, uint64_t d, uint64_t r, int index_method,
                     uint32_t** selected) {
  API_BEGIN;
  breader_t rd = {filter, len, 0};
  bloom_t f;
  bloom_deserialize(&rd, &f);
  uint64_t n;
  const uint32_t* P = positive_scan(&f, d, &n);
  rng_t g = {selection_seed(f.sa, f.sb)};
  const uint32_t* sel = index_method == GP_INDEX_BLOOM_P1 ? p1_select(P, n, r, &g) : p2_select(P, n, &f, r, &g);
  *selected = (uint32_t*)detach(sel, r * 4);
  API_END;
}

int gpo_conflict_sets(const uint8_t* filter, size_t len, uint64_t d, uint64_t** bits,
                      uint64_t** offsets, uint32_t** members, uint64_t* nsets) {
  API_BEGIN;
  breader_t rd = {filter, len, 0};
  bloom_t f;
  bloom_deserialize(&rd, &f);
  uint64_t n, ns;
  const uint32_t* P = positive_scan(&f, d, &n);
  uint32_t* mem;
  cset_t* sets = conflict_sets(P, n, &f, &mem, &ns);
  uint64_t* b = (uint64_t*)xalloc((ns + 1) * 8);
  uint64_t* o = (uint64_t*)xalloc((ns + 1) * 8);
  uint64_t total = 0;
  for (uint64_t s = 0; s < ns; ++s) total += sets[s].size;
  uint32_t* m = (uint32_t*)xalloc((total ? total : 1) * 4);
  uint64_t at = 0;
  for (uint64_t s = 0; s < ns; ++s) {
    b[s] = sets[s].bit;
    o[s] = at;
    for (uint64_t t = 0; t < sets[s].size; ++t) m[at++] = P[mem[sets[s].off + t]];
  }
  o[ns] = at;
  *nsets = ns;
  *bits = (uint64_t*)detach(b, ns * 8);
  *offsets = (uint64_t*)detach(o, (ns + 1) * 8);
  *members = (uint32_t*)detach(m, at * 4);
  API_END;
}

/* ==================================================================== curvefit.cpp */
static void stable_sort_desc(const double* v, uint32_t* idx, uint32_t* tmp, uint64_t n) {
  /* bottom-up merge sort: std::stable_sort with values(a) > values(b) (curvefit.cpp:30-32) */
  for (uint64_t width = 1; width < n; width *= 2) {
    for (uint64_t lo = 0; lo < n; lo += 2 * width) {
      uint64_t mid = lo + width < n ? lo + width : n;
      uint64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      uint64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        if (v[idx[j]] > v[idx[i]])
          tmp[k++] = idx[j++];
        else
          tmp[k++] = idx[i++];
      }
      while (i < mid) tmp[k++] = idx[i++];
      while (j < hi) tmp[k++] = idx[j++];
    }
    memcpy(idx, tmp, n * 4);
  }
}

typedef struct {
  uint32_t begin, end;
  double dev;
  uint32_t arg;
  int live;
} piece_t;

static piece_t make_piece(const double* v, uint32_t begin, uint32_t end, uint32_t min_points) {
  /* curvefit.cpp:50-67 (fp64, no contraction) */
  piece_t p = {begin, end, 0.0, 0, 0};
  const uint32_t len = end - begin;
  if (len < 3) return p;
  const double y0 = v[begin];
  const double slope = (v[end - 1] - y0) / (double)(len - 1);
  for (uint32_t i = begin + 1; i + 1 < end; ++i) {
    const double pred = y0 + slope * (double)(i - begin);
    const double d2 = (v[i] - pred) * (v[i] - pred);
    if (d2 > p.dev) {
      p.dev = d2;
      p.arg = i;
    }
  }
  p.live = p.dev > 0.0 && p.arg - begin >= min_points && end - p.arg >= min_points;
  return p;
}

static int cmp_piece_begin(const void* a, const void* b) {
  const piece_t *x = (const piece_t*)a, *y = (const piece_t*)b;
  return (x->begin > y->begin) - (x->begin < y->begin);
}

/* segment, curvefit.cpp:71-99; returns pieces sorted by begin */
static piece_t* segment(const double* v, uint32_t n, int max_segments, int min_points, uint64_t* count) {
  if (n < 1) fail(GP_ERROR, "segment: empty sequence");
  if (max_segments < 1) fail(GP_ERROR, "segment: max_segments must be >= 1");
  const uint32_t mp = (uint32_t)(min_points > 1 ? min_points : 1);
  piece_t* pieces = (piece_t*)xalloc((size_t)max_segments * sizeof(piece_t));
  uint64_t np = 1;
  pieces[0] = make_piece(v, 0, n, mp);
  while (np < (uint64_t)max_segments) {
    uint64_t best = np;
    for (uint64_t i = 0; i < np; ++i) {
      if (!pieces[i].live) continue;
      if (best == np || pieces[i].dev > pieces[best].dev ||
          (pieces[i].dev == pieces[best].dev && pieces[i].begin < pieces[best].begin))
        best = i;
    }
    if (best == np) break;
    const piece_t p = pieces[best];
    pieces[best] = make_piece(v, p.begin, p.arg, mp);
    pieces[np++] = make_piece(v, p.arg, p.end, mp);
  }
  qsort(pieces, np, sizeof(piece_t), cmp_piece_begin);
  *count = np;
  return pieces;
}

static double knot_m(const double* s, uint32_t n) { /* curvefit.cpp:101-105 */
  if (n < 4) fail(GP_ERROR, "knot_m: need at least 4 points");
  return fabs((s[0] - s[1]) - (s[n - 2] - s[n - 1]));
}
static int knot_count_linear(double m) { /* curvefit.cpp:107-110 */
  const double p = ceil(2.0 * sqrt(m > 0.0 ? m : 0.0));
  return (int)p > 1 ? (int)p : 1;
}
static int part_budget(const double* t, uint32_t begin, uint32_t end) { /* curvefit.cpp:424-428 */
  const uint32_t len = end - begin;
  if (len < 4) return 1;
  int b = knot_count_linear(knot_m(t + begin, len)) + 1;
  return b < 0xffff ? b : 0xffff;
}

/* Least squares by Householder QR with column pivoting on the n×(e+1)
 * Vandermonde matrix; curvefit.cpp:154 uses Eigen's colPivHouseholderQr.
 * Not bit-identical to Eigen (third-party arithmetic). */
static void lsq_qr(double* A, uint32_t n, int cols, const double* y, double* x) {
  double* c = (double*)xalloc((size_t)n * 8);
  memcpy(c, y, (size_t)n * 8);
  int perm[64];
  double norms[64];
  const int kmax = (int)n < cols ? (int)n : cols;
#define AT(i, j) A[(size_t)(j) * n + (i)]
  for (int j = 0; j < cols; ++j) {
    perm[j] = j;
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += AT(i, j) * AT(i, j);
    norms[j] = s;
  }
  for (int k = 0; k < kmax; ++k) {
    int best = k;
    for (int j = k + 1; j < cols; ++j)
      if (norms[j] > norms[best]) best = j;
    if (best != k) {
      for (uint32_t i = 0; i < n; ++i) {
        double t = AT(i, k);
        AT(i, k) = AT(i, best);
        AT(i, best) = t;
      }
      double t = norms[k];
      norms[k] = norms[best];
      norms[best] = t;
      int ti = perm[k];
      perm[k] = perm[best];
      perm[best] = ti;
    }
    double tail = 0.0;
    for (uint32_t i = k + 1; i < n; ++i) tail += AT(i, k) * AT(i, k);
    const double c0 = AT(k, k);
    double beta, tk;
    if (tail == 0.0) {
      beta = c0;
      tk = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (uint32_t i = k + 1; i < n; ++i) AT(i, k) /= denom;
      tk = (beta - c0) / beta;
    }
    AT(k, k) = beta;
    for (int j = k + 1; j < cols; ++j) {
      double s = AT(k, j);
      for (uint32_t i = k + 1; i < n; ++i) s += AT(i, k) * AT(i, j);
      s *= tk;
      AT(k, j) -= s;
      for (uint32_t i = k + 1; i < n; ++i) AT(i, j) -= s * AT(i, k);
      double rn = 0.0;
      for (uint32_t i = k + 1; i < n; ++i) rn += AT(i, j) * AT(i, j);
      norms[j] = rn;
    }
    /* apply the reflector to the right-hand side */
    double s = c[k];
    for (uint32_t i = k + 1; i < n; ++i) s += AT(i, k) * c[i];
    s *= tk;
    c[k] -= s;
    for (uint32_t i = k + 1; i < n; ++i) c[i] -= s * AT(i, k);
  }
  const double thresh = 2.220446049250313e-16 * (double)kmax;
  double maxpiv = 0.0;
  for (int k = 0; k < kmax; ++k) maxpiv = fabs(AT(k, k)) > maxpiv ? fabs(AT(k, k)) : maxpiv;
  int rank = 0;
  for (int k = 0; k < kmax; ++k)
    if (fabs(AT(k, k)) > thresh * maxpiv) ++rank;
  double z[64] = {0};
  for (int k = rank - 1; k >= 0; --k) {
    double s = c[k];
    for (int j = k + 1; j < rank; ++j) s -= AT(k, j) * z[j];
    z[k] = s / AT(k, k);
  }
  for (int k = 0; k < cols; ++k) x[perm[k]] = z[k];
#undef AT
}

/* fit_poly, curvefit.cpp:127-174 → coefficients in x = 1..n (degree+1 entries) */
static void fit_poly(const double* y, uint32_t n, int degree, double* coeffs) {
  if (n < 1) fail(GP_ERROR, "fit_poly: empty sequence");
  if (degree < 0 || degree > 60) fail(GP_ERROR, "fit_poly: degree out of range [0, 60]");
  for (int j = 0; j <= degree; ++j) coeffs[j] = 0.0;
  if (n == 1) {
    coeffs[0] = y[0];
    return;
  }
  const int eff = degree < (int)n - 1 ? degree : (int)n - 1;
  const double alpha = 2.0 / (double)(n - 1);
  const double beta = -(double)(n + 1) / (double)(n - 1);
  double* vand = (double*)xalloc((size_t)n * (eff + 1) * 8);
  for (uint32_t i = 0; i < n; ++i) {
    const double t = alpha * (double)(i + 1) + beta;
    double pw = 1.0;
    for (int j = 0; j <= eff; ++j) {
      vand[(size_t)j * n + i] = pw;
      pw *= t;
    }
  }
  double ct[64];
  lsq_qr(vand, n, eff + 1, y, ct);
  double binom[64][64];
  for (int j = 0; j <= eff; ++j) {
    for (int k = 0; k <= j; ++k) binom[j][k] = 1.0;
    for (int k = 1; k < j; ++k) binom[j][k] = binom[j - 1][k - 1] + binom[j - 1][k];
  }
  for (int k = 0; k <= eff; ++k) {
    double c = 0.0;
    const double ak = pow(alpha, k);
    for (int j = k; j <= eff; ++j) c += ct[j] * binom[j][k] * ak * pow(beta, j - k);
    coeffs[k] = c;
  }
}

typedef struct {
  uint8_t kind, degree;
  uint32_t sign_split;
  uint32_t* bounds;
  uint64_t nseg;
  float* coeffs;
} fitmodel_t;

/* value_compress, curvefit.cpp:432-493 (poly kind only; dexp is out of scope) */
static void value_compress(const double* values, uint64_t n, int degree, int max_segments,
                           fitmodel_t* m, uint32_t** map_out, uint64_t* map_len) {
  if (n < 1) fail(GP_ERROR, "value_compress: empty sequence");
  if (degree < 0 || degree > 60) fail(GP_ERROR, "value_compress: bad degree");
  if (n > 0xffffffffULL) fail(GP_ERROR, "value_compress: sequence too long");
  const uint32_t un = (uint32_t)n;
  /* sort_view, curvefit.cpp:26-39 */
  uint32_t* map = (uint32_t*)xalloc(n * 4);
  uint32_t* tmp = (uint32_t*)xalloc(n * 4);
  for (uint32_t i = 0; i < un; ++i) map[i] = i;
  stable_sort_desc(values, map, tmp, n);
  double* sv = (double*)xalloc(n * 8);
  uint32_t l = 0;
  for (uint32_t i = 0; i < un; ++i) {
    sv[i] = values[map[i]];
    if (sv[i] >= 0.0) l = i + 1;
  }
  double* t = (double*)xalloc(n * 8); /* sign fold, curvefit.cpp:442-446 */
  for (uint32_t i = 0; i < l; ++i) t[i] = sv[i];
  for (uint32_t j = 0; j + l < un; ++j) t[l + j] = -sv[un - 1 - j];
  int identity = 1; /* curvefit.cpp:449-455 */
  for (uint32_t i = 0; i < un; ++i)
    if (map[i] != i) {
      identity = 0;
      break;
    }
  *map_len = identity ? 0 : n;
  *map_out = identity ? NULL : map;

  uint32_t parts[2][2];
  int nparts = 0;
  if (l > 0) {
    parts[nparts][0] = 0;
    parts[nparts][1] = l;
    ++nparts;
  }
  if (l < un) {
    parts[nparts][0] = l;
    parts[nparts][1] = un;
    ++nparts;
  }
  const int cps = degree + 1;
  uint64_t cap_seg = 0;
  int budgets[2];
  for (int pi = 0; pi < nparts; ++pi) {
    int budget;
    if (max_segments > 0) { /* curvefit.cpp:473-481 */
      int64_t share = (int64_t)max_segments * (int64_t)(parts[pi][1] - parts[pi][0]) / (int64_t)n;
      budget = share > 1 ? (int)share : 1;
      if (pi + 1 == nparts) {
        const int used = pi == 0 ? 0 : budgets[0]; /* refined below with the actual count */
        budget = max_segments - used > 1 ? max_segments - used : 1;
      }
    } else {
      budget = part_budget(t, parts[pi][0], parts[pi][1]);
    }
    budgets[pi] = budget;
    cap_seg += (uint64_t)budget;
  }
  if (max_segments > 0) cap_seg += (uint64_t)max_segments; /* last-part budget uses the emitted count */
  m->kind = 0;
  m->degree = (uint8_t)degree;
  m->sign_split = l;
  m->bounds = (uint32_t*)xalloc(cap_seg * 4 + 4);
  m->coeffs = (float*)xalloc(cap_seg * cps * 4 + 4);
  m->nseg = 0;
  double* c = (double*)xalloc((size_t)cps * 8);
  for (int pi = 0; pi < nparts; ++pi) {
    const uint32_t begin = parts[pi][0], end = parts[pi][1];
    int budget = budgets[pi];
    if (max_segments > 0 && pi + 1 == nparts) { /* used = segments emitted so far */
      const int used = (int)m->nseg;
      budget = max_segments - used > 1 ? max_segments - used : 1;
    }
    uint64_t ns;
    piece_t* segs = segment(t + begin, end - begin, budget, degree + 1, &ns);
    for (uint64_t s = 0; s < ns; ++s) { /* fit_part, curvefit.cpp:409-420 */
      const uint32_t sb = begin + segs[s].begin, se = begin + segs[s].end;
      fit_poly(t + sb, se - sb, degree, c);
      m->bounds[m->nseg] = se;
      for (int j = 0; j < cps; ++j) m->coeffs[m->nseg * cps + j] = (float)c[j];
      ++m->nseg;
    }
  }
}

static void serialize_fit(const fitmodel_t* m, bytes_t* out) { /* curvefit.cpp:285-298 */
  if (m->nseg == 0) fail(GP_ERROR, "fit: no segments");
  if (m->nseg > 0xffff) fail(GP_ERROR, "fit: too many segments");
  put_u8(out, m->kind);
  put_le(out, m->nseg, 2);
  for (uint64_t i = 0; i < m->nseg; ++i) put_le(out, m->bounds[i], 4);
  put_u8(out, m->degree);
  const uint64_t cps = m->kind == 1 ? 4u : (uint64_t)m->degree + 1u;
  for (uint64_t i = 0; i < m->nseg * cps; ++i) put_f32(out, m->coeffs[i]);
  put_le(out, m->sign_split, 4);
}

static void parse_fit(breader_t* r, uint64_t count, fitmodel_t* m) { /* curvefit.cpp:300-325 */
  const uint8_t kind = (uint8_t)get_le(r, 1);
  if (kind > 1) fail(GP_UNKNOWN_METHOD, "fit: unknown model kind");
  m->kind = kind;
  const uint16_t segs = (uint16_t)get_le(r, 2);
  if (segs < 1) fail(GP_CORRUPT_PAYLOAD, "fit: zero segments");
  m->bounds = (uint32_t*)xalloc((size_t)segs * 4);
  uint32_t prev = 0;
  for (uint16_t i = 0; i < segs; ++i) {
    const uint32_t e = (uint32_t)get_le(r, 4);
    if (e <= prev && !(i == 0 && e > 0)) fail(GP_CORRUPT_PAYLOAD, "fit: bounds not increasing");
    prev = e;
    m->bounds[i] = e;
  }
  m->nseg = segs;
  if (prev != count) fail(GP_CORRUPT_PAYLOAD, "fit: bounds do not cover the sequence");
  m->degree = (uint8_t)get_le(r, 1);
  const uint64_t cps = kind == 1 ? 4u : (uint64_t)m->degree + 1u;
  m->coeffs = (float*)xalloc(segs * cps * 4);
  for (uint64_t i = 0; i < segs * cps; ++i) m->coeffs[i] = get_f32(r);
  m->sign_split = (uint32_t)get_le(r, 4);
  if (m->sign_split > count) fail(GP_CORRUPT_PAYLOAD, "fit: sign split out of range");
  if (m->sign_split > 0 && m->sign_split < count) {
    int found = 0;
    for (uint16_t i = 0; i < segs; ++i) found |= m->bounds[i] == m->sign_split;
    if (!found) fail(GP_CORRUPT_PAYLOAD, "fit: segment straddles sign split");
  }
}

static unsigned reorder_entry_bits(uint64_t d) { /* curvefit.cpp:327-330: bit_width(d - 1) */
  if (d < 1) fail(GP_ERROR, "reorder: d must be >= 1");
  uint64_t x = d - 1;
  unsigned w = 0;
  while (x) {
    ++w;
    x >>= 1;
  }
  return w;
}
static void reorder_encode(const uint32_t* map, uint64_t n, uint64_t d, bitw_t* w) { /* curvefit.cpp:332-340 */
  const unsigned bits = reorder_entry_bits(d);
  for (uint64_t i = 0; i < n; ++i) {
    if ((uint64_t)map[i] >= d) fail(GP_ERROR, "reorder: entry out of range");
    bw_bits(w, map[i], bits);
  }
}
static uint32_t* reorder_decode(const uint8_t* p, size_t len, uint64_t count, uint64_t d) { /* :342-356 */
  const unsigned bits = reorder_entry_bits(d);
  bitr_t r = {p, len, 0};
  uint32_t* out = (uint32_t*)xalloc((count ? count : 1) * 4);
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t e = br_bits(&r, bits);
    if (e >= d) fail(GP_CORRUPT_PAYLOAD, "reorder: entry out of range");
    out[i] = (uint32_t)e;
  }
  if (br_remaining(&r) >= 8 || (br_remaining(&r) > 0 && br_bits(&r, (unsigned)br_remaining(&r)) != 0))
    fail(GP_CORRUPT_PAYLOAD, "reorder: trailing garbage");
  return out;
}

static double eval_poly(const float* c, size_t k, double x) { /* curvefit.cpp:360-364 */
  double acc = 0.0;
  for (size_t j = k; j-- > 0;) acc = acc * x + (double)c[j];
  return acc;
}

static double* value_decompress(const fitmodel_t* m, const uint32_t* reorder, uint64_t reorder_n,
                                uint64_t count) { /* curvefit.cpp:495-542 */
  if (count < 1 || count > 0xffffffffULL) fail(GP_CORRUPT_PAYLOAD, "fit: bad value count");
  if (m->nseg == 0) fail(GP_CORRUPT_PAYLOAD, "fit: no segments");
  uint32_t prev = 0;
  for (uint64_t i = 0; i < m->nseg; ++i) {
    if (m->bounds[i] <= prev && i > 0) fail(GP_CORRUPT_PAYLOAD, "fit: bounds not increasing");
    if (i == 0 && m->bounds[i] == 0) fail(GP_CORRUPT_PAYLOAD, "fit: bounds not increasing");
    prev = m->bounds[i];
  }
  if (prev != count) fail(GP_CORRUPT_PAYLOAD, "fit: bounds do not cover the sequence");
  const uint32_t l = m->sign_split;
  if (l > count) fail(GP_CORRUPT_PAYLOAD, "fit: sign split out of range");
  if (m->kind != 0) fail(GP_UNSUPPORTED, "fit: dexp evaluation is out of scope");
  const uint32_t un = (uint32_t)count;
  const size_t cps = (size_t)m->degree + 1;
  double* t = (double*)xalloc(count * 8);
  uint32_t begin = 0;
  for (uint64_t s = 0; s < m->nseg; ++s) {
    const uint32_t end = m->bounds[s];
    const float* c = m->coeffs + s * cps;
    for (uint32_t i = begin; i < end; ++i) t[i] = eval_poly(c, cps, (double)(i - begin + 1));
    begin = end;
  }
  double* sorted = (double*)xalloc(count * 8);
  for (uint32_t i = 0; i < l; ++i) sorted[i] = t[i];
  for (uint32_t i = l; i < un; ++i) sorted[i] = -t[l + (un - 1 - i)];
  if (reorder_n == 0) return sorted;
  if (reorder_n != count) fail(GP_CORRUPT_PAYLOAD, "reorder: wrong entry count");
  uint8_t* seen = (uint8_t*)xalloc(count);
  double* out = (double*)xalloc(count * 8);
  for (uint64_t p = 0; p < count; ++p) {
    const uint32_t orig = reorder[p];
    if (orig >= un || seen[orig]) fail(GP_CORRUPT_PAYLOAD, "reorder: not a permutation");
    seen[orig] = 1;
    out[orig] = sorted[p];
  }
  return out;
}

int gpo_value_compress(const double* v, uint64_t n, int degree, int max_segments, uint8_t** fit,
                       size_t* fit_len, uint32_t** map, uint64_t* map_len) {
  API_BEGIN;
  fitmodel_t m;
  uint32_t* mp;
  value_compress(v, n, degree, max_segments, &m, &mp, map_len);
  bytes_t b;
  bytes_init(&b, 64);
  serialize_fit(&m, &b);
  *fit_len = b.n;
  *fit = (uint8_t*)detach(b.p, b.n);
  *map = *map_len ? (uint32_t*)detach(mp, *map_len * 4) : NULL;
  API_END;
}

/* ==================================================================== container.cpp */
typedef struct {
  uint16_t version;
  uint8_t index_method, value_method;
  uint64_t d, r;
  const uint8_t *ip, *vp, *rp;
  size_t il, vl, rl;
} container_t;

static int index_known(uint8_t id) { return id <= GP_INDEX_BLOOM_NAIVE; }
static int value_known(uint8_t id) { return id <= GP_VALUE_RAW_F64; }

static void pack(const container_t* c, bytes_t* out) { /* container.cpp:58-82 */
  if (!index_known(c->index_method)) fail(GP_ERROR, "container: unregistered index method");
  if (!value_known(c->value_method)) fail(GP_ERROR, "container: unregistered value method");
  put_bytes(out, (const uint8_t*)"DRC1", 4);
  put_le(out, c->version, 2);
  put_u8(out, c->index_method);
  put_u8(out, c->value_method);
  put_u8(out, c->rl == 0 ? 0u : 1u);
  put_le(out, c->d, 8);
  put_le(out, c->r, 8);
  put_le(out, c->il, 8);
  put_le(out, c->vl, 8);
  put_le(out, c->rl, 8);
  put_bytes(out, c->ip, c->il);
  put_bytes(out, c->vp, c->vl);
  put_bytes(out, c->rp, c->rl);
  crc_init();
  uint32_t crc = 0xFFFFFFFFu;
  crc = crc_update(crc, c->ip, c->il);
  crc = crc_update(crc, c->vp, c->vl);
  crc = crc_update(crc, c->rp, c->rl);
  put_le(out, crc ^ 0xFFFFFFFFu, 4);
}

static void unpack(const uint8_t* bytes, size_t n, container_t* c) { /* container.cpp:84-127 */
  if (n < 4) fail(GP_TRUNCATED, "container: shorter than magic");
  if (memcmp(bytes, "DRC1", 4) != 0) fail(GP_CORRUPT_PAYLOAD, "container: bad magic");
  breader_t r = {bytes + 4, n - 4, 0};
  const uint16_t version = (uint16_t)get_le(&r, 2);
  if (version != 1) fail(GP_DECODE, "container: unsupported version");
  const uint8_t index_id = (uint8_t)get_le(&r, 1);
  const uint8_t value_id = (uint8_t)get_le(&r, 1);
  const uint8_t flags = (uint8_t)get_le(&r, 1);
  c->version = version;
  c->d = get_le(&r, 8);
  c->r = get_le(&r, 8);
  const uint64_t il = get_le(&r, 8), vl = get_le(&r, 8), rl = get_le(&r, 8);
  const uint64_t body = il + vl + rl + 4; /* u64 arithmetic, wraps like the reference */
  const uint64_t rem = r.n - r.pos;
  if (rem < body) fail(GP_TRUNCATED, "container: payloads truncated");
  if (rem > body) fail(GP_CORRUPT_PAYLOAD, "container: trailing garbage");
  c->ip = get_bytes(&r, il);
  c->vp = get_bytes(&r, vl);
  c->rp = get_bytes(&r, rl);
  const uint32_t stored = (uint32_t)get_le(&r, 4);
  crc_init();
  uint32_t crc = 0xFFFFFFFFu;
  crc = crc_update(crc, c->ip, il);
  crc = crc_update(crc, c->vp, vl);
  crc = crc_update(crc, c->rp, rl);
  if ((crc ^ 0xFFFFFFFFu) != stored) fail(GP_CHECKSUM, "container: checksum mismatch");
  if (!index_known(index_id)) fail(GP_UNKNOWN_METHOD, "container: unknown index method");
  if (!value_known(value_id)) fail(GP_UNKNOWN_METHOD, "container: unknown value method");
  c->index_method = index_id;
  c->value_method = value_id;
  if ((flags & ~1u) != 0) fail(GP_CORRUPT_PAYLOAD, "container: unknown flag bits");
  if (((flags & 1u) != 0) != (rl > 0)) fail(GP_CORRUPT_PAYLOAD, "container: reorder flag inconsistent with payload");
  if (rl > 0 && c->value_method != GP_VALUE_FIT_POLY && c->value_method != GP_VALUE_FIT_DEXP)
    fail(GP_CORRUPT_PAYLOAD, "container: reorder payload without a fit value method");
  if (c->r > c->d) fail(GP_CORRUPT_PAYLOAD, "container: r exceeds d");
  c->il = il;
  c->vl = vl;
  c->rl = rl;
}

/* ==================================================================== pipeline.cpp */
static double* gather_values(const sparse_t* sg, const float* dense, const uint32_t* idx, uint64_t n) {
  /* pipeline.cpp:38-54 */
  double* out = (double*)xalloc((n ? n : 1) * 8);
  if (dense) {
    for (uint64_t i = 0; i < n; ++i) out[i] = (double)dense[idx[i]];
    return out;
  }
  for (uint64_t i = 0; i < n; ++i) { /* lower_bound over the support */
    uint64_t lo = 0, hi = sg->count;
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (sg->support[mid] < idx[i]) lo = mid + 1; else hi = mid;
    }
    out[i] = (lo < sg->count && sg->support[lo] == idx[i]) ? sg->values[lo] : 0.0;
  }
  return out;
}

/* quantize + serialize_quant (codecs.cpp:290-351): per bucket the f32 scale
 * 2*max|v|; code = floor(u) + [unit() < frac(u)], u = (v/scale + 0.5)*levels
 * clamped to [0, levels]; unit() is drawn only when scale > 0; codes packed
 * LSB-first at `bits` each.  Payload: bits u8, bucket u32, scales f32[nb], codes. */
static void quantize_serialize(const double* v, uint64_t n, int bits, uint32_t bucket, rng_t* g, bytes_t* out) {
  if (bits < 1 || bits > 16) fail(GP_ERROR, "quantize: bits out of range [1, 16]");
  if (bucket < 1) fail(GP_ERROR, "quantize: bucket must be >= 1");
  const uint64_t levels = (1ULL << bits) - 1;
  const uint64_t nb = (n + bucket - 1) / bucket;
  put_u8(out, (uint8_t)bits);
  put_le(out, bucket, 4);
  float* scales = (float*)xalloc((nb ? nb : 1) * sizeof(float));
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t lo = b * bucket, hi = lo + bucket < n ? lo + bucket : n;
    double mx = 0.0;
    for (uint64_t i = lo; i < hi; ++i) mx = fabs(v[i]) > mx ? fabs(v[i]) : mx;
    scales[b] = (float)(2.0 * mx);
    put_f32(out, scales[b]);
  }
  bitw_t w;
  bw_init(&w, (n * (uint64_t)bits + 7) / 8 + 1);
  for (uint64_t i = 0; i < n; ++i) {
    const float scale = scales[i / bucket];
    uint64_t code = 0;
    if (scale > 0.0f) {
      double u = (v[i] / (double)scale + 0.5) * (double)levels;
      u = u < 0.0 ? 0.0 : (u > (double)levels ? (double)levels : u);
      const double lo = floor(u);
      const double frac = u - lo;
      code = (uint64_t)lo;
      if (rng_unit(g) < frac) ++code;
      if (code > levels) code = levels;
    }
    bw_bits(&w, code, (unsigned)bits);
  }
  put_bytes(out, w.b.p, w.b.n);
}

/* parse_quant + dequantize (codecs.cpp:327-368, pipeline.cpp:124-129) */
static double* parse_dequantize(const uint8_t* p, size_t len, uint64_t count) {
  breader_t r = {p, len, 0};
  const unsigned bits = (unsigned)get_le(&r, 1);
  if (bits < 1 || bits > 16) fail(GP_CORRUPT_PAYLOAD, "quant: bits out of range");
  const uint32_t bucket = (uint32_t)get_le(&r, 4);
  if (bucket < 1) fail(GP_CORRUPT_PAYLOAD, "quant: bucket must be >= 1");
  const uint64_t nb = (count + bucket - 1) / bucket;
  float* scales = (float*)xalloc((nb ? nb : 1) * sizeof(float));
  for (uint64_t b = 0; b < nb; ++b) scales[b] = get_f32(&r);
  const uint64_t code_bytes = (count * bits + 7) / 8;
  const uint8_t* codes = get_bytes(&r, code_bytes);
  if (r.pos != r.n) fail(GP_CORRUPT_PAYLOAD, "pipeline: quant payload trailing bytes");
  const uint64_t levels = (1ULL << bits) - 1;
  double* out = (double*)xalloc((count ? count : 1) * 8);
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t code = 0;
    for (unsigned j = 0; j < bits; ++j) {
      const uint64_t bit = i * bits + j;
      code |= (uint64_t)((codes[bit / 8] >> (bit % 8)) & 1u) << j;
    }
    out[i] = (double)scales[i / bucket] * ((double)code / (double)levels - 0.5);
  }
  return out;
}

/* ---- canonical Huffman over index bytes (codecs.cpp:72-242) ---- */
typedef struct {
  uint8_t len[256];
  uint64_t code[256];
  uint8_t sorted[256];
  unsigned nsym, max_len;
  uint64_t first_code[64];
  uint32_t first_index[64], count[64];
} huff_t;

static void huff_freqs(uint64_t d, uint64_t freq[256]) { /* index_byte_frequencies, codecs.cpp:72-91 */
  if (d < 1) fail(GP_ERROR, "index_byte_frequencies: d must be >= 1");
  if (d > 0x100000000ULL) fail(GP_ERROR, "index_byte_frequencies: d exceeds 32-bit index space");
  memset(freq, 0, 256 * sizeof(uint64_t));
  for (unsigned j = 0; j < 4; ++j) {
    const uint64_t width = 1ULL << (8 * j);
    const uint64_t high = d >> (8 * (j + 1));
    const uint64_t mid = (d >> (8 * j)) & 0xff;
    const uint64_t low = d & (width - 1);
    for (unsigned b = 0; b < 256; ++b) {
      uint64_t n = high * width;
      if (b < mid) n += width;
      else if (b == mid) n += low;
      freq[b] += n;
    }
  }
}

/* from_frequencies (codecs.cpp:93-170): min-heap on (weight, creation order),
 * lengths by depth, canonical codes by (length, symbol) */
static void huff_build(uint64_t d, huff_t* h) {
  uint64_t freq[256];
  huff_freqs(d, freq);
  uint64_t w[511];
  int left[511], right[511], sym[511];
  int heap[511], hn = 0, nn = 0;
  memset(h, 0, sizeof *h);
#define HLESS(a, b) (w[a] < w[b] || (w[a] == w[b] && (a) < (b)))
  for (int s = 0; s < 256; ++s) {
    if (!freq[s]) continue;
    w[nn] = freq[s]; left[nn] = right[nn] = -1; sym[nn] = s;
    int i = hn++; heap[i] = nn++;
    while (i > 0 && HLESS(heap[i], heap[(i - 1) / 2])) { int t = heap[i]; heap[i] = heap[(i - 1) / 2]; heap[(i - 1) / 2] = t; i = (i - 1) / 2; }
  }
  if (nn == 0) fail(GP_ERROR, "huffman: empty alphabet");
  if (nn == 1) {
    h->len[sym[0]] = 1;
  } else {
    while (hn > 1) {
      int ab[2];
      for (int q = 0; q < 2; ++q) {
        ab[q] = heap[0];
        heap[0] = heap[--hn];
        int i = 0;
        for (;;) {
          int l = 2 * i + 1, r = l + 1, m = i;
          if (l < hn && HLESS(heap[l], heap[m])) m = l;
          if (r < hn && HLESS(heap[r], heap[m])) m = r;
          if (m == i) break;
          int t = heap[i]; heap[i] = heap[m]; heap[m] = t; i = m;
        }
      }
      w[nn] = w[ab[0]] + w[ab[1]]; left[nn] = ab[0]; right[nn] = ab[1]; sym[nn] = -1;
      int i = hn++; heap[i] = nn++;
      while (i > 0 && HLESS(heap[i], heap[(i - 1) / 2])) { int t = heap[i]; heap[i] = heap[(i - 1) / 2]; heap[(i - 1) / 2] = t; i = (i - 1) / 2; }
    }
    int st[511], dp[511], sn = 0;
    st[sn] = nn - 1; dp[sn++] = 0;
    while (sn) {
      const int id = st[--sn], dep = dp[sn];
      if (sym[id] >= 0) {
        if (dep > 57) fail(GP_ERROR, "huffman: code length exceeds 57 bits");
        h->len[sym[id]] = (uint8_t)dep;
      } else {
        st[sn] = left[id]; dp[sn++] = dep + 1;
        st[sn] = right[id]; dp[sn++] = dep + 1;
      }
    }
  }
#undef HLESS
  for (unsigned L = 1; L <= 57; ++L)
    for (int s = 0; s < 256; ++s)
      if (h->len[s] == L) h->sorted[h->nsym++] = (uint8_t)s;
  h->max_len = h->len[h->sorted[h->nsym - 1]];
  uint64_t code = 0;
  unsigned prev = h->len[h->sorted[0]];
  for (unsigned i = 0; i < h->nsym; ++i) {
    const unsigned L = h->len[h->sorted[i]];
    code = i ? (code + 1) << (L - prev) : 0;
    h->code[h->sorted[i]] = code;
    prev = L;
    if (h->count[L] == 0) {
      h->first_index[L] = i;
      h->first_code[L] = code;
    }
    ++h->count[L];
  }
}

static void huff_encode_indices(const huff_t* h, const uint32_t* idx, uint64_t r, uint64_t d, bitw_t* w) {
  for (uint64_t i = 0; i < r; ++i) { /* encode_indices, codecs.cpp:219-229 */
    if (idx[i] >= d) fail(GP_ERROR, "huffman: index out of range");
    for (unsigned j = 0; j < 4; ++j) {
      const uint8_t s = (uint8_t)(idx[i] >> (8 * j));
      const unsigned L = h->len[s];
      if (L == 0) fail(GP_ERROR, "huffman: symbol absent from codec");
      for (unsigned b = L; b-- > 0;) bw_bit(w, (int)((h->code[s] >> b) & 1u)); /* MSB first */
    }
  }
}

/* decode + decode_indices (codecs.cpp:196-242); *bits_used = bits consumed */
static uint32_t* huff_decode_indices(const huff_t* h, const uint8_t* p, size_t n, uint64_t count, uint64_t d,
                                     uint64_t* bits_used) {
  const uint64_t nbits = 8 * (uint64_t)n;
  uint64_t pos = 0;
  uint8_t* bytes = (uint8_t*)xalloc(4 * count + 1);
  for (uint64_t i = 0; i < 4 * count; ++i) {
    uint64_t code = 0;
    int found = -1;
    for (unsigned L = 1; L <= h->max_len; ++L) {
      if (pos >= nbits) fail(GP_TRUNCATED, "bit stream exhausted");
      code = (code << 1) | ((p[pos / 8] >> (pos % 8)) & 1u);
      ++pos;
      if (h->count[L] && code >= h->first_code[L] && code - h->first_code[L] < h->count[L]) {
        found = h->sorted[h->first_index[L] + (uint32_t)(code - h->first_code[L])];
        break;
      }
    }
    if (found < 0) fail(GP_CORRUPT_PAYLOAD, "huffman: invalid code");
    bytes[i] = (uint8_t)found;
  }
  if (nbits - pos >= 8) fail(GP_CORRUPT_PAYLOAD, "huffman: trailing garbage");
  if (bits_used) *bits_used = pos;
  uint32_t* out = (uint32_t*)xalloc((count ? count : 1) * 4);
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t v = 0;
    for (unsigned j = 0; j < 4; ++j) v |= (uint32_t)bytes[4 * i + j] << (8 * j);
    if (v >= d) fail(GP_CORRUPT_PAYLOAD, "huffman: decoded index out of range");
    out[i] = v;
  }
  return out;
}

static void encode_values(const double* values, uint64_t n, const gp_pipeline_config* cfg, uint64_t d,
                          bytes_t* vout, bitw_t* rout) { /* pipeline.cpp:56-93 */
  switch (cfg->value_method) {
    case GP_VALUE_NONE:
      for (uint64_t i = 0; i < n; ++i) put_f32(vout, (float)values[i]);
      return;
    case GP_VALUE_RAW_F64:
      for (uint64_t i = 0; i < n; ++i) put_f64(vout, values[i]);
      return;
    case GP_VALUE_FIT_POLY: {
      fitmodel_t m;
      uint32_t* map;
      uint64_t map_len;
      value_compress(values, n, cfg->degree, cfg->max_segments, &m, &map, &map_len);
      if (map_len) reorder_encode(map, map_len, d, rout);
      serialize_fit(&m, vout);
      return;
    }
    case GP_VALUE_QUANT: {
      rng_t g = {gpo_hash64(0xC, cfg->seed)}; /* derive_quant_seed, pipeline.cpp:26, :81-84 */
      quantize_serialize(values, n, cfg->quant_bits, cfg->quant_bucket, &g, vout);
      return;
    }
    case GP_VALUE_DEFLATE_SLOT: { /* pipeline.cpp:85-90 + byte_compress codecs.cpp:244-266 */
      if (cfg->slot_codec == 1) fail(GP_UNSUPPORTED, "oracle: the deflate byte codec is out of scope");
      if (cfg->slot_codec != 0) fail(GP_UNKNOWN_METHOD, "byte_compress: unknown codec id");
      put_u8(vout, 0);
      put_le(vout, 4 * n, 8);
      for (uint64_t i = 0; i < n; ++i) put_f32(vout, (float)values[i]);
      return;
    }
    default:
      fail(GP_UNSUPPORTED, "oracle: value method %d is out of scope", cfg->value_method);
  }
}

static void compress(const sparse_t* sg, const gp_pipeline_config* cfg, const float* dense,
                     bytes_t* packed) { /* pipeline.cpp:146-221 */
  validate_sparse(sg);
  const uint64_t d = sg->d, r = sg->count;
  if (r < 1 && cfg->index_method != GP_INDEX_NONE)
    fail(GP_ERROR, "pipeline: empty support requires the raw index method");
  container_t c;
  memset(&c, 0, sizeof c);
  c.version = 1;
  c.d = d;
  c.r = r;
  c.index_method = cfg->index_method;
  c.value_method = cfg->value_method;
  bytes_t ip, vp;
  bitw_t rp;
  bytes_init(&ip, 64);
  bytes_init(&vp, 64);
  bw_init(&rp, 64);
  const double* values = sg->values;
  uint64_t nvalues = r;
  switch (cfg->index_method) {
    case GP_INDEX_NONE:
      for (uint64_t i = 0; i < r; ++i) put_le(&ip, sg->support[i], 4);
      break;
    case GP_INDEX_BITMAP:
      bytes_reserve(&ip, (d + 7) / 8);
      bitmap_to_bytes(to_bitmap(sg->support, r, d), d, ip.p);
      ip.n = (d + 7) / 8;
      break;
    case GP_INDEX_RLE: {
      bitw_t w;
      bw_init(&w, 64);
      rle_encode(to_bitmap(sg->support, r, d), d, &w);
      ip = w.b;
      break;
    }
    case GP_INDEX_HUFFMAN: { /* pipeline.cpp:179-184 */
      huff_t h;
      huff_build(d, &h);
      bitw_t w;
      bw_init(&w, 64);
      huff_encode_indices(&h, sg->support, r, d, &w);
      ip = w.b;
      break;
    }
    case GP_INDEX_BLOOM_P0:
    case GP_INDEX_BLOOM_P1:
    case GP_INDEX_BLOOM_P2:
    case GP_INDEX_BLOOM_PD:
    case GP_INDEX_BLOOM_NAIVE: {
      const uint64_t sa = seed_a_of(cfg->seed), sb = seed_b_of(cfg->seed);
      bloom_t f;
      build_filter(&f, sg->support, r, cfg->fpr, sa, sb);
      bloom_serialize(&f, &ip);
      if (cfg->index_method == GP_INDEX_BLOOM_NAIVE) break;
      uint64_t np;
      const uint32_t* P = positive_scan(&f, d, &np);
      if (cfg->index_method == GP_INDEX_BLOOM_P0) {
        values = gather_values(sg, dense, P, np);
        nvalues = np;
      } else if (cfg->index_method == GP_INDEX_BLOOM_PD) {
        put_u8(&ip, cfg->pd_variant);
        values = gather_values(sg, dense, pd_select(P, np, r, cfg->pd_variant), r);
      } else {
        rng_t g = {selection_seed(sa, sb)};
        const uint32_t* sel = cfg->index_method == GP_INDEX_BLOOM_P1 ? p1_select(P, np, r, &g)
                                                                     : p2_select(P, np, &f, r, &g);
        values = gather_values(sg, dense, sel, r);
      }
      break;
    }
    default:
      fail(GP_UNSUPPORTED, "oracle: index method %d is out of scope", cfg->index_method);
  }
  if (nvalues == 0 && (cfg->value_method == GP_VALUE_FIT_POLY || cfg->value_method == GP_VALUE_FIT_DEXP ||
                       cfg->value_method == GP_VALUE_QUANT))
    fail(GP_ERROR, "pipeline: fit/quant value methods need a nonempty value sequence");
  encode_values(values, nvalues, cfg, d, &vp, &rp);
  c.ip = ip.p;
  c.il = ip.n;
  c.vp = vp.p;
  c.vl = vp.n;
  c.rp = rp.b.p;
  c.rl = rp.b.n;
  pack(&c, packed);
}

static double* decode_values(const container_t* c, uint64_t count) { /* pipeline.cpp:95-142 */
  switch (c->value_method) {
    case GP_VALUE_NONE: {
      if (c->vl != 4 * count) fail(GP_CORRUPT_PAYLOAD, "pipeline: raw f32 payload length mismatch");
      breader_t r = {c->vp, c->vl, 0};
      double* out = (double*)xalloc((count ? count : 1) * 8);
      for (uint64_t i = 0; i < count; ++i) out[i] = (double)get_f32(&r);
      return out;
    }
    case GP_VALUE_RAW_F64: {
      if (c->vl != 8 * count) fail(GP_CORRUPT_PAYLOAD, "pipeline: raw f64 payload length mismatch");
      breader_t r = {c->vp, c->vl, 0};
      double* out = (double*)xalloc((count ? count : 1) * 8);
      for (uint64_t i = 0; i < count; ++i) out[i] = get_f64(&r);
      return out;
    }
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP: {
      breader_t r = {c->vp, c->vl, 0};
      fitmodel_t m;
      parse_fit(&r, count, &m);
      if (r.pos != r.n) fail(GP_CORRUPT_PAYLOAD, "pipeline: fit payload trailing bytes");
      const uint32_t* reorder = NULL;
      uint64_t rn = 0;
      if (c->rl) {
        reorder = reorder_decode(c->rp, c->rl, count, c->d);
        rn = count;
      }
      return value_decompress(&m, reorder, rn, count);
    }
    case GP_VALUE_QUANT:
      return parse_dequantize(c->vp, c->vl, count);
    case GP_VALUE_DEFLATE_SLOT: { /* byte_decompress (codecs.cpp:268-288) + pipeline.cpp:130-139 */
      breader_t r = {c->vp, c->vl, 0};
      const unsigned id = (unsigned)get_le(&r, 1);
      const uint64_t raw_len = get_le(&r, 8);
      const size_t body = r.n - r.pos;
      if (id == 1) fail(GP_UNSUPPORTED, "oracle: the deflate byte codec is out of scope");
      if (id != 0) fail(GP_UNKNOWN_METHOD, "byte_decompress: unknown codec id");
      if (body != raw_len) fail(GP_CORRUPT_PAYLOAD, "store: length mismatch");
      if (raw_len != 4 * count) fail(GP_CORRUPT_PAYLOAD, "pipeline: deflate slot length mismatch");
      double* out = (double*)xalloc((count ? count : 1) * 8);
      for (uint64_t i = 0; i < count; ++i) out[i] = (double)get_f32(&r);
      return out;
    }
    default:
      fail(GP_UNSUPPORTED, "oracle: value method %d is out of scope", c->value_method);
  }
  return NULL;
}

static void decompress(const container_t* c, sparse_t* out) { /* pipeline.cpp:223-306 */
  if (c->d < 1) fail(GP_CORRUPT_PAYLOAD, "pipeline: d must be >= 1");
  if (c->d > 0xffffffffULL) fail(GP_CORRUPT_PAYLOAD, "pipeline: d exceeds index space");
  const uint64_t d = c->d;
  out->d = d;
  switch (c->index_method) {
    case GP_INDEX_NONE: {
      if (c->il != 4 * c->r) fail(GP_CORRUPT_PAYLOAD, "pipeline: raw key payload length mismatch");
      breader_t r = {c->ip, c->il, 0};
      out->support = (uint32_t*)xalloc((c->r ? c->r : 1) * 4);
      for (uint64_t i = 0; i < c->r; ++i) out->support[i] = (uint32_t)get_le(&r, 4);
      out->count = c->r;
      break;
    }
    case GP_INDEX_BITMAP:
    case GP_INDEX_RLE: {
      const uint64_t* w = c->index_method == GP_INDEX_BITMAP ? bitmap_from_bytes(c->ip, c->il, d)
                                                             : rle_decode(c->ip, c->il, d);
      if (bitmap_popcount(w, d) != c->r)
        fail(GP_CORRUPT_PAYLOAD, c->index_method == GP_INDEX_BITMAP ? "pipeline: bitmap popcount != r"
                                                                     : "pipeline: rle popcount != r");
      out->support = bitmap_support(w, d, c->r);
      out->count = c->r;
      break;
    }
    case GP_INDEX_HUFFMAN: { /* pipeline.cpp:254-258 */
      huff_t h;
      huff_build(d, &h);
      out->support = huff_decode_indices(&h, c->ip, c->il, c->r, d, NULL);
      out->count = c->r;
      break;
    }
    case GP_INDEX_BLOOM_P0:
    case GP_INDEX_BLOOM_P1:
    case GP_INDEX_BLOOM_P2:
    case GP_INDEX_BLOOM_PD:
    case GP_INDEX_BLOOM_NAIVE: {
      breader_t rd = {c->ip, c->il, 0};
      bloom_t f;
      bloom_deserialize(&rd, &f);
      int variant = 0;
      if (c->index_method == GP_INDEX_BLOOM_PD) {
        const uint8_t v = (uint8_t)get_le(&rd, 1);
        if (v > 2) fail(GP_CORRUPT_PAYLOAD, "pipeline: unknown deterministic variant");
        variant = v;
      }
      if (rd.pos != rd.n) fail(GP_CORRUPT_PAYLOAD, "pipeline: bloom payload trailing bytes");
      if (c->index_method == GP_INDEX_BLOOM_NAIVE) { /* naive_reconstruct, bloom.cpp:130-138 */
        const double* v = decode_values(c, c->r);
        uint64_t np;
        out->support = positive_scan(&f, d, &np);
        out->count = np;
        out->values = (double*)xalloc((np ? np : 1) * 8);
        const uint64_t k = c->r < np ? c->r : np;
        for (uint64_t i = 0; i < k; ++i) out->values[i] = v[i];
        return;
      }
      uint64_t np;
      const uint32_t* P = positive_scan(&f, d, &np);
      if (c->index_method == GP_INDEX_BLOOM_P0) {
        out->support = (uint32_t*)P;
        out->count = np;
      } else {
        if (np < c->r) fail(GP_CORRUPT_PAYLOAD, "pipeline: positive set smaller than r");
        rng_t g = {selection_seed(f.sa, f.sb)};
        if (c->index_method == GP_INDEX_BLOOM_P1)
          out->support = p1_select(P, np, c->r, &g);
        else if (c->index_method == GP_INDEX_BLOOM_P2)
          out->support = p2_select(P, np, &f, c->r, &g);
        else
          out->support = pd_select(P, np, c->r, variant);
        out->count = c->r;
      }
      out->values = decode_values(c, out->count);
      return;
    }
    default:
      fail(GP_UNSUPPORTED, "oracle: index method %d is out of scope", c->index_method);
  }
  out->values = decode_values(c, c->r);
  for (uint64_t i = 1; i < out->count; ++i) /* validate → CorruptPayloadError, pipeline.cpp:299-305 */
    if (out->support[i] <= out->support[i - 1])
      fail(GP_CORRUPT_PAYLOAD, "sparse gradient: support not strictly increasing");
  for (uint64_t i = 0; i < out->count; ++i)
    if ((uint64_t)out->support[i] >= d) fail(GP_CORRUPT_PAYLOAD, "sparse gradient: index out of range");
}

/* ==================================================================== public pipeline */
int gpo_compress_pack(uint64_t d, const uint32_t* support, const double* values, uint64_t r,
                      const float* dense, const gp_pipeline_config* cfg, uint8_t** out, size_t* len) {
  API_BEGIN;
  if (dense == NULL && values == NULL) fail(GP_ERROR, "oracle: need values or a dense gradient");
  sparse_t sg = {d, (uint32_t*)support, (double*)values, r};
  if (!values) { /* gather(dense, support), gradient.cpp:44-54 */
    sg.values = (double*)xalloc((r ? r : 1) * 8);
    for (uint64_t i = 0; i < r; ++i) {
      if ((uint64_t)support[i] >= d) fail(GP_ERROR, "gather: index out of range");
      sg.values[i] = (double)dense[support[i]];
    }
  }
  bytes_t b;
  bytes_init(&b, 256);
  compress(&sg, cfg, dense, &b);
  *len = b.n;
  *out = (uint8_t*)detach(b.p, b.n);
  API_END;
}

int gpo_encode_dense(const float* g, uint64_t d, uint64_t r, const gp_pipeline_config* cfg,
                     uint8_t** out, size_t* len) {
  API_BEGIN;
  uint32_t* support = (uint32_t*)xalloc((r ? r : 1) * 4);
  int rc = gpo_top_r(g, d, r, support);
  if (rc != GP_OK) fail(rc, "%s", g_msg);
  rc = gpo_compress_pack(d, support, NULL, r, g, cfg, out, len);
  if (rc != GP_OK) fail(rc, "%s", g_msg);
  API_END;
}

int gpo_decode(const uint8_t* bytes, size_t len, uint64_t* d, uint32_t** support, double** values,
               uint64_t* n) {
  API_BEGIN;
  container_t c;
  unpack(bytes, len, &c);
  sparse_t sg;
  memset(&sg, 0, sizeof sg);
  decompress(&c, &sg);
  *d = sg.d;
  *n = sg.count;
  *support = (uint32_t*)detach(sg.support, sg.count * 4);
  *values = (double*)detach(sg.values, sg.count * 8);
  API_END;
}

int gpo_decode_accumulate(const uint8_t* bytes, size_t len, double* dense, uint64_t d, double scale) {
  API_BEGIN;
  container_t c;
  unpack(bytes, len, &c);
  sparse_t sg;
  memset(&sg, 0, sizeof sg);
  decompress(&c, &sg);
  if (sg.d != d) fail(GP_ERROR, "decode_accumulate: dimension mismatch");
  for (uint64_t i = 0; i < sg.count; ++i) dense[sg.support[i]] += scale * sg.values[i];
  API_END;
}

static void fit_shape(const uint8_t* p, size_t n, uint64_t* ncoeff, uint64_t* last) { /* container.cpp:131-145 */
  breader_t r = {p, n, 0};
  const uint8_t kind = (uint8_t)get_le(&r, 1);
  if (kind > 1) fail(GP_UNKNOWN_METHOD, "fit: unknown model kind");
  const uint16_t segs = (uint16_t)get_le(&r, 2);
  if (segs < 1) fail(GP_CORRUPT_PAYLOAD, "fit: zero segments");
  uint32_t l = 0;
  for (uint16_t i = 0; i < segs; ++i) l = (uint32_t)get_le(&r, 4);
  const uint8_t degree = (uint8_t)get_le(&r, 1);
  *ncoeff = (uint64_t)segs * (kind == 1 ? 4u : degree + 1u);
  *last = l;
}

int gpo_volume(const uint8_t* bytes, size_t len, gpo_volume_report* v) { /* container.cpp:148-243 */
  API_BEGIN;
  container_t c;
  unpack(bytes, len, &c);
  memset(v, 0, sizeof *v);
  const uint64_t header = 4 + 2 + 1 + 1 + 1 + 8 + 8 + 8 + 8 + 8;
  v->total_bits = 8 * (header + c.il + c.vl + c.rl + 4);
  switch (c.index_method) {
    case GP_INDEX_NONE:
      if (c.il != 4 * c.r) fail(GP_CORRUPT_PAYLOAD, "container: raw key payload length mismatch");
      v->index_bits = 32 * c.r;
      break;
    case GP_INDEX_BITMAP:
      if (c.il != (c.d + 7) / 8) fail(GP_CORRUPT_PAYLOAD, "container: bitmap payload length mismatch");
      v->index_bits = c.d;
      break;
    case GP_INDEX_RLE:
      if (c.il == 0) fail(GP_CORRUPT_PAYLOAD, "container: empty rle payload");
      v->index_bits = 8 * c.il - 7;
      break;
    case GP_INDEX_HUFFMAN: { /* container.cpp:171-178: bits of the 4r decoded codes */
      huff_t h;
      huff_build(c.d, &h);
      uint64_t used = 0;
      huff_decode_indices(&h, c.ip, c.il, c.r, c.d, &used);
      v->index_bits = used;
      break;
    }
    default: {
      breader_t r = {c.ip, c.il, 0};
      v->index_bits = get_le(&r, 8);
      break;
    }
  }
  uint64_t value_count = c.r;
  switch (c.value_method) {
    case GP_VALUE_NONE:
      if (c.vl % 4 != 0) fail(GP_CORRUPT_PAYLOAD, "container: raw f32 payload length mismatch");
      value_count = c.vl / 4;
      v->value_bits = 8 * c.vl;
      break;
    case GP_VALUE_RAW_F64:
      if (c.vl % 8 != 0) fail(GP_CORRUPT_PAYLOAD, "container: raw f64 payload length mismatch");
      value_count = c.vl / 8;
      v->value_bits = 8 * c.vl;
      break;
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP: {
      uint64_t ncoeff, cnt;
      fit_shape(c.vp, c.vl, &ncoeff, &cnt);
      value_count = cnt;
      v->value_bits = 32 * ncoeff;
      break;
    }
    case GP_VALUE_DEFLATE_SLOT:
      if (c.vl < 9) fail(GP_CORRUPT_PAYLOAD, "container: deflate slot payload too short");
      v->value_bits = 8 * (c.vl - 9);
      break;
    case GP_VALUE_QUANT: { /* container.cpp:213-225 */
      if (c.index_method == GP_INDEX_BLOOM_P0) {
        breader_t br = {c.ip, c.il, 0};
        bloom_t f;
        bloom_deserialize(&br, &f);
        uint64_t np = 0;
        positive_scan(&f, c.d, &np);  /* arena allocations, released on return */
        value_count = np;
      }
      breader_t r = {c.vp, c.vl, 0};
      const unsigned bits = (unsigned)get_le(&r, 1);
      const uint32_t bucket = (uint32_t)get_le(&r, 4);
      if (bits < 1 || bucket < 1) fail(GP_CORRUPT_PAYLOAD, "container: bad quant header");
      const uint64_t nb = (value_count + bucket - 1) / bucket;
      v->value_bits = 32 * nb + (uint64_t)bits * value_count;
      break;
    }
    default:
      fail(GP_UNSUPPORTED, "oracle: value method %d is out of scope", c.value_method);
  }
  if (c.rl) {
    const unsigned width = reorder_entry_bits(c.d);
    v->reorder_bits = value_count * width;
    if (c.rl != (v->reorder_bits + 7) / 8) fail(GP_CORRUPT_PAYLOAD, "container: reorder payload length mismatch");
  }
  v->metadata_bits = v->total_bits - v->index_bits - v->value_bits - v->reorder_bits;
  if (c.d > 0) v->ratio_dense = (double)v->total_bits / (32.0 * (double)c.d);
  if (c.r > 0) v->ratio_sparse = (double)v->total_bits / (64.0 * (double)c.r);
  API_END;
}
