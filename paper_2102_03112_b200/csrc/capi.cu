// capi.cu — the C-ABI (include/gradpack_b200.h): context, workspace, and the
// host orchestration of encode (top_r → compress_gradient → pack) and decode
// (unpack → decompress_gradient → to_dense accumulate).
//
// The host side only enqueues.  Method dispatch is decided on the host from
// the config (encode) or from the container header (decode: either a caller
// hint that the device verifies after the CRC, or a synchronous 75-byte
// header peek when no hint is given).  No CPU fallback exists: if the CUDA
// device or this library is unavailable, every entry point fails.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>

#include "gp_ctx.hpp"
#include "huffman.cuh"
#include "gp_device.cuh"

namespace gp {

int set_error(gp_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

int check_launch(gp_ctx* ctx, const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ctx, GP_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GP_OK;
}

void stage_begin(gp_ctx* ctx, int stage, cudaStream_t s) {
  Profiler& p = ctx->prof;
  if (!p.on || p.next + 2 > p.pool.size()) return;
  p.open_stage = stage;
  p.open_event = p.next;
  cudaEventRecord(p.pool[p.next++], s);
}

void stage_end(gp_ctx* ctx, cudaStream_t s) {
  Profiler& p = ctx->prof;
  if (!p.on || p.open_stage < 0) return;
  cudaEventRecord(p.pool[p.next++], s);
  p.stage.push_back(p.open_stage);
  p.first.push_back(p.open_event);
  p.open_stage = -1;
}

bool g_pdl = !getenv("GP_PDL") || atoi(getenv("GP_PDL")) != 0;

namespace {
__global__ void fill_bytes(uint8_t* p, uint32_t word, uint64_t bytes) {
  gp_pdl_wait();
  const uint64_t head = (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15;
  const uint64_t h = head < bytes ? head : bytes;
  const uint64_t n16 = (bytes - h) / 16;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint4* q = reinterpret_cast<uint4*>(p + h);
  for (uint64_t i = tid; i < n16; i += stride) q[i] = make_uint4(word, word, word, word);
  if (tid < h) p[tid] = static_cast<uint8_t>(word);
  const uint64_t tail = h + 16 * n16;
  if (tid < bytes - tail) p[tail + tid] = static_cast<uint8_t>(word);
}
}  // namespace

void fill_async(gp_ctx* ctx, void* p, int value, size_t bytes, cudaStream_t s) {
  static const bool kern = !getenv("GP_FILL_KERNEL") || atoi(getenv("GP_FILL_KERNEL")) != 0;
  if (!kern) {
    cudaMemsetAsync(p, value, bytes, s);
    return;
  }
  if (bytes == 0) return;
  const uint32_t b = static_cast<uint32_t>(value) & 0xFFu;
  GP_LAUNCH(ctx, fill_bytes, grid_for(ctx, (bytes + 15) / 16, 256), 256, 0, s, static_cast<uint8_t*>(p),
            b * 0x01010101u, static_cast<uint64_t>(bytes));
}

void reset_scan(gp_ctx* ctx, cudaStream_t s, uint64_t ntiles_bound) {
  Workspace& w = ctx->ws;
  const uint64_t n = ntiles_bound < w.tiles_cap ? ntiles_bound : w.tiles_cap;
  fill_async(ctx, w.scan_base, 0, 128 + n * 8, s);
}

namespace {

bool is_bloom(int m) { return m >= GP_INDEX_BLOOM_P0 && m <= GP_INDEX_BLOOM_NAIVE; }

// Methods with a device implementation on this path (the rest of FORMAT.md's
// registry returns GP_UNSUPPORTED).
bool index_supported(int m) {
  return m == GP_INDEX_NONE || m == GP_INDEX_BITMAP || m == GP_INDEX_RLE || m == GP_INDEX_HUFFMAN ||
         m == GP_INDEX_BLOOM_P0 ||
         m == GP_INDEX_BLOOM_P1 ||
         m == GP_INDEX_BLOOM_P2 ||
         m == GP_INDEX_BLOOM_PD || m == GP_INDEX_BLOOM_NAIVE;
}
bool value_supported(int m) {
  return m == GP_VALUE_NONE || m == GP_VALUE_RAW_F64 || m == GP_VALUE_FIT_POLY || m == GP_VALUE_FIT_DEXP ||
         m == GP_VALUE_QUANT || m == GP_VALUE_DEFLATE_SLOT;
}

struct PlanInit {
  uint64_t d, r, il, n_values;
  uint64_t m, seed_a, seed_b, minv;
  uint64_t seed;
  const uint64_t* seed_dev;  // non-null: the pipeline seed is read here at execution time
  uint32_t k;
  uint8_t index_method, value_method, pd_variant;
};

__global__ void init_plan(Plan* plan, PlanInit p) {
  gp_pdl_wait();
  plan->d = p.d;
  plan->r = p.r;
  plan->index_method = p.index_method;
  plan->value_method = p.value_method;
  plan->pd_variant = p.pd_variant;
  plan->flags = 0;
  plan->il = p.il;
  plan->vl = 0;
  plan->rl = 0;
  plan->n_values = p.n_values;
  plan->n_sel = p.r;
  plan->off_index = 49;
  plan->off_value = 49 + p.il;
  plan->off_reorder = 49 + p.il;
  plan->m = p.m;
  plan->k = p.k;
  // derive_filter_seed_a/b (pipeline.cpp:21-22) from the pipeline seed, on
  // the device so a captured graph can replay with a new seed per step
  const uint64_t seed = p.seed_dev ? *p.seed_dev : p.seed;
  plan->seed = seed;
  plan->seed_a = hash64(0xA, seed);
  plan->seed_b = hash64(0xB, seed);
  plan->minv = p.minv;
  plan->scan_lo = 0;  // full-range positive scans unless gp_bloom_scan_range narrows it
  plan->scan_hi = 0;
  // the value codec's accumulators and flags (values_fit.cu)
  plan->sign_split = 0;
  plan->identity = 1;
  plan->fit_kind = 0;
  plan->dexp_fail = 0;
}

// Simulation::pipeline_seed(seed, worker, *step) (harness.cpp:201-203, over
// Problem::batch_seed :47-51) into seed_out[0], on the device; with buckets,
// seed_out[b] = hash64(b, that seed) (the bucketed convention of dp.py).
__global__ void pipeline_seed_kernel(uint64_t* seed_out, const uint64_t* step, uint64_t seed, uint32_t worker,
                                     uint32_t buckets) {
  gp_pdl_wait();
  const uint64_t key = (static_cast<uint64_t>(worker) << 32) | (*step & 0xFFFFFFFFULL);
  const uint64_t ps = hash64(0xC0DEC, hash64(key, hash64(0xDA7A, seed)));
  if (buckets == 0) {
    if (threadIdx.x == 0) *seed_out = ps;
    return;
  }
  for (uint32_t b = threadIdx.x; b < buckets; b += blockDim.x) seed_out[b] = hash64(b, ps);
}

// compress_gradient's validate(sg) (gradient.cpp:19-30) + gather(dense, support)
__global__ void take_support(const float* __restrict__ dense, const uint32_t* __restrict__ support, uint64_t r,
                             uint64_t d, uint32_t* ws_support, float* ws_values, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = support[i];
    if (static_cast<uint64_t>(s) >= d || (i > 0 && s <= support[i - 1])) {
      latch(status, GP_ERROR);
      return;
    }
    ws_support[i] = s;
    if (dense) ws_values[i] = dense[s];
  }
}

// component calls: the filter payload starts at offset 0 of the caller's buffer
__global__ void component_offsets(Plan* plan) {
  gp_pdl_wait();
  plan->off_index = 0;
  plan->off_value = plan->il;
  plan->off_reorder = plan->il;
}

// P (ascending positives) to the caller, |P| to *count; GP_CAPACITY past cap
__global__ void copy_positions(const uint32_t* __restrict__ pos, const Plan* plan, uint32_t* __restrict__ out,
                               uint64_t cap, uint64_t* count, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = plan->n_pos;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *count = n;
    if (n > cap) latch(status, GP_CAPACITY);
  }
  if (n > cap) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = pos[i];
}

// ---------------------------------------------------------------- workspace
struct Carver {
  uint8_t* base;
  size_t off;
  template <typename T>
  T* take(uint64_t n) {
    off = (off + 255) & ~static_cast<size_t>(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += n * sizeof(T);
    return p;
  }
};

void carve(Workspace& w, uint8_t* base, uint64_t D) {
  Carver c{base, 0};
  w.plan = c.take<Plan>(1);
  w.status = c.take<uint32_t>(64);
  w.status_pre = c.take<uint32_t>(64);
  w.tiles_cap = 4 * (D / 1024) + 4096;
  w.scan_base = c.take<uint8_t>(128 + w.tiles_cap * 8);
  w.ticket = reinterpret_cast<uint32_t*>(w.scan_base);
  w.tiles = reinterpret_cast<uint64_t*>(w.scan_base ? w.scan_base + 128 : nullptr);
  w.hist = c.take<uint32_t>(32768 + 256 + 65536 + 256);
  w.cand_idx = c.take<uint32_t>(D);
  w.cand_val = c.take<float>(D);
  w.support = c.take<uint32_t>(D);
  w.values = c.take<float>(D);
  w.m_cap = 48 * D + 4096;
  w.filter = c.take<uint32_t>(w.m_cap / 32 + 1);
  w.pos = c.take<uint32_t>(D);
  w.sel = c.take<uint32_t>(D);
  w.flags = c.take<uint8_t>(D);
  w.selbits = c.take<uint32_t>(D / 32 + 1);
  w.set_cap = 2 * D;
  w.pair_cap = 4 * D;
  w.p2_count = c.take<uint32_t>(w.set_cap + 1);
  w.p2_off = c.take<uint32_t>(w.set_cap + 1);
  w.p2_alloc = c.take<uint32_t>(64);
  w.p2_sets = c.take<uint32_t>(w.set_cap);
  w.p2_table = c.take<uint32_t>(256 * (w.set_cap / 4096 + 1) + 256);
  w.pairs = c.take<uint32_t>(w.pair_cap);
  w.p2_rank = c.take<uint32_t>(w.pair_cap);
  w.p2_members = c.take<uint32_t>(w.pair_cap);
  w.first_touch = c.take<uint32_t>(D);
  w.u32a = c.take<uint32_t>(D);
  w.u32b = c.take<uint32_t>(D);
  w.u32c = c.take<uint32_t>(D);
  w.u32d = c.take<uint32_t>(D);
  w.f64a = c.take<double>(D);
  w.f64b = c.take<double>(D);
  w.seg_cap = std::min<uint64_t>(2 * kFitMaxSeg, D) + 2;
  w.node_cap = static_cast<uint32_t>(std::min<uint64_t>(4 * (kFitMaxSeg + 1), 2 * D) + 64);
  w.partial = c.take<double>((D / 2048 + w.seg_cap + 2) * 44);
  w.sort_table = c.take<uint32_t>(2 * 256 * (D / kSortTileKeys + 2));  // per-tile digit aggregates + inclusive prefixes
  w.sort_flags = c.take<uint32_t>(64 + D / kSortTileKeys + 2);        // 8 tickets, 1024 histogram bins follow below
  w.sort_hist = c.take<uint32_t>(4 * 256);
  w.seg_dev = c.take<double>(4 * 2048);
  w.seg_arg = c.take<uint32_t>(4 * 2048);
  w.seg_end = c.take<uint32_t>(w.seg_cap);
  w.coeffs = c.take<float>(w.seg_cap * kFitMaxCps);
  w.seg_nodes = c.take<uint8_t>(32ull * w.node_cap);
  w.seg_heap = c.take<uint32_t>(w.node_cap);
  w.seg_pend = c.take<uint32_t>(w.node_cap);
  w.seg_off = c.take<uint64_t>(w.node_cap + 1);
  w.seg_state = c.take<uint32_t>(8);
  w.seg_chunk = c.take<uint64_t>(w.seg_cap + 1);
  w.fit_scratch = c.take<double>(static_cast<uint64_t>(kWideBlocks) * 3 * kFitMaxCps * kFitMaxCps);
  w.crc_cap = 2 * ((64 * D + (1 << 20)) / (64 * 256) + 64);
  w.crc_digits = c.take<uint32_t>(13 * 256 + kCrcSmallTabWords);  // 5 byte-digit shift tables + the full and small grids' lane-stride multiply tables + crc_tail's tables
  w.crc_acc = c.take<uint32_t>(64 + 256);  // [0] XOR accumulator, [1] block counter, [2] crc_tail ticket, [64, 320) crc_tail partials
  w.scratch = c.take<uint8_t>(2 * D);
  w.huff = c.take<HuffTable>(1);
  w.huff_res = c.take<uint64_t>(16);
  w.bytes_total = c.off;
}

}  // namespace
}  // namespace gp

using namespace gp;

extern "C" {

void gp_pipeline_config_default(gp_pipeline_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->index_method = GP_INDEX_NONE;
  cfg->value_method = GP_VALUE_NONE;
  cfg->pd_variant = 0;
  cfg->slot_codec = 1;
  cfg->degree = 5;
  cfg->max_segments = 0;
  cfg->quant_bits = 7;
  cfg->quant_bucket = 512;
  cfg->fpr = 0.01;
  cfg->seed = 0;
}

int gp_ctx_create(int device, uint64_t max_d, gp_ctx** out) {
  if (!out) return GP_ERROR;
  *out = nullptr;
  if (max_d < 1 || max_d > 0xFFFFFFFFULL) return GP_ERROR;
  auto* ctx = new (std::nothrow) gp_ctx();
  if (!ctx) return GP_ERROR;
  ctx->device = device;
  ctx->max_d = max_d;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) {  // kernel attributes are per device: set them for this one
    kernel_attrs_bloom();
    kernel_attrs_p2();
    kernel_attrs_topr();
    kernel_attrs_dense();
    kernel_attrs_topr64();
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    delete ctx;
    return GP_CUDA;
  }
  const uint64_t D = max_d < 4096 ? 4096 : max_d;
  carve(ctx->ws, nullptr, D);
  const size_t bytes = ctx->ws.bytes_total;
  void* base = nullptr;
  e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) {
    delete ctx;
    return GP_CUDA;
  }
  carve(ctx->ws, static_cast<uint8_t*>(base), D);
  ctx->ws.base = base;
  ctx->ws.bytes = bytes;
  e = cudaMemset(ctx->ws.status, 0, 64 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(ctx->ws.plan, 0, sizeof(Plan));
  if (e == cudaSuccess) e = cudaMemset(ctx->ws.huff, 0, sizeof(HuffTable));  // empty Huffman table cache
  if (e == cudaSuccess) e = cudaMemset(ctx->ws.seg_state, 0, 8 * sizeof(uint32_t));  // fit segmentation control words
  if (e == cudaSuccess) e = cudaMemset(ctx->ws.status_pre, 0, 64 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess || crc_tables_init(ctx) != GP_OK) {
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    cudaFree(base);
    delete ctx;
    return GP_CUDA;
  }
  *out = ctx;
  return GP_OK;
}

void gp_ctx_destroy(gp_ctx* ctx) {
  if (!ctx) return;
  for (auto& e : ctx->prof.pool) cudaEventDestroy(e);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ws.base) cudaFree(ctx->ws.base);
  delete ctx;
}

int gp_ctx_set_index_event(gp_ctx* ctx, void* event) {
  if (!ctx) return GP_ERROR;
  ctx->index_event = static_cast<cudaEvent_t>(event);
  return GP_OK;
}

int gp_ctx_set_decode_overwrite(gp_ctx* ctx, int on) {
  if (!ctx) return GP_ERROR;
  ctx->decode_overwrite = on != 0;
  return GP_OK;
}

int gp_ctx_set_seed_source(gp_ctx* ctx, const uint64_t* d_seed) {
  if (!ctx) return GP_ERROR;
  ctx->seed_dev = d_seed;
  return GP_OK;
}

int gp_pipeline_seed_device(uint64_t* d_seed, const uint64_t* d_step, uint64_t seed, uint32_t worker,
                            uint32_t buckets, void* stream) {
  if (!d_seed || !d_step) return GP_ERROR;
  pipeline_seed_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_seed, d_step, seed, worker, buckets);
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_CUDA;
}

const char* gp_last_error(const gp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

uint64_t gp_ctx_launch_count(const gp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int gp_ctx_status(gp_ctx* ctx, void* stream) {
  if (!ctx) return GP_ERROR;
  auto s = static_cast<cudaStream_t>(stream);
  uint32_t st = 0;
  cudaError_t e = cudaMemcpyAsync(&st, ctx->ws.status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(ctx, GP_CUDA, std::string("status: ") + cudaGetErrorString(e));
  if (st != 0) {
    fill_async(ctx, ctx->ws.status, 0, sizeof(uint32_t), s);
    cudaStreamSynchronize(s);
    static const char* names[] = {"ok", "Error", "DecodeError", "TruncatedError", "ChecksumError",
                                  "UnknownMethodError", "CorruptPayloadError", "FitError", "CUDA",
                                  "unsupported method on the device path", "device capacity exceeded"};
    return set_error(ctx, static_cast<int>(st),
                     std::string("device: ") + (st < 11 ? names[st] : "unknown status"));
  }
  return GP_OK;
}

int gp_ctx_profile(gp_ctx* ctx, int on) {
  if (!ctx) return GP_ERROR;
  Profiler& p = ctx->prof;
  if (on && p.pool.empty()) {
    p.pool.resize(8192);
    for (auto& e : p.pool)
      if (cudaEventCreate(&e) != cudaSuccess) return set_error(ctx, GP_CUDA, "event pool");
  }
  p.on = on != 0;
  p.next = 0;
  p.stage.clear();
  p.first.clear();
  return GP_OK;
}

int gp_ctx_stage_times(gp_ctx* ctx, double* ms, uint64_t* counts, int n) {
  if (!ctx) return GP_ERROR;
  Profiler& p = ctx->prof;
  if (!p.stage.empty()) {
    if (cudaEventSynchronize(p.pool[p.next - 1]) != cudaSuccess) return set_error(ctx, GP_CUDA, "event sync");
    for (size_t i = 0; i < p.stage.size(); ++i) {
      float t = 0.0f;
      cudaEventElapsedTime(&t, p.pool[p.first[i]], p.pool[p.first[i] + 1]);
      if (p.stage[i] < n) {
        if (ms) ms[p.stage[i]] += t;
        if (counts) counts[p.stage[i]] += 1;
      }
    }
  }
  p.next = 0;
  p.stage.clear();
  p.first.clear();
  return GP_OK;
}

const char* gp_stage_name(int stage) {
  static const char* names[] = {"topr", "index", "bloom_build", "bloom_scan", "p2_sets", "p2_engine", "select",
                                "gather", "values", "pack_crc", "dec_parse_crc", "dec_index", "dec_bloom_scan",
                                "dec_p2_sets", "dec_p2_engine", "dec_select", "dec_values", "dec_scatter"};
  return stage >= 0 && stage < ST_COUNT ? names[stage] : "";
}

int gp_bloom_params(double epsilon, uint64_t r, uint64_t* m, uint32_t* k) {
  // bloom.cpp:22-31; evaluated on the host exactly as the reference does
  if (!(epsilon > 0.0 && epsilon < 1.0) || r < 1) return GP_ERROR;
  const double ln2 = 0.693147180559945309417232121458176568;
  const double lninv = std::log(1.0 / epsilon);
  if (m) *m = static_cast<uint64_t>(std::ceil(static_cast<double>(r) * lninv / (ln2 * ln2)));
  if (k) *k = static_cast<uint32_t>(std::ceil(lninv / ln2));
  return GP_OK;
}

uint64_t gp_max_container_bytes(uint64_t d, uint64_t r, const gp_pipeline_config* cfg) {
  if (!cfg) return 0;
  uint64_t il = 0, n = r;
  switch (cfg->index_method) {
    case GP_INDEX_NONE: il = 4 * r; break;
    case GP_INDEX_BITMAP: il = (d + 7) / 8; break;
    case GP_INDEX_RLE: il = d + 2; break;  // <= one group per coordinate, + the polarity byte
    case GP_INDEX_HUFFMAN: il = huffman_il_bound(d, r) + 8; break;  // 4 codes of <= max_len bits per key
    default: {
      uint64_t m = 0;
      uint32_t k = 0;
      gp_bloom_params(cfg->fpr, r < 1 ? 1 : r, &m, &k);
      il = 26 + (m + 7) / 8 + 1;
      if (cfg->index_method == GP_INDEX_BLOOM_P0) n = d;
    }
  }
  uint64_t vl = 0, rl = 0;
  switch (cfg->value_method) {
    case GP_VALUE_RAW_F64: vl = 8 * n; break;
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP: {
      const uint64_t segs = std::min<uint64_t>(kFitMaxSeg, n < 1 ? 1 : n);
      vl = 1 + 2 + 4 * segs + 1 + 4 * segs * (static_cast<uint64_t>(cfg->degree) + 1) + 4;
      uint64_t w = 0;
      for (uint64_t x = d - 1; x; x >>= 1) ++w;
      rl = (n * w + 7) / 8;
      break;
    }
    case GP_VALUE_QUANT: {
      const uint64_t bits = cfg->quant_bits < 1 ? 1 : (cfg->quant_bits > 16 ? 16 : cfg->quant_bits);
      const uint64_t bucket = cfg->quant_bucket < 1 ? 1 : cfg->quant_bucket;
      vl = 5 + 4 * ((n + bucket - 1) / bucket) + (n * bits + 7) / 8;
      break;
    }
    case GP_VALUE_DEFLATE_SLOT: vl = cfg->slot_codec == 1 ? deflate_slot_bound(n) : 9 + 4 * n; break;
    default: vl = 4 * n; break;
  }
  return 49 + il + vl + rl + 4;
}

static int encode_common(gp_ctx* ctx, const float* d_dense, uint64_t d, const uint32_t* d_support, uint64_t r,
                         const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap, uint64_t* d_len,
                         void* stream, float* ef_residual = nullptr, const double* d_values64 = nullptr,
                         const double* d_dense64 = nullptr, double* ef_residual64 = nullptr) {
  // f64 value sequences: compress_gradient's Vector values (gp_encode_sparse)
  // or the f64 error-feedback input (gp_encode_topr_ef64)
  const bool f64 = d_values64 || ef_residual64;
  if (!ctx || !cfg || !d_out || (!d_dense && !f64) || (ef_residual64 && !d_dense))
    return set_error(ctx, GP_ERROR, "encode: null argument");
  ctx->vals64 = nullptr;  // per-encode launch inputs (set below, cleared at the end): never stale
  ctx->gather_dense = nullptr;
  auto s = static_cast<cudaStream_t>(stream);
  if (d < 1) return set_error(ctx, GP_ERROR, "sparsifier: dim must be >= 1");
  if (d > 0xFFFFFFFFULL) return set_error(ctx, GP_ERROR, "sparsifier: dim exceeds 32-bit index space");
  if (d_values64 && r == 0) {  // compress_gradient of an empty support (pipeline.cpp:152-154, :215-218)
    if (cfg->index_method != GP_INDEX_NONE)
      return set_error(ctx, GP_ERROR, "pipeline: empty support requires the raw index method");
    if (cfg->value_method == GP_VALUE_FIT_POLY || cfg->value_method == GP_VALUE_FIT_DEXP ||
        cfg->value_method == GP_VALUE_QUANT)
      return set_error(ctx, GP_ERROR, "pipeline: fit/quant value methods need a nonempty value sequence");
  } else if (r < 1 || r > d) {
    return set_error(ctx, GP_ERROR, "sparsifier: r out of range [1, d]");
  }
  if (d > ctx->max_d) return set_error(ctx, GP_CAPACITY, "encode: d exceeds the context's max_d");
  const int im = cfg->index_method, vm = cfg->value_method;
  if (im > GP_INDEX_BLOOM_NAIVE || vm > GP_VALUE_RAW_F64)
    return set_error(ctx, GP_ERROR, "container: unregistered method");
  if (!index_supported(im) || !value_supported(vm))
    return set_error(ctx, GP_UNSUPPORTED, "method not implemented on the device path");
  if (vm == GP_VALUE_FIT_POLY || vm == GP_VALUE_FIT_DEXP) {
    if (cfg->degree < 0 || cfg->degree > 60) return set_error(ctx, GP_ERROR, "value_compress: bad degree");
  }
  if (vm == GP_VALUE_QUANT) {
    if (cfg->quant_bits < 1 || cfg->quant_bits > 16) return set_error(ctx, GP_ERROR, "quantize: bits out of range [1, 16]");
    if (cfg->quant_bucket < 1) return set_error(ctx, GP_ERROR, "quantize: bucket must be >= 1");
  }
  if (vm == GP_VALUE_DEFLATE_SLOT && cfg->slot_codec > 1)
    return set_error(ctx, GP_UNKNOWN_METHOD, "byte_compress: unknown codec id");
  const uint64_t bound = gp_max_container_bytes(d, r, cfg);
  if (cap < bound) return set_error(ctx, GP_CAPACITY, "encode: output capacity below gp_max_container_bytes");

  PlanInit pi{};
  pi.d = d;
  pi.r = r;
  pi.index_method = static_cast<uint8_t>(im);
  pi.value_method = static_cast<uint8_t>(vm);
  pi.pd_variant = cfg->pd_variant;
  pi.n_values = r;
  if (is_bloom(im)) {
    uint64_t m = 0;
    uint32_t k = 0;
    if (gp_bloom_params(cfg->fpr, r, &m, &k) != GP_OK)
      return set_error(ctx, GP_ERROR, "bloom_params: epsilon must be in (0, 1)");
    if (m >= (1ULL << 32) || m > ctx->ws.m_cap || k > 0xFFFF)
      return set_error(ctx, GP_CAPACITY, "bloom filter exceeds the context's filter capacity");
    if (im == GP_INDEX_BLOOM_PD && cfg->pd_variant > 2) return set_error(ctx, GP_ERROR, "pd_select: unknown variant");
    pi.m = m;
    pi.k = k;
    pi.minv = ~0ULL / m;
    pi.il = 26 + (m + 7) / 8 + (im == GP_INDEX_BLOOM_PD ? 1 : 0);
  } else {
    pi.il = im == GP_INDEX_NONE ? 4 * r : im == GP_INDEX_HUFFMAN ? 0 : (d + 7) / 8;  // Huffman: set on the device
  }
  pi.seed = cfg->seed;
  pi.seed_dev = ctx->seed_dev;
  GP_LAUNCH(ctx, init_plan, 1, 1, 0, s, ctx->ws.plan, pi);

  // dense-selection fast path (dense.cu): one pass writes bitmap + raw values
  // when top_r(g, r) is the nonzero set; the general kernels below then run
  // against the gate word and return at once (or run, when r != nnz)
  const bool nz = !d_support && !ef_residual && !f64 && nz_fast_path_eligible(d, r, im, vm);
  uint32_t* const real_status = ctx->ws.status;
  if (nz) {
    GP_STAGE(ctx, ST_INDEX, s, launch_nz_encode(ctx, d_dense, d, r, d_out, s));
    ctx->ws.status = gate_word(ctx);
  }
  const double* dense64 = d_dense64;
  if (d_support) {
    GP_LAUNCH(ctx, take_support, grid_for(ctx, r, 256), 256, 0, s, f64 ? nullptr : d_dense, d_support, r, d,
              ctx->ws.support, ctx->ws.values, ctx->ws.status);
    ctx->vals64 = d_values64;  // sg.values in support order (a Bloom gather below replaces them)
  } else if (ef_residual64) {
    GP_STAGE(ctx, ST_TOPR, s, launch_top_r64(ctx, d_dense, ef_residual64, d, r, s));
    dense64 = ef_residual64;  // the input g + e, written by top-r's first pass
    ctx->vals64 = ctx->ws.f64a;
  } else {
    GP_STAGE(ctx, ST_TOPR, s, launch_top_r(ctx, d_dense, d, r, s, ef_residual));
    if (ef_residual) d_dense = ef_residual;  // the input g + e, written by top-r's first pass
  }
  switch (im) {
    case GP_INDEX_NONE: launch_index_none(ctx, d_out, r, s); break;
    case GP_INDEX_BITMAP: launch_index_bitmap(ctx, d_out, d, r, s); break;
    case GP_INDEX_RLE: GP_STAGE(ctx, ST_INDEX, s, launch_index_rle(ctx, d_out, d, r, s)); break;
    case GP_INDEX_HUFFMAN:
      GP_STAGE(ctx, ST_INDEX, s, launch_index_huffman(ctx, d_out, r, huffman_il_bound(d, r) + 8, s));
      break;
    default: {
      GP_STAGE(ctx, ST_BLOOM_BUILD, s, launch_bloom_build(ctx, d_out, pi.m, r, s));
      if (ctx->index_event) cudaEventRecord(ctx->index_event, s);  // the filter payload is final
      if (im == GP_INDEX_BLOOM_NAIVE) break;  // values stay in support order (pipeline.cpp:196-199)
      GP_STAGE(ctx, ST_BLOOM_SCAN, s, launch_bloom_scan(ctx, d, pi.m, false, s));
      if (im == GP_INDEX_BLOOM_P2)
        launch_select_p2(ctx, d, pi.m, pi.k, false, s, r + static_cast<uint64_t>(cfg->fpr * static_cast<double>(d)));
      else if (im == GP_INDEX_BLOOM_P1)
        GP_STAGE(ctx, ST_SELECT, s, launch_select_p1(ctx, d, r, s));
      else
        GP_STAGE(ctx, ST_SELECT, s, launch_select_slice(ctx, d, s));
      if (f64) {
        GP_STAGE(ctx, ST_GATHER, s, launch_gather_values64(ctx, dense64, d_support, d_values64, r, d, s));
        ctx->vals64 = ctx->ws.f64a;
      } else if (vm == GP_VALUE_FIT_POLY || vm == GP_VALUE_FIT_DEXP) {
        ctx->gather_dense = d_dense;  // the fit's key kernel gathers v[j] = dense[sel[j]] itself
      } else {
        GP_STAGE(ctx, ST_GATHER, s, launch_gather_values(ctx, d_dense, d, s));
      }
    }
  }
  const uint64_t n_bound = im == GP_INDEX_BLOOM_P0 ? d : r;
  switch (vm) {
    case GP_VALUE_NONE:
    case GP_VALUE_RAW_F64: launch_values_raw(ctx, d_out, vm == GP_VALUE_RAW_F64, n_bound, s); break;
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP:
      GP_STAGE(ctx, ST_VALUES, s, launch_values_fit(ctx, d_out, cfg->degree, cfg->max_segments, n_bound, s,
                                                    vm == GP_VALUE_FIT_DEXP));
      break;
    case GP_VALUE_QUANT:  // derive_quant_seed (pipeline.cpp:26)
      GP_STAGE(ctx, ST_VALUES, s,
               launch_values_quant(ctx, d_out, cfg->quant_bits, cfg->quant_bucket, n_bound, s));
      break;
    case GP_VALUE_DEFLATE_SLOT:
      if (cfg->slot_codec == 1)
        GP_STAGE(ctx, ST_VALUES, s, launch_values_deflate(ctx, d_out, n_bound, s));
      else
        launch_values_slot(ctx, d_out, n_bound, s);
      break;
    default: break;
  }
  if (nz) {
    ctx->ws.status = real_status;
    launch_gate_merge(ctx, s);
  }
  GP_STAGE(ctx, ST_PACK, s, launch_finish_container(ctx, d_out, cap, d_len, bound, s));
  ctx->vals64 = nullptr;  // captured by the launches above
  ctx->gather_dense = nullptr;
  return check_launch(ctx, "encode");
}

int gp_encode_topr(gp_ctx* ctx, const float* d_grad, uint64_t d, uint64_t r, const gp_pipeline_config* cfg,
                   uint8_t* d_out, uint64_t cap, uint64_t* d_len, void* stream) {
  return encode_common(ctx, d_grad, d, nullptr, r, cfg, d_out, cap, d_len, stream);
}

int gp_encode_support(gp_ctx* ctx, const float* d_dense, uint64_t d, const uint32_t* d_support, uint64_t r,
                      const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap, uint64_t* d_len,
                      void* stream) {
  if (!d_support) return set_error(ctx, GP_ERROR, "encode_support: null support");
  return encode_common(ctx, d_dense, d, d_support, r, cfg, d_out, cap, d_len, stream);
}

// own: the container this context just encoded (error feedback).  The index
// stage is skipped where the encoder's state already holds the decoded
// support — the selection in ws.sel for Bloom P0/P1/P2/Pd, the top-r support
// for none/bitmap/RLE (copied to ws.sel) — since decoding the index payload
// reproduces exactly that set; Bloom-naive (whose decoded support is all of P,
// never computed by the encoder) takes the full decode.
static int decode_common(gp_ctx* ctx, const uint8_t* d_in, uint64_t len, const uint64_t* d_len,
                         const gp_pipeline_config* hint,
                         float* d_dense, uint64_t dense_d, float scale, uint32_t* d_support, double* d_values,
                         uint64_t cap, uint64_t* d_count, uint64_t* d_dim, void* stream, bool own = false,
                         bool scatter = true, double* d_dense64 = nullptr) {
  if (!ctx || !d_in) return set_error(ctx, GP_ERROR, "decode: null argument");
  auto s = static_cast<cudaStream_t>(stream);
  gp_pipeline_config h{};
  if (hint) {
    h = *hint;
  } else {
    // synchronous header peek: method ids drive the host-side dispatch
    uint8_t hdr[8] = {0};
    const uint64_t n = len < 8 ? len : 8;
    if (n) {
      cudaError_t e = cudaMemcpyAsync(hdr, d_in, n, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return set_error(ctx, GP_CUDA, std::string("decode peek: ") + cudaGetErrorString(e));
    }
    h.index_method = hdr[6];
    h.value_method = hdr[7];
  }
  // parse, then the CRC verdict; the decode work that does not touch the
  // caller's output (index and value decoders, into workspace buffers) runs
  // on the context's side stream concurrently with the CRC, its errors held
  // in a second status word and merged after the verdict in stream order
  // (container.cu parse_container / merge_status), so error precedence is
  // the reference's: header, checksum, post-CRC checks, method decoders
  GP_STAGE(ctx, ST_DEC_PARSE, s, launch_parse_container(ctx, d_in, len, d_len, hint ? &h : nullptr, s);
           cudaEventRecord(ctx->ev_fork, s); launch_verify_crc(ctx, d_in, len, s));
  cudaStream_t ps = ctx->side;
  cudaStreamWaitEvent(ps, ctx->ev_fork, 0);
  auto join = [&]() {
    cudaEventRecord(ctx->ev_join, ps);
    cudaStreamWaitEvent(s, ctx->ev_join, 0);
  };
  const int im = h.index_method, vm = h.value_method;
  const bool known = im <= GP_INDEX_BLOOM_NAIVE && vm <= GP_VALUE_RAW_F64;
  if (known && (!index_supported(im) || !value_supported(vm))) {
    join();
    // surface header/CRC errors first, then report the unsupported method
    const int st = gp_ctx_status(ctx, stream);
    if (st != GP_OK) return st;
    return set_error(ctx, GP_UNSUPPORTED, "method not implemented on the device path");
  }
  if (!known) {  // the CRC verdict step latches UnknownMethod
    join();
    return check_launch(ctx, "decode");
  }
  const uint64_t bound = ctx->max_d;
  // bitmap + raw values into a dense buffer (or a prepare for one): the fused
  // dense path (dense.cu) — per-tile counts and checks now, one scatter pass
  // reading bitmap words and value runs, no materialised support
  const bool fused = im == GP_INDEX_BITMAP && (vm == GP_VALUE_NONE || vm == GP_VALUE_RAW_F64) && !own &&
                     !d_support && !d_dense64 && (d_dense || !scatter);
  Workspace& w = ctx->ws;
  uint32_t* const main_status = w.status;
  w.status = w.status_pre;  // every pre-verdict launch latches into the second word
  if (own && im != GP_INDEX_BLOOM_NAIVE) {
    if (!is_bloom(im)) launch_own_support(ctx, bound, ps);
  } else switch (im) {
    case GP_INDEX_NONE: launch_decode_index_none(ctx, d_in, bound, ps); break;
    case GP_INDEX_BITMAP:
      if (fused) {
        GP_STAGE(ctx, ST_DEC_INDEX, ps, launch_decode_bitmap_check(ctx, d_in, ps); launch_bm_prepare(ctx, d_in, bound, ps));
      } else {
        launch_decode_index_bitmap(ctx, d_in, bound, ps);
      }
      break;
    case GP_INDEX_RLE: GP_STAGE(ctx, ST_DEC_INDEX, ps, launch_decode_index_rle(ctx, d_in, len, bound, ps)); break;
    case GP_INDEX_HUFFMAN: GP_STAGE(ctx, ST_DEC_INDEX, ps, launch_decode_index_huffman(ctx, d_in, len, ps)); break;
    default: {
      GP_STAGE(ctx, ST_DEC_BLOOM_SCAN, ps, launch_bloom_parse(ctx, d_in, ctx->ws.m_cap, ps);
                                           launch_bloom_scan(ctx, bound, 0, true, ps));
      if (im == GP_INDEX_BLOOM_P2)
        launch_select_p2(ctx, bound, ctx->ws.set_cap, 64, true, ps);
      else if (im == GP_INDEX_BLOOM_P1)
        GP_STAGE(ctx, ST_DEC_SELECT, ps, launch_select_p1(ctx, bound, bound, ps));
      else
        GP_STAGE(ctx, ST_DEC_SELECT, ps, launch_select_slice(ctx, bound, ps));
    }
  }
  switch (vm) {
    case GP_VALUE_NONE:
    case GP_VALUE_RAW_F64: launch_values_raw_check(ctx, ps); break;
    case GP_VALUE_FIT_POLY:
    case GP_VALUE_FIT_DEXP: GP_STAGE(ctx, ST_DEC_VALUES, ps, launch_decode_fit(ctx, d_in, bound, ps)); break;
    case GP_VALUE_QUANT: GP_STAGE(ctx, ST_DEC_VALUES, ps, launch_decode_quant(ctx, d_in, bound, ps)); break;
    case GP_VALUE_DEFLATE_SLOT:
      launch_decode_slot(ctx, d_in, ps);
      GP_STAGE(ctx, ST_DEC_VALUES, ps, launch_decode_inflate(ctx, d_in, bound, ps));
      break;
    default: break;
  }
  if ((im == GP_INDEX_NONE || im == GP_INDEX_HUFFMAN) && !own) launch_validate_support(ctx, bound, ps);
  w.status = main_status;
  join();
  launch_merge_status(ctx, s);
  if (scatter && fused) {
    GP_STAGE(ctx, ST_DEC_SCATTER, s,
             launch_bm_scatter(ctx, d_in, bound, d_dense, dense_d, scale, ctx->decode_overwrite, s));
    return check_launch(ctx, "decode");
  }
  if (scatter && d_dense && ctx->decode_overwrite) launch_dense_zero(ctx, d_dense, dense_d, s);
  if (scatter)
    GP_STAGE(ctx, ST_DEC_SCATTER, s,
             launch_decode_scatter(ctx, d_in, bound, d_dense, dense_d, scale, d_support, d_values, cap, d_count, d_dim, s,
                                   d_dense64));
  return check_launch(ctx, "decode");
}

int gp_decode_accumulate(gp_ctx* ctx, const uint8_t* d_container, uint64_t len, float* d_dense, uint64_t d,
                         float scale, void* stream) {
  return decode_common(ctx, d_container, len, nullptr, nullptr, d_dense, d, scale, nullptr, nullptr, 0, nullptr,
                       nullptr, stream);
}

int gp_decode_accumulate_dlen(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap, const uint64_t* d_len,
                              const gp_pipeline_config* hint, float* d_dense, uint64_t d, float scale, void* stream) {
  if (!hint || !d_len) return set_error(ctx, GP_ERROR, "decode_accumulate_dlen: needs a hint and a length word");
  return decode_common(ctx, d_container, cap, d_len, hint, d_dense, d, scale, nullptr, nullptr, 0, nullptr, nullptr,
                       stream);
}

int gp_decode_accumulate_hint(gp_ctx* ctx, const uint8_t* d_container, uint64_t len, const gp_pipeline_config* hint,
                              float* d_dense, uint64_t d, float scale, void* stream) {
  return decode_common(ctx, d_container, len, nullptr, hint, d_dense, d, scale, nullptr, nullptr, 0, nullptr,
                       nullptr, stream);
}

int gp_decode_prepare(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap, const uint64_t* d_len,
                      const gp_pipeline_config* hint, void* stream) {
  if (!hint) return set_error(ctx, GP_ERROR, "decode_prepare: needs a hint");
  return decode_common(ctx, d_container, cap, d_len, hint, nullptr, 0, 0.0f, nullptr, nullptr, 0, nullptr, nullptr,
                       stream, false, false);
}

int gp_decode_finish(gp_ctx* ctx, const uint8_t* d_container, float* d_dense, uint64_t d, float scale,
                     void* stream) {
  if (!ctx || !d_container || !d_dense) return set_error(ctx, GP_ERROR, "decode_finish: null argument");
  auto s = static_cast<cudaStream_t>(stream);
  // the prepare chose the path on the device: exactly one of the two scatters runs
  if (ctx->decode_overwrite) launch_dense_zero(ctx, d_dense, d, s);
  launch_bm_scatter(ctx, d_container, ctx->max_d, d_dense, d, scale, ctx->decode_overwrite, s);
  GP_STAGE(ctx, ST_DEC_SCATTER, s,
           launch_decode_scatter(ctx, d_container, ctx->max_d, d_dense, d, scale, nullptr, nullptr, 0, nullptr, nullptr,
                                 s));
  return check_launch(ctx, "decode_finish");
}

int gp_decode_sparse(gp_ctx* ctx, const uint8_t* d_container, uint64_t len, uint32_t* d_support, double* d_values,
                     uint64_t cap, uint64_t* d_count, uint64_t* d_dim, void* stream) {
  if (!d_support || !d_values) return set_error(ctx, GP_ERROR, "decode_sparse: null output");
  return decode_common(ctx, d_container, len, nullptr, nullptr, nullptr, 0, 0.0f, d_support, d_values, cap, d_count,
                       d_dim, stream);
}

int gp_encode_topr_ef(gp_ctx* ctx, const float* d_grad, float* d_residual, uint64_t d, uint64_t r,
                      const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap, uint64_t* d_len, void* stream) {
  if (!d_residual || !d_grad) return set_error(ctx, GP_ERROR, "encode_topr_ef: null argument");
  const int rc = encode_common(ctx, d_grad, d, nullptr, r, cfg, d_out, cap, d_len, stream, d_residual);
  if (rc != GP_OK) return rc;
  // residual <- input - decode(container)  (harness.cpp:269-271)
  return decode_common(ctx, d_out, cap, d_len, cfg, d_residual, d, -1.0f, nullptr, nullptr, 0, nullptr, nullptr,
                       stream, true);
}

int gp_encode_topr_ef64(gp_ctx* ctx, const float* d_grad, double* d_residual, uint64_t d, uint64_t r,
                        const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap, uint64_t* d_len, void* stream) {
  if (!d_residual || !d_grad) return set_error(ctx, GP_ERROR, "encode_topr_ef64: null argument");
  const int rc = encode_common(ctx, d_grad, d, nullptr, r, cfg, d_out, cap, d_len, stream, nullptr, nullptr, nullptr,
                               d_residual);
  if (rc != GP_OK) return rc;
  // residual <- input - to_dense(decode(container)), all f64 (harness.cpp:269-271)
  return decode_common(ctx, d_out, cap, d_len, cfg, nullptr, d, -1.0f, nullptr, nullptr, 0, nullptr, nullptr, stream,
                       true, true, d_residual);
}

int gp_encode_sparse(gp_ctx* ctx, uint64_t d, const uint32_t* d_support, const double* d_values, uint64_t r,
                     const double* d_dense, const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap,
                     uint64_t* d_len, void* stream) {
  if (r > 0 && (!d_support || !d_values)) return set_error(ctx, GP_ERROR, "encode_sparse: null support or values");
  // r = 0 (index None only): the kernels read no support or value; any
  // non-null pointer selects the caller-support path
  static const uint32_t kNoSupport = 0;
  static const double kNoValue = 0.0;
  return encode_common(ctx, nullptr, d, r ? d_support : &kNoSupport, r, cfg, d_out, cap, d_len, stream, nullptr,
                       r ? d_values : &kNoValue, d_dense);
}

int gp_top_r(gp_ctx* ctx, const float* d_grad, uint64_t d, uint64_t r, uint32_t* d_support, float* d_values,
             void* stream) {
  if (!ctx || !d_grad || !d_support) return set_error(ctx, GP_ERROR, "top_r: null argument");
  if (d < 1) return set_error(ctx, GP_ERROR, "sparsifier: dim must be >= 1");
  if (d > 0xFFFFFFFFULL) return set_error(ctx, GP_ERROR, "sparsifier: dim exceeds 32-bit index space");
  if (r < 1 || r > d) return set_error(ctx, GP_ERROR, "sparsifier: r out of range [1, d]");
  if (d > ctx->max_d) return set_error(ctx, GP_CAPACITY, "top_r: d exceeds the context's max_d");
  auto s = static_cast<cudaStream_t>(stream);
  launch_top_r(ctx, d_grad, d, r, s);
  cudaMemcpyAsync(d_support, ctx->ws.support, r * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  if (d_values) cudaMemcpyAsync(d_values, ctx->ws.values, r * sizeof(float), cudaMemcpyDeviceToDevice, s);
  return check_launch(ctx, "top_r");
}

int gp_crc32c(gp_ctx* ctx, const uint8_t* d_data, uint64_t n, uint32_t* d_crc, void* stream) {
  if (!ctx || (!d_data && n) || !d_crc) return set_error(ctx, GP_ERROR, "crc32c: null argument");
  launch_crc_host_range(ctx, d_data, n, d_crc, static_cast<cudaStream_t>(stream));
  return check_launch(ctx, "crc32c");
}

// Component calls over a bare serialized filter (no container): the plan is
// set up as for a decode whose index payload is the filter at offset 0.
static int bloom_component(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d, uint64_t r,
                           int method, cudaStream_t s) {
  if (d < 1 || d > ctx->max_d) return set_error(ctx, GP_CAPACITY, "bloom: d exceeds the context's max_d");
  PlanInit pi{};
  pi.d = d;
  pi.r = r;
  pi.il = filter_len;
  pi.index_method = static_cast<uint8_t>(method);
  pi.value_method = GP_VALUE_NONE;
  GP_LAUNCH(ctx, init_plan, 1, 1, 0, s, ctx->ws.plan, pi);  // the filter seeds come from its payload
  GP_LAUNCH(ctx, component_offsets, 1, 1, 0, s, ctx->ws.plan);
  launch_bloom_parse(ctx, d_filter, ctx->ws.m_cap, s);
  launch_bloom_scan(ctx, d, 0, false, s);
  return GP_OK;
}

int gp_bloom_positive_scan(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                           uint32_t* d_positives, uint64_t cap, uint64_t* d_count, void* stream) {
  if (!ctx || !d_filter || !d_positives || !d_count) return set_error(ctx, GP_ERROR, "positive_scan: null argument");
  auto s = static_cast<cudaStream_t>(stream);
  const int rc = bloom_component(ctx, d_filter, filter_len, d, 0, GP_INDEX_BLOOM_P0, s);
  if (rc != GP_OK) return rc;
  GP_LAUNCH(ctx, copy_positions, grid_for(ctx, d, 256), 256, 0, s, ctx->ws.pos, ctx->ws.plan, d_positives, cap,
            d_count, ctx->ws.status);
  return check_launch(ctx, "positive_scan");
}

__global__ void set_scan_range(Plan* plan, uint64_t lo, uint64_t hi) {
  gp_pdl_wait();
  plan->scan_lo = lo;
  plan->scan_hi = hi;
}

// caller positives -> ws.pos, |P| from a device word (the sharded decode)
__global__ void take_positions(const uint32_t* __restrict__ src, const uint64_t* __restrict__ count, Plan* plan,
                               uint32_t* __restrict__ pos, uint64_t cap, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status)) return;
  const uint64_t n = *count;
  if (n > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_CAPACITY);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) plan->n_pos = n;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    pos[i] = src[i];
}

int gp_bloom_scan_range(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d, uint64_t lo,
                        uint64_t hi, uint32_t* d_positives, uint64_t cap, uint64_t* d_count, void* stream) {
  if (!ctx || !d_filter || !d_positives || !d_count) return set_error(ctx, GP_ERROR, "scan_range: null argument");
  if (lo > hi || hi > d) return set_error(ctx, GP_ERROR, "scan_range: need lo <= hi <= d");
  if (d < 1 || d > ctx->max_d) return set_error(ctx, GP_CAPACITY, "bloom: d exceeds the context's max_d");
  auto s = static_cast<cudaStream_t>(stream);
  PlanInit pi{};
  pi.d = d;
  pi.il = filter_len;
  pi.index_method = GP_INDEX_BLOOM_P0;
  pi.value_method = GP_VALUE_NONE;
  GP_LAUNCH(ctx, init_plan, 1, 1, 0, s, ctx->ws.plan, pi);
  GP_LAUNCH(ctx, component_offsets, 1, 1, 0, s, ctx->ws.plan);
  launch_bloom_parse(ctx, d_filter, ctx->ws.m_cap, s);
  if (hi == lo) {  // empty slice: |P| = 0 (the scan treats hi = 0 as "all of d")
    GP_LAUNCH(ctx, set_scan_range, 1, 1, 0, s, ctx->ws.plan, 0, 0);
    fill_async(ctx, d_count, 0, sizeof(uint64_t), s);
    return check_launch(ctx, "scan_range");
  }
  GP_LAUNCH(ctx, set_scan_range, 1, 1, 0, s, ctx->ws.plan, lo, hi);
  launch_bloom_scan(ctx, hi - lo, 0, false, s);
  GP_LAUNCH(ctx, set_scan_range, 1, 1, 0, s, ctx->ws.plan, 0, 0);
  GP_LAUNCH(ctx, copy_positions, grid_for(ctx, hi - lo, 256), 256, 0, s, ctx->ws.pos, ctx->ws.plan, d_positives,
            cap, d_count, ctx->ws.status);
  return check_launch(ctx, "scan_range");
}

int gp_decode_index_from_positions(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                                   uint64_t r, int index_method, const uint32_t* d_positives,
                                   const uint64_t* d_count, void* stream) {
  if (!ctx || !d_filter || !d_positives || !d_count) return set_error(ctx, GP_ERROR, "index_from_positions: null");
  if (index_method < GP_INDEX_BLOOM_P0 || index_method > GP_INDEX_BLOOM_PD)
    return set_error(ctx, GP_ERROR, "index_from_positions: index_method must be Bloom P0, P1, P2 or Pd");
  if (r < 1) return set_error(ctx, GP_ERROR, "index_from_positions: r must be >= 1");
  if (d < 1 || d > ctx->max_d) return set_error(ctx, GP_CAPACITY, "bloom: d exceeds the context's max_d");
  auto s = static_cast<cudaStream_t>(stream);
  PlanInit pi{};
  pi.d = d;
  pi.r = r;
  pi.il = filter_len;
  pi.index_method = static_cast<uint8_t>(index_method);
  pi.value_method = GP_VALUE_NONE;
  GP_LAUNCH(ctx, init_plan, 1, 1, 0, s, ctx->ws.plan, pi);
  GP_LAUNCH(ctx, component_offsets, 1, 1, 0, s, ctx->ws.plan);
  launch_bloom_parse(ctx, d_filter, ctx->ws.m_cap, s);
  GP_LAUNCH(ctx, take_positions, grid_for(ctx, d, 256), 256, 0, s, d_positives, d_count, ctx->ws.plan, ctx->ws.pos,
            ctx->max_d, ctx->ws.status);
  launch_bloom_after_scan(ctx, false, s);
  if (index_method == GP_INDEX_BLOOM_P2)
    launch_select_p2(ctx, d, ctx->ws.set_cap, 64, false, s);
  else if (index_method == GP_INDEX_BLOOM_P1)
    launch_select_p1(ctx, d, d, s);
  else
    launch_select_slice(ctx, d, s);
  return check_launch(ctx, "index_from_positions");
}

int gp_decode_index_prepare(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d, uint64_t r,
                            int index_method, void* stream) {
  if (!ctx || !d_filter) return set_error(ctx, GP_ERROR, "decode_index_prepare: null argument");
  if (index_method < GP_INDEX_BLOOM_P0 || index_method > GP_INDEX_BLOOM_PD)
    return set_error(ctx, GP_ERROR, "decode_index_prepare: index_method must be Bloom P0, P1, P2 or Pd");
  if (r < 1) return set_error(ctx, GP_ERROR, "decode_index_prepare: r must be >= 1");
  auto s = static_cast<cudaStream_t>(stream);
  const int rc = bloom_component(ctx, d_filter, filter_len, d, r, index_method, s);
  if (rc != GP_OK) return rc;
  if (index_method == GP_INDEX_BLOOM_P2)
    launch_select_p2(ctx, d, ctx->ws.set_cap, 64, false, s);
  else if (index_method == GP_INDEX_BLOOM_P1)
    launch_select_p1(ctx, d, d, s);
  else
    launch_select_slice(ctx, d, s);
  return check_launch(ctx, "decode_index_prepare");
}

int gp_decode_accumulate_own(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap, const uint64_t* d_len,
                             const gp_pipeline_config* hint, float* d_dense, uint64_t d, float scale, void* stream) {
  if (!hint || !d_len) return set_error(ctx, GP_ERROR, "decode_accumulate_own: needs a hint and a length word");
  if (hint->index_method < GP_INDEX_BLOOM_P0 || hint->index_method > GP_INDEX_BLOOM_PD)
    return set_error(ctx, GP_ERROR, "decode_accumulate_own: Bloom P0, P1, P2 or Pd containers only");
  return decode_common(ctx, d_container, cap, d_len, hint, d_dense, d, scale, nullptr, nullptr, 0, nullptr, nullptr,
                       stream, true);
}

int gp_bloom_select(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d, uint64_t r,
                    int index_method, uint32_t* d_selected, void* stream) {
  if (!ctx || !d_filter || !d_selected) return set_error(ctx, GP_ERROR, "bloom_select: null argument");
  if (index_method != GP_INDEX_BLOOM_P1 && index_method != GP_INDEX_BLOOM_P2)
    return set_error(ctx, GP_ERROR, "bloom_select: index_method must be P1 (5) or P2 (6)");
  if (r < 1) return set_error(ctx, GP_ERROR, "bloom_select: r must be >= 1");
  auto s = static_cast<cudaStream_t>(stream);
  const int rc = bloom_component(ctx, d_filter, filter_len, d, r, index_method, s);
  if (rc != GP_OK) return rc;
  if (index_method == GP_INDEX_BLOOM_P2)
    launch_select_p2(ctx, d, ctx->ws.set_cap, 64, false, s);
  else
    launch_select_p1(ctx, d, d, s);
  cudaMemcpyAsync(d_selected, ctx->ws.sel, r * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
  return check_launch(ctx, "bloom_select");
}

}  // extern "C"
