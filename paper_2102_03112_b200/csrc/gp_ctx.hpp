// gp_ctx.hpp — host-side context: device workspace, device plan, launch accounting.
//
// One gp_ctx per (device, stream user).  Everything a step needs is carved out
// of one cudaMalloc made at gp_ctx_create, sized for gradients of up to max_d
// elements, so no allocation (and no implicit synchronisation) happens inside
// encode/decode.  Data-dependent sizes (|P|, payload lengths, segment counts)
// never travel to the host: kernels read them from the device-resident Plan
// and size their grid-stride loops from it.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gradpack_b200.h"

#ifdef __CUDACC__
// first statement of every kernel: wait for the grid this launch depends on
// (a no-op without programmatic dependent launch)
__device__ __forceinline__ void gp_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

namespace gp {

// Device-resident step descriptor, rewritten by each encode/decode call.
struct Plan {
  // ---- shared
  uint64_t d, r;
  uint8_t index_method, value_method, flags, pd_variant;
  uint32_t pad0;
  uint64_t il, vl, rl;          // payload lengths (bytes)
  uint64_t total_len;           // container length
  uint64_t n_values;            // value count (|P| for bloom-p0, else r)
  uint64_t n_sel;               // selected coordinates written to `sel`
  // ---- top-r
  uint32_t bin_star, full_bin;  // threshold bin of key >> kTopShift; bin fully kept?
  uint32_t thresh, tie_cut;     // exact threshold key; last kept index among ties
  uint64_t above, n_cand;       // keys in bins above bin_star; candidates emitted
  uint64_t thresh64;            // f64 input (topr64.cu): exact threshold key
  uint64_t r64_prefix, r64_need;  // topr64 refine: 32-bit key prefix of T, rank under it
  uint32_t r64_n, r64_pad;        // keys under that prefix
  uint64_t tie_q;               // keep the first tie_q keys == thresh (index order)
  uint32_t tie_all, pad2;       // every key == thresh is kept
  // ---- bloom
  uint64_t m, seed_a, seed_b, minv;
  uint64_t seed;                // the pipeline seed of this encode
  uint32_t k, pad1;
  uint64_t n_pos;               // |P|
  uint64_t scan_lo, scan_hi;    // positive scan over [scan_lo, scan_hi) only (0, 0: all of [0, d))
  uint64_t n_pairs, n_sets, n_multi, n_single_sel;
  uint64_t n_large;             // conflict sets of >= 255 members (ordered by a second pass)
  // ---- rle
  uint64_t n_runs, n_groups;
  // ---- value codec
  uint32_t sign_split, identity;
  uint32_t nseg, degree;
  uint64_t fit_bounds_at, fit_coeffs_at;  // decode: container offsets of the fit bounds / coefficients
  uint32_t q_bits, q_bucket;    // quantizer header (decode)
  uint32_t fit_kind, dexp_fail; // fit model kind (0 poly, 1 dexp); a dexp part failed (fallback)
  uint32_t slot_id, fused_bitmap;  // byte codec of a value-id-4 slot (0 store, 1 deflate; decode);
                                   // bitmap decode on the fused dense path (dense.cu), else 0
  // ---- decode
  uint64_t crc_stored;
  uint32_t crc_calc, post_crc_error;
  uint64_t off_index, off_value, off_reorder;
};

// fit models: up to 0xffff segments (u16 in the payload, curvefit.cpp:287)
// of up to 61 coefficients (degree <= 60, curvefit.cpp:130)
constexpr uint64_t kFitMaxSeg = 0xffff;
constexpr uint64_t kFitMaxCps = 61;
constexpr uint32_t kWideBlocks = 160;  // fit_solve_wide grid (its per-block scratch)
constexpr uint64_t kSortTileKeys = 2048;  // radix sort tile (sort.cu kTile): sizes sort_table / sort_flags

struct HuffTable;  // huffman.cuh

struct Workspace {
  void* base = nullptr;
  size_t bytes = 0;
  size_t bytes_total = 0;
  Plan* plan = nullptr;
  uint32_t* status = nullptr;
  uint32_t* status_pre = nullptr;  // status of the decode work launched before the CRC verdict (container.cu)
  uint8_t* scan_base = nullptr;   // [128 B tickets | tile descriptors], zeroed per scan
  uint32_t* ticket = nullptr;     // 32 tickets (first 128 B of scan_base)
  uint64_t* tiles = nullptr;      // scan tile descriptors
  size_t tiles_cap = 0;
  uint32_t* hist = nullptr;       // 32768 bins of key >> 16 + 65536 low-bit bins of the threshold bin
  uint32_t* cand_idx = nullptr;   // [D]
  float* cand_val = nullptr;      // [D]
  uint32_t* support = nullptr;    // [D]
  float* values = nullptr;        // [D]
  uint32_t* filter = nullptr;     // filter words, m_cap bits
  uint64_t m_cap = 0;
  uint32_t* pos = nullptr;        // P [D]
  uint32_t* sel = nullptr;        // selection [D]
  uint8_t* flags = nullptr;       // per-P flags [D]
  uint32_t* selbits = nullptr;    // selection bitset over P positions [D/32]
  // conflict sets (p2.cu)
  uint64_t set_cap = 0;           // max filter width m for P2
  uint32_t* p2_count = nullptr;   // [set_cap + 1]
  uint32_t* p2_off = nullptr;     // [set_cap + 1]
  uint32_t* p2_alloc = nullptr;   // bucket-space allocator word
  uint32_t* p2_sets = nullptr;    // [set_cap]
  uint32_t* p2_table = nullptr;   // [256 * set_cap / 4096 + 256]
  uint32_t* p2_members = nullptr; // [pair_cap]
  uint32_t* first_touch = nullptr; // per-P earliest visit of a window [D]
  uint32_t* bucket = nullptr;     // per-bit counters [m_cap + 1]
  uint32_t* bucket_off = nullptr; // per-bit offsets [m_cap + 1]
  uint32_t* pairs = nullptr;      // conflict pairs [pair_cap]
  uint32_t* p2_rank = nullptr;    // each pair's slot in its set [pair_cap]
  uint64_t pair_cap = 0;
  uint32_t* set_bit = nullptr;    // multi-member sets (bit) [m_cap]
  uint32_t* set_key = nullptr;    // sort keys [m_cap]
  uint32_t* set_tmp = nullptr;    // [m_cap]
  uint32_t* set_tmp2 = nullptr;   // [m_cap]
  uint32_t* u32a = nullptr;       // generic [D]
  uint32_t* u32b = nullptr;       // generic [D]
  uint32_t* u32c = nullptr;       // generic [D]
  uint32_t* u32d = nullptr;       // generic [D]
  double* f64a = nullptr;         // [D]
  double* f64b = nullptr;         // [D]
  double* partial = nullptr;      // fit chunk partial sums [(D/2048 + 128) * 44]
  uint32_t* sort_table = nullptr; // onesweep per-tile digit state [2][tiles][256]
  uint32_t* sort_flags = nullptr; // [0,8): pass tickets, [64, 64+tiles): tile flags
  uint32_t* sort_hist = nullptr;  // global digit histograms [4][256]
  double* seg_dev = nullptr;      // segmentation sweep partials [4 * 2048]
  uint32_t* seg_arg = nullptr;    // [4 * 2048]
  uint32_t* seg_end = nullptr;    // fit segment bounds [seg_cap]
  float* coeffs = nullptr;        // fit coefficients, segment-major [seg_cap * 61]
  uint64_t seg_cap = 0;           // segments both sign parts may produce before the 0xffff check
  uint8_t* seg_nodes = nullptr;   // segmentation tree, 32-byte nodes [node_cap]
  uint32_t* seg_heap = nullptr;   // [node_cap]
  uint32_t* seg_pend = nullptr;   // pending nodes / traversal stack [node_cap]
  uint64_t* seg_off = nullptr;    // interior-length prefix of the pending nodes [node_cap + 1]
  uint32_t node_cap = 0;
  uint32_t* seg_state = nullptr;  // SegState control words [8]
  uint64_t* seg_chunk = nullptr;  // accumulate chunk starts per segment [seg_cap + 1]
  double* fit_scratch = nullptr;  // fit_solve_wide per-block matrices [kWideBlocks * 3 * 61 * 61]
  uint32_t* crc_digits = nullptr; // CRC shift-operator digit tables [5 * 256] + lane-stride multiply [4 * 256]
  uint32_t* crc_acc = nullptr;    // XOR accumulator + block counter [2]
  bool crc_ready = false;
  uint64_t crc_cap = 0;
  uint8_t* scratch = nullptr;     // generic byte scratch [2 * D]
  HuffTable* huff = nullptr;      // Huffman index table of the current container
  uint64_t* huff_res = nullptr;   // Huffman decode verdict words + round flags [16]
};

}  // namespace gp

namespace gp {
// Pipeline stages timed with CUDA events when profiling is on (gp_ctx_profile).
enum Stage {
  ST_TOPR, ST_INDEX, ST_BLOOM_BUILD, ST_BLOOM_SCAN, ST_P2_SETS, ST_P2_ENGINE, ST_SELECT, ST_GATHER, ST_VALUES,
  ST_PACK, ST_DEC_PARSE, ST_DEC_INDEX, ST_DEC_BLOOM_SCAN, ST_DEC_P2_SETS, ST_DEC_P2_ENGINE, ST_DEC_SELECT,
  ST_DEC_VALUES, ST_DEC_SCATTER, ST_COUNT
};
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<int> stage;   // per recorded pair
  std::vector<size_t> first;
  int open_stage = -1;
  size_t open_event = 0;
};
}  // namespace gp

struct gp_ctx {
  int device = 0;
  int sm_count = 148;
  uint64_t max_d = 0;
  gp::Workspace ws;
  std::string last_error;
  uint64_t launches = 0;
  gp::Profiler prof;
  const uint64_t* seed_dev = nullptr;  // gp_ctx_set_seed_source: pipeline seed read on the device
  cudaEvent_t index_event = nullptr;   // gp_ctx_set_index_event: recorded once encode's index payload is final
  bool decode_overwrite = false;
  const double* vals64 = nullptr;      // this encode's f64 value sequence (null: ws.values, f32)
  const float* gather_dense = nullptr;  // Bloom + fit encode: the key kernel gathers dense[sel[j]] (values_fit.cu)
  cudaStream_t side = nullptr;         // decode work before the CRC verdict runs here, beside the CRC
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;       // gp_ctx_set_decode_overwrite: dense = scale * decoded (zeros off the support)
};

namespace gp {

// Every kernel launch goes through this macro so gp_ctx_launch_count() can
// report how many native kernels a step enqueued.  Launches carry the
// programmatic-stream-serialization attribute (programmatic dependent launch,
// also inside captured graphs): a kernel's launch and block scheduling
// overlap the end of the kernel before it on the stream, and every kernel
// begins with gp_pdl_wait() (griddepcontrol.wait: the preceding grid has
// completed and its memory is visible) before it reads anything.  GP_PDL=0
// launches without the attribute.
extern bool g_pdl;
template <typename... P, typename... A>
inline void launch_k(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<A&&>(a)...);
}
#define GP_LAUNCH(ctx, kernel, grid, block, smem, stream, ...)                         \
  do {                                                                                \
    ::gp::launch_k(kernel, (grid), (block), (smem), (stream), __VA_ARGS__);           \
    ++(ctx)->launches;                                                                \
  } while (0)

// cudaMemsetAsync as a PDL-chained kernel (a memset node between two kernels
// breaks their programmatic launch overlap); GP_FILL_KERNEL=0 uses the memset
void fill_async(gp_ctx* ctx, void* p, int value, size_t bytes, cudaStream_t s);

// Grid for a grid-stride loop over n items: enough blocks to cover n, capped
// at 8 resident blocks per SM.
inline int grid_for(const gp_ctx* ctx, uint64_t n, int block) {
  const uint64_t g = (n + block - 1) / block;
  const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

int set_error(gp_ctx* ctx, int code, const std::string& msg);
void stage_begin(gp_ctx* ctx, int stage, cudaStream_t s);
void stage_end(gp_ctx* ctx, cudaStream_t s);
// Times `call` as `stage` when profiling is on (events on the launch stream).
#define GP_STAGE(ctx, stage, s, call)         \
  do {                                        \
    ::gp::stage_begin((ctx), (stage), (s));   \
    call;                                     \
    ::gp::stage_end((ctx), (s));              \
  } while (0)
int check_launch(gp_ctx* ctx, const char* what);

// ---- host launchers, grouped by translation unit ----
void reset_scan(gp_ctx* ctx, cudaStream_t s, uint64_t ntiles_bound);  // capi.cu
// dynamic shared-memory opt-ins, per device (called by gp_ctx_create)
void kernel_attrs_bloom();
void kernel_attrs_p2();
void kernel_attrs_topr();
void kernel_attrs_dense();
void kernel_attrs_topr64();

// topr.cu: ws.support / ws.values <- top-r of grad
void launch_top_r(gp_ctx* ctx, const float* grad, uint64_t d, uint64_t r, cudaStream_t s, float* residual = nullptr);
void launch_own_support(gp_ctx* ctx, uint64_t r_bound, cudaStream_t s);
// topr64.cu: ws.support / ws.f64a <- top-r of double(grad) + residual (written over residual)
void launch_top_r64(gp_ctx* ctx, const float* grad, double* residual, uint64_t d, uint64_t r, cudaStream_t s);

// container.cu
void launch_crc_range(gp_ctx* ctx, const uint8_t* base, const uint64_t* off_dev, uint64_t off_host,
                      const uint64_t* la, const uint64_t* lb, const uint64_t* lc, uint64_t len_host,
                      uint64_t len_bound, uint32_t* out, cudaStream_t s);
constexpr int kCrcSmallTabWords = 4 * 256 + 17 * 128;  // crc_tail: slice-by-4 tables, 17 nibble-table constants
int crc_tables_init(gp_ctx* ctx);  // container.cu (gp_ctx_create)
bool nz_fast_path_eligible(uint64_t d, uint64_t r, int index_method, int value_method);  // dense.cu
uint32_t* gate_word(gp_ctx* ctx);
void launch_nz_encode(gp_ctx* ctx, const float* g, uint64_t d, uint64_t r, uint8_t* out, cudaStream_t s);
void launch_gate_merge(gp_ctx* ctx, cudaStream_t s);
void launch_dense_zero(gp_ctx* ctx, float* dense, uint64_t n, cudaStream_t s);
void launch_decode_bitmap_check(gp_ctx* ctx, const uint8_t* in, cudaStream_t s);  // indexcodec.cu
void launch_bm_prepare(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, cudaStream_t s);
void launch_bm_scatter(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, float* dense, uint64_t dense_d, float scale,
                       bool overwrite, cudaStream_t s);
void launch_crc_host_range(gp_ctx* ctx, const uint8_t* data, uint64_t n, uint32_t* out, cudaStream_t s);
void launch_finish_container(gp_ctx* ctx, uint8_t* out, uint64_t cap, uint64_t* d_len, uint64_t len_bound,
                             cudaStream_t s);
void launch_parse_container(gp_ctx* ctx, const uint8_t* in, uint64_t len, const uint64_t* len_dev,
                            const gp_pipeline_config* hint, cudaStream_t s);
void launch_verify_crc(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, cudaStream_t s);
void launch_merge_status(gp_ctx* ctx, cudaStream_t s);

// indexcodec.cu
void launch_index_none(gp_ctx* ctx, uint8_t* out, uint64_t r, cudaStream_t s);
void launch_index_bitmap(gp_ctx* ctx, uint8_t* out, uint64_t d, uint64_t r, cudaStream_t s);
void launch_decode_index_none(gp_ctx* ctx, const uint8_t* in, uint64_t r_bound, cudaStream_t s);
void launch_validate_support(gp_ctx* ctx, uint64_t r_bound, cudaStream_t s);
void launch_decode_index_bitmap(gp_ctx* ctx, const uint8_t* in, uint64_t d_bound, cudaStream_t s);
void launch_index_rle(gp_ctx* ctx, uint8_t* out, uint64_t d, uint64_t r, cudaStream_t s);          // rle.cu
void launch_index_huffman(gp_ctx* ctx, uint8_t* out, uint64_t r, uint64_t il_bound, cudaStream_t s);  // huffman.cu
void launch_decode_index_huffman(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, cudaStream_t s);
uint64_t huffman_il_bound(uint64_t d, uint64_t r);
void launch_decode_index_rle(gp_ctx* ctx, const uint8_t* in, uint64_t len_bound, uint64_t d_bound, cudaStream_t s);

// bloom.cu / p2.cu
void launch_bloom_build(gp_ctx* ctx, uint8_t* out, uint64_t m, uint64_t r, cudaStream_t s);
void launch_bloom_parse(gp_ctx* ctx, const uint8_t* in, uint64_t m_bound, cudaStream_t s);
void launch_bloom_scan(gp_ctx* ctx, uint64_t d_bound, uint64_t m_host, bool decoding, cudaStream_t s);
void launch_select_slice(gp_ctx* ctx, uint64_t n_bound, cudaStream_t s);
void launch_bloom_after_scan(gp_ctx* ctx, bool decoding, cudaStream_t s);
void launch_select_p1(gp_ctx* ctx, uint64_t n_bound, uint64_t r_bound, cudaStream_t s);
void launch_flags_compact(gp_ctx* ctx, int method, uint64_t n_bound, cudaStream_t s);
void launch_select_p2(gp_ctx* ctx, uint64_t n_bound, uint64_t m_bound, uint32_t k_bound, bool decoding,
                      cudaStream_t s, uint64_t n_expect = 0);

// sort.cu
void launch_table_scan(gp_ctx* ctx, uint32_t* table, const uint64_t* n_dev, uint64_t n_bound, int tile_shift,
                       cudaStream_t s);

// values.cu
void launch_gather_values(gp_ctx* ctx, const float* dense, uint64_t n_bound, cudaStream_t s);
void launch_gather_values64(gp_ctx* ctx, const double* dense, const uint32_t* sup, const double* sval, uint64_t r,
                            uint64_t n_bound, cudaStream_t s);
void launch_values_raw(gp_ctx* ctx, uint8_t* out, bool f64, uint64_t n_bound, cudaStream_t s);
void launch_values_raw_check(gp_ctx* ctx, cudaStream_t s);
void launch_values_fit(gp_ctx* ctx, uint8_t* out, int degree, int max_segments, uint64_t n_bound, cudaStream_t s,
                       bool dexp = false);
void launch_decode_fit(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s);
void launch_values_quant(gp_ctx* ctx, uint8_t* out, int bits, uint32_t bucket, uint64_t n_bound,
                         cudaStream_t s);                                                            // values_quant.cu
void launch_decode_quant(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s);
void launch_values_slot(gp_ctx* ctx, uint8_t* out, uint64_t n_bound, cudaStream_t s);
void launch_values_deflate(gp_ctx* ctx, uint8_t* out, uint64_t n_bound, cudaStream_t s);  // deflate.cu
uint64_t deflate_slot_bound(uint64_t n);
void launch_decode_slot(gp_ctx* ctx, const uint8_t* in, cudaStream_t s);
void launch_decode_inflate(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s);
void launch_decode_scatter(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, float* dense, uint64_t dense_d,
                           float scale,
                           uint32_t* out_support, double* out_values, uint64_t cap, uint64_t* d_count,
                           uint64_t* d_dim, cudaStream_t s, double* dense64 = nullptr);

}  // namespace gp
