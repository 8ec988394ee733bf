/*
 * gradpack_b200.h — C-ABI of the B200-native DeepReduce sparse-gradient path.
 *
 * Drop-in boundary for the reference's C++ compressor API (gradpack,
 * /root/reference/proj).  Every entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only: device pointers are
 * prefixed d_, host pointers h_; `stream` is a cudaStream_t passed as void*.
 *
 * Asynchrony contract: functions that take a stream only ENQUEUE work and
 * return GP_OK when the launch succeeded.  Errors that depend on device data
 * (checksums, payload validation) are latched in a per-context device status
 * word; gp_ctx_status() synchronises the stream and returns the first one, in
 * the reference's check order (container.cpp:84-127, pipeline.cpp:223-306).
 * Host-detectable misuse (bad config, capacity) is returned immediately.
 */
#ifndef GRADPACK_B200_H_
#define GRADPACK_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GP_API __attribute__((visibility("default")))
#else
#define GP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, 1:1 with the exception classes of errors.hpp:21-53. */
enum gp_status {
  GP_OK = 0,
  GP_ERROR = 1,              /* gradpack::Error            errors.hpp:21 */
  GP_DECODE = 2,             /* gradpack::DecodeError      errors.hpp:26 */
  GP_TRUNCATED = 3,          /* gradpack::TruncatedError   errors.hpp:31 */
  GP_CHECKSUM = 4,           /* gradpack::ChecksumError    errors.hpp:36 */
  GP_UNKNOWN_METHOD = 5,     /* gradpack::UnknownMethodError errors.hpp:41 */
  GP_CORRUPT_PAYLOAD = 6,    /* gradpack::CorruptPayloadError errors.hpp:46 */
  GP_FIT = 7,                /* gradpack::FitError         errors.hpp:51 */
  GP_CUDA = 8,               /* CUDA runtime failure (no reference equivalent) */
  GP_UNSUPPORTED = 9,        /* method id registered in FORMAT.md but not on this device path */
  GP_CAPACITY = 10,          /* device workspace / output buffer too small */
  GP_NCCL = 11               /* NCCL failure / library not loadable (no reference equivalent) */
};

/* Stable wire ids (container.hpp:23-43, FORMAT.md:46-89). */
enum gp_index_method {
  GP_INDEX_NONE = 0, GP_INDEX_BITMAP = 1, GP_INDEX_RLE = 2, GP_INDEX_HUFFMAN = 3,
  GP_INDEX_BLOOM_P0 = 4, GP_INDEX_BLOOM_P1 = 5, GP_INDEX_BLOOM_P2 = 6,
  GP_INDEX_BLOOM_PD = 7, GP_INDEX_BLOOM_NAIVE = 8
};
enum gp_value_method {
  GP_VALUE_NONE = 0, GP_VALUE_FIT_POLY = 1, GP_VALUE_FIT_DEXP = 2, GP_VALUE_QUANT = 3,
  GP_VALUE_DEFLATE_SLOT = 4, GP_VALUE_RAW_F64 = 5
};

/* POD mirror of gradpack::PipelineConfig (pipeline.hpp:28-39), same defaults. */
typedef struct gp_pipeline_config {
  uint8_t index_method;   /* gp_index_method, default NONE */
  uint8_t value_method;   /* gp_value_method, default NONE */
  uint8_t pd_variant;     /* 0 leftmost, 1 middle, 2 rightmost */
  uint8_t slot_codec;     /* 0 store, 1 deflate (default 1) */
  int32_t degree;         /* fit polynomial degree, default 5 */
  int32_t max_segments;   /* fit cap, 0 = knot heuristic */
  int32_t quant_bits;     /* default 7 */
  uint32_t quant_bucket;  /* default 512 */
  double fpr;             /* Bloom target FPR, default 0.01 */
  uint64_t seed;          /* pipeline seed */
} gp_pipeline_config;

GP_API void gp_pipeline_config_default(gp_pipeline_config* cfg);

/* ---------------------------------------------------------------- context */
typedef struct gp_ctx gp_ctx;

/* One context per (device, stream user).  The workspace is sized once for
 * gradients of up to max_d elements; no allocation happens inside a step.
 * The context also owns a second stream: a decode forks its index and value
 * decoders onto it beside the CRC verdict (event fork/join, so the caller's
 * stream — captured into a CUDA graph or not — sees one ordered call). */
GP_API int gp_ctx_create(int device, uint64_t max_d, gp_ctx** out);
GP_API void gp_ctx_destroy(gp_ctx* ctx);
GP_API const char* gp_last_error(const gp_ctx* ctx);
/* Synchronise `stream`, return and clear the first latched device status. */
GP_API int gp_ctx_status(gp_ctx* ctx, void* stream);
/* Number of kernel launches this context has enqueued since creation. */
GP_API uint64_t gp_ctx_launch_count(const gp_ctx* ctx);

/* Stage profiling: with on != 0 every pipeline stage enqueued by this
 * context is bracketed by CUDA events on its stream.  gp_ctx_stage_times
 * synchronises, ADDS the elapsed ms and counts per stage into the caller's
 * arrays (index = stage id, see gp_stage_name) and resets the record. */
GP_API int gp_ctx_profile(gp_ctx* ctx, int on);
GP_API int gp_ctx_stage_times(gp_ctx* ctx, double* ms, uint64_t* counts, int n_stages);
GP_API const char* gp_stage_name(int stage);

/* Upper bound of pack(compress_gradient(...)) for a gradient of d elements with
 * r kept (container.cpp:58-82 layout).  Host-only arithmetic. */
GP_API uint64_t gp_max_container_bytes(uint64_t d, uint64_t r, const gp_pipeline_config* cfg);

/* Seed source for CUDA-graph replay.  With a non-null d_seed, every encode on
 * this context reads its pipeline seed from the device word *d_seed when the
 * step executes (cfg->seed is ignored), so one captured step replays with a
 * new seed per step.  NULL restores cfg->seed.  Host-only bookkeeping. */
GP_API int gp_ctx_set_seed_source(gp_ctx* ctx, const uint64_t* d_seed);

/* d_seed[0] = Simulation::pipeline_seed(seed, worker, *d_step)
 * (harness.cpp:201-203) computed on the device (one tiny kernel on `stream`):
 * the per-(worker, step) seed of the DP loop without a host round trip.  With
 * buckets > 0, d_seed[b] = hash64(b, that seed) for b < buckets (the bucketed
 * step's per-bucket seeds). */
GP_API int gp_pipeline_seed_device(uint64_t* d_seed, const uint64_t* d_step, uint64_t seed, uint32_t worker,
                                   uint32_t buckets, void* stream);

/* ---------------------------------------------------------------- encode */
/* top_r (sparsify.cpp:32-46) + compress_gradient(sg, cfg, &dense)
 * (pipeline.cpp:146-221) + pack (container.cpp:58-82), fused.
 * d_grad: f32[d] on device.  Writes the container to d_out (capacity cap) and
 * its byte length to the device word *d_len.  r == 0 is invalid (Error). */
GP_API int gp_encode_topr(gp_ctx* ctx, const float* d_grad, uint64_t d, uint64_t r,
                   const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap,
                   uint64_t* d_len, void* stream);

/* Error-feedback encode, the compensation step of the reference worker loop
 * (harness.cpp:230 input = g + residual; :250 compress_gradient(top_r(input),
 * cfg, &input) + pack; :269-271 residual = input - to_dense(decode(wire))).
 * d_grad: f32[d]; d_residual: f32[d], read as e and overwritten with the new
 * residual.  The add is fused into top-r's first pass (f32, round to
 * nearest); the subtraction is the decode scatter with scale -1.  Writes the
 * container and its length word as gp_encode_topr does. */
GP_API int gp_encode_topr_ef(gp_ctx* ctx, const float* d_grad, float* d_residual, uint64_t d, uint64_t r,
                             const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap,
                             uint64_t* d_len, void* stream);

/* The same step in the reference's own precision: d_residual is f64[d]
 * (Simulation::residual_, a VectorXd, gradient.hpp:29), input = double(g) +
 * residual in f64, top_r over the f64 input (63-bit keys), the value codec on
 * the f64 values, and residual = input - decoded in f64.  Containers and
 * residuals are bit-identical to the reference loop fed double(g). */
GP_API int gp_encode_topr_ef64(gp_ctx* ctx, const float* d_grad, double* d_residual, uint64_t d, uint64_t r,
                               const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap,
                               uint64_t* d_len, void* stream);

/* compress_gradient(sg, cfg, dense) + pack with the reference's own value
 * type (pipeline.cpp:146-221): sg = (d, d_support u32[r] strictly increasing,
 * d_values f64[r]); d_dense f64[d] or NULL.  Bloom policies take values from
 * d_dense when given, else from sg with zeros off its support
 * (pipeline.cpp:38-54).  r = 0 is legal for index method NONE with raw value
 * methods (empty payloads), an Error otherwise, as in the reference. */
GP_API int gp_encode_sparse(gp_ctx* ctx, uint64_t d, const uint32_t* d_support, const double* d_values,
                            uint64_t r, const double* d_dense, const gp_pipeline_config* cfg, uint8_t* d_out,
                            uint64_t cap, uint64_t* d_len, void* stream);

/* compress_gradient(sg, cfg, &dense) + pack for a caller-chosen support:
 * d_support: u32[r] strictly increasing (validated, gradient.cpp:19-30),
 * values are gathered from d_dense (pipeline.cpp:38-54). */
GP_API int gp_encode_support(gp_ctx* ctx, const float* d_dense, uint64_t d, const uint32_t* d_support,
                      uint64_t r, const gp_pipeline_config* cfg, uint8_t* d_out, uint64_t cap,
                      uint64_t* d_len, void* stream);

/* ---------------------------------------------------------------- decode */
/* unpack (container.cpp:84-127) + decompress_gradient (pipeline.cpp:223-306)
 * + to_dense accumulate: d_dense[support[i]] += scale * value[i] (f32).
 * This is the per-peer step of the harness mean (harness.cpp:274-284). */
GP_API int gp_decode_accumulate(gp_ctx* ctx, const uint8_t* d_container, uint64_t len,
                         float* d_dense, uint64_t d, float scale, void* stream);

/* As gp_decode_accumulate, but dispatches the device pipeline for the
 * methods in `hint` without peeking the header on the host (no host sync).
 * The device verifies the container's method ids against the hint after the
 * CRC check; a mismatch latches GP_UNSUPPORTED and leaves d_dense untouched,
 * and the caller may retry without a hint. */
GP_API int gp_decode_accumulate_hint(gp_ctx* ctx, const uint8_t* d_container, uint64_t len,
                              const gp_pipeline_config* hint, float* d_dense, uint64_t d,
                              float scale, void* stream);

/* As gp_decode_accumulate_hint, with the container length read on the device
 * from *d_len (e.g. the length word gp_encode_topr wrote); `cap` is the
 * buffer capacity.  Fully asynchronous: no host round trip at all. */
GP_API int gp_decode_accumulate_dlen(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap,
                                     const uint64_t* d_len, const gp_pipeline_config* hint,
                                     float* d_dense, uint64_t d, float scale, void* stream);

/* Overwrite mode (on = 1) for this context's following decodes into a dense
 * buffer: d_dense = scale * decoded on the support and 0 elsewhere — exactly
 * what zeroing the buffer and accumulating would produce (the first container
 * of a DP step's mean, harness.cpp:274-284), without the separate zero pass.
 * Bitmap + raw containers then write the whole buffer in one pass (dense.cu).
 * When a decode latches an error the buffer's contents are unspecified. */
GP_API int gp_ctx_set_decode_overwrite(gp_ctx* ctx, int on);

/* Early index decode (one rank's own container, N = 1 and the own peer at
 * N > 1): the Bloom filter payload of a container is final as soon as its
 * encode built the filter, so its positive scan and P0/P1/P2/Pd selection can
 * run on a second context and stream while the encode finishes (selection,
 * values, pack).  gp_ctx_set_index_event(enc_ctx, ev) makes encode record the
 * CUDA event `ev` at that point; gp_decode_index_prepare(dec_ctx, filter at
 * container + 49, 26 + ceil(m/8) [+1 for Pd], d, r, method, stream) runs the
 * index stage; gp_decode_accumulate_own(dec_ctx, ...) then decodes the finished
 * container (parse, CRC, method check, values, scatter) with that prepared
 * index stage.  The work is the full decode; only its schedule moves. */
GP_API int gp_ctx_set_index_event(gp_ctx* ctx, void* event);
GP_API int gp_decode_index_prepare(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                                   uint64_t r, int index_method, void* stream);
GP_API int gp_decode_accumulate_own(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap, const uint64_t* d_len,
                                    const gp_pipeline_config* hint, float* d_dense, uint64_t d, float scale,
                                    void* stream);

/* A decode split in two for concurrent peers: gp_decode_prepare runs everything
 * of gp_decode_accumulate_dlen but the final scatter (parse, CRC, index and
 * value decode, validation) into the context's workspace; gp_decode_finish
 * then applies d_dense[support[i]] += scale * value[i] from that state.  With
 * one context per container, the prepares of several peers run concurrently
 * on their own streams while the finishes keep the rank order of the
 * accumulation (each finish must follow its prepare; a context holds one
 * prepared container at a time). */
GP_API int gp_decode_prepare(gp_ctx* ctx, const uint8_t* d_container, uint64_t cap, const uint64_t* d_len,
                             const gp_pipeline_config* hint, void* stream);
GP_API int gp_decode_finish(gp_ctx* ctx, const uint8_t* d_container, float* d_dense, uint64_t d, float scale,
                            void* stream);

/* unpack + decompress_gradient to sparse form.  Writes up to cap entries of
 * support (u32) and values (f64) and the count to the device word *d_count.
 * *d_dim receives the container's d. */
GP_API int gp_decode_sparse(gp_ctx* ctx, const uint8_t* d_container, uint64_t len,
                     uint32_t* d_support, double* d_values, uint64_t cap,
                     uint64_t* d_count, uint64_t* d_dim, void* stream);

/* ---------------------------------------------------------------- components */
/* top_r (sparsify.cpp:32-46): ascending support of the r largest |g|, ties to
 * the lower index; values gathered alongside (gradient.cpp:44-54). */
GP_API int gp_top_r(gp_ctx* ctx, const float* d_grad, uint64_t d, uint64_t r, uint32_t* d_support,
             float* d_values, void* stream);

/* crc32c (container.cpp:30-48) of n device bytes into the device word *d_crc. */
GP_API int gp_crc32c(gp_ctx* ctx, const uint8_t* d_data, uint64_t n, uint32_t* d_crc, void* stream);

/* positive_scan (bloom.cpp:123-128) of a serialized filter (bloom.cpp:84-94,
 * FORMAT.md:58-75) over [0, d): ascending positives, count to *d_count. */
GP_API int gp_bloom_positive_scan(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len,
                           uint64_t d, uint32_t* d_positives, uint64_t cap, uint64_t* d_count,
                           void* stream);

/* p1_select / p2_select (bloom.cpp:140-154, :175-222) over the positives of a
 * serialized filter, with the selection stream seeded as
 * derive_selection_seed(seed_a, seed_b) (pipeline.cpp:23-25, :205, :286).
 * index_method selects P1 (5) or P2 (6).  Output: r ascending keys. */
GP_API int gp_bloom_select(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                    uint64_t r, int index_method, uint32_t* d_selected, void* stream);

/* volume (container.cpp:148-243) of a HOST copy of a packed container: exact
 * bit accounting; bits per nonzero = total_bits / r.  Host-only. */
typedef struct gp_volume_report {
  uint64_t index_bits, value_bits, reorder_bits, metadata_bits, total_bits;
  double ratio_dense;   /* total / (32 d) */
  double ratio_sparse;  /* total / (64 r); 0 when r = 0 */
} gp_volume_report;
GP_API int gp_volume(const uint8_t* h_container, uint64_t len, gp_volume_report* out);

/* bloom_params (bloom.cpp:22-31).  Host arithmetic, returns GP_ERROR on bad args. */
GP_API int gp_bloom_params(double epsilon, uint64_t r, uint64_t* m, uint32_t* k);

/* Sharded decode index stage (the N > 1 exchange): positive_scan
 * (bloom.cpp:123-128) of a serialized filter over the coordinate slice
 * [lo, hi) only — the ascending positives there, global coordinates — so the
 * N ranks of a step split the scans of all N filters by coordinate range
 * instead of each scanning every filter over all of [0, d); and the
 * selection (P0/Pd slice, P1, P2 replay, bloom.cpp:140-222) from a complete
 * positive list assembled by the caller (d_count: |P| in device memory),
 * finished by gp_decode_accumulate_own on the same context. */
GP_API int gp_bloom_scan_range(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                               uint64_t lo, uint64_t hi, uint32_t* d_positives, uint64_t cap,
                               uint64_t* d_count, void* stream);
GP_API int gp_decode_index_from_positions(gp_ctx* ctx, const uint8_t* d_filter, uint64_t filter_len, uint64_t d,
                                          uint64_t r, int index_method, const uint32_t* d_positives,
                                          const uint64_t* d_count, void* stream);

/* ---------------------------------------------------------------- data-parallel step
 * Simulation::step's exchange between real workers (harness.cpp:219-293),
 * one process (or host thread) per GPU: encode own gradient (with
 * compensation: gp_encode_topr_ef64 on a device-resident f64 residual), the
 * container lengths allgathered, ONE host sync on them (and on this rank's
 * encode status), the containers allgathered padded to the longest, then every
 * rank's container decoded in rank order into the dense mean
 * (dense = fmaf(1/N, v, dense), the first overwriting).  Replaces the worker
 * loop + pairwise mean of harness.cpp:227-284; the mean is the f32 sequential
 * accumulation (within N ulp(f32) of the reference's f64 pairwise tree).
 *
 * gp_dp_unique_id: ncclGetUniqueId (rank 0), to be shared by the caller.
 * gp_dp_create: NCCL communicator of `nranks` (libnccl.so.2 resolved at run
 * time), device buffers sized by gp_max_container_bytes(d, r, cfg).
 * gp_dp_create_local: an in-process group over `nranks` contexts (one host
 * thread per rank must call gp_dp_step concurrently): the allgathers are
 * device copies ordered by events — the same step on one GPU.
 * gp_dp_step: pipeline seed = Simulation::pipeline_seed(seed, rank, step)
 * (harness.cpp:201-203); d_grad f32[d]; d_mean f32[d] receives the mean.
 * An encode error is returned at the host sync; the group cannot continue
 * (peers block in the exchange), as an exception ends the reference's loop. */
#define GP_DP_UNIQUE_ID_BYTES 128
typedef struct gp_dp gp_dp;
GP_API int gp_dp_unique_id(uint8_t* out_id);
GP_API int gp_dp_create(gp_ctx* ctx, const uint8_t* id, int nranks, int rank, uint64_t d, uint64_t r,
                        const gp_pipeline_config* cfg, int ef, gp_dp** out);
GP_API int gp_dp_create_local(gp_ctx** ctxs, int nranks, uint64_t d, uint64_t r, const gp_pipeline_config* cfg,
                              int ef, gp_dp** out);
GP_API int gp_dp_step(gp_dp* dp, const float* d_grad, uint64_t seed, int step, float* d_mean, void* stream);
GP_API const double* gp_dp_residual(const gp_dp* dp);
GP_API int gp_dp_destroy(gp_dp* dp);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* GRADPACK_B200_H_ */
