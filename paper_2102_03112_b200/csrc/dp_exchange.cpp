// dp_exchange.cpp — the data-parallel step of Simulation::step between real
// workers (harness.cpp:219-293), host C++ over the C-ABI:
//
//   encode own gradient (top_r + compress_gradient + pack; with compensation
//   the f64 error-feedback step, harness.cpp:230/:269-271) → allgather of the
//   container lengths → one host sync (the lengths, and this rank's encode
//   status) → allgather of the containers padded to the longest (NCCL has no
//   allgatherv) → decode of every rank's container in rank order into the
//   dense mean, dense = fmaf(1/N, v, dense), the first one overwriting.
//
// Transports: NCCL, resolved at run time from libnccl.so.2 (no link-time
// dependency; inside a process that already loaded torch's NCCL the loader
// hands back that library), and an in-process group of contexts (one host
// thread per rank) whose allgather is device copies ordered by CUDA events —
// the same step on one GPU, for tests and single-process multi-context use.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "gp_ctx.hpp"

namespace gp {

namespace {

uint64_t mix64_h(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t hash64_h(uint64_t x, uint64_t seed) { return mix64_h(x ^ (seed + 0x9E3779B97F4A7C15ULL)); }

// Simulation::pipeline_seed (harness.cpp:201-203) over Problem::batch_seed (:47-51)
uint64_t pipeline_seed_h(uint64_t seed, int worker, int step) {
  const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(worker)) << 32) | static_cast<uint32_t>(step);
  return hash64_h(0xC0DEC, hash64_h(key, hash64_h(0xDA7A, seed)));
}

struct Transport {
  virtual ~Transport() = default;
  // recv[k * bytes, (k + 1) * bytes) <- rank k's send[0, bytes), on `s`
  virtual int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s, std::string& err) = 0;
};

// ---------------------------------------------------------------- NCCL
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok() const { return all_gather != nullptr; }
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.h, "ncclAllGather"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.error_string) a.all_gather = nullptr;
    return a;
  }();
  return api;
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  bool owned = false;
  ~NcclTransport() override {
    if (owned && comm) nccl().comm_destroy(comm);
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s, std::string& err) override {
    const ncclResult_t r = nccl().all_gather(send, recv, bytes, ncclUint8, comm, s);
    if (r != ncclSuccess) {
      err = std::string("ncclAllGather: ") + nccl().error_string(r);
      return GP_NCCL;
    }
    return GP_OK;
  }
};

// ---------------------------------------------------------------- in-process group
// One generation-counted host barrier plus per-rank receive buffers and events.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<void*> recv;            // each rank's current receive buffer
  std::vector<cudaEvent_t> copied;    // rank k's copies into every peer issued
  std::vector<cudaEvent_t> recv_free; // rank k finished reading its receive buffer
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct LocalTransport : Transport {
  std::shared_ptr<LocalGroup> g;
  int rank = 0;
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t s, std::string& err) override {
    LocalGroup& G = *g;
    G.recv[rank] = recv;
    G.barrier();  // every rank published its receive buffer (and its last recv_free record)
    for (int k = 0; k < G.n; ++k) {
      cudaStreamWaitEvent(s, G.recv_free[k], 0);  // peer k is done reading its previous contents
      const cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t*>(G.recv[k]) + static_cast<size_t>(rank) * bytes,
                                            send, bytes, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) {
        err = std::string("local allgather: ") + cudaGetErrorString(e);
        return GP_CUDA;
      }
    }
    cudaEventRecord(G.copied[rank], s);
    G.barrier();  // every rank recorded its copies
    for (int k = 0; k < G.n; ++k) cudaStreamWaitEvent(s, G.copied[k], 0);
    G.barrier();  // no rank re-records `copied` before every peer waited on it
    return GP_OK;
  }
  void release(cudaStream_t s) { cudaEventRecord(g->recv_free[rank], s); }
};

}  // namespace
}  // namespace gp

struct gp_dp {
  gp_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  uint64_t d = 0, r = 0;
  gp_pipeline_config cfg{};
  int ef = 0;                        // 1: f64 error feedback (gp_encode_topr_ef64)
  std::unique_ptr<gp::Transport> tr;
  gp::LocalTransport* local = nullptr;
  uint64_t cap = 0;                  // gp_max_container_bytes
  uint8_t* send = nullptr;           // [cap]
  uint8_t* recv = nullptr;           // [nranks * cap]
  uint64_t* len = nullptr;           // device length word [1] + gathered lengths [nranks]
  double* residual = nullptr;        // [d] with ef
  uint64_t* h_sizes = nullptr;       // pinned [nranks + 1]: lengths + this rank's status word
  std::string err;
};

using namespace gp;

namespace {

int dp_alloc(gp_dp* dp) {
  dp->cap = gp_max_container_bytes(dp->d, dp->r, &dp->cfg);
  cudaError_t e = cudaSetDevice(dp->ctx->device);
  if (e == cudaSuccess) e = cudaMalloc(&dp->send, dp->cap);
  if (e == cudaSuccess && dp->nranks > 1) e = cudaMalloc(&dp->recv, dp->cap * dp->nranks);
  if (e == cudaSuccess) e = cudaMalloc(&dp->len, sizeof(uint64_t) * (dp->nranks + 1));
  if (e == cudaSuccess && dp->ef) e = cudaMalloc(&dp->residual, sizeof(double) * dp->d);
  if (e == cudaSuccess && dp->ef) e = cudaMemset(dp->residual, 0, sizeof(double) * dp->d);
  if (e == cudaSuccess) e = cudaMallocHost(&dp->h_sizes, sizeof(uint64_t) * (dp->nranks + 1));
  if (e != cudaSuccess) return set_error(dp->ctx, GP_CUDA, std::string("dp: ") + cudaGetErrorString(e));
  return GP_OK;
}

void dp_free(gp_dp* dp) {
  cudaFree(dp->send);
  cudaFree(dp->recv);
  cudaFree(dp->len);
  cudaFree(dp->residual);
  if (dp->h_sizes) cudaFreeHost(dp->h_sizes);
}

int dp_check(gp_ctx* ctx, uint64_t d, uint64_t r, const gp_pipeline_config* cfg, int nranks, int rank) {
  if (!ctx || !cfg) return GP_ERROR;
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(ctx, GP_ERROR, "dp: bad rank / world size");
  if (d < 1 || r < 1 || r > d || d > ctx->max_d) return set_error(ctx, GP_ERROR, "dp: bad d / r for this context");
  return GP_OK;
}

}  // namespace

extern "C" {

int gp_dp_unique_id(uint8_t* out_id) {
  if (!out_id) return GP_ERROR;
  if (!nccl().ok()) return GP_NCCL;
  ncclUniqueId id;
  if (nccl().get_unique_id(&id) != ncclSuccess) return GP_NCCL;
  static_assert(sizeof(ncclUniqueId) == GP_DP_UNIQUE_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out_id, &id, sizeof(id));
  return GP_OK;
}

int gp_dp_create(gp_ctx* ctx, const uint8_t* id, int nranks, int rank, uint64_t d, uint64_t r,
                 const gp_pipeline_config* cfg, int ef, gp_dp** out) {
  if (!out) return GP_ERROR;
  *out = nullptr;
  int rc = dp_check(ctx, d, r, cfg, nranks, rank);
  if (rc != GP_OK) return rc;
  if (nranks > 1 && !id) return set_error(ctx, GP_ERROR, "dp: NCCL unique id required");
  auto* dp = new gp_dp;
  dp->ctx = ctx;
  dp->nranks = nranks;
  dp->rank = rank;
  dp->d = d;
  dp->r = r;
  dp->cfg = *cfg;
  dp->ef = ef ? 1 : 0;
  if (nranks > 1) {
    if (!nccl().ok()) {
      delete dp;
      return set_error(ctx, GP_NCCL, "dp: libnccl.so.2 not loadable");
    }
    auto t = std::make_unique<NcclTransport>();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    cudaSetDevice(ctx->device);
    const ncclResult_t nr = nccl().comm_init_rank(&t->comm, nranks, uid, rank);
    if (nr != ncclSuccess) {
      delete dp;
      return set_error(ctx, GP_NCCL, std::string("ncclCommInitRank: ") + nccl().error_string(nr));
    }
    t->owned = true;
    dp->tr = std::move(t);
  }
  rc = dp_alloc(dp);
  if (rc != GP_OK) {
    dp_free(dp);
    delete dp;
    return rc;
  }
  *out = dp;
  return GP_OK;
}

int gp_dp_create_local(gp_ctx** ctxs, int nranks, uint64_t d, uint64_t r, const gp_pipeline_config* cfg, int ef,
                       gp_dp** out) {
  if (!ctxs || !out || nranks < 1) return GP_ERROR;
  auto g = std::make_shared<LocalGroup>();
  g->n = nranks;
  g->recv.assign(nranks, nullptr);
  g->copied.assign(nranks, nullptr);
  g->recv_free.assign(nranks, nullptr);
  int rc = GP_OK;
  for (int k = 0; k < nranks && rc == GP_OK; ++k) {
    out[k] = nullptr;
    rc = dp_check(ctxs[k], d, r, cfg, nranks, k);
    if (rc != GP_OK) break;
    cudaSetDevice(ctxs[k]->device);
    cudaEventCreateWithFlags(&g->copied[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->recv_free[k], cudaEventDisableTiming);
    auto* dp = new gp_dp;
    dp->ctx = ctxs[k];
    dp->nranks = nranks;
    dp->rank = k;
    dp->d = d;
    dp->r = r;
    dp->cfg = *cfg;
    dp->ef = ef ? 1 : 0;
    auto t = std::make_unique<LocalTransport>();
    t->g = g;
    t->rank = k;
    dp->local = t.get();
    dp->tr = std::move(t);
    rc = dp_alloc(dp);
    out[k] = dp;
  }
  if (rc != GP_OK) {
    for (int k = 0; k < nranks; ++k)
      if (out[k]) gp_dp_destroy(out[k]), out[k] = nullptr;
  }
  return rc;
}

int gp_dp_step(gp_dp* dp, const float* d_grad, uint64_t seed, int step, float* d_mean, void* stream) {
  if (!dp || !d_grad || !d_mean) return GP_ERROR;
  gp_ctx* ctx = dp->ctx;
  auto s = static_cast<cudaStream_t>(stream);
  gp_pipeline_config cfg = dp->cfg;
  cfg.seed = pipeline_seed_h(seed, dp->rank, step);
  const int n = dp->nranks;
  int rc = dp->ef ? gp_encode_topr_ef64(ctx, d_grad, dp->residual, dp->d, dp->r, &cfg, dp->send, dp->cap, dp->len,
                                        stream)
                  : gp_encode_topr(ctx, d_grad, dp->d, dp->r, &cfg, dp->send, dp->cap, dp->len, stream);
  if (rc != GP_OK) return rc;
  if (n == 1) {  // no exchange: the device-side length drives the decode, no host sync
    gp_ctx_set_decode_overwrite(ctx, 1);
    rc = gp_decode_accumulate_dlen(ctx, dp->send, dp->cap, dp->len, &dp->cfg, d_mean, dp->d, 1.0f, stream);
    gp_ctx_set_decode_overwrite(ctx, 0);
    return rc;
  }
  // lengths first
  rc = dp->tr->allgather(dp->len, dp->len + 1, sizeof(uint64_t), s, dp->err);
  if (rc != GP_OK) return set_error(ctx, rc, dp->err);
  // the step's one host sync: the lengths and this rank's encode status
  cudaMemcpyAsync(dp->h_sizes, dp->len + 1, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s);
  const int st = gp_ctx_status(ctx, stream);  // synchronises the stream
  if (st != GP_OK) {
    if (dp->local) dp->local->release(s);
    return st;
  }
  uint64_t mx = 0;
  for (int k = 0; k < n; ++k) mx = std::max<uint64_t>(mx, dp->h_sizes[k]);
  if (mx > dp->cap) return set_error(ctx, GP_CAPACITY, "dp: a peer's container exceeds this rank's capacity");
  rc = dp->tr->allgather(dp->send, dp->recv, mx, s, dp->err);
  if (rc != GP_OK) return set_error(ctx, rc, dp->err);
  const float scale = 1.0f / static_cast<float>(n);
  for (int k = 0; k < n && rc == GP_OK; ++k) {  // worker order (harness.cpp:274-284)
    gp_ctx_set_decode_overwrite(ctx, k == 0 ? 1 : 0);
    rc = gp_decode_accumulate_hint(ctx, dp->recv + static_cast<size_t>(k) * mx, dp->h_sizes[k], &dp->cfg, d_mean,
                                   dp->d, scale, stream);
  }
  gp_ctx_set_decode_overwrite(ctx, 0);
  if (dp->local) dp->local->release(s);
  return rc;
}

const double* gp_dp_residual(const gp_dp* dp) { return dp ? dp->residual : nullptr; }

int gp_dp_destroy(gp_dp* dp) {
  if (!dp) return GP_ERROR;
  cudaSetDevice(dp->ctx->device);
  cudaDeviceSynchronize();
  dp_free(dp);
  delete dp;
  return GP_OK;
}

}  // extern "C"
