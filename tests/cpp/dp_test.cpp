// dp_test.cpp — drives gp_dp_step (the C-ABI data-parallel step) from C++,
// one host thread per rank (TEST PROGRAM, tests/test_gpu_cpp_dp.py).
//
//   dp_test local|nccl NRANKS D R INDEX VALUE FPR STEPS EF INDIR OUTDIR
//
// Reads INDIR/g_<k>.bin (f32[D]) per rank; `local` runs an in-process group
// of NRANKS contexts on device 0 (gp_dp_create_local), `nccl` a single-rank
// NCCL communicator per process (NRANKS must be 1 here: one GPU).  After each
// step every rank's dense mean goes to OUTDIR/mean_<k>_<step>.bin (and, with
// EF, the f64 residual to OUTDIR/res_<k>_<step>.bin).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gradpack_b200.h"

static void die(const char* what, int rc, gp_ctx* ctx = nullptr) {
  std::fprintf(stderr, "%s failed: %d %s\n", what, rc, ctx ? gp_last_error(ctx) : "");
  std::exit(1);
}

template <typename T>
static std::vector<T> read_file(const std::string& path, size_t n) {
  std::vector<T> v(n);
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f || std::fread(v.data(), sizeof(T), n, f) != n) {
    std::fprintf(stderr, "cannot read %s\n", path.c_str());
    std::exit(1);
  }
  std::fclose(f);
  return v;
}

template <typename T>
static void write_file(const std::string& path, const std::vector<T>& v) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f || std::fwrite(v.data(), sizeof(T), v.size(), f) != v.size()) {
    std::fprintf(stderr, "cannot write %s\n", path.c_str());
    std::exit(1);
  }
  std::fclose(f);
}

int main(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: dp_test local|nccl NRANKS D R INDEX VALUE FPR STEPS EF INDIR OUTDIR\n");
    return 2;
  }
  const std::string mode = argv[1];
  const int n = std::atoi(argv[2]);
  const uint64_t d = std::strtoull(argv[3], nullptr, 10), r = std::strtoull(argv[4], nullptr, 10);
  gp_pipeline_config cfg;
  gp_pipeline_config_default(&cfg);
  cfg.index_method = static_cast<uint8_t>(std::atoi(argv[5]));
  cfg.value_method = static_cast<uint8_t>(std::atoi(argv[6]));
  cfg.fpr = std::atof(argv[7]);
  const int steps = std::atoi(argv[8]), ef = std::atoi(argv[9]);
  const std::string indir = argv[10], outdir = argv[11];

  std::vector<gp_ctx*> ctx(n, nullptr);
  std::vector<gp_dp*> dp(n, nullptr);
  std::vector<float*> grad(n, nullptr), mean(n, nullptr);
  std::vector<cudaStream_t> st(n);
  for (int k = 0; k < n; ++k) {
    int rc = gp_ctx_create(0, d, &ctx[k]);
    if (rc) die("gp_ctx_create", rc);
    const std::vector<float> g = read_file<float>(indir + "/g_" + std::to_string(k) + ".bin", d);
    cudaMalloc(&grad[k], d * sizeof(float));
    cudaMalloc(&mean[k], d * sizeof(float));
    cudaMemcpy(grad[k], g.data(), d * sizeof(float), cudaMemcpyHostToDevice);
    cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking);
  }
  if (mode == "local") {
    const int rc = gp_dp_create_local(ctx.data(), n, d, r, &cfg, ef, dp.data());
    if (rc) die("gp_dp_create_local", rc, ctx[0]);
  } else {
    if (n != 1) die("nccl mode on one GPU needs NRANKS = 1", 1);
    uint8_t id[GP_DP_UNIQUE_ID_BYTES];
    int rc = gp_dp_unique_id(id);
    if (rc) die("gp_dp_unique_id", rc);
    rc = gp_dp_create(ctx[0], id, 1, 0, d, r, &cfg, ef, &dp[0]);
    if (rc) die("gp_dp_create", rc, ctx[0]);
  }
  for (int step = 0; step < steps; ++step) {
    std::vector<int> rcs(n, 0);
    std::vector<std::thread> th;
    for (int k = 0; k < n; ++k)
      th.emplace_back([&, k] { rcs[k] = gp_dp_step(dp[k], grad[k], 1, step, mean[k], st[k]); });
    for (auto& t : th) t.join();
    for (int k = 0; k < n; ++k) {
      if (rcs[k]) die("gp_dp_step", rcs[k], ctx[k]);
      const int s2 = gp_ctx_status(ctx[k], st[k]);
      if (s2) die("device status", s2, ctx[k]);
      std::vector<float> h(d);
      cudaMemcpy(h.data(), mean[k], d * sizeof(float), cudaMemcpyDeviceToHost);
      write_file(outdir + "/mean_" + std::to_string(k) + "_" + std::to_string(step) + ".bin", h);
      if (ef) {
        std::vector<double> e(d);
        cudaMemcpy(e.data(), gp_dp_residual(dp[k]), d * sizeof(double), cudaMemcpyDeviceToHost);
        write_file(outdir + "/res_" + std::to_string(k) + "_" + std::to_string(step) + ".bin", e);
      }
    }
  }
  for (int k = 0; k < n; ++k) {
    gp_dp_destroy(dp[k]);
    gp_ctx_destroy(ctx[k]);
  }
  std::printf("ok\n");
  return 0;
}
