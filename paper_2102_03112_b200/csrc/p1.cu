// p1.cu — K8: P1 random selection (p1_select, bloom.cpp:140-154), bit-exact.
//
// Reference: partial Fisher-Yates over a copy of P — for i < r:
// j_i = i + below(n - i) (CounterRng stream, rng.hpp:52-59), swap(pool[i],
// pool[j_i]) — then sort(pool[0, r)).  Parallel form:
//   * every draw at once: draw i uses stream position i unless an earlier
//     below() rejected (probability ~n/2^64 per draw); any rejection sends the
//     whole draw list through an exact sequential kernel instead;
//   * slot i is final after step i (later steps only touch slots > i), and it
//     receives the value slot j_i held just before step i.  Slot s holds,
//     before step i, B(i') for the latest i' < i with j_i' = s, else P[s],
//     where B(t) is the value slot t held just before step t (same rule with
//     s = t).  Sorting the (j_i, i) pairs stably by j groups the steps per
//     target, so both lookups are short walks; each selected value is found by
//     following its chain;
//   * the r final values (indices into P) are flagged and compacted in P
//     order, which is the reference's final sort.
#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace gp {

namespace {

__device__ __forceinline__ bool p1_active(const Plan* plan) { return plan->index_method == GP_INDEX_BLOOM_P1; }

__global__ void p1_draws(Plan* plan, uint32_t* __restrict__ jkey, uint32_t* __restrict__ step, uint32_t* reject,
                         const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p1_active(plan)) return;
  const uint64_t n = plan->n_pos, r = plan->r;
  const uint64_t seed = hash64(plan->seed_a, plan->seed_b);  // derive_selection_seed (pipeline.cpp:23-25)
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t span = n - i;
    const uint64_t v = rng_at(seed, i);
    if (v > below_bound(span)) *reject = 1;
    jkey[i] = static_cast<uint32_t>(i + v % span);
    step[i] = static_cast<uint32_t>(i);
  }
}

// exact fallback: sequential stream with rejections (taken with probability ~r*n/2^64)
__global__ void p1_draws_serial(Plan* plan, uint32_t* __restrict__ jkey, const uint32_t* reject,
                                const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p1_active(plan) || !*reject || threadIdx.x != 0) return;
  const uint64_t n = plan->n_pos, r = plan->r;
  const uint64_t seed = hash64(plan->seed_a, plan->seed_b);
  uint64_t pos = 0;
  for (uint64_t i = 0; i < r; ++i) {
    const uint64_t span = n - i, bound = below_bound(span);
    uint64_t v = rng_at(seed, pos++);
    while (v > bound) v = rng_at(seed, pos++);
    jkey[i] = static_cast<uint32_t>(i + v % span);
  }
}

__global__ void p1_reset(uint32_t* reject) {
  gp_pdl_wait(); *reject = 0; }

// end (inclusive) of each target's group in the sorted pairs
__global__ void p1_groups(const Plan* plan, const uint32_t* __restrict__ skey, uint32_t* __restrict__ gend,
                          const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p1_active(plan)) return;
  const uint64_t r = plan->r;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < r;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (t + 1 == r || skey[t + 1] != skey[t]) gend[skey[t]] = static_cast<uint32_t>(t);
}

// latest step i' < i that targeted slot s, or UINT32_MAX
__device__ __forceinline__ uint32_t latest_before(const uint32_t* skey, const uint32_t* sstep, const uint32_t* gend,
                                                  uint32_t s, uint32_t i) {
  uint32_t e = gend[s];
  if (e == 0xFFFFFFFFu) return 0xFFFFFFFFu;
  while (true) {
    if (skey[e] != s) return 0xFFFFFFFFu;
    if (sstep[e] < i) return sstep[e];
    if (e == 0) return 0xFFFFFFFFu;
    --e;
  }
}

__global__ void p1_resolve(const Plan* plan, const uint32_t* __restrict__ jkey, const uint32_t* __restrict__ skey,
                           const uint32_t* __restrict__ sstep, const uint32_t* __restrict__ gend,
                           uint8_t* __restrict__ flags, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p1_active(plan)) return;
  const uint64_t r = plan->r;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < r;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = jkey[i];
    uint32_t t = latest_before(skey, sstep, gend, s, static_cast<uint32_t>(i));
    uint32_t value = s;  // index into P: P[s] unless an earlier step wrote slot s
    while (t != 0xFFFFFFFFu) {  // value = B(t): slot t just before step t
      value = t;
      t = latest_before(skey, sstep, gend, t, t);
    }
    flags[value] = 1;
  }
}

__global__ void p1_bits(const Plan* plan, const uint8_t* __restrict__ flags, uint32_t* __restrict__ selbits,
                        const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !p1_active(plan)) return;
  const uint64_t n = plan->n_pos;
  const uint64_t nw = (n + 31) / 32;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32; w < nw; w += warps) {
    const uint64_t p = 32 * w + (threadIdx.x & 31);
    const unsigned bits = __ballot_sync(kFull, p < n && flags[p]);
    if ((threadIdx.x & 31) == 0) selbits[w] = bits;
  }
}

}  // namespace

void launch_radix_sort(gp_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* ktmp, uint32_t* vtmp,
                       const uint64_t* n_dev, uint64_t n_bound, int bits, cudaStream_t s, bool hist_ready = false,
                       const float* fit_v = nullptr, double* fit_t = nullptr);
void launch_flags_compact(gp_ctx* ctx, int method, uint64_t n_bound, cudaStream_t s);

void launch_select_p1(gp_ctx* ctx, uint64_t n_bound, uint64_t r_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  uint32_t* reject = w.p2_alloc + 1;
  GP_LAUNCH(ctx, p1_reset, 1, 1, 0, s, reject);
  GP_LAUNCH(ctx, p1_draws, grid_for(ctx, r_bound, 256), 256, 0, s, w.plan, w.u32a, w.u32b, reject, w.status);
  GP_LAUNCH(ctx, p1_draws_serial, 1, 32, 0, s, w.plan, w.u32a, reject, w.status);
  // stable sort of (target, step) by target; a copy of the targets stays in u32d... sort in place on copies
  cudaMemcpyAsync(w.f64a, w.u32a, r_bound * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);  // unsorted targets
  int bits = 8;
  while (bits < 32 && (1ull << bits) < n_bound) bits += 8;
  launch_radix_sort(ctx, w.u32a, w.u32b, w.u32c, w.u32d, &w.plan->r, r_bound, bits, s);
  fill_async(ctx, w.first_touch, 0xFF, n_bound * sizeof(uint32_t), s);
  fill_async(ctx, w.flags, 0, n_bound, s);
  GP_LAUNCH(ctx, p1_groups, grid_for(ctx, r_bound, 256), 256, 0, s, w.plan, w.u32a, w.first_touch, w.status);
  GP_LAUNCH(ctx, p1_resolve, grid_for(ctx, r_bound, 256), 256, 0, s, w.plan,
            reinterpret_cast<const uint32_t*>(w.f64a), w.u32a, w.u32b, w.first_touch, w.flags, w.status);
  GP_LAUNCH(ctx, p1_bits, grid_for(ctx, n_bound, 256), 256, 0, s, w.plan, w.flags, w.selbits, w.status);
  launch_flags_compact(ctx, GP_INDEX_BLOOM_P1, n_bound, s);
}

}  // namespace gp
