// values_fit.cu — K11-K15: the piecewise-polynomial value codec
// (value_compress / value_decompress, curvefit.cpp:26-174, :285-356, :388-542).
//
// Encode (values in ws.values, n = plan->n_values):
//   fit_keys     : descending, stable sort keys (-0.0 canonicalised to +0.0, the
//                  reference comparator treats them as equal) + sign split l
//   radix sort   : 4 x 8-bit stable passes → map[sorted_pos] = original pos
//   fit_prepare  : identity flag; folded sequence t (negatives reversed and
//                  negated behind the sign split, curvefit.cpp:442-446)
//   fit_segment  : greedy max-chord-deviation splitting per sign part, fp64
//                  with no contraction and lowest-index ties (curvefit.cpp:50-99)
//                  — bit-exact boundaries
//   fit_accumulate / fit_solve : least squares per segment on t in [-1, 1]
//                  (degree <= 7 in registers; degree 8..60: fit_solve_wide).  The reference solves the Vandermonde system
//                  with Eigen's column-pivoted QR (curvefit.cpp:154); here the
//                  normal equations are formed in the Legendre basis (Gram
//                  matrix ~ diagonal, condition ~ 2*degree+1) with fixed-order
//                  fp64 reductions, solved by Cholesky, mapped to t-monomials,
//                  then expanded to x-monomials exactly as curvefit.cpp:157-172.
//                  Coefficients agree with the reference within f32 rounding
//                  (tolerance-checked).
//   fit_emit / reorder_pack : serialize_fit + the bit-packed map
// Decode: fit_parse (parse_fit + reorder checks), fit_unpack_eval (reorder
// entries + permutation check, fp64 Horner without FMA, sign unfold,
// permutation scatter, one pass) — bit-exact for a given container.
#include <cooperative_groups.h>

#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace cg = cooperative_groups;

namespace gp {

namespace {

constexpr int kMaxDeg = 7;                  // register path (fit_accumulate / fit_solve)
constexpr int kCps = kMaxDeg + 1;
constexpr int kWideDeg = 60;                // fit_poly's range (curvefit.cpp:130)
constexpr int kWideCps = kWideDeg + 1;
constexpr int kChunk = 2048;                // points per accumulate block
constexpr int kAcc = 36 + 8;                // Gram upper triangle (<= 36) + rhs (<= 8)

// coefficients of segment s live at coeffs[s * cps + j], cps = the serialized
// coeffs_per_segment (FORMAT.md: degree + 1 for poly, 4 for dexp)
__device__ __forceinline__ uint32_t cps_of(const Plan* plan) { return plan->fit_kind ? 4u : plan->degree + 1u; }

__device__ __forceinline__ bool fit_active(const Plan* plan) {
  return plan->value_method == GP_VALUE_FIT_POLY || plan->value_method == GP_VALUE_FIT_DEXP;
}
// the piecewise-polynomial encode stages: skipped when a dexp model stands
__device__ __forceinline__ bool poly_active(const Plan* plan) { return fit_active(plan) && plan->fit_kind == 0; }

constexpr double kExpClamp = 700.0;
__device__ __forceinline__ double safe_exp(double x) { return exp(x < kExpClamp ? x : kExpClamp); }

// eval_dexp (curvefit.cpp:365-368)
__device__ __forceinline__ double eval_dexp(const float* c, double x) {
  return __dadd_rn(__dmul_rn(static_cast<double>(c[0]), safe_exp(__dmul_rn(static_cast<double>(c[1]), x))),
                   __dmul_rn(static_cast<double>(c[2]), safe_exp(__dmul_rn(static_cast<double>(c[3]), x))));
}

// Sort keys of sort_view (curvefit.cpp:26-39): descending, stable, -0.0 equal
// to +0.0 (operator>).  f32 values: one 32-bit key.  f64 values: the 64-bit
// key is sorted as two stable 32-bit LSD passes — the low word here (pass 1),
// the high word gathered through pass 1's permutation by fit_keys_hi.
__device__ __forceinline__ uint64_t desc_key64(double v) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  if (b == 0x8000000000000000ull) b = 0;
  const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}

// ghist != null (f32 values): the radix sort's four digit histograms are
// accumulated here too (shared bins, warp-aggregated), so the sort skips its
// own histogram pass over the keys
//
// gdense != null: the values are gathered here, v[j] = gdense[gsel[j]]
// (gather_values, pipeline.cpp:38-54), and stored to vout for the later passes.
__global__ void fit_keys(const ValSrc values, Plan* plan, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ idx, uint32_t* __restrict__ ghist, const float* __restrict__ gdense,
                         const uint32_t* __restrict__ gsel, float* __restrict__ vout, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t cnt;
  __shared__ uint32_t h[4][256];
  if (failed(status) || !fit_active(plan)) return;
  if (threadIdx.x == 0) cnt = 0;
  if (ghist)
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) h[i >> 8][i & 255] = 0;
  __syncthreads();
  const uint64_t n = plan->n_values;
  const int lane = threadIdx.x & 31;
  uint32_t nonneg = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x); i0 < n; i0 += stride) {  // warp-uniform
    const uint64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    uint32_t key = 0;
    if (ok) {
      if (values.f64) {
        const double v = values.f64[i];
        key = static_cast<uint32_t>(desc_key64(v));
        nonneg += v >= 0.0 ? 1u : 0u;
      } else {
        float v;
        if (gdense) {
          v = gdense[gsel[i]];
          vout[i] = v;
        } else {
          v = values.f32[i];
        }
        uint32_t b = __float_as_uint(v);
        if (b == 0x80000000u) b = 0;  // -0.0 == +0.0 under operator>
        const uint32_t asc = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
        key = ~asc;  // ascending key order == descending value order
        nonneg += v >= 0.0f ? 1u : 0u;
      }
      keys[i] = key;
      idx[i] = static_cast<uint32_t>(i);
    }
    if (ghist) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t dig = ok ? (key >> (8 * p)) & 255u : 256u;
        const unsigned peers = __match_any_sync(kFull, dig);
        if (ok && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&h[p][dig], __popc(peers));
      }
    }
  }
  nonneg = warp_sum(nonneg);
  if ((threadIdx.x & 31) == 0 && nonneg) atomicAdd(&cnt, nonneg);
  __syncthreads();
  if (threadIdx.x == 0 && cnt) atomicAdd(&plan->sign_split, cnt);
  if (ghist)
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
      if (h[i >> 8][i & 255]) atomicAdd(&ghist[i], h[i >> 8][i & 255]);
}

// f64 pass 2 keys: the high words in pass 1's order
__global__ void fit_keys_hi(const double* __restrict__ v64, const Plan* plan, const uint32_t* __restrict__ idx,
                            uint32_t* __restrict__ keys, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !fit_active(plan)) return;
  const uint64_t n = plan->n_values;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = static_cast<uint32_t>(desc_key64(v64[idx[i]]) >> 32);
}

// t[s] and the identity flag; map = sorted idx
__global__ void fit_prepare(const ValSrc values, const uint32_t* __restrict__ map, Plan* plan,
                            double* __restrict__ t, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !fit_active(plan)) return;
  const uint64_t n = plan->n_values;
  const uint64_t l = plan->sign_split;
  bool ident = true;
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (map[s] != s) ident = false;
    t[s] = s < l ? values[map[s]] : -values[map[n - 1 - (s - l)]];
  }
  // one plain store per block at most (per-warp atomics on the flag serialised: ~10 us at C4)
  if (__syncthreads_or(!ident) && threadIdx.x == 0) plan->identity = 0;
}

// ---------------------------------------------------------------- segmentation
// segment() (curvefit.cpp:69-99) is a best-first expansion: repeatedly split
// the live piece of largest deviation (ties: lowest begin) until the budget is
// reached.  The device keeps the expansion tree in global memory and runs it
// in ROUNDS inside one cooperative kernel:
//   1. evaluate the pending nodes (make_piece: max squared chord deviation,
//      lowest index on ties) — a grid sweep over the disjoint ranges;
//   2. one thread replays the reference's selection loop on a binary heap
//      keyed (dev desc, begin asc), popping while the top's children are
//      known (the budget's last split needs none);
//   3. when it stalls, the children of EVERY heap node not yet expanded
//      become the next round's pending nodes (only heap nodes can ever be
//      popped, and their ranges are disjoint, so a round sweeps <= n points).
// A round costs one sweep however many pieces it evaluates, so budgets up to
// 0xffff (part_budget, curvefit.cpp:424-428) take about log2(budget) rounds on
// balanced data instead of one sweep per split.  Segments are the unsplit
// nodes in tree (= begin) order.
struct SegNode {
  uint32_t begin, end;  // part-relative range
  uint32_t arg, live;
  double dev;
  uint32_t left, split;  // first child id (right = left + 1) or kNoChild; popped by the replay
};
constexpr uint32_t kNoChild = 0xFFFFFFFFu;
constexpr int kFewRanges = 8;  // rounds with <= 8 pending nodes reduce partials instead of atomics
constexpr int kSmallBudget = 64;  // budgets up to this run the replicated piece list (no tree)

// control words shared by the blocks of fit_segment_coop (global memory)
struct SegState {
  uint32_t npend, nnodes, heapn, pops, done, overflow, pad0, pad1;
};

__device__ __forceinline__ bool seg_before(const SegNode& a, const SegNode& b) {  // a pops before b
  return a.dev > b.dev || (a.dev == b.dev && a.begin < b.begin);
}

__device__ void heap_push(uint32_t* heap, uint32_t& n, const SegNode* nodes, uint32_t id) {
  uint32_t i = n++;
  while (i > 0) {
    const uint32_t p = (i - 1) / 2;
    if (!seg_before(nodes[id], nodes[heap[p]])) break;
    heap[i] = heap[p];
    i = p;
  }
  heap[i] = id;
}

__device__ uint32_t heap_pop(uint32_t* heap, uint32_t& n, const SegNode* nodes) {
  const uint32_t top = heap[0];
  const uint32_t last = heap[--n];
  uint32_t i = 0;
  while (true) {
    const uint32_t l = 2 * i + 1;
    if (l >= n) break;
    const uint32_t c = (l + 1 < n && seg_before(nodes[heap[l + 1]], nodes[heap[l]])) ? l + 1 : l;
    if (!seg_before(nodes[heap[c]], nodes[last])) break;
    heap[i] = heap[c];
    i = c;
  }
  if (n) heap[i] = last;
  return top;
}

__device__ __forceinline__ void make_live(SegNode& p, uint32_t mp) {
  if (!(p.dev > 0.0)) p.arg = 0;
  p.live = (p.dev > 0.0 && p.arg - p.begin >= mp && p.end - p.arg >= mp) ? 1u : 0u;
}

// Few pending ranges: every block scans a slice of each, writes its block-best
// (dev, arg) to a double-buffered partial array; after grid.sync() block 0
// reduces the partials in block order (same tie rule) into the nodes.
// Every block reduces (replicated, identical results in sres); block 0 also
// stores them in the nodes.  rb/re give the ranges when nodes is null.
__device__ void seg_sweep_few(const double* __restrict__ t, SegNode* nodes, const uint32_t* pend, int nr,
                              const uint32_t* rb, const uint32_t* re, double* pdev, uint32_t* parg, double* sdev,
                              uint32_t* sarg, double* sres_dev, uint32_t* sres_arg, cg::grid_group& grid) {
  const uint32_t G = gridDim.x;
  for (int q = 0; q < nr; ++q) {
    const uint32_t b = nodes ? nodes[pend[q]].begin : rb[q], e = nodes ? nodes[pend[q]].end : re[q];
    const uint32_t len = e - b;
    double best = 0.0;
    uint32_t arg = 0;
    if (len >= 3) {
      const double y0 = t[b];
      const double slope = __ddiv_rn(__dsub_rn(t[e - 1], y0), static_cast<double>(len - 1));
      for (uint32_t i = b + 1 + blockIdx.x * blockDim.x + threadIdx.x; i + 1 < e; i += G * blockDim.x) {
        const double pred = __dadd_rn(y0, __dmul_rn(slope, static_cast<double>(i - b)));
        const double d = __dsub_rn(t[i], pred);
        const double d2 = __dmul_rn(d, d);
        if (d2 > best) {
          best = d2;
          arg = i;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(kFull, best, o);
      const uint32_t oa = __shfl_xor_sync(kFull, arg, o);
      if (ob > best || (ob == best && ob > 0.0 && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      sdev[threadIdx.x >> 5] = best;
      sarg[threadIdx.x >> 5] = arg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = 0.0;
      uint32_t aa = 0;
      for (uint32_t w = 0; w < blockDim.x / 32; ++w)
        if (sdev[w] > bb || (sdev[w] == bb && bb > 0.0 && sarg[w] < aa)) {
          bb = sdev[w];
          aa = sarg[w];
        }
      pdev[q * G + blockIdx.x] = bb;
      parg[q * G + blockIdx.x] = aa;
    }
    __syncthreads();
  }
  grid.sync();
  for (int q = 0; q < nr; ++q) {
    double best = 0.0;
    uint32_t arg = 0;
    for (uint32_t j = threadIdx.x; j < G; j += blockDim.x) {
      const double v = __ldcg(&pdev[q * G + j]);
      const uint32_t a = __ldcg(&parg[q * G + j]);
      if (v > best || (v == best && best > 0.0 && a < arg)) {
        best = v;
        arg = a;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(kFull, best, o);
      const uint32_t oa = __shfl_xor_sync(kFull, arg, o);
      if (ob > best || (ob == best && ob > 0.0 && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      sdev[threadIdx.x >> 5] = best;
      sarg[threadIdx.x >> 5] = arg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bb = 0.0;
      uint32_t aa = 0;
      for (uint32_t w = 0; w < blockDim.x / 32; ++w)
        if (sdev[w] > bb || (sdev[w] == bb && bb > 0.0 && sarg[w] < aa)) {
          bb = sdev[w];
          aa = sarg[w];
        }
      sres_dev[q] = bb;
      sres_arg[q] = aa;
      if (nodes && blockIdx.x == 0) {
        nodes[pend[q]].dev = bb;
        nodes[pend[q]].arg = aa;
      }
    }
    __syncthreads();
  }
}

// Many pending ranges: the interior points of all of them, concatenated
// (off = exclusive prefix of interior lengths), 32 consecutive points per
// thread; the maximum by atomicMax on the non-negative doubles' bit patterns,
// then the lowest index attaining it by atomicMin (two sweeps, exact ties).
constexpr uint32_t kSweepRun = 32;
__device__ __forceinline__ uint32_t find_pend(const uint64_t* off, uint32_t npend, uint64_t j) {
  uint32_t lo = 0, hi = npend;  // last q with off[q] <= j
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (off[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

template <bool kArg>
__device__ void seg_sweep_many_pass(const double* __restrict__ t, SegNode* nodes, const uint32_t* pend,
                                    const uint64_t* off, uint32_t npend) {
  const uint64_t total = off[npend];
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j0 = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * kSweepRun; j0 < total;
       j0 += nthreads * kSweepRun) {
    const uint64_t j1 = j0 + kSweepRun < total ? j0 + kSweepRun : total;
    uint32_t q = find_pend(off, npend, j0);
    uint64_t qend = off[q + 1];
    while (true) {
      SegNode* nd = &nodes[pend[q]];
      const uint32_t b = nd->begin, e = nd->end;
      const double y0 = t[b];
      const double slope = __ddiv_rn(__dsub_rn(t[e - 1], y0), static_cast<double>(e - b - 1));
      const double target = kArg ? __longlong_as_double(static_cast<long long>(
                                       *reinterpret_cast<volatile unsigned long long*>(&nd->dev)))
                                 : 0.0;
      const uint64_t stop = qend < j1 ? qend : j1;
      double best = 0.0;
      for (uint64_t j = j0; j < stop; ++j) {
        const uint32_t i = b + 1 + static_cast<uint32_t>(j - off[q]);
        const double pred = __dadd_rn(y0, __dmul_rn(slope, static_cast<double>(i - b)));
        const double d = __dsub_rn(t[i], pred);
        const double d2 = __dmul_rn(d, d);
        if (kArg) {
          if (d2 == target && target > 0.0) {
            atomicMin(&nd->arg, i);
            break;  // the run's lowest index
          }
        } else if (d2 > best) {
          best = d2;
        }
      }
      if (!kArg && best > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(&nd->dev),
                  static_cast<unsigned long long>(__double_as_longlong(best)));
      if (stop >= j1) break;
      j0 = stop;
      ++q;
      qend = off[q + 1];
    }
  }
}

__global__ void __launch_bounds__(256) fit_segment_coop(Plan* plan, const double* __restrict__ t, int degree,
                                                        int max_segments, double* pdev, uint32_t* parg,
                                                        SegNode* nodes, uint32_t* heap, uint32_t* pend,
                                                        uint64_t* off, SegState* st, uint32_t* seg_end,
                                                        uint64_t* chunk, uint32_t node_cap, uint32_t seg_cap,
                                                        uint32_t* status) {
  gp_pdl_wait();
  cg::grid_group grid = cg::this_grid();
  __shared__ double sdev[32];
  __shared__ uint32_t sarg[32];
  __shared__ double sres_dev[kFewRanges];
  __shared__ uint32_t sres_arg[kFewRanges];
  __shared__ uint64_t sh[40];
  __shared__ SegNode small[kSmallBudget];
  __shared__ int s_best;
  // uniform exit decisions only (every block must reach every grid.sync)
  if (failed(status) || !poly_active(plan)) return;
  const uint64_t n = plan->n_values;
  const uint32_t l = plan->sign_split;
  const uint32_t un = static_cast<uint32_t>(n);
  uint32_t pb[2], pe[2];
  int nparts = 0;
  if (l > 0) {
    pb[nparts] = 0;
    pe[nparts++] = l;
  }
  if (l < un) {
    pb[nparts] = l;
    pe[nparts++] = un;
  }
  const uint32_t mp = static_cast<uint32_t>(degree + 1 > 1 ? degree + 1 : 1);
  const uint32_t G = gridDim.x;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  int sweep = 0;
  uint32_t nseg = 0;  // replicated in every block
  bool overflow = false;
  // Automatic budgets (max_segments 0) depend only on each part's end points:
  // when every part gets at most one split (the BASELINE configs), the parts'
  // root sweeps share one grid sweep and one barrier, not one each
  bool joint = max_segments <= 0 && nparts > 0;
  long long jbudget[2] = {1, 1};
  for (int pi = 0; pi < nparts && joint; ++pi) {
    const uint32_t b = pb[pi], e = pe[pi], len = e - b;
    if (len >= 4) {  // part_budget (curvefit.cpp:101-110, :424-428)
      const double km = fabs(__dsub_rn(__dsub_rn(t[b], t[b + 1]), __dsub_rn(t[e - 2], t[e - 1])));
      const double p = ceil(2.0 * sqrt(km > 0.0 ? km : 0.0));
      const int kc = static_cast<int>(p) > 1 ? static_cast<int>(p) : 1;
      jbudget[pi] = kc + 1 < 0xffff ? kc + 1 : 0xffff;
    }
    joint = jbudget[pi] <= 2;
  }
  if (joint) {
    uint32_t rb[2], re[2];
    int nr = 0, slot[2] = {-1, -1};
    for (int pi = 0; pi < nparts; ++pi)
      if (jbudget[pi] == 2) {
        slot[pi] = nr;
        rb[nr] = pb[pi];
        re[nr++] = pe[pi];
      }
    if (nr > 0) {
      seg_sweep_few(t, nullptr, nullptr, nr, rb, re, pdev, parg, sdev, sarg, sres_dev, sres_arg, grid);
      ++sweep;
    }
    for (int pi = 0; pi < nparts; ++pi) {
      const uint32_t b = pb[pi], e = pe[pi], len = e - b;
      uint32_t split = 0;
      if (slot[pi] >= 0) {
        const double dv = sres_dev[slot[pi]];
        SegNode root{0, len, dv > 0.0 ? sres_arg[slot[pi]] - b : 0u, 0u, dv, kNoChild, 0u};
        make_live(root, mp);
        if (root.live) split = root.arg;
      }
      if (nseg + 2 > seg_cap) {
        overflow = true;
        break;
      }
      if (leader) {
        if (split) seg_end[nseg] = b + split;
        seg_end[nseg + (split ? 1 : 0)] = e;
      }
      nseg += split ? 2 : 1;
    }
    nparts = 0;  // done: skip the general loop below
  }
  for (int pi = 0; pi < nparts; ++pi) {
    const uint32_t b = pb[pi], e = pe[pi], len = e - b;
    long long budget;
    if (max_segments > 0) {  // curvefit.cpp:473-481
      const long long share = static_cast<long long>(max_segments) * static_cast<long long>(len) /
                              static_cast<long long>(n);
      budget = share > 1 ? share : 1;
      if (pi + 1 == nparts) {
        const long long used = static_cast<long long>(nseg);  // segments of part 0
        budget = max_segments - used > 1 ? max_segments - used : 1;
      }
    } else if (len < 4) {
      budget = 1;
    } else {  // part_budget (curvefit.cpp:101-110, :424-428)
      const double km = fabs(__dsub_rn(__dsub_rn(t[b], t[b + 1]), __dsub_rn(t[e - 2], t[e - 1])));
      const double p = ceil(2.0 * sqrt(km > 0.0 ? km : 0.0));
      const int kc = static_cast<int>(p) > 1 ? static_cast<int>(p) : 1;
      budget = kc + 1 < 0xffff ? kc + 1 : 0xffff;
    }
    if (budget <= 2) {  // at most one split: the root's, decided in every block (no tree, no replay)
      uint32_t split = 0;
      if (budget == 2) {
        const uint32_t rb = 0, re = len;
        seg_sweep_few(t + b, nullptr, nullptr, 1, &rb, &re, pdev + (sweep & 1) * kFewRanges * G,
                      parg + (sweep & 1) * kFewRanges * G, sdev, sarg, sres_dev, sres_arg, grid);
        ++sweep;
        SegNode root{0, len, sres_arg[0], 0u, sres_dev[0], kNoChild, 0u};
        make_live(root, mp);
        if (root.live) split = root.arg;
      }
      if (nseg + 2 > seg_cap) {
        overflow = true;
        break;
      }
      if (leader) {
        if (split) seg_end[nseg] = b + split;
        seg_end[nseg + (split ? 1 : 0)] = e;
      }
      nseg += split ? 2 : 1;
      continue;
    }
    if (budget <= kSmallBudget) {
      // small budgets (C5's max_segments = 8): the reference's loop with the piece
      // list replicated in every block — each split one sweep of its two
      // children, decided identically everywhere; no tree, no leader, no extra
      // grid barriers
      int np = 1;
      {
        const uint32_t rb = 0, re = len;
        seg_sweep_few(t + b, nullptr, nullptr, 1, &rb, &re, pdev + (sweep & 1) * kFewRanges * G,
                      parg + (sweep & 1) * kFewRanges * G, sdev, sarg, sres_dev, sres_arg, grid);
        ++sweep;
        if (threadIdx.x == 0) {
          small[0] = SegNode{0, len, sres_arg[0], 0u, sres_dev[0], kNoChild, 0u};
          make_live(small[0], mp);
        }
      }
      __syncthreads();
      while (np < budget) {
        if (threadIdx.x == 0) {
          int best = -1;
          for (int i = 0; i < np; ++i) {
            if (!small[i].live) continue;
            if (best < 0 || seg_before(small[i], small[best])) best = i;
          }
          s_best = best;
        }
        __syncthreads();
        const int best = s_best;
        if (best < 0) break;
        const SegNode pp = small[best];
        SegNode left{pp.begin, pp.arg, 0, 0u, 0.0, kNoChild, 0u}, right{pp.arg, pp.end, 0, 0u, 0.0, kNoChild, 0u};
        if (np + 1 < budget) {  // another split may follow: evaluate both children
          const uint32_t rb[2] = {pp.begin, pp.arg}, re[2] = {pp.arg, pp.end};
          seg_sweep_few(t + b, nullptr, nullptr, 2, rb, re, pdev + (sweep & 1) * kFewRanges * G,
                        parg + (sweep & 1) * kFewRanges * G, sdev, sarg, sres_dev, sres_arg, grid);
          ++sweep;
          left.arg = sres_arg[0];
          left.dev = sres_dev[0];
          right.arg = sres_arg[1];
          right.dev = sres_dev[1];
          make_live(left, mp);
          make_live(right, mp);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          small[best] = left;
          small[np] = right;
        }
        ++np;
        __syncthreads();
      }
      if (nseg + np > seg_cap) {
        overflow = true;
        break;
      }
      if (leader) {
        for (int i = 1; i < np; ++i) {  // by begin
          const SegNode v = small[i];
          int j = i;
          while (j > 0 && small[j - 1].begin > v.begin) {
            small[j] = small[j - 1];
            --j;
          }
          small[j] = v;
        }
        for (int i = 0; i < np; ++i) seg_end[nseg + i] = b + small[i].end;
      }
      nseg += static_cast<uint32_t>(np);
      __syncthreads();
      continue;
    }
    if (leader) {
      nodes[0] = SegNode{0, len, kNoChild, 0u, 0.0, kNoChild, 0u};
      pend[0] = 0;
      off[0] = 0;
      off[1] = len >= 3 ? len - 2 : 0;
      st->npend = 1u;
      st->nnodes = 1;
      st->heapn = 0;
      st->pops = 0;
      st->done = 0u;
      st->pad0 = nseg;
    }
    grid.sync();
    while (!ld_relaxed_u32(&st->done)) {
      const uint32_t npend = ld_relaxed_u32(&st->npend);
      if (npend <= kFewRanges) {
        seg_sweep_few(t + b, nodes, pend, static_cast<int>(npend), nullptr, nullptr,
                      pdev + (sweep & 1) * kFewRanges * G, parg + (sweep & 1) * kFewRanges * G, sdev, sarg,
                      sres_dev, sres_arg, grid);
        ++sweep;
      } else {
        seg_sweep_many_pass<false>(t + b, nodes, pend, off, npend);
        grid.sync();
        seg_sweep_many_pass<true>(t + b, nodes, pend, off, npend);
        grid.sync();
      }
      if (leader) {  // the reference's selection loop, resumed
        for (uint32_t q = 0; q < npend; ++q) make_live(nodes[pend[q]], mp);
        uint32_t heapn = st->heapn, pops = st->pops, nnodes = st->nnodes;
        if (pops == 0 && heapn == 0 && nodes[0].live && nodes[0].split == 0) heap_push(heap, heapn, nodes, 0);
        bool stall = false;
        while (pops + 1 < budget && heapn > 0) {
          const uint32_t top = heap[0];
          const bool last = pops + 2 >= budget;  // this pop reaches the budget
          if (nodes[top].left == kNoChild && !last) {
            stall = true;
            break;
          }
          heap_pop(heap, heapn, nodes);
          ++pops;
          nodes[top].split = 1;
          if (nodes[top].left == kNoChild) {  // the budget's last split: ranges only
            if (nnodes + 2 > node_cap) {
              overflow = true;
              break;
            }
            nodes[nnodes] = SegNode{nodes[top].begin, nodes[top].arg, kNoChild, 0u, 0.0, kNoChild, 0u};
            nodes[nnodes + 1] = SegNode{nodes[top].arg, nodes[top].end, kNoChild, 0u, 0.0, kNoChild, 0u};
            nodes[top].left = nnodes;
            nnodes += 2;
          } else {
            const uint32_t c = nodes[top].left;
            if (nodes[c].live) heap_push(heap, heapn, nodes, c);
            if (nodes[c + 1].live) heap_push(heap, heapn, nodes, c + 1);
          }
        }
        uint32_t np = 0;
        if (stall && !overflow) {  // expand every heap node with unknown children
          uint64_t acc = 0;
          for (uint32_t h = 0; h < heapn; ++h) {
            const uint32_t id = heap[h];
            if (nodes[id].left != kNoChild) continue;
            if (nnodes + 2 > node_cap) {
              overflow = true;
              break;
            }
            const SegNode pn = nodes[id];
            nodes[nnodes] = SegNode{pn.begin, pn.arg, kNoChild, 0u, 0.0, kNoChild, 0u};
            nodes[nnodes + 1] = SegNode{pn.arg, pn.end, kNoChild, 0u, 0.0, kNoChild, 0u};
            nodes[id].left = nnodes;
            for (int c = 0; c < 2; ++c) {
              const uint32_t cl = nodes[nnodes + c].end - nodes[nnodes + c].begin;
              pend[np] = nnodes + c;
              off[np] = acc;
              acc += cl >= 3 ? cl - 2 : 0;
              ++np;
            }
            nnodes += 2;
          }
          off[np] = acc;
        }
        st->heapn = heapn;
        st->pops = pops;
        st->nnodes = nnodes;
        st->npend = np;
        st->done = (!stall || overflow) ? 1u : 0u;
        if (overflow) st->overflow = 1;
      }
      grid.sync();
    }
    if (leader && !st->overflow) {  // unsplit nodes in tree order = segments by begin
      uint32_t sp = 0;
      nseg = st->pad0;
      pend[sp++] = 0;
      while (sp) {
        const uint32_t id = pend[--sp];
        if (nodes[id].split) {
          pend[sp++] = nodes[id].left + 1;
          pend[sp++] = nodes[id].left;
        } else {
          if (nseg >= seg_cap) {
            st->overflow = 1;
            break;
          }
          seg_end[nseg++] = b + nodes[id].end;
        }
      }
      st->pad0 = nseg;  // every block's segment count
    }
    if (leader && st->overflow) st->pad0 = nseg;
    grid.sync();
    nseg = ld_relaxed_u32(&st->pad0);
    if (ld_relaxed_u32(&st->overflow)) {
      overflow = true;
      break;
    }
  }
  if (blockIdx.x != 0) return;
  if (threadIdx.x == 0) {
    // more pieces than the node / segment arrays hold means more than 0xffff
    // segments: serialize_fit's "too many segments" (curvefit.cpp:287)
    if (overflow || st->overflow) latch(status, GP_ERROR);
    plan->nseg = nseg;
    plan->degree = static_cast<uint32_t>(degree);
    st->overflow = 0;
    st->pad0 = 0;
  }
  if (overflow) return;
  // fit_accumulate's chunk starts: chunk[s] = sum over earlier segments of ceil(len / kChunk)
  uint64_t carry = 0;
  for (uint32_t base = 0; base < nseg; base += blockDim.x) {
    const uint32_t q = base + threadIdx.x;
    uint64_t c = 0;
    if (q < nseg) {
      const uint32_t sb = q == 0 ? 0 : seg_end[q - 1];
      c = (seg_end[q] - sb + kChunk - 1) / kChunk;
    }
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum<uint64_t, 256>(c, sh, tot);
    if (q < nseg) chunk[q] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) chunk[nseg] = carry;
}

// ---------------------------------------------------------------- least squares
__device__ __forceinline__ void seg_range(const uint32_t* seg_end, uint32_t s, uint32_t& b, uint32_t& e) {
  b = s == 0 ? 0 : seg_end[s - 1];
  e = seg_end[s];
}

__device__ __forceinline__ uint32_t chunk_segment(const uint64_t* chunk, uint32_t S, uint64_t c) {
  uint32_t lo = 0, hi = S;  // last s with chunk[s] <= c
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (chunk[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// degree <= 7: Legendre Gram upper triangle + rhs per 2048-point chunk, fixed-order sums
__global__ void __launch_bounds__(256) fit_accumulate(const Plan* plan, const double* __restrict__ t,
                                                      const uint32_t* __restrict__ seg_end,
                                                      const uint64_t* __restrict__ chunk,
                                                      double* __restrict__ partial, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ double red[8][kAcc];
  if (failed(status) || !poly_active(plan) || plan->degree > kMaxDeg) return;
  const uint32_t S = plan->nseg;
  const uint64_t nchunks = chunk[S];
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t seg = chunk_segment(chunk, S, c);
    uint32_t b, e;
    seg_range(seg_end, seg, b, e);
    const uint32_t start = b + static_cast<uint32_t>((c - chunk[seg]) * kChunk);
    const uint32_t stop = start + kChunk < e ? start + kChunk : e;
    const uint32_t len = e - b;
    const int deg = static_cast<int>(plan->degree);
    const int eff = deg < static_cast<int>(len) - 1 ? deg : static_cast<int>(len) - 1;
    double acc[kAcc];
#pragma unroll
    for (int j = 0; j < kAcc; ++j) acc[j] = 0.0;
    if (len > 1) {
      const double alpha = 2.0 / static_cast<double>(len - 1);
      const double beta = -static_cast<double>(len + 1) / static_cast<double>(len - 1);
      for (uint32_t i = start + threadIdx.x; i < stop; i += 256) {
        const double x = alpha * static_cast<double>(i - b + 1) + beta;  // t in [-1, 1]
        const double y = t[i];
        double P[kCps];
        P[0] = 1.0;
        P[1] = x;
#pragma unroll
        for (int j = 1; j < kMaxDeg; ++j) P[j + 1] = ((2 * j + 1) * x * P[j] - j * P[j - 1]) / (j + 1);
        int a = 0;
#pragma unroll
        for (int j = 0; j <= kMaxDeg; ++j)
#pragma unroll
          for (int q = j; q <= kMaxDeg; ++q, ++a)
            if (q <= eff) acc[a] += P[j] * P[q];
#pragma unroll
        for (int j = 0; j <= kMaxDeg; ++j)
          if (j <= eff) acc[36 + j] += P[j] * y;
      }
    }
    // fixed-order reduction: warp tree, then warps in index order
#pragma unroll
    for (int j = 0; j < kAcc; ++j) {
      double v = acc[j];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < kAcc) {
      double v = 0.0;
      for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
      partial[c * kAcc + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// Legendre → t-monomial coefficients, P_{j+1} = ((2j+1) t P_j - j P_{j-1}) /
// (j+1), evaluated at compile time with the same double operations the
// solver used to run per segment (36 fp64 divisions off its serial path).
struct LegendreTable {
  double c[kCps][kCps];
};
constexpr LegendreTable make_legendre() {
  LegendreTable T{};
  for (int j = 0; j < kCps; ++j)
    for (int p = 0; p < kCps; ++p) T.c[j][p] = 0.0;
  T.c[0][0] = 1.0;
  T.c[1][1] = 1.0;
  for (int j = 1; j + 1 < kCps; ++j)
    for (int p = 0; p <= j + 1; ++p)
      T.c[j + 1][p] = ((2 * j + 1) * (p > 0 ? T.c[j][p - 1] : 0.0) - j * T.c[j - 1][p]) / (j + 1);
  return T;
}
__constant__ LegendreTable kLegendre = make_legendre();

// degree <= 7: one segment per block iteration; thread 0 solves (sizes <= 8x8)
// emit_out != null: the model is also serialised here (fit_emit's layout,
// curvefit.cpp:285-298): each segment's block writes its bound and
// coefficients, block 0 the header fields — one launch fewer on the encode.
__global__ void fit_solve(Plan* plan, const double* __restrict__ t, const uint32_t* __restrict__ seg_end,
                          const uint64_t* __restrict__ chunk, const double* __restrict__ partial, float* coeffs,
                          uint8_t* emit_out, uint32_t* status) {
  gp_pdl_wait();
  __shared__ double sacc[kAcc];
  __shared__ double spow[2][kCps];  // alpha^k, beta^k (curvefit.cpp:157-172's pow values), one lane each
  if (failed(status) || !poly_active(plan) || plan->degree > kMaxDeg) return;
  const uint32_t S = plan->nseg;
  const int deg = static_cast<int>(plan->degree);
  const uint32_t cps = static_cast<uint32_t>(deg) + 1;
  uint8_t* ep = nullptr;  // the value payload (emit_out + 49 + il) and its coefficient array
  uint8_t* eq = nullptr;
  if (emit_out) {
    if (S > 0xffff) {  // curvefit.cpp:287
      if (blockIdx.x == 0 && threadIdx.x == 0) latch(status, GP_ERROR);
      return;
    }
    ep = emit_out + 49 + plan->il;
    eq = ep + 3 + 4ull * S + 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ep[0] = 0;  // piecewise polynomial
      ep[1] = static_cast<uint8_t>(S);
      ep[2] = static_cast<uint8_t>(S >> 8);
      eq[-1] = static_cast<uint8_t>(deg);
      const uint64_t nc = static_cast<uint64_t>(S) * cps;
      st_u32_unaligned(eq + 4 * nc, plan->sign_split);
      plan->vl = 1 + 2 + 4ull * S + 1 + 4ull * S * cps + 4;
      uint32_t w = 0;
      for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
      plan->rl = plan->identity ? 0 : (plan->n_values * w + 7) / 8;
    }
  }
  for (uint32_t seg = blockIdx.x; seg < S; seg += gridDim.x) {
    uint32_t b, e;
    seg_range(seg_end, seg, b, e);
    if (e - b > 1 && threadIdx.x >= 32 && threadIdx.x < 32 + 2 * kCps) {
      const uint32_t len = e - b, q = threadIdx.x - 32, k = q % kCps;
      const double alpha = 2.0 / static_cast<double>(len - 1);
      const double beta = -static_cast<double>(len + 1) / static_cast<double>(len - 1);
      spow[q / kCps][k] = pow(q < kCps ? alpha : beta, static_cast<double>(k));
    }
    {  // chunk partials of this segment, summed in chunk order, one accumulator per thread
      const uint64_t c0 = chunk[seg], ncs = chunk[seg + 1] - c0;
      if (threadIdx.x < kAcc) {
        // in chunk order; the loads of 8 chunks issue before their adds (a
        // dependent load-add chain was ~0.2 us per chunk)
        double v = 0.0;
        const double* src = partial + c0 * kAcc + threadIdx.x;
        uint64_t c = 0;
        for (; c + 8 <= ncs; c += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = src[(c + u) * kAcc];
#pragma unroll
          for (int u = 0; u < 8; ++u) v += x[u];
        }
        for (; c < ncs; ++c) v += src[c * kAcc];
        sacc[threadIdx.x] = v;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const uint32_t len = e - b;
      float* out = coeffs + static_cast<uint64_t>(seg) * cps;
      for (int j = 0; j <= deg; ++j) out[j] = 0.0f;
      if (len == 1) {  // curvefit.cpp:134-138
        out[0] = static_cast<float>(t[b]);
      } else {
        const int eff = deg < static_cast<int>(len) - 1 ? deg : static_cast<int>(len) - 1;
        const int m = eff + 1;
        // Every loop below runs over the fixed bound kCps with an `< m` guard and is
        // fully unrolled, so the 8x8 systems live in registers, not local memory.
        double G[kCps][kCps], rhs[kCps];
        {
          int a = 0;
#pragma unroll
          for (int j = 0; j <= kMaxDeg; ++j)
#pragma unroll
            for (int q = j; q <= kMaxDeg; ++q, ++a) G[j][q] = G[q][j] = sacc[a];
        }
#pragma unroll
        for (int j = 0; j < kCps; ++j) rhs[j] = sacc[36 + j];
        // Cholesky G = L L^T (SPD: the Legendre columns are independent for len > eff)
        double L[kCps][kCps];
#pragma unroll
        for (int j = 0; j < kCps; ++j)
#pragma unroll
          for (int i = 0; i < kCps; ++i) L[j][i] = 0.0;
#pragma unroll
        for (int j = 0; j < kCps; ++j) {
          if (j < m) {
            double s2 = G[j][j];
#pragma unroll
            for (int q = 0; q < j; ++q) s2 -= L[j][q] * L[j][q];
            L[j][j] = sqrt(s2 > 0.0 ? s2 : 0.0);
#pragma unroll
            for (int i = j + 1; i < kCps; ++i) {
              if (i < m) {
                double v = G[i][j];
#pragma unroll
                for (int q = 0; q < j; ++q) v -= L[i][q] * L[j][q];
                L[i][j] = L[j][j] > 0.0 ? v / L[j][j] : 0.0;
              }
            }
          }
        }
        double z[kCps], aL[kCps];
#pragma unroll
        for (int i = 0; i < kCps; ++i) {
          double v = rhs[i];
#pragma unroll
          for (int q = 0; q < i; ++q) v -= L[i][q] * z[q];
          z[i] = (i < m && L[i][i] > 0.0) ? v / L[i][i] : 0.0;
        }
#pragma unroll
        for (int i = kCps - 1; i >= 0; --i) {
          double v = z[i];
#pragma unroll
          for (int q = i + 1; q < kCps; ++q) v -= L[q][i] * aL[q];  // L[q][i] = 0 for q >= m
          aL[i] = (i < m && L[i][i] > 0.0) ? v / L[i][i] : 0.0;
        }
        double ct[kCps];
#pragma unroll
        for (int p = 0; p < kCps; ++p) {
          double v = 0.0;
#pragma unroll
          for (int j = p; j < kCps; ++j) v += aL[j] * kLegendre.c[j][p];  // aL[j] = 0 for j >= m
          ct[p] = v;
        }
        // t-monomials → x-monomials, curvefit.cpp:157-172 (the same pow() values)
        double pa[kCps], pb[kCps];
#pragma unroll
        for (int k = 0; k < kCps; ++k) {
          pa[k] = k < m ? spow[0][k] : 0.0;
          pb[k] = k < m ? spow[1][k] : 0.0;
        }
        constexpr double kBinom[kCps][kCps] = {{1, 0, 0, 0, 0, 0, 0, 0},       {1, 1, 0, 0, 0, 0, 0, 0},
                                               {1, 2, 1, 0, 0, 0, 0, 0},       {1, 3, 3, 1, 0, 0, 0, 0},
                                               {1, 4, 6, 4, 1, 0, 0, 0},       {1, 5, 10, 10, 5, 1, 0, 0},
                                               {1, 6, 15, 20, 15, 6, 1, 0},    {1, 7, 21, 35, 35, 21, 7, 1}};
#pragma unroll
        for (int k = 0; k < kCps; ++k) {
          if (k < m) {
            double c = 0.0;
#pragma unroll
            for (int j = k; j < kCps; ++j)
              if (j < m) c += ct[j] * kBinom[j][k] * pa[k] * pb[j - k];
            out[k] = static_cast<float>(c);
          }
        }
      }
      if (ep) {
        st_u32_unaligned(ep + 3 + 4ull * seg, e);
        for (uint32_t j = 0; j < cps; ++j)
          st_u32_unaligned(eq + 4 * (static_cast<uint64_t>(seg) * cps + j), __float_as_uint(out[j]));
      }
    }
    __syncthreads();
  }
}

// Degree 8..60 (fit_poly's range, curvefit.cpp:130): one block per segment.
// The normal equations in the Legendre basis are accumulated in batches of 64
// points whose basis values sit in shared memory; each thread owns a fixed
// set of Gram / rhs entries and sums them in point order (deterministic).
// Cholesky, Legendre → t-monomials and the x expansion (Pascal binomials in
// double, as curvefit.cpp:159-165 builds them) run in one thread on the
// block's global scratch.  The Vandermonde system the reference hands to
// Eigen's QR is ill-conditioned at these degrees, so the coefficients are not
// expected to match it beyond the reconstructed values' tolerance.
constexpr int kWideBatch = 64;
constexpr int kWideEntries = kWideCps * (kWideCps + 1) / 2 + kWideCps;  // 1891 + 61
constexpr int kWideScratch = 3 * kWideCps * kWideCps;                    // G | L | Lc (doubles)
__global__ void __launch_bounds__(256) fit_solve_wide(Plan* plan, const double* __restrict__ t,
                                                      const uint32_t* __restrict__ seg_end, float* coeffs,
                                                      double* scratch, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ double V[kWideBatch][kWideCps];
  __shared__ double Y[kWideBatch];
  __shared__ int16_t ej[kWideEntries], eq[kWideEntries];  // entry → (row, column); column -1 = rhs
  if (failed(status) || !poly_active(plan) || plan->degree <= kMaxDeg) return;
  const uint32_t S = plan->nseg;
  const int deg = static_cast<int>(plan->degree);
  const uint32_t cps = static_cast<uint32_t>(deg) + 1;
  double* G = scratch + static_cast<uint64_t>(blockIdx.x) * kWideScratch;
  double* L = G + kWideCps * kWideCps;
  double* Lc = L + kWideCps * kWideCps;
  for (uint32_t seg = blockIdx.x; seg < S; seg += gridDim.x) {
    uint32_t b, e;
    seg_range(seg_end, seg, b, e);
    const uint32_t len = e - b;
    float* out = coeffs + static_cast<uint64_t>(seg) * cps;
    if (len == 1) {
      if (threadIdx.x == 0) {
        for (int j = 0; j <= deg; ++j) out[j] = 0.0f;
        out[0] = static_cast<float>(t[b]);
      }
      continue;
    }
    const int eff = deg < static_cast<int>(len) - 1 ? deg : static_cast<int>(len) - 1;
    const int m = eff + 1;
    const int ne = m * (m + 1) / 2 + m;
    if (threadIdx.x == 0) {
      int a = 0;
      for (int j = 0; j < m; ++j)
        for (int q = j; q < m; ++q, ++a) {
          ej[a] = static_cast<int16_t>(j);
          eq[a] = static_cast<int16_t>(q);
        }
      for (int j = 0; j < m; ++j, ++a) {
        ej[a] = static_cast<int16_t>(j);
        eq[a] = -1;
      }
    }
    __syncthreads();
    constexpr int kOwn = (kWideEntries + 255) / 256;
    double acc[kOwn];
#pragma unroll
    for (int u = 0; u < kOwn; ++u) acc[u] = 0.0;
    const double alpha = 2.0 / static_cast<double>(len - 1);
    const double beta = -static_cast<double>(len + 1) / static_cast<double>(len - 1);
    for (uint32_t p0 = 0; p0 < len; p0 += kWideBatch) {
      const uint32_t nb = len - p0 < kWideBatch ? len - p0 : kWideBatch;
      if (threadIdx.x < nb) {
        const uint32_t i = p0 + threadIdx.x;
        const double x = alpha * static_cast<double>(i + 1) + beta;
        V[threadIdx.x][0] = 1.0;
        if (m > 1) V[threadIdx.x][1] = x;
        for (int j = 1; j + 1 < m; ++j)
          V[threadIdx.x][j + 1] = ((2 * j + 1) * x * V[threadIdx.x][j] - j * V[threadIdx.x][j - 1]) / (j + 1);
        Y[threadIdx.x] = t[b + i];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kOwn; ++u) {
        const int a = threadIdx.x + 256 * u;
        if (a < ne) {
          const int j = ej[a], q = eq[a];
          double v = acc[u];
          if (q >= 0)
            for (uint32_t k = 0; k < nb; ++k) v += V[k][j] * V[k][q];
          else
            for (uint32_t k = 0; k < nb; ++k) v += V[k][j] * Y[k];
          acc[u] = v;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < kOwn; ++u) {
      const int a = threadIdx.x + 256 * u;
      if (a < ne) {
        const int j = ej[a], q = eq[a];
        if (q >= 0) {
          G[j * kWideCps + q] = acc[u];
          G[q * kWideCps + j] = acc[u];
        } else {
          Lc[j] = acc[u];  // rhs, parked in the Lc area until the solve
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double rhs[kWideCps], z[kWideCps], aL[kWideCps], ct[kWideCps];
      for (int j = 0; j < m; ++j) rhs[j] = Lc[j];
      for (int j = 0; j < m; ++j) {  // Cholesky
        double s2 = G[j * kWideCps + j];
        for (int q = 0; q < j; ++q) s2 -= L[j * kWideCps + q] * L[j * kWideCps + q];
        L[j * kWideCps + j] = sqrt(s2 > 0.0 ? s2 : 0.0);
        for (int i = j + 1; i < m; ++i) {
          double v = G[i * kWideCps + j];
          for (int q = 0; q < j; ++q) v -= L[i * kWideCps + q] * L[j * kWideCps + q];
          L[i * kWideCps + j] = L[j * kWideCps + j] > 0.0 ? v / L[j * kWideCps + j] : 0.0;
        }
      }
      for (int i = 0; i < m; ++i) {
        double v = rhs[i];
        for (int q = 0; q < i; ++q) v -= L[i * kWideCps + q] * z[q];
        z[i] = L[i * kWideCps + i] > 0.0 ? v / L[i * kWideCps + i] : 0.0;
      }
      for (int i = m - 1; i >= 0; --i) {
        double v = z[i];
        for (int q = i + 1; q < m; ++q) v -= L[q * kWideCps + i] * aL[q];
        aL[i] = L[i * kWideCps + i] > 0.0 ? v / L[i * kWideCps + i] : 0.0;
      }
      // Legendre → t-monomials, row by row in the Lc area
      for (int j = 0; j < m; ++j)
        for (int p = 0; p < m; ++p) Lc[j * kWideCps + p] = 0.0;
      Lc[0] = 1.0;
      if (m > 1) Lc[kWideCps + 1] = 1.0;
      for (int j = 1; j + 1 < m; ++j)
        for (int p = 0; p <= j + 1; ++p)
          Lc[(j + 1) * kWideCps + p] =
              ((2 * j + 1) * (p > 0 ? Lc[j * kWideCps + p - 1] : 0.0) - j * Lc[(j - 1) * kWideCps + p]) / (j + 1);
      for (int p = 0; p < m; ++p) {
        double v = 0.0;
        for (int j = p; j < m; ++j) v += aL[j] * Lc[j * kWideCps + p];
        ct[p] = v;
      }
      // binomials by Pascal's rule (curvefit.cpp:159-165) into the L area
      double* B = L;
      for (int j = 0; j < m; ++j) {
        for (int k = 0; k <= j; ++k) B[j * kWideCps + k] = 1.0;
        for (int k = 1; k < j; ++k) B[j * kWideCps + k] = B[(j - 1) * kWideCps + k - 1] + B[(j - 1) * kWideCps + k];
      }
      for (int j = 0; j <= deg; ++j) out[j] = 0.0f;
      for (int k = 0; k < m; ++k) {
        double c = 0.0;
        const double ak = pow(alpha, static_cast<double>(k));
        for (int j = k; j < m; ++j) c += ct[j] * B[j * kWideCps + k] * ak * pow(beta, static_cast<double>(j - k));
        out[k] = static_cast<float>(c);
      }
    }
    __syncthreads();
  }
}

// serialize_fit (curvefit.cpp:285-298) + reorder payload size; vl, rl, flags
__global__ void fit_emit(Plan* plan, uint8_t* out, int cfg_degree, const uint32_t* __restrict__ seg_end,
                         const float* __restrict__ coeffs, uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !fit_active(plan)) return;
  const uint32_t kind = plan->fit_kind;
  const uint32_t S = plan->nseg, deg = kind ? static_cast<uint32_t>(cfg_degree) : plan->degree;
  const uint32_t cps = kind ? 4 : deg + 1;  // coeffs_per_segment
  if (S > 0xffff) {  // curvefit.cpp:287
    if (threadIdx.x == 0) latch(status, GP_ERROR);
    return;
  }
  uint8_t* p = out + 49 + plan->il;
  if (threadIdx.x == 0) {
    p[0] = static_cast<uint8_t>(kind);  // 0 piecewise polynomial, 1 double exponential
    p[1] = static_cast<uint8_t>(S);
    p[2] = static_cast<uint8_t>(S >> 8);
  }
  for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) st_u32_unaligned(p + 3 + 4ull * s, seg_end[s]);
  uint8_t* q = p + 3 + 4ull * S;
  if (threadIdx.x == 0) *q = static_cast<uint8_t>(deg);
  ++q;
  const uint64_t nc = static_cast<uint64_t>(S) * cps;
  for (uint64_t i = threadIdx.x; i < nc; i += blockDim.x) st_u32_unaligned(q + 4 * i, __float_as_uint(coeffs[i]));
  if (threadIdx.x == 0) {
    st_u32_unaligned(q + 4 * nc, plan->sign_split);
    plan->vl = 1 + 2 + 4ull * S + 1 + 4ull * S * cps + 4;
    uint32_t w = 0;
    for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
    plan->rl = plan->identity ? 0 : (plan->n_values * w + 7) / 8;
  }
}

// reorder_encode (curvefit.cpp:332-340): entries of w bits, LSB-first
__global__ void reorder_pack(const uint32_t* __restrict__ map, Plan* plan, uint8_t* out, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || !fit_active(plan) || plan->identity) return;
  const uint64_t rl = plan->rl, n = plan->n_values;
  uint32_t w = 0;
  for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
  if (w == 0) return;
  uint8_t* p = out + 49 + plan->il + plan->vl;
  for (uint64_t byte = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; byte < rl;
       byte += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t v = 0;
    uint64_t bit = 8 * byte;
    int filled = 0;
    while (filled < 8) {
      const uint64_t e = bit / w;
      if (e >= n) break;
      const uint32_t off = static_cast<uint32_t>(bit - e * w);
      const int take = static_cast<int>(w - off) < 8 - filled ? static_cast<int>(w - off) : 8 - filled;
      v |= ((map[e] >> off) & ((1u << take) - 1u)) << filled;
      filled += take;
      bit += take;
    }
    p[byte] = static_cast<uint8_t>(v);
  }
}

// ---------------------------------------------------------------- decode
// parse_fit (curvefit.cpp:300-325), pipeline.cpp:117-118 trailing bytes, and
// the reorder_decode length/slack rules (curvefit.cpp:342-356).  One block:
// the sequential parse's first failure is the lowest failing bound index
// (truncation before bound i, or bound i not increasing), found in parallel.
__global__ void __launch_bounds__(256) fit_parse(const uint8_t* __restrict__ in, Plan* plan, uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t s_first;
  __shared__ uint32_t s_found;
  __shared__ int s_err;
  if (failed(status) || !fit_active(plan)) return;
  const uint8_t* p = in + plan->off_value;
  const uint64_t vl = plan->vl, count = plan->n_values;
  if (threadIdx.x == 0) {
    s_err = 0;
    s_first = 0xFFFFFFFFu;
    s_found = 0;
    if (vl < 1) s_err = GP_TRUNCATED;
    else if (p[0] > 1) s_err = GP_UNKNOWN_METHOD;
    else if (vl < 3) s_err = GP_TRUNCATED;
    else if ((p[1] | (p[2] << 8)) < 1) s_err = GP_CORRUPT_PAYLOAD;
  }
  __syncthreads();
  if (s_err) {
    if (threadIdx.x == 0) latch(status, s_err);
    return;
  }
  const uint8_t kind = p[0];
  const uint32_t S = p[1] | (p[2] << 8);
  for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
    bool bad = vl < 3 + 4ull * (i + 1);
    if (!bad) {
      const uint32_t e = ld_u32_unaligned(p + 3 + 4ull * i);
      const uint32_t prev = i == 0 ? 0u : ld_u32_unaligned(p + 3 + 4ull * (i - 1));
      bad = e <= prev && !(i == 0 && e > 0);
    }
    if (bad) atomicMin(&s_first, i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t f = s_first;
    if (f != 0xFFFFFFFFu) {
      s_err = vl < 3 + 4ull * (f + 1) ? GP_TRUNCATED : GP_CORRUPT_PAYLOAD;
    } else if (ld_u32_unaligned(p + 3 + 4ull * (S - 1)) != count) {
      s_err = GP_CORRUPT_PAYLOAD;
    }
  }
  __syncthreads();
  if (s_err) {
    if (threadIdx.x == 0) latch(status, s_err);
    return;
  }
  uint64_t at = 3 + 4ull * S;
  if (vl < at + 1) {
    if (threadIdx.x == 0) latch(status, GP_TRUNCATED);
    return;
  }
  const uint32_t deg = p[at++];
  const uint64_t cps = kind == 1 ? 4 : deg + 1;
  const uint64_t nc = S * cps;
  if (vl < at + 4 * nc) {
    if (threadIdx.x == 0) latch(status, GP_TRUNCATED);
    return;
  }
  const uint64_t coeff_at = at;
  at += 4 * nc;
  if (vl < at + 4) {
    if (threadIdx.x == 0) latch(status, GP_TRUNCATED);
    return;
  }
  const uint32_t l = ld_u32_unaligned(p + at);
  at += 4;
  if (l > count) {
    if (threadIdx.x == 0) latch(status, GP_CORRUPT_PAYLOAD);
    return;
  }
  if (l > 0 && l < count) {  // binary_search over the (increasing) bounds
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x)
      if (ld_u32_unaligned(p + 3 + 4ull * i) == l) s_found = 1;
    __syncthreads();
    if (!s_found) {
      if (threadIdx.x == 0) latch(status, GP_CORRUPT_PAYLOAD);
      return;
    }
  }
  if (at != vl) {
    if (threadIdx.x == 0) latch(status, GP_CORRUPT_PAYLOAD);
    return;
  }
  // reorder_decode structure: count entries of w bits, < 8 slack bits, zero slack
  if (plan->rl) {
    uint32_t w = 0;
    for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
    const uint64_t need = count * w, have = 8 * plan->rl;
    int err = 0;
    if (have < need) err = GP_TRUNCATED;
    else if (have - need >= 8) err = GP_CORRUPT_PAYLOAD;
    else if (have > need && (in[plan->off_reorder + plan->rl - 1] >> (need % 8))) err = GP_CORRUPT_PAYLOAD;
    if (err) {
      if (threadIdx.x == 0) latch(status, err);
      return;
    }
  }
  if (threadIdx.x == 0) {  // fit_unpack_eval reads bounds and coefficients from the payload itself
    plan->fit_bounds_at = plan->off_value + 3;
    plan->fit_coeffs_at = plan->off_value + coeff_at;
    plan->nseg = S;
    plan->degree = deg;
    plan->fit_kind = kind;
    plan->sign_split = l;
  }
}

// value_decompress (curvefit.cpp:517-541) in one pass: per value s, the
// reorder entry (entry >= d or >= n → corrupt; permutation check by an
// atomicOr bitset, :531-538), evaluate + unfold, store at the entry.  Bounds
// and coefficients come straight from the payload (any degree byte and up to
// 0xffff segments); models of <= 64 segments and <= 8 coefficients are staged
// in shared memory, larger ones searched in place (binary search of the
// bounds).  Errors latch the pre-verdict status; nothing reaches the caller's
// dense vector before the verdict (decode_common).
constexpr int kEvalSmemSeg = 64;
__global__ void fit_unpack_eval(const uint8_t* __restrict__ in, const Plan* plan, uint32_t* __restrict__ map,
                                uint32_t* seen, double* __restrict__ out, uint32_t* status) {
  gp_pdl_wait();
  __shared__ uint32_t sb[kEvalSmemSeg];
  __shared__ float sc[kEvalSmemSeg * kCps];
  if (failed(status) || !fit_active(plan)) return;
  const uint32_t S = plan->nseg, cps = cps_of(plan);
  const uint8_t* bp = in + plan->fit_bounds_at;
  const uint8_t* cp = in + plan->fit_coeffs_at;
  const bool dexp = plan->fit_kind == 1;
  const bool small = S <= kEvalSmemSeg && cps <= kCps;
  if (small) {
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) sb[i] = ld_u32_unaligned(bp + 4ull * i);
    for (uint32_t i = threadIdx.x; i < S * cps; i += blockDim.x) sc[i] = __uint_as_float(ld_u32_unaligned(cp + 4ull * i));
    __syncthreads();
  }
  const uint64_t n = plan->n_values, d = plan->d;
  const uint64_t l = plan->sign_split;
  const bool reorder = plan->rl != 0;
  uint32_t w = 0;
  for (uint64_t x = d - 1; x; x >>= 1) ++w;
  const uint8_t* rp = in + plan->off_reorder;
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t dst = s;
    if (reorder) {
      uint64_t v = 0;
      const uint64_t bit0 = s * w;
      for (uint32_t j = 0; j < w; ++j) {
        const uint64_t bit = bit0 + j;
        v |= static_cast<uint64_t>((rp[bit >> 3] >> (bit & 7)) & 1u) << j;
      }
      if (v >= d || v >= n) {
        latch(status, GP_CORRUPT_PAYLOAD);
        continue;
      }
      map[s] = static_cast<uint32_t>(v);
      if (atomicOr(&seen[v >> 5], 1u << (v & 31)) & (1u << (v & 31))) latch(status, GP_CORRUPT_PAYLOAD);
      dst = v;
    }
    const uint64_t j = s < l ? s : l + (n - 1 - s);  // position in the folded sequence
    uint32_t seg, begin;
    double acc = 0.0;
    if (small) {
      seg = 0;
      while (sb[seg] <= j) ++seg;
      begin = seg == 0 ? 0 : sb[seg - 1];
      const double x = static_cast<double>(j - begin + 1);
      const float* c = sc + seg * cps;
      if (dexp)
        acc = eval_dexp(c, x);
      else
        for (int q = static_cast<int>(cps) - 1; q >= 0; --q)
          acc = __dadd_rn(__dmul_rn(acc, x), static_cast<double>(c[q]));
    } else {  // first bound > j
      uint32_t lo = 0, hi = S - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (ld_u32_unaligned(bp + 4ull * mid) > j) hi = mid; else lo = mid + 1;
      }
      seg = lo;
      begin = seg == 0 ? 0 : ld_u32_unaligned(bp + 4ull * (seg - 1));
      const double x = static_cast<double>(j - begin + 1);
      const uint8_t* c = cp + 4ull * seg * cps;
      if (dexp) {
        float cc[4];
        for (int q = 0; q < 4; ++q) cc[q] = __uint_as_float(ld_u32_unaligned(c + 4 * q));
        acc = eval_dexp(cc, x);
      } else {
        for (int q = static_cast<int>(cps) - 1; q >= 0; --q)
          acc = __dadd_rn(__dmul_rn(acc, x), static_cast<double>(__uint_as_float(ld_u32_unaligned(c + 4ull * q))));
      }
    }
    out[dst] = s < l ? acc : -acc;
  }
}

// ---------------------------------------------------------------- dexp
// fit_dexp (curvefit.cpp:225-283) of one sign part per block: log-linear
// starts on the two halves (:194-221), then Levenberg-Marquardt with the
// reference's damping schedule, acceptance and convergence tests; every sum
// over the part is a block reduction in fp64.  The 4x4 damped system is solved
// by LDLT (SPD for lambda > 0; Eigen's pivoted LDLT gives the same solution up
// to rounding).  A part shorter than 4 points or a non-finite fit makes the
// whole model fall back to the polynomial fit (value_compress, :464-491).
constexpr int kDexpBlock = 1024;

template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) sh[warp * N + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double a = 0.0;
    for (int w = 0; w < kDexpBlock / 32; ++w) a += sh[w * N + k];
    v[k] = a;
  }
  __syncthreads();
}

__device__ double dexp_sse(const double* y, uint32_t n, const double* p, double* sh) {
  double v[1] = {0.0};
  for (uint32_t i = threadIdx.x; i < n; i += kDexpBlock) {
    const double x = static_cast<double>(i + 1);
    const double r = p[0] * safe_exp(p[1] * x) + p[2] * safe_exp(p[3] * x) - y[i];
    v[0] += r * r;
  }
  block_sum<1>(v, sh);
  return v[0];
}

// amp * e^{rate x} over 1-based positions begin+1 .. begin+len (positive samples)
__device__ void log_linear(const double* y, uint32_t begin, uint32_t len, double* sh, double& amp, double& rate) {
  double v[5] = {0, 0, 0, 0, 0};  // sx, sy, sxx, sxy, m
  double lastpos = -1.0;          // index of the last positive sample
  for (uint32_t i = begin + threadIdx.x; i < begin + len; i += kDexpBlock) {
    if (!(y[i] > 0.0)) continue;
    const double x = static_cast<double>(i + 1), ly = log(y[i]);
    v[0] += x;
    v[1] += ly;
    v[2] += x * x;
    v[3] += x * ly;
    v[4] += 1.0;
    lastpos = static_cast<double>(i);
  }
  double lp[1] = {lastpos};
  block_sum<5>(v, sh);
  {  // max over threads of the last positive index
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) lp[0] = fmax(lp[0], __shfl_xor_sync(kFull, lp[0], o));
    if (lane == 0) sh[warp] = lp[0];
    __syncthreads();
    double a = -1.0;
    for (int w = 0; w < kDexpBlock / 32; ++w) a = fmax(a, sh[w]);
    lp[0] = a;
    __syncthreads();
  }
  const double m = v[4];
  if (m >= 2) {
    const double denom = m * v[2] - v[0] * v[0];
    if (fabs(denom) > 1e-12) {
      const double r = (m * v[3] - v[0] * v[1]) / denom;
      const double lamp = (v[1] - r * v[0]) / m;
      if (isfinite(r) && isfinite(lamp)) {
        amp = exp(fmin(fmax(lamp, -kExpClamp), kExpClamp));
        rate = r;
        return;
      }
    }
  }
  if (m >= 1) {
    amp = y[static_cast<uint32_t>(lp[0])];
    rate = 0.0;
    return;
  }
  amp = 1e-12;
  rate = 0.0;
}

__global__ void __launch_bounds__(kDexpBlock) dexp_fit(Plan* plan, const double* __restrict__ t, uint32_t* seg_end,
                                                        float* coeffs, const uint32_t* status) {
  gp_pdl_wait();
  __shared__ double sh[(kDexpBlock / 32) * 14];
  __shared__ double sp[4], scand[4], sbest, slambda;
  __shared__ int sflag;  // bit0 accepted, bit1 converged, bit2 stop attempts
  if (failed(status) || plan->value_method != GP_VALUE_FIT_DEXP) return;
  const uint32_t n = static_cast<uint32_t>(plan->n_values), l = plan->sign_split;
  uint32_t parts[2][2], np = 0;
  if (l > 0) { parts[np][0] = 0; parts[np][1] = l; ++np; }
  if (l < n) { parts[np][0] = l; parts[np][1] = n; ++np; }
  if (blockIdx.x >= np) return;
  const uint32_t begin = parts[blockIdx.x][0], len = parts[blockIdx.x][1] - begin;
  if (len < 4) {
    if (threadIdx.x == 0) atomicOr(&plan->dexp_fail, 1u);
    return;
  }
  const double* y = t + begin;
  const uint32_t half = len / 2;
  double a0, b0, c0, d0;
  log_linear(y, 0, half, sh, a0, b0);
  log_linear(y, half, len - half, sh, c0, d0);
  if (threadIdx.x == 0) {
    sp[0] = a0; sp[1] = b0; sp[2] = c0; sp[3] = d0;
    slambda = 1e-3;
  }
  __syncthreads();
  double best = dexp_sse(y, len, sp, sh);
  if (!isfinite(best)) {
    if (threadIdx.x == 0) atomicOr(&plan->dexp_fail, 1u);
    return;
  }
  bool converged = false;
  for (int it = 0; it < 300 && !converged; ++it) {
    double v[14];
#pragma unroll
    for (int k = 0; k < 14; ++k) v[k] = 0.0;
    const double p0 = sp[0], p1 = sp[1], p2 = sp[2], p3 = sp[3];
    for (uint32_t i = threadIdx.x; i < len; i += kDexpBlock) {
      const double x = static_cast<double>(i + 1);
      const double eb = safe_exp(p1 * x), ed = safe_exp(p3 * x);
      const double j[4] = {eb, p0 * x * eb, ed, p2 * x * ed};
      const double r = p0 * eb + p2 * ed - y[i];
      int q = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b) v[q++] += j[a] * j[b];
#pragma unroll
      for (int a = 0; a < 4; ++a) v[10 + a] += j[a] * r;
    }
    block_sum<14>(v, sh);
    bool accepted = false;
    for (int attempt = 0; attempt < 24; ++attempt) {
      if (threadIdx.x == 0) {
        // (JtJ + lambda I) delta = -Jtr by LDLT
        double A[4][4];
        int q = 0;
        for (int a = 0; a < 4; ++a)
          for (int b = a; b < 4; ++b) {
            A[a][b] = A[b][a] = v[q++];
          }
        for (int a = 0; a < 4; ++a) A[a][a] += slambda;
        double L[4][4] = {}, D[4];
        for (int j2 = 0; j2 < 4; ++j2) {
          double dd = A[j2][j2];
          for (int k2 = 0; k2 < j2; ++k2) dd -= L[j2][k2] * L[j2][k2] * D[k2];
          D[j2] = dd;
          L[j2][j2] = 1.0;
          for (int i2 = j2 + 1; i2 < 4; ++i2) {
            double s2 = A[i2][j2];
            for (int k2 = 0; k2 < j2; ++k2) s2 -= L[i2][k2] * L[j2][k2] * D[k2];
            L[i2][j2] = s2 / dd;
          }
        }
        double z[4], delta[4];
        for (int i2 = 0; i2 < 4; ++i2) {
          double s2 = -v[10 + i2];
          for (int k2 = 0; k2 < i2; ++k2) s2 -= L[i2][k2] * z[k2];
          z[i2] = s2;
        }
        for (int i2 = 3; i2 >= 0; --i2) {
          double s2 = z[i2] / D[i2];
          for (int k2 = i2 + 1; k2 < 4; ++k2) s2 -= L[k2][i2] * delta[k2];
          delta[i2] = s2;
        }
        for (int a = 0; a < 4; ++a) scand[a] = sp[a] + delta[a];
        double dn = 0.0;
        for (int a = 0; a < 4; ++a) dn += delta[a] * delta[a];
        sh[(kDexpBlock / 32) * 14 - 1] = sqrt(dn);  // |delta|, read back by thread 0 below
      }
      __syncthreads();
      const double dnorm = sh[(kDexpBlock / 32) * 14 - 1];
      __syncthreads();
      const double sse = dexp_sse(y, len, scand, sh);
      if (threadIdx.x == 0) {
        int f = 0;
        if (isfinite(sse) && sse < best) {
          const double gain = best - sse;
          double pn = 0.0;
          for (int a = 0; a < 4; ++a) {
            sp[a] = scand[a];
            pn += sp[a] * sp[a];
          }
          sbest = sse;
          slambda = fmax(slambda / 10.0, 1e-12);
          f = 1;
          if (gain <= 1e-14 * (sse + 1e-300) || dnorm <= 1e-12 * (1.0 + sqrt(pn))) f |= 2;
        } else {
          slambda *= 10.0;
          if (slambda > 1e14) f = 4;
        }
        sflag = f;
      }
      __syncthreads();
      const int f = sflag;
      if (f & 1) {
        best = sbest;
        accepted = true;
        converged = (f & 2) != 0;
        break;
      }
      if (f & 4) break;
    }
    if (!accepted) break;
  }
  if (threadIdx.x == 0) {
    double a = sp[0], b = sp[1], c = sp[2], d = sp[3];
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d) && isfinite(best))) {
      atomicOr(&plan->dexp_fail, 1u);
      return;
    }
    if (b > d) {  // the slower exponential first (curvefit.cpp:277-281)
      double tmp = a; a = c; c = tmp;
      tmp = b; b = d; d = tmp;
    }
    float* co = coeffs + blockIdx.x * 4;
    co[0] = static_cast<float>(a);
    co[1] = static_cast<float>(b);
    co[2] = static_cast<float>(c);
    co[3] = static_cast<float>(d);
    seg_end[blockIdx.x] = parts[blockIdx.x][1];
  }
}

// dexp model or the polynomial fallback (value_compress attempt 1)
__global__ void dexp_decide(Plan* plan, const uint32_t* status) {
  gp_pdl_wait();
  if (failed(status) || plan->value_method != GP_VALUE_FIT_DEXP) return;
  if (plan->dexp_fail) return;  // fit_kind stays 0: the polynomial path runs
  const uint32_t n = static_cast<uint32_t>(plan->n_values), l = plan->sign_split;
  plan->nseg = (l > 0 ? 1u : 0u) + (l < n ? 1u : 0u);
  plan->fit_kind = 1;
}

}  // namespace

void launch_radix_sort(gp_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* ktmp, uint32_t* vtmp,
                       const uint64_t* n_dev, uint64_t n_bound, int bits, cudaStream_t s, bool hist_ready = false,
                       const float* fit_v = nullptr, double* fit_t = nullptr);

static_assert(sizeof(SegNode) == 32, "workspace sizes SegNode at 32 bytes");
static_assert(sizeof(SegState) == 32, "workspace sizes SegState at 32 bytes");

void launch_values_fit(gp_ctx* ctx, uint8_t* out, int degree, int max_segments, uint64_t n_bound, cudaStream_t s,
                       bool dexp) {
  Workspace& w = ctx->ws;
  // sign_split / identity / fit_kind / dexp_fail: reset by the encode's init_plan (capi.cu)
  const ValSrc vals{w.values, ctx->vals64};
  // f32 values: the keys kernel also builds the sort's digit histograms
  uint32_t* ghist = ctx->vals64 ? nullptr : w.sort_hist;
  if (ghist) fill_async(ctx, ghist, 0, 4 * 256 * sizeof(uint32_t), s);
  const float* gdense = ctx->vals64 ? nullptr : ctx->gather_dense;
  GP_LAUNCH(ctx, fit_keys, std::min(grid_for(ctx, n_bound, 256), 2 * ctx->sm_count), 256, 0, s, vals, w.plan, w.u32a,
            w.u32b, ghist, gdense, w.sel, w.values, w.status);
  // f32: the sort's last pass also writes fit_prepare's folded sequence t and the identity flag
  launch_radix_sort(ctx, w.u32a, w.u32b, w.u32c, w.u32d, &w.plan->n_values, n_bound, 32, s, ghist != nullptr,
                    ghist ? w.values : nullptr, ghist ? w.f64b : nullptr);
  if (ctx->vals64) {  // the high words, stable on top of the low-word order
    GP_LAUNCH(ctx, fit_keys_hi, grid_for(ctx, n_bound, 256), 256, 0, s, ctx->vals64, w.plan, w.u32b, w.u32a, w.status);
    launch_radix_sort(ctx, w.u32a, w.u32b, w.u32c, w.u32d, &w.plan->n_values, n_bound, 32, s);
  }
  if (!ghist) GP_LAUNCH(ctx, fit_prepare, grid_for(ctx, n_bound, 256), 256, 0, s, vals, w.u32b, w.plan, w.f64b, w.status);
  if (dexp) {
    GP_LAUNCH(ctx, dexp_fit, 2, kDexpBlock, 0, s, w.plan, w.f64b, w.seg_end, w.coeffs, w.status);
    GP_LAUNCH(ctx, dexp_decide, 1, 1, 0, s, w.plan, w.status);
  }
  {  // cooperative launch: every block of the grid must be resident
    static int grid = 0;
    if (!grid) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_segment_coop, 256, 0);
      grid = std::max(1, std::min(per_sm, 2)) * ctx->sm_count;
    }
    const double* t = w.f64b;
    Plan* plan = w.plan;
    double* pdev = w.seg_dev;
    uint32_t* parg = w.seg_arg;
    SegNode* nodes = reinterpret_cast<SegNode*>(w.seg_nodes);
    uint32_t* heap = w.seg_heap;
    uint32_t* pend = w.seg_pend;
    uint64_t* off = w.seg_off;
    SegState* st = reinterpret_cast<SegState*>(w.seg_state);
    uint32_t* seg_end = w.seg_end;
    uint64_t* chunk = w.seg_chunk;
    uint32_t node_cap = w.node_cap;
    uint32_t seg_cap = static_cast<uint32_t>(w.seg_cap);
    uint32_t* status = w.status;
    void* args[] = {&plan, &t, &degree, &max_segments, &pdev, &parg, &nodes, &heap, &pend, &off, &st,
                    &seg_end, &chunk, &node_cap, &seg_cap, &status};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fit_segment_coop), grid, 256, args, 0, s);
    ++ctx->launches;
  }
  const uint64_t seg_bound = std::min<uint64_t>(n_bound, w.seg_cap);
  // 140 registers: one resident block per SM, so a grid beyond the SM count
  // only adds waves of blocks that find no chunk (grid-stride over chunks)
  GP_LAUNCH(ctx, fit_accumulate,
            static_cast<int>(std::min<uint64_t>(n_bound / kChunk + seg_bound + 1, static_cast<uint64_t>(ctx->sm_count))),
            256, 0, s, w.plan,
            w.f64b, w.seg_end, w.seg_chunk, w.partial, w.status);
  const bool fused_emit = !dexp && degree <= kMaxDeg;  // fit_solve serialises the model itself
  GP_LAUNCH(ctx, fit_solve, grid_for(ctx, seg_bound * 64, 64), 64, 0, s, w.plan, w.f64b, w.seg_end, w.seg_chunk,
            w.partial, w.coeffs, fused_emit ? out : nullptr, w.status);
  if (degree > kMaxDeg)
    GP_LAUNCH(ctx, fit_solve_wide, static_cast<int>(std::min<uint64_t>(seg_bound, kWideBlocks)), 256, 0, s, w.plan,
              w.f64b, w.seg_end, w.coeffs, w.fit_scratch, w.status);
  if (!fused_emit) GP_LAUNCH(ctx, fit_emit, 1, 256, 0, s, w.plan, out, degree, w.seg_end, w.coeffs, w.status);
  GP_LAUNCH(ctx, reorder_pack, grid_for(ctx, n_bound * 4, 256), 256, 0, s, w.u32b, w.plan, out, w.status);
}

void launch_decode_fit(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  fill_async(ctx, w.u32c, 0, ((n_bound + 31) / 32) * 4, s);  // before fit_parse: the kernels chain by PDL
  GP_LAUNCH(ctx, fit_parse, 1, 256, 0, s, in, w.plan, w.status);
  GP_LAUNCH(ctx, fit_unpack_eval, grid_for(ctx, n_bound, 256), 256, 0, s, in, w.plan, w.u32b, w.u32c, w.f64a,
            w.status);
}

}  // namespace gp
