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
//   fit_accumulate / fit_solve : least squares of degree <= 7 per segment on
//                  t in [-1, 1].  The reference solves the Vandermonde system
//                  with Eigen's column-pivoted QR (curvefit.cpp:154); here the
//                  normal equations are formed in the Legendre basis (Gram
//                  matrix ~ diagonal, condition ~ 2*degree+1) with fixed-order
//                  fp64 reductions, solved by Cholesky, mapped to t-monomials,
//                  then expanded to x-monomials exactly as curvefit.cpp:157-172.
//                  Coefficients agree with the reference within f32 rounding
//                  (tolerance-checked).
//   fit_emit / reorder_pack : serialize_fit + the bit-packed map
// Decode: fit_parse (parse_fit + reorder checks), reorder_unpack (entries,
// permutation check), fit_eval (fp64 Horner without FMA, sign unfold,
// permutation scatter) — bit-exact for a given container.
#include <cooperative_groups.h>

#include "gp_ctx.hpp"
#include "gp_device.cuh"

namespace cg = cooperative_groups;

namespace gp {

namespace {

constexpr int kMaxDeg = 7;
constexpr int kCps = kMaxDeg + 1;           // coefficient stride in Plan::coeffs
constexpr int kChunk = 2048;                // points per accumulate block
constexpr int kAcc = 36 + 8;                // Gram upper triangle (<= 36) + rhs (<= 8)

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

__global__ void fit_keys(const float* __restrict__ values, Plan* plan, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ idx, const uint32_t* status) {
  __shared__ uint32_t cnt;
  if (failed(status) || !fit_active(plan)) return;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const uint64_t n = plan->n_values;
  uint32_t nonneg = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float v = values[i];
    uint32_t b = __float_as_uint(v);
    if (b == 0x80000000u) b = 0;  // -0.0 == +0.0 under operator>
    const uint32_t asc = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    keys[i] = ~asc;  // ascending key order == descending value order
    idx[i] = static_cast<uint32_t>(i);
    nonneg += v >= 0.0f ? 1u : 0u;
  }
  nonneg = warp_sum(nonneg);
  if ((threadIdx.x & 31) == 0 && nonneg) atomicAdd(&cnt, nonneg);
  __syncthreads();
  if (threadIdx.x == 0 && cnt) atomicAdd(&plan->sign_split, cnt);
}

// t[s] and the identity flag; map = sorted idx
__global__ void fit_prepare(const float* __restrict__ values, const uint32_t* __restrict__ map, Plan* plan,
                            double* __restrict__ t, const uint32_t* status) {
  if (failed(status) || !fit_active(plan)) return;
  const uint64_t n = plan->n_values;
  const uint64_t l = plan->sign_split;
  bool ident = true;
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (map[s] != s) ident = false;
    t[s] = s < l ? static_cast<double>(values[map[s]]) : -static_cast<double>(values[map[n - 1 - (s - l)]]);
  }
  if (__any_sync(kFull, !ident) && (threadIdx.x & 31) == 0) atomicAnd(&plan->identity, 0u);
}

// ---------------------------------------------------------------- segmentation
struct Piece {
  uint32_t begin, end, arg, live;
  double dev;
};

// Grid-cooperative segmentation: every make_piece (curvefit.cpp:50-67) is one
// sweep in which all blocks scan a slice of the piece, write their block-best
// (dev, arg) to a double-buffered partial array, grid.sync(), and every block
// reduces the partials in block order (same result everywhere, same tie rule:
// max dev, lowest index).  The piece list is replicated per block; children
// of a split are only evaluated when another split can follow.
struct SweepRange {
  uint32_t begin, end;
};

__device__ void seg_sweep(const double* __restrict__ t, const SweepRange* rr, int nr, uint32_t mp, double* pdev,
                          uint32_t* parg, Piece* out, double* sdev, uint32_t* sarg, cg::grid_group& grid) {
  const uint32_t G = gridDim.x;
  for (int q = 0; q < nr; ++q) {
    const uint32_t b = rr[q].begin, e = rr[q].end, len = e - b;
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
  // every block reduces the G partials of each range, all threads in parallel
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
      Piece p{rr[q].begin, rr[q].end, aa, 0u, bb};
      p.live = (bb > 0.0 && aa - p.begin >= mp && p.end - aa >= mp) ? 1u : 0u;
      out[q] = p;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) fit_segment_coop(Plan* plan, const double* __restrict__ t, int degree,
                                                        int max_segments, double* pdev, uint32_t* parg,
                                                        uint32_t* status) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sdev[32];
  __shared__ uint32_t sarg[32];
  __shared__ Piece pieces[kMaxSeg];
  __shared__ Piece res[2];
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
  int sweep = 0;
  uint32_t nseg = 0;
  bool overflow = false;
  for (int pi = 0; pi < nparts && !overflow; ++pi) {
    const uint32_t b = pb[pi], e = pe[pi], len = e - b;
    int budget;
    if (max_segments > 0) {  // curvefit.cpp:473-481
      const long long share = static_cast<long long>(max_segments) * static_cast<long long>(len) /
                              static_cast<long long>(n);
      budget = share > 1 ? static_cast<int>(share) : 1;
      if (pi + 1 == nparts) budget = max_segments - static_cast<int>(nseg) > 1 ? max_segments - static_cast<int>(nseg) : 1;
    } else if (len < 4) {
      budget = 1;
    } else {  // part_budget (curvefit.cpp:101-110, :424-428)
      const double km = fabs(__dsub_rn(__dsub_rn(t[b], t[b + 1]), __dsub_rn(t[e - 2], t[e - 1])));
      const double p = ceil(2.0 * sqrt(km > 0.0 ? km : 0.0));
      const int kc = static_cast<int>(p) > 1 ? static_cast<int>(p) : 1;
      budget = kc + 1 < 0xffff ? kc + 1 : 0xffff;
    }
    int np = 1;
    if (budget > 1) {
      SweepRange r0{0, len};
      seg_sweep(t + b, &r0, 1, mp, pdev + (sweep & 1) * 2 * G, parg + (sweep & 1) * 2 * G, res, sdev, sarg, grid);
      ++sweep;
      if (threadIdx.x == 0) pieces[0] = res[0];
    } else if (threadIdx.x == 0) {
      pieces[0] = Piece{0, len, 0, 0u, 0.0};
    }
    __syncthreads();
    while (np < budget) {
      if (threadIdx.x == 0) {
        int best = -1;
        for (int i = 0; i < np; ++i) {
          if (!pieces[i].live) continue;
          if (best < 0 || pieces[i].dev > pieces[best].dev ||
              (pieces[i].dev == pieces[best].dev && pieces[i].begin < pieces[best].begin))
            best = i;
        }
        s_best = best;
      }
      __syncthreads();
      const int best = s_best;
      if (best < 0) break;
      if (nseg + np + 1 > static_cast<uint32_t>(kMaxSeg)) {
        overflow = true;
        break;
      }
      const Piece pp = pieces[best];
      Piece left{pp.begin, pp.arg, 0, 0u, 0.0}, right{pp.arg, pp.end, 0, 0u, 0.0};
      if (np + 1 < budget) {  // another split may follow: evaluate both children
        SweepRange rr[2] = {{pp.begin, pp.arg}, {pp.arg, pp.end}};
        seg_sweep(t + b, rr, 2, mp, pdev + (sweep & 1) * 2 * G, parg + (sweep & 1) * 2 * G, res, sdev, sarg, grid);
        ++sweep;
        left = res[0];
        right = res[1];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        pieces[best] = left;
        pieces[np] = right;
      }
      ++np;
      __syncthreads();
    }
    if (overflow) break;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      for (int i = 1; i < np; ++i) {  // sort by begin
        const Piece v = pieces[i];
        int j = i;
        while (j > 0 && pieces[j - 1].begin > v.begin) {
          pieces[j] = pieces[j - 1];
          --j;
        }
        pieces[j] = v;
      }
      for (int i = 0; i < np; ++i) plan->seg_end[nseg + i] = b + pieces[i].end;
    }
    nseg += static_cast<uint32_t>(np);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (overflow) latch(status, GP_CAPACITY);
    plan->nseg = nseg;
    plan->degree = static_cast<uint32_t>(degree);
  }
}

// ---------------------------------------------------------------- least squares
__device__ __forceinline__ void seg_range(const Plan* plan, uint32_t s, uint32_t& b, uint32_t& e) {
  b = s == 0 ? 0 : plan->seg_end[s - 1];
  e = plan->seg_end[s];
}

// chunk c of the concatenated per-segment chunk lists → (segment, start)
__device__ bool locate_chunk(const Plan* plan, uint64_t c, uint32_t& seg, uint32_t& start, uint32_t& stop) {
  uint64_t acc = 0;
  for (uint32_t s = 0; s < plan->nseg; ++s) {
    uint32_t b, e;
    seg_range(plan, s, b, e);
    const uint64_t nc = (e - b + kChunk - 1) / kChunk;
    if (c < acc + nc) {
      seg = s;
      start = b + static_cast<uint32_t>((c - acc) * kChunk);
      stop = start + kChunk < e ? start + kChunk : e;
      return true;
    }
    acc += nc;
  }
  return false;
}

__global__ void __launch_bounds__(256) fit_accumulate(const Plan* plan, const double* __restrict__ t,
                                                      double* __restrict__ partial, const uint32_t* status) {
  __shared__ double red[8][kAcc];
  if (failed(status) || !poly_active(plan)) return;
  uint32_t seg, start, stop;
  if (!locate_chunk(plan, blockIdx.x, seg, start, stop)) return;
  uint32_t b, e;
  seg_range(plan, seg, b, e);
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
    partial[static_cast<uint64_t>(blockIdx.x) * kAcc + threadIdx.x] = v;
  }
}

// one block per segment; thread 0 solves (sizes are <= 8x8)
__global__ void fit_solve(Plan* plan, const double* __restrict__ t, const double* __restrict__ partial,
                          const uint32_t* status) {
  __shared__ double sacc[kAcc];
  if (failed(status) || !poly_active(plan)) return;
  const uint32_t seg = blockIdx.x;
  if (seg >= plan->nseg) return;
  uint32_t b, e;
  seg_range(plan, seg, b, e);
  {  // chunk partials of this segment, summed in chunk order, one accumulator per thread
    uint64_t c0 = 0;
    for (uint32_t s2 = 0; s2 < seg; ++s2) {
      uint32_t bb, ee;
      seg_range(plan, s2, bb, ee);
      c0 += (ee - bb + kChunk - 1) / kChunk;
    }
    const uint64_t ncs = (e - b + kChunk - 1) / kChunk;
    if (threadIdx.x < kAcc) {
      double v = 0.0;
      for (uint64_t c = 0; c < ncs; ++c) v += partial[(c0 + c) * kAcc + threadIdx.x];
      sacc[threadIdx.x] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const uint32_t len = e - b;
  const int deg = static_cast<int>(plan->degree);
  float* out = plan->coeffs + seg * kCps;
  for (int j = 0; j <= deg; ++j) out[j] = 0.0f;
  if (len == 1) {  // curvefit.cpp:134-138
    out[0] = static_cast<float>(t[b]);
    return;
  }
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
      double s = G[j][j];
#pragma unroll
      for (int q = 0; q < j; ++q) s -= L[j][q] * L[j][q];
      L[j][j] = sqrt(s > 0.0 ? s : 0.0);
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
  // Legendre → t-monomials: P_{j+1} = ((2j+1) t P_j - j P_{j-1}) / (j+1)
  double Lc[kCps][kCps];
#pragma unroll
  for (int j = 0; j < kCps; ++j)
#pragma unroll
    for (int p = 0; p < kCps; ++p) Lc[j][p] = 0.0;
  Lc[0][0] = 1.0;
  Lc[1][1] = 1.0;
#pragma unroll
  for (int j = 1; j + 1 < kCps; ++j)
#pragma unroll
    for (int p = 0; p <= j + 1; ++p)
      Lc[j + 1][p] = ((2 * j + 1) * (p > 0 ? Lc[j][p - 1] : 0.0) - j * Lc[j - 1][p]) / (j + 1);
  double ct[kCps];
#pragma unroll
  for (int p = 0; p < kCps; ++p) {
    double v = 0.0;
#pragma unroll
    for (int j = p; j < kCps; ++j) v += aL[j] * Lc[j][p];  // aL[j] = 0 for j >= m
    ct[p] = v;
  }
  // t-monomials → x-monomials, curvefit.cpp:157-172 (the same pow() values)
  const double alpha = 2.0 / static_cast<double>(len - 1);
  const double beta = -static_cast<double>(len + 1) / static_cast<double>(len - 1);
  double pa[kCps], pb[kCps];
#pragma unroll
  for (int k = 0; k < kCps; ++k) {
    pa[k] = k < m ? pow(alpha, static_cast<double>(k)) : 0.0;
    pb[k] = k < m ? pow(beta, static_cast<double>(k)) : 0.0;
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

// serialize_fit (curvefit.cpp:285-298) + reorder payload size; vl, rl, flags
__global__ void fit_emit(Plan* plan, uint8_t* out, int cfg_degree, const uint32_t* status) {
  if (failed(status) || !fit_active(plan) || threadIdx.x != 0) return;
  const uint32_t kind = plan->fit_kind;
  const uint32_t S = plan->nseg, deg = kind ? static_cast<uint32_t>(cfg_degree) : plan->degree;
  const uint32_t cps = kind ? 4 : deg + 1;  // coeffs_per_segment
  uint8_t* p = out + 49 + plan->il;
  p[0] = static_cast<uint8_t>(kind);  // 0 piecewise polynomial, 1 double exponential
  p[1] = static_cast<uint8_t>(S);
  p[2] = static_cast<uint8_t>(S >> 8);
  uint8_t* q = p + 3;
  for (uint32_t s = 0; s < S; ++s, q += 4) st_u32_unaligned(q, plan->seg_end[s]);
  *q++ = static_cast<uint8_t>(deg);
  for (uint32_t s = 0; s < S; ++s)
    for (uint32_t j = 0; j < cps; ++j, q += 4) st_u32_unaligned(q, __float_as_uint(plan->coeffs[s * kCps + j]));
  st_u32_unaligned(q, plan->sign_split);
  plan->vl = 1 + 2 + 4ull * S + 1 + 4ull * S * cps + 4;
  uint32_t w = 0;
  for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
  plan->rl = plan->identity ? 0 : (plan->n_values * w + 7) / 8;
}

// reorder_encode (curvefit.cpp:332-340): entries of w bits, LSB-first
__global__ void reorder_pack(const uint32_t* __restrict__ map, Plan* plan, uint8_t* out, const uint32_t* status) {
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
// the reorder_decode length/slack rules (curvefit.cpp:342-356).
__global__ void fit_parse(const uint8_t* __restrict__ in, Plan* plan, uint32_t* status) {
  if (failed(status) || !fit_active(plan)) return;
  const uint8_t* p = in + plan->off_value;
  const uint64_t vl = plan->vl, count = plan->n_values;
  if (vl < 1) return latch(status, GP_TRUNCATED);
  if (p[0] > 1) return latch(status, GP_UNKNOWN_METHOD);
  const uint8_t kind = p[0];
  if (vl < 3) return latch(status, GP_TRUNCATED);
  const uint32_t S = p[1] | (p[2] << 8);
  if (S < 1) return latch(status, GP_CORRUPT_PAYLOAD);
  uint32_t prev = 0;
  for (uint32_t i = 0; i < S; ++i) {
    if (vl < 3 + 4ull * (i + 1)) return latch(status, GP_TRUNCATED);
    const uint32_t e = ld_u32_unaligned(p + 3 + 4 * i);
    if (e <= prev && !(i == 0 && e > 0)) return latch(status, GP_CORRUPT_PAYLOAD);
    prev = e;
    if (i < kMaxSeg) plan->seg_end[i] = e;
  }
  if (prev != count) return latch(status, GP_CORRUPT_PAYLOAD);
  uint64_t at = 3 + 4ull * S;
  if (vl < at + 1) return latch(status, GP_TRUNCATED);
  const uint32_t deg = p[at++];
  const uint64_t cps = kind == 1 ? 4 : deg + 1;
  if (vl < at + 4 * S * cps) return latch(status, GP_TRUNCATED);
  const uint64_t coeff_at = at;
  at += 4 * S * cps;
  if (vl < at + 4) return latch(status, GP_TRUNCATED);
  const uint32_t l = ld_u32_unaligned(p + at);
  at += 4;
  if (l > count) return latch(status, GP_CORRUPT_PAYLOAD);
  if (l > 0 && l < count) {
    bool found = false;
    for (uint32_t i = 0; i < S; ++i) found |= ld_u32_unaligned(p + 3 + 4 * i) == l;
    if (!found) return latch(status, GP_CORRUPT_PAYLOAD);
  }
  if (at != vl) return latch(status, GP_CORRUPT_PAYLOAD);
  // reorder_decode structure: count entries of w bits, < 8 slack bits, zero slack
  if (plan->rl) {
    uint32_t w = 0;
    for (uint64_t x = plan->d - 1; x; x >>= 1) ++w;
    const uint64_t need = count * w, have = 8 * plan->rl;
    if (have < need) return latch(status, GP_TRUNCATED);
    if (have - need >= 8) return latch(status, GP_CORRUPT_PAYLOAD);
    if (have > need) {
      const uint8_t last = in[plan->off_reorder + plan->rl - 1];
      if (last >> (need % 8)) return latch(status, GP_CORRUPT_PAYLOAD);
    }
  }
  if (S > kMaxSeg || (kind == 0 && deg > kMaxDeg)) return latch(status, GP_CAPACITY);
  plan->nseg = S;
  plan->degree = deg;
  plan->fit_kind = kind;
  plan->sign_split = l;
  for (uint32_t s = 0; s < S; ++s)
    for (uint32_t j = 0; j < cps; ++j)
      plan->coeffs[s * kCps + j] = __uint_as_float(ld_u32_unaligned(p + coeff_at + 4 * (s * cps + j)));
}

// reorder entries (entry >= d → corrupt) + permutation check (curvefit.cpp:531-538)
__global__ void reorder_unpack(const uint8_t* __restrict__ in, Plan* plan, uint32_t* __restrict__ map,
                               uint32_t* seen, uint32_t* status) {
  if (failed(status) || !fit_active(plan) || plan->rl == 0) return;
  const uint64_t n = plan->n_values, d = plan->d;
  uint32_t w = 0;
  for (uint64_t x = d - 1; x; x >>= 1) ++w;
  const uint8_t* p = in + plan->off_reorder;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t v = 0;
    const uint64_t bit0 = i * w;
    for (uint32_t j = 0; j < w; ++j) {
      const uint64_t bit = bit0 + j;
      v |= static_cast<uint64_t>((p[bit >> 3] >> (bit & 7)) & 1u) << j;
    }
    if (v >= d || v >= n) {
      latch(status, GP_CORRUPT_PAYLOAD);
      continue;
    }
    map[i] = static_cast<uint32_t>(v);
    if (atomicOr(&seen[v >> 5], 1u << (v & 31)) & (1u << (v & 31))) latch(status, GP_CORRUPT_PAYLOAD);
  }
}

// value_decompress evaluate + unfold + scatter (curvefit.cpp:517-541)
__global__ void fit_eval(const Plan* plan, const uint32_t* __restrict__ map, double* __restrict__ out,
                         const uint32_t* status) {
  __shared__ uint32_t bounds[kMaxSeg];
  __shared__ float coeffs[kMaxSeg * kCps];
  if (failed(status) || !fit_active(plan)) return;
  const uint32_t S = plan->nseg, cps = plan->degree + 1;
  const bool dexp = plan->fit_kind == 1;
  for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) bounds[i] = plan->seg_end[i];
  for (uint32_t i = threadIdx.x; i < S * kCps; i += blockDim.x) coeffs[i] = plan->coeffs[i];
  __syncthreads();
  const uint64_t n = plan->n_values;
  const uint64_t l = plan->sign_split;
  const bool reorder = plan->rl != 0;
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = s < l ? s : l + (n - 1 - s);  // position in the folded sequence
    uint32_t seg = 0;
    while (bounds[seg] <= j) ++seg;
    const uint32_t begin = seg == 0 ? 0 : bounds[seg - 1];
    const double x = static_cast<double>(j - begin + 1);
    const float* c = coeffs + seg * kCps;
    double acc = 0.0;
    if (dexp)
      acc = eval_dexp(c, x);
    else
      for (int q = static_cast<int>(cps) - 1; q >= 0; --q) acc = __dadd_rn(__dmul_rn(acc, x), static_cast<double>(c[q]));
    const double v = s < l ? acc : -acc;
    out[reorder ? map[s] : s] = v;
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

__global__ void __launch_bounds__(kDexpBlock) dexp_fit(Plan* plan, const double* __restrict__ t,
                                                        const uint32_t* status) {
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
    float* co = plan->coeffs + blockIdx.x * kCps;
    co[0] = static_cast<float>(a);
    co[1] = static_cast<float>(b);
    co[2] = static_cast<float>(c);
    co[3] = static_cast<float>(d);
    plan->seg_end[blockIdx.x] = parts[blockIdx.x][1];
  }
}

// dexp model or the polynomial fallback (value_compress attempt 1)
__global__ void dexp_decide(Plan* plan, const uint32_t* status) {
  if (failed(status) || plan->value_method != GP_VALUE_FIT_DEXP) return;
  if (plan->dexp_fail) return;  // fit_kind stays 0: the polynomial path runs
  const uint32_t n = static_cast<uint32_t>(plan->n_values), l = plan->sign_split;
  plan->nseg = (l > 0 ? 1u : 0u) + (l < n ? 1u : 0u);
  plan->fit_kind = 1;
}

}  // namespace

void launch_radix_sort(gp_ctx* ctx, uint32_t* keys, uint32_t* vals, uint32_t* ktmp, uint32_t* vtmp,
                       const uint64_t* n_dev, uint64_t n_bound, int bits, cudaStream_t s);

__global__ void fit_reset(Plan* plan) {
  plan->sign_split = 0;
  plan->identity = 1;
  plan->fit_kind = 0;
  plan->dexp_fail = 0;
}

void launch_values_fit(gp_ctx* ctx, uint8_t* out, int degree, int max_segments, uint64_t n_bound, cudaStream_t s,
                       bool dexp) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, fit_reset, 1, 1, 0, s, w.plan);
  GP_LAUNCH(ctx, fit_keys, grid_for(ctx, n_bound, 256), 256, 0, s, w.values, w.plan, w.u32a, w.u32b, w.status);
  launch_radix_sort(ctx, w.u32a, w.u32b, w.u32c, w.u32d, &w.plan->n_values, n_bound, 32, s);
  GP_LAUNCH(ctx, fit_prepare, grid_for(ctx, n_bound, 256), 256, 0, s, w.values, w.u32b, w.plan, w.f64b, w.status);
  if (dexp) {
    GP_LAUNCH(ctx, dexp_fit, 2, kDexpBlock, 0, s, w.plan, w.f64b, w.status);
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
    uint32_t* st = w.status;
    void* args[] = {&plan, &t, &degree, &max_segments, &pdev, &parg, &st};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fit_segment_coop), grid, 256, args, 0, s);
    ++ctx->launches;
  }
  const uint64_t chunks = n_bound / kChunk + kMaxSeg + 1;
  GP_LAUNCH(ctx, fit_accumulate, static_cast<int>(chunks), 256, 0, s, w.plan, w.f64b, w.partial, w.status);
  GP_LAUNCH(ctx, fit_solve, kMaxSeg, 64, 0, s, w.plan, w.f64b, w.partial, w.status);
  GP_LAUNCH(ctx, fit_emit, 1, 32, 0, s, w.plan, out, degree, w.status);
  GP_LAUNCH(ctx, reorder_pack, grid_for(ctx, n_bound * 4, 256), 256, 0, s, w.u32b, w.plan, out, w.status);
}

void launch_decode_fit(gp_ctx* ctx, const uint8_t* in, uint64_t n_bound, cudaStream_t s) {
  Workspace& w = ctx->ws;
  GP_LAUNCH(ctx, fit_parse, 1, 1, 0, s, in, w.plan, w.status);
  cudaMemsetAsync(w.u32c, 0, ((n_bound + 31) / 32) * 4, s);
  GP_LAUNCH(ctx, reorder_unpack, grid_for(ctx, n_bound, 256), 256, 0, s, in, w.plan, w.u32b, w.u32c, w.status);
  GP_LAUNCH(ctx, fit_eval, grid_for(ctx, n_bound, 256), 256, 0, s, w.plan, w.u32b, w.f64a, w.status);
}

}  // namespace gp
