// fluence.cu — fluence products and coverage.
//
//   k_nonzero   ordered list of columns with t_k != 0 (LP plans are sparse)
//   k_gemv_n    μ = A·t  (Eq. 5): each thread owns 4 consecutive rows
//               (one float4 per column, coalesced 512 B per warp per column),
//               walks the nonzero columns in order, fp64 accumulation -> the
//               summation order is fixed (deterministic); HBM-bound
//   k_gemv_t    g = Aᵀ·y (the LP's adjoint product): one CTA per 4
//               columns, float4 row chunks, y read once per 4 columns, fixed
//               tree reduction in fp64; HBM-bound
//   k_gemv_multi  μ = A·x, A·𝟙 and Aᵀ·y in ONE pass over A (uvd_fluence_multi,
//               the bench step's three products): register row sums, a butterfly
//               reduce-scatter of the column dots into per-warp partials,
//               k_gemv_t_reduce in a fixed chunked order; HBM-bound, deterministic
//   k_coverage  Σ|s_i|[μ_i ≥ μ_min], Σ|s_i|, Σ|s_i|[rowsum_i > 0] (P:9),
//               fixed-shape two-level reduction
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <vector>

#include "uvd_internal.cuh"

namespace uvd {

__global__ void __launch_bounds__(1024) k_nonzero(const double* __restrict__ x, int64_t k,
                                                  int32_t* __restrict__ idx, double* __restrict__ val,
                                                  int32_t* __restrict__ cnt) {
  __shared__ int32_t part[1024];
  int64_t per = (k + 1023) / 1024;
  int64_t s = threadIdx.x * per, e = s + per < k ? s + per : k;
  int32_t c = 0;
  for (int64_t i = s; i < e; ++i) c += x[i] != 0.0;
  part[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = s; i < e; ++i)
    if (x[i] != 0.0) { idx[run] = (int32_t)i; val[run] = x[i]; ++run; }
  if (threadIdx.x == 1023) *cnt = part[1023];
}

constexpr int kGemvThreads = 256;

// μ = A·t over the nonzero columns.  Each thread owns 4 consecutive rows
// (float4 loads, 512 B per warp per column, 8 columns in flight); when there are
// too few row quads to keep enough bytes in flight (Little's law: ~6.5 MB at
// 6.5 TB/s and ~1 µs), the column list is split over gridDim.y chunks whose
// partial sums are added in chunk order by k_gemv_n_reduce (deterministic).
__global__ void __launch_bounds__(kGemvThreads) k_gemv_n(const float* __restrict__ A, int64_t ld,
                                                         int64_t n, const int32_t* __restrict__ idx,
                                                         const double* __restrict__ val,
                                                         const int32_t* __restrict__ cnt, int64_t chunk,
                                                         double* __restrict__ out) {
  const int64_t q = blockIdx.x * (int64_t)kGemvThreads + threadIdx.x;  // row quad
  const int64_t r0 = 4 * q;
  if (r0 >= n) return;
  const int32_t nz = *cnt;
  const int64_t kb = (int64_t)blockIdx.y * chunk;
  const int64_t ke = kb + chunk < (int64_t)nz ? kb + chunk : (int64_t)nz;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const float4* __restrict__ A4 = reinterpret_cast<const float4*>(A);
  const int64_t ld4 = ld / 4;
  int64_t k = kb;
  for (; k + 8 <= ke; k += 8) {  // 8 columns in flight
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(A4 + (int64_t)idx[k + u] * ld4 + q);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double t = val[k + u];
      a0 += (double)v[u].x * t; a1 += (double)v[u].y * t; a2 += (double)v[u].z * t; a3 += (double)v[u].w * t;
    }
  }
  for (; k < ke; ++k) {
    float4 v = __ldcs(A4 + (int64_t)idx[k] * ld4 + q);
    double t = val[k];
    a0 += (double)v.x * t; a1 += (double)v.y * t; a2 += (double)v.z * t; a3 += (double)v.w * t;
  }
  double* o = out + (int64_t)blockIdx.y * n;
  o[r0] = a0;
  if (r0 + 1 < n) o[r0 + 1] = a1;
  if (r0 + 2 < n) o[r0 + 2] = a2;
  if (r0 + 3 < n) o[r0 + 3] = a3;
}

__global__ void k_gemv_n_reduce(const double* __restrict__ part, int s, int64_t n, double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int k = 0; k < s; ++k) v += part[k * n + r];
    out[r] = v;
  }
}

// g = Aᵀ·y: one CTA per 4 columns, float4 row chunks, y read once per 4
// columns (L2-resident), fixed tree reduction.  (16 columns per CTA measured
// 27 % slower: 190 registers, one CTA per SM.)
constexpr int kGemvTCols = 4;

__global__ void __launch_bounds__(kGemvThreads) k_gemv_t(const float* __restrict__ A, int64_t ld,
                                                         int64_t n, int64_t k,
                                                         const double* __restrict__ y,
                                                         double* __restrict__ out) {
  __shared__ double red[kGemvTCols][kGemvThreads / 32];
  const int64_t c0 = (int64_t)blockIdx.x * kGemvTCols;
  const int nc = (int)(k - c0 < kGemvTCols ? k - c0 : kGemvTCols);
  const float4* __restrict__ A4 = reinterpret_cast<const float4*>(A);
  const int64_t ld4 = ld / 4, nq = (n + 3) / 4;
  double acc[kGemvTCols];
#pragma unroll
  for (int c = 0; c < kGemvTCols; ++c) acc[c] = 0.0;
  for (int64_t q = threadIdx.x; q < nq; q += kGemvThreads) {
    const int64_t r = 4 * q;
    const double y0 = y[r];
    const double y1 = r + 1 < n ? y[r + 1] : 0.0;
    const double y2 = r + 2 < n ? y[r + 2] : 0.0;
    const double y3 = r + 3 < n ? y[r + 3] : 0.0;
    if (nc == kGemvTCols) {
      float4 v[kGemvTCols];
#pragma unroll
      for (int c = 0; c < kGemvTCols; ++c) v[c] = __ldcs(A4 + (c0 + c) * ld4 + q);
#pragma unroll
      for (int c = 0; c < kGemvTCols; ++c)
        acc[c] += (double)v[c].x * y0 + (double)v[c].y * y1 + (double)v[c].z * y2 + (double)v[c].w * y3;
    } else {
#pragma unroll
      for (int c = 0; c < kGemvTCols; ++c)
        if (c < nc) {
          const float4 v = __ldcs(A4 + (c0 + c) * ld4 + q);
          acc[c] += (double)v.x * y0 + (double)v.y * y1 + (double)v.z * y2 + (double)v.w * y3;
        }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kGemvTCols; ++c) {
    double v = acc[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < nc) {
    double v = 0.0;
    for (int w = 0; w < kGemvThreads / 32; ++w) v += red[threadIdx.x][w];
    out[c0 + threadIdx.x] = v;
  }
}

// The three products of one step in ONE pass over a dense A (uvd_fluence_multi):
// μ = A·x, A·𝟙 and g = Aᵀ·y.  A thread owns 4 rows across all columns (one
// float4 per column, 8 columns in flight): μ and A·𝟙 accumulate in registers in
// column order — the same fp64 sums as k_gemv_n over all columns (x_j = 0 adds
// an exact 0).  For Aᵀ·y each warp reduces its 128 rows' dots of the 8 columns
// with a butterfly reduce-scatter (lanes trade half their columns at each of
// the first three steps: 9 shuffles for 8 columns instead of 40) and writes the
// 8 partials as one contiguous 64-byte row of part[warp][k]; k_gemv_t_reduce
// sums the warps in order.  No block barrier; deterministic; HBM-bound: A is
// read once instead of once per product.
static __global__ void k_fill_value(double* __restrict__ p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

#ifndef UVD_MULTI_THREADS
#define UVD_MULTI_THREADS 128  // 128 / 64 / 256 / 512: 8.4–8.5 / 8.5 / 9.2 / 9.4 ms per C5 pass
#endif
constexpr int kMultiThreads = UVD_MULTI_THREADS;
constexpr int kMultiCols = 8;  // columns in flight per thread (the reduce-scatter is written for 8)

__device__ __forceinline__ double shfl_x(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

template <bool X, bool ONE, bool Y>
__global__ void __launch_bounds__(kMultiThreads) k_gemv_multi(const float* __restrict__ A, int64_t ld, int64_t n,
                                                              int64_t k, const double* __restrict__ x,
                                                              const double* __restrict__ y,
                                                              double* __restrict__ ax, double* __restrict__ a1,
                                                              double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * kMultiThreads + threadIdx.x;  // row quad
  const int64_t gw = q >> 5;                                           // global warp
  const int64_t r0 = 4 * q;
  const bool in = r0 < n;
  const float4* __restrict__ A4 = reinterpret_cast<const float4*>(A) + q;
  const int64_t ld4 = ld / 4;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
  if (Y && in) {
    y0 = y[r0];
    y1 = r0 + 1 < n ? y[r0 + 1] : 0.0;
    y2 = r0 + 2 < n ? y[r0 + 2] : 0.0;
    y3 = r0 + 3 < n ? y[r0 + 3] : 0.0;
  }
  // after the reduce-scatter, lane l holds column c(l) = bits 4, 3, 2 of l (as
  // 4·b4 + 2·b3 + b2) summed over lanes l ^ {0, 1, 2, 3}; lanes with l % 4 == 0 write
  const int cl = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  // software-pipelined: the next 8 columns are in flight while this group's
  // sums and the shuffle chain of its reduce-scatter run
  float4 v[kMultiCols], vn[kMultiCols];
#pragma unroll
  for (int u = 0; u < kMultiCols; ++u)
    v[u] = (in && u < k) ? __ldcs(A4 + (int64_t)u * ld4) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t c0 = 0; c0 < k; c0 += kMultiCols) {
    const int nc = (int)(k - c0 < kMultiCols ? k - c0 : kMultiCols);
    const int64_t c1 = c0 + kMultiCols;
#pragma unroll
    for (int u = 0; u < kMultiCols; ++u)
      vn[u] = (in && c1 + u < k) ? __ldcs(A4 + (c1 + u) * ld4) : make_float4(0.f, 0.f, 0.f, 0.f);
    double d[kMultiCols];
#pragma unroll
    for (int u = 0; u < kMultiCols; ++u) {
      if (X && u < nc) {
        const double t = x[c0 + u];
        m0 += (double)v[u].x * t; m1 += (double)v[u].y * t; m2 += (double)v[u].z * t; m3 += (double)v[u].w * t;
      }
      if (ONE) { s0 += (double)v[u].x; s1 += (double)v[u].y; s2 += (double)v[u].z; s3 += (double)v[u].w; }
      d[u] = Y ? (double)v[u].x * y0 + (double)v[u].y * y1 + (double)v[u].z * y2 + (double)v[u].w * y3 : 0.0;
    }
    if (Y) {
      // step 1 (xor 16): keep columns 0-3 (bit 4 clear) or 4-7, send the other half
      const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
      double e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double mine = h4 ? d[u + 4] : d[u], other = h4 ? d[u] : d[u + 4];
        e[u] = mine + shfl_x(other, 16);
      }
      double f[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double mine = h3 ? e[u + 2] : e[u], other = h3 ? e[u] : e[u + 2];
        f[u] = mine + shfl_x(other, 8);
      }
      double g = (h2 ? f[1] : f[0]) + shfl_x(h2 ? f[0] : f[1], 4);
      g += shfl_x(g, 2);
      g += shfl_x(g, 1);
      if ((lane & 3) == 0 && cl < nc) part[gw * k + c0 + cl] = g;
    }
#pragma unroll
    for (int u = 0; u < kMultiCols; ++u) v[u] = vn[u];
  }
  if (!in) return;
  if (X) {
    ax[r0] = m0;
    if (r0 + 1 < n) ax[r0 + 1] = m1;
    if (r0 + 2 < n) ax[r0 + 2] = m2;
    if (r0 + 3 < n) ax[r0 + 3] = m3;
  }
  if (ONE) {
    a1[r0] = s0;
    if (r0 + 1 < n) a1[r0 + 1] = s1;
    if (r0 + 2 < n) a1[r0 + 2] = s2;
    if (r0 + 3 < n) a1[r0 + 3] = s3;
  }
}

// Σ over the warps' partials in a fixed order: gridDim.y chunks of warps
// (chunk sums to part2[chunk][k]), then the chunks in order (deterministic)
__global__ void k_gemv_t_reduce(const double* __restrict__ part, int64_t nw, int64_t k, double* __restrict__ out) {
  const int64_t per = (nw + gridDim.y - 1) / gridDim.y, w0 = blockIdx.y * per;
  const int64_t w1 = w0 + per < nw ? w0 + per : nw;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t w = w0; w < w1; ++w) v += part[w * k + j];
    out[(int64_t)blockIdx.y * k + j] = v;
  }
}

// CSC: μ += A[:,c]·t_c for the nonzero columns (one block per column, fp64
// atomics: the order of the per-row additions is not fixed, so results may
// differ from the dense kernel by a few fp64 ulps); g_c = Σ_e vals·y[row]
// (one block per column, fixed tree reduction)
__global__ void k_csc_n(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                        const float* __restrict__ vals, const int32_t* __restrict__ idx,
                        const double* __restrict__ val, const int32_t* __restrict__ cnt,
                        double* __restrict__ out) {
  for (int32_t q = blockIdx.x; q < *cnt; q += gridDim.x) {
    const int64_t c = idx[q];
    const double t = val[q];
    for (int64_t e = colptr[c] + threadIdx.x; e < colptr[c + 1]; e += blockDim.x)
      atomicAdd(out + rowidx[e], (double)vals[e] * t);
  }
}

__global__ void __launch_bounds__(kGemvThreads) k_csc_t(const int64_t* __restrict__ colptr,
                                                        const int32_t* __restrict__ rowidx,
                                                        const float* __restrict__ vals,
                                                        const double* __restrict__ y,
                                                        double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  double s = 0.0;
  for (int64_t e = colptr[c] + threadIdx.x; e < colptr[c + 1]; e += kGemvThreads)
    s += (double)vals[e] * y[rowidx[e]];
  __shared__ double red[kGemvThreads];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kGemvThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

// coverage: per-block partials, then one block combines them in fixed order
constexpr int kCovThreads = 256;
__global__ void __launch_bounds__(kCovThreads) k_coverage_part(const double* __restrict__ mu,
                                                               const double* __restrict__ area,
                                                               const double* __restrict__ rowsum,
                                                               int64_t n, double mu_min,
                                                               double* __restrict__ part) {
  __shared__ double s[3][kCovThreads];
  double c = 0.0, t = 0.0, v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kCovThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kCovThreads) {
    double a = area[i];
    t += a;
    if (mu[i] >= mu_min) c += a;             // inclusive (Q16)
    if (!rowsum || rowsum[i] > 0.0) v += a;  // ever visible
  }
  s[0][threadIdx.x] = c; s[1][threadIdx.x] = t; s[2][threadIdx.x] = v;
  __syncthreads();
  for (int off = kCovThreads / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
      for (int k = 0; k < 3; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x < 3) part[3 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_coverage_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += part[3 * b + threadIdx.x];
    out[threadIdx.x] = v;
  }
}

// NEXT-4 static single-point baseline (P:7): per
// column j of a dense shard, out[3j..3j+2] = {Σ_i |s_i| [A_ij > 0] (visible
// area), min_{A_ij > 0} A_ij (+inf if none), Σ_i |s_i| [A_ij·T ≥ μ_min]
// (area covered by a static lamp left at j for T)}.  One block per column
// (contiguous column reads), fixed-order reduction.
constexpr int kStaticThreads = 256;
__global__ void __launch_bounds__(kStaticThreads) k_static_cols(const float* __restrict__ A, int64_t ld, int64_t n,
                                                                const double* __restrict__ area, double t_budget,
                                                                double mu_min, double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const float* col = A + c * ld;
  double vis = 0.0, cov = 0.0, mn = INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += kStaticThreads) {
    const double a = (double)__ldcs(col + i);
    if (a > 0.0) {
      vis += area[i];
      mn = fmin(mn, a);
      if (a * t_budget >= mu_min) cov += area[i];  // inclusive (Q16)
    }
  }
  __shared__ double s[3][kStaticThreads];
  s[0][threadIdx.x] = vis; s[1][threadIdx.x] = mn; s[2][threadIdx.x] = cov;
  __syncthreads();
  for (int o = kStaticThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s[0][threadIdx.x] += s[0][threadIdx.x + o];
      s[1][threadIdx.x] = fmin(s[1][threadIdx.x], s[1][threadIdx.x + o]);
      s[2][threadIdx.x] += s[2][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x < 3) out[3 * c + threadIdx.x] = s[threadIdx.x][0];
}


// NEXT-4 choice (reading Q24): the column with the largest visible area, ties
// to the shorter dwell μ_min / min A, then the lower index; and the column
// covering most area within the budget, ties to the lower index.  One block
// and a total order: the result is unique and deterministic.
struct StaticPick {
  double vis, dwell, cov;
  int64_t j;
};
__device__ __forceinline__ bool better_vis(const StaticPick& a, const StaticPick& b) {
  if (a.vis != b.vis) return a.vis > b.vis;
  if (a.dwell != b.dwell) return a.dwell < b.dwell;
  return a.j < b.j;
}
__device__ __forceinline__ bool better_cov(const StaticPick& a, const StaticPick& b) {
  if (a.cov != b.cov) return a.cov > b.cov;
  return a.j < b.j;
}
__global__ void __launch_bounds__(kStaticThreads) k_static_choose(const double* __restrict__ cols3, int64_t k,
                                                                  double mu_min, double* __restrict__ res) {
  StaticPick bv{-1.0, INFINITY, -1.0, INT64_MAX}, bc = bv;
  for (int64_t j = threadIdx.x; j < k; j += kStaticThreads) {
    const double mn = cols3[3 * j + 1];
    const StaticPick c{cols3[3 * j], isinf(mn) ? INFINITY : mu_min / mn, cols3[3 * j + 2], j};
    if (better_vis(c, bv)) bv = c;
    if (better_cov(c, bc)) bc = c;
  }
  __shared__ StaticPick sv[kStaticThreads], sc[kStaticThreads];
  sv[threadIdx.x] = bv;
  sc[threadIdx.x] = bc;
  __syncthreads();
  for (int o = kStaticThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      if (better_vis(sv[threadIdx.x + o], sv[threadIdx.x])) sv[threadIdx.x] = sv[threadIdx.x + o];
      if (better_cov(sc[threadIdx.x + o], sc[threadIdx.x])) sc[threadIdx.x] = sc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    res[0] = (double)sv[0].j;
    res[1] = sv[0].dwell;
    res[2] = (double)sc[0].j;
  }
}

// The allocator of a matrix's scratch: the caller's (A->allocator) or the
// ABI's default, cudaMallocAsync / cudaFreeAsync on the call's stream.
Alloc matrix_alloc(const uvd_matrix_out* A, int dev, cudaStream_t st) {
  Alloc al;
  al.device = dev;
  al.stream = st;
  if (A && A->allocator && A->allocator->alloc && A->allocator->free) {
    al.user = *A->allocator;
    al.has_user = true;
  }
  return al;
}

// Column split of A·t when the row quads alone cannot keep HBM busy.
static int64_t gemv_split(int64_t n, int64_t k, bool csc, int dev) {
  const int sms = sm_count(dev);
  const int64_t quads = (n + 3) / 4;
  const int64_t rblocks = (quads + kGemvThreads - 1) / kGemvThreads;
  int64_t split = csc ? 1 : std::max<int64_t>(1, std::min<int64_t>((8 * sms + rblocks - 1) / rblocks, 16));
  split = std::max<int64_t>(1, std::min<int64_t>(split, k / 8));
  while (split > 1 && (size_t)split * n * 8 > ((size_t)64 << 20)) --split;
  return split;
}

static size_t gemv_part_off(int64_t k) { return ((size_t)k * 12 + 256 + 255) & ~(size_t)255; }

size_t fluence_ws_bytes(int64_t n, int64_t k, bool csc, int dev) {
  const int64_t split = gemv_split(n, std::max<int64_t>(k, 1), csc, dev);
  return gemv_part_off(std::max<int64_t>(k, 1)) + (split > 1 ? (size_t)split * n * 8 : 0);
}

// One fluence product on `st` with a caller-provided workspace `ws` of at least
// fluence_ws_bytes(n, k) bytes (used by A·t only).  No allocation: uvd_lp_solve
// captures these launches in a CUDA graph.
int fluence_run(const uvd_matrix_out* A, int64_t n, int64_t k, int transpose, const double* x, double* out,
                cudaStream_t st, void* ws) {
  const bool csc = A->format == UVD_CSC;
  if (!transpose) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t quads = (n + 3) / 4;
    const int64_t rblocks = (quads + kGemvThreads - 1) / kGemvThreads;
    const int64_t split = gemv_split(n, k, csc, dev);
    char* sp = (char*)ws;
    double* val = (double*)sp;
    int32_t* idx = (int32_t*)(sp + (size_t)k * 8);
    int32_t* cnt = (int32_t*)(sp + (size_t)k * 12 + 128);
    double* part = (double*)(sp + gemv_part_off(k));
    k_nonzero<<<1, 1024, 0, st>>>(x, k, idx, val, cnt);
    note_launch();
    if (csc) {
      UVD_CUDA_TRY(cudaMemsetAsync(out, 0, n * sizeof(double), st));
      k_csc_n<<<(unsigned)std::min<int64_t>(k, 4096), kGemvThreads, 0, st>>>(A->colptr, A->rowidx, A->values,
                                                                              idx, val, cnt, out);
    } else {
      const int64_t chunk = (k + split - 1) / split;
      dim3 grid((unsigned)rblocks, (unsigned)split);
      k_gemv_n<<<grid, kGemvThreads, 0, st>>>(A->values, A->ld, n, idx, val, cnt, chunk, split > 1 ? part : out);
      if (split > 1) {
        k_gemv_n_reduce<<<(unsigned)std::min<int64_t>((n + 255) / 256, 8 * sm_count(dev)), 256, 0, st>>>(
            part, (int)split, n, out);
        note_launch();
      }
    }
    note_launch();
  } else {
    if (csc)
      k_csc_t<<<(unsigned)k, kGemvThreads, 0, st>>>(A->colptr, A->rowidx, A->values, x, out);
    else
      k_gemv_t<<<(unsigned)((k + kGemvTCols - 1) / kGemvTCols), kGemvThreads, 0, st>>>(A->values, A->ld, n, k, x,
                                                                                      out);
    note_launch();
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

int fluence_check(const uvd_matrix_out* A, int64_t n, int64_t k, const double* x) {
  if (k > 0 && n > 0 && !x) { set_error("uvd_fluence: null x"); return UVD_ERR_INVALID; }
  if (A->format == UVD_CSC) {
    if (!A->colptr || !A->rowidx || !A->values) {
      set_error("uvd_fluence: CSC A needs colptr, rowidx and values");
      return UVD_ERR_INVALID;
    }
  } else if (A->format != UVD_DENSE_COLMAJOR) {
    set_error("uvd_fluence: unknown format %d", A->format);
    return UVD_ERR_INVALID;
  } else if (!A->values || A->ld < n || A->ld % 4 != 0 || ((uintptr_t)A->values & 15)) {
    set_error("uvd_fluence: dense A needs 16-B aligned values and ld >= n, ld %% 4 == 0");
    return UVD_ERR_INVALID;
  }
  return UVD_OK;
}

}  // namespace uvd

using namespace uvd;

extern "C" int uvd_fluence(const uvd_matrix_out* A, int64_t n, int64_t k, int transpose,
                           const double* x, double* out, void* stream) {
  clear_error();
  if (!A || !out || n < 0 || k < 0) { set_error("uvd_fluence: bad argument"); return UVD_ERR_INVALID; }
  DeviceGuard dg(pointer_device(out));
  NvtxRange nv(transpose ? "uvd_fluence(A^T y)" : "uvd_fluence(A t)");
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) return UVD_OK;
  if (k == 0) {  // empty shard: μ = 0, g is empty
    if (!transpose) UVD_CUDA_TRY(cudaMemsetAsync(out, 0, n * sizeof(double), st));
    return UVD_OK;
  }
  UVD_TRY(fluence_check(A, n, k, x));
  int dev = 0;
  cudaGetDevice(&dev);
  void* ws = nullptr;
  Scratch sc(matrix_alloc(A, dev, st), st);  // returned to the allocator at every exit
  if (!transpose) {
    ws = sc.get(fluence_ws_bytes(n, k, A->format == UVD_CSC, dev));
    if (!ws) { set_error("uvd_fluence: out of device memory"); return UVD_ERR_NOMEM; }
  }
  return fluence_run(A, n, k, transpose, x, out, st, ws);
}

extern "C" int uvd_fluence_multi(const uvd_matrix_out* A, int64_t n, int64_t k, const double* x,
                                 const double* y, double* ax, double* a1, double* aty, void* stream) {
  clear_error();
  double* any = ax ? ax : a1 ? a1 : aty;
  if (!A || n < 0 || k < 0 || (!any && n > 0 && k > 0) || (ax && !x && k > 0) || (aty && !y && n > 0)) {
    set_error("uvd_fluence_multi: bad argument (an output needs its input vector)");
    return UVD_ERR_INVALID;
  }
  if (!any) return UVD_OK;  // nothing to compute (an empty shard asked only for its empty Aᵀ·y)
  DeviceGuard dg(pointer_device(any));
  NvtxRange nv("uvd_fluence_multi");
  cudaStream_t st = (cudaStream_t)stream;
  if (A->format != UVD_DENSE_COLMAJOR) { set_error("uvd_fluence_multi: dense A only"); return UVD_ERR_INVALID; }
  if (n == 0 || k == 0) {  // empty: A·x = A·𝟙 = 0 (n rows), Aᵀ·y = 0 (k columns)
    if (ax && n) UVD_CUDA_TRY(cudaMemsetAsync(ax, 0, n * sizeof(double), st));
    if (a1 && n) UVD_CUDA_TRY(cudaMemsetAsync(a1, 0, n * sizeof(double), st));
    if (aty && k) UVD_CUDA_TRY(cudaMemsetAsync(aty, 0, k * sizeof(double), st));
    return UVD_OK;
  }
  UVD_TRY(fluence_check(A, n, k, x ? x : y ? y : any));
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t quads = (n + 3) / 4, nw = (quads + 31) / 32;
  const size_t part_bytes = aty ? (size_t)nw * k * sizeof(double) : 0;
  Scratch sc(matrix_alloc(A, dev, st), st);
  size_t part_max = (size_t)4 << 30;
  if (const char* e = getenv("UVD_MULTI_PART_MAX")) part_max = (size_t)atoll(e);  // tests
  if (part_bytes > part_max) {  // the warp partials would exceed 4 GB: one pass per product
    void* ws = (ax || a1) ? sc.get(fluence_ws_bytes(n, k, false, dev)) : nullptr;
    double* ones = a1 ? (double*)sc.get((size_t)k * sizeof(double)) : nullptr;
    if (((ax || a1) && !ws) || (a1 && !ones)) { set_error("uvd_fluence_multi: out of device memory"); return UVD_ERR_NOMEM; }
    if (ax) UVD_TRY(fluence_run(A, n, k, 0, x, ax, st, ws));
    if (a1) {
      k_fill_value<<<(unsigned)std::min<int64_t>((k + 255) / 256, 1024), 256, 0, st>>>(ones, k, 1.0);
      note_launch();
      UVD_TRY(fluence_run(A, n, k, 0, ones, a1, st, ws));
    }
    if (aty) UVD_TRY(fluence_run(A, n, k, 1, y, aty, st, nullptr));
    return UVD_OK;
  }
  double* part = nullptr;
  double* part2 = nullptr;
  // the warp partials are summed in chunks: enough blocks to stream them at HBM speed
  const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(64, (8 * sm_count(dev) * 256 + k - 1) / std::max<int64_t>(k, 1)));
  if (aty) {
    part = (double*)sc.get(part_bytes);
    part2 = chunks > 1 ? (double*)sc.get((size_t)chunks * k * sizeof(double)) : nullptr;
    if (!part || (chunks > 1 && !part2)) { set_error("uvd_fluence_multi: out of device memory"); return UVD_ERR_NOMEM; }
  }
  const int sel = (ax ? 4 : 0) | (a1 ? 2 : 0) | (aty ? 1 : 0);
  auto kern = sel == 7 ? k_gemv_multi<true, true, true> : sel == 6 ? k_gemv_multi<true, true, false>
            : sel == 5 ? k_gemv_multi<true, false, true> : sel == 4 ? k_gemv_multi<true, false, false>
            : sel == 3 ? k_gemv_multi<false, true, true> : sel == 2 ? k_gemv_multi<false, true, false>
                       : k_gemv_multi<false, false, true>;
  kern<<<(unsigned)((quads + kMultiThreads - 1) / kMultiThreads), kMultiThreads, 0, st>>>(A->values, A->ld, n, k, x,
                                                                                         y, ax, a1, part);
  note_launch();
  if (aty) {
    const unsigned gx = (unsigned)std::min<int64_t>((k + 255) / 256, 8 * sm_count(dev));
    k_gemv_t_reduce<<<dim3(gx, (unsigned)chunks), 256, 0, st>>>(part, nw, k, chunks > 1 ? part2 : aty);
    if (chunks > 1) k_gemv_t_reduce<<<dim3(gx, 1), 256, 0, st>>>(part2, chunks, k, aty);
    note_launch(chunks > 1 ? 2 : 1);
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

extern "C" int uvd_coverage(const uvd_scene* s, const double* mu, double mu_min,
                            const double* a_rowsum, double out[3], void* stream) {
  clear_error();
  if (!s || !mu || !out) { set_error("uvd_coverage: null argument"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_coverage");
  cudaStream_t st = (cudaStream_t)stream;
  int nb = (int)std::min<int64_t>((s->N + kCovThreads - 1) / kCovThreads, std::min(2 * sm_count(s->alloc.device), kCovBlocksMax));
  nb = std::max(nb, 1);
  // partials: one buffer per stream (calls on different streams never share
  // one; calls on one stream are ordered by it), kept for the scene's lifetime
  double* part = nullptr;
  {
    uvd_scene* ms = const_cast<uvd_scene*>(s);  // internal cache only: results do not depend on it
    std::lock_guard<std::mutex> lk(ms->cov_mu);
    for (const auto& c : ms->cov_part)
      if (c.stream == st) part = c.p;
    if (!part) {
      Alloc al = ms->alloc;
      al.stream = st;
      part = (double*)al.get((3 * kCovBlocksMax + 3) * sizeof(double));
      if (!part) { set_error("uvd_coverage: out of device memory"); return UVD_ERR_NOMEM; }
      ms->cov_part.push_back({st, part});
    }
  }
  double* dout = part + 3 * kCovBlocksMax;
  k_coverage_part<<<nb, kCovThreads, 0, st>>>(mu, s->area, a_rowsum, s->N, mu_min, part);
  note_launch();
  k_coverage_final<<<1, 32, 0, st>>>(part, nb, dout);
  note_launch();
  double* h = (double*)host_stage();
  if (!h) { set_error("uvd_coverage: out of pinned host memory"); return UVD_ERR_NOMEM; }
  UVD_CUDA_TRY(cudaMemcpyAsync(h, dout, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  UVD_CUDA_TRY(cudaGetLastError());
  out[0] = h[0]; out[1] = h[1]; out[2] = h[2];
  return UVD_OK;
}

extern "C" int uvd_static_columns(const uvd_scene* s, const uvd_matrix_out* A, int64_t k, double t_budget,
                                  double mu_min, double* out, int64_t choice[2], double* dwell, void* stream) {
  clear_error();
  if (!s || !A || !out || k < 0 || !(mu_min > 0.0) || !(t_budget >= 0.0)) {
    set_error("uvd_static_columns: bad argument");
    return UVD_ERR_INVALID;
  }
  if (A->format != UVD_DENSE_COLMAJOR || !A->values || A->ld < s->N) {
    set_error("uvd_static_columns: needs a dense A with ld >= N");
    return UVD_ERR_INVALID;
  }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_static_columns");
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 0) {
    if (choice) choice[0] = choice[1] = -1;
    if (dwell) *dwell = INFINITY;
    return UVD_OK;
  }
  k_static_cols<<<(unsigned)k, kStaticThreads, 0, st>>>(A->values, A->ld, s->N, s->area, t_budget, mu_min, out);
  note_launch();
  if (choice || dwell) {
    Scratch sc(matrix_alloc(A, s->alloc.device, st), st);
    double* res = (double*)sc.get(3 * sizeof(double));
    double* h = (double*)host_stage();
    if (!res || !h) { set_error("uvd_static_columns: out of memory"); return UVD_ERR_NOMEM; }
    k_static_choose<<<1, kStaticThreads, 0, st>>>(out, k, mu_min, res);
    note_launch();
    UVD_CUDA_TRY(cudaMemcpyAsync(h, res, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    if (choice) { choice[0] = (int64_t)h[0]; choice[1] = (int64_t)h[2]; }
    if (dwell) *dwell = h[1];
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}
