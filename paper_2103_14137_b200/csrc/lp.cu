// lp.cu — NEXT-1: the relaxed dwell-time LP of Eq. 9
// (P:262–272), the first stage of the paper's two-stage planner (§IV-D), solved
// on the GPU by the primal–dual hybrid gradient method instead of the paper's
// Gurobi interior point.
//
//   primal  min cᵀx  s.t. Kx ≥ q, x ≥ 0      x = (t ∈ R^k, σ ∈ R^n)
//   dual    max qᵀy  s.t. Kᵀy ≤ c, y ≥ 0      y = (y ∈ R^n, y_b)
//   K = [[A, I], [−𝟙ᵀ, 0]],  c = (𝟙, p),  q = (μ_min 𝟙, −T_max)
//
// PDHG (Chambolle & Pock 2011), with their diagonal preconditioners for
// α = 1 — T_j = η / Σ_i |K_ij|, Σ_i = η / Σ_j |K_ij|, which bound
// ‖Σ^½ K T^½‖ ≤ η < 1 — and a primal weight ω (steps T/ω, Σω):
//   x⁺ = max(0, x − (T/ω)(c − Kᵀy))
//   y⁺ = max(0, y + (Σω)(q − K(2x⁺ − x)))
// plus PDLP-style adaptive restarts (Applegate et al. 2021): every
// `check_every` iterations the current iterate and the running average are
// scored by their ω-weighted KKT error; the better one becomes the restart
// point on sufficient (×0.2) or stalled necessary (×0.8) decay or after 36 % of
// the iterations; ω is then updated from the primal and dual movement.
//
// One iteration = Aᵀ·y (k_gemv_t) + A·t⁺ (k_nonzero + k_gemv_n, zero-t columns
// skipped) + two fused fp64 vector kernels (k_lp_primal: t-update, Σt and the
// running averages; k_lp_dual: σ- and y-updates, K(2x⁺−x) formed from the
// stored A·t, and the averages).  Bandwidth: one pass over A for Aᵀ·y plus the
// nonzero-t columns for A·t; single-process solves replay `check_every`
// iterations as one CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "uvd_internal.cuh"

namespace uvd {

struct LpScal {  // device-resident scalars of the iteration
  double y2, S, y2_avg, S_avg, y2_last;  // budget dual y_b, Σt (global), their averages, restart anchor
  double omega;                         // primal weight ω
  double w;                             // averaging weight of the current iteration, 1/(m+1)
  double m;                             // iterates averaged since the last restart
};

struct LpVec {
  double *t, *gT, *t_avg, *gT_avg, *t_last, *tau;                          // [k]
  double *sig, *y1, *mu, *buf, *sig_avg, *mu_avg, *y_avg, *sig_last, *y_last, *sig1, *pen;  // [n] (buf n+1)
  LpScal* sc;
  double* part;      // [kLpBlocks][8] row partials
  double* rows_out;  // [8]
  double* cols_out;  // [4] (summed across ranks)
};

constexpr int kLpBlocks = 296;  // 2 x 148 SMs: fixed grid -> fixed reduction order
constexpr int kLpThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  // fixed-order block reduction (blockDim.x a multiple of 32, <= 1024)
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s += sh[i];
  return s;  // valid in thread 0
}

// x-update of the t block, running averages of t and of Kᵀy's A-part, Σt⁺.
__global__ void __launch_bounds__(1024) k_lp_primal(LpVec v, int64_t k, int64_t n) {
  __shared__ double sh[32];
  LpScal* s = v.sc;
  const double m = s->m, w = 1.0 / (m + 1.0), om = s->omega, y2 = s->y2;
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double g = v.gT[j];
    const double tn = fmax(0.0, v.t[j] - v.tau[j] / om * (1.0 - g + y2));  // c_t − (Kᵀy)_t = 1 − (Aᵀy)_k + y_b
    v.t_avg[j] += w * (tn - v.t_avg[j]);
    v.gT_avg[j] += w * (g - v.gT_avg[j]);
    v.t[j] = tn;
    acc += tn;
  }
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    v.buf[n] = tot;  // this rank's Σt⁺ (summed across ranks with A·t⁺)
    s->y2_avg += w * (y2 - s->y2_avg);
    s->w = w;
    s->m = m + 1.0;
  }
}

// σ-update, y-update from K(2x⁺ − x) = 2(A t⁺ + σ⁺) − (A t + σ), averages.
__global__ void __launch_bounds__(kLpThreads) k_lp_dual(LpVec v, int64_t n, double mu_min, double t_max,
                                                       double sig2, double eta) {
  const LpScal* s = v.sc;
  const double w = s->w, om = s->omega;
  for (int64_t i = blockIdx.x * (int64_t)kLpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kLpThreads) {
    const double mun = v.buf[i], so = v.sig[i], yo = v.y1[i];
    const double sn = fmax(0.0, so - eta / om * (v.pen[i] - yo));  // c_σ − (Kᵀy)_σ = p − y
    const double kxo = v.mu[i] + so, kxn = mun + sn;
    const double yn = fmax(0.0, yo + om * v.sig1[i] * (mu_min - 2.0 * kxn + kxo));
    v.sig_avg[i] += w * (sn - v.sig_avg[i]);
    v.mu_avg[i] += w * (mun - v.mu_avg[i]);
    v.y_avg[i] += w * (yo - v.y_avg[i]);
    v.mu[i] = mun;
    v.sig[i] = sn;
    v.y1[i] = yn;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LpScal* sw = v.sc;
    const double Sn = v.buf[n];
    const double y2n = fmax(0.0, sw->y2 + om * sig2 * (2.0 * Sn - sw->S - t_max));  // row −Σt ≥ −T_max
    sw->S_avg += w * (Sn - sw->S_avg);
    sw->S = Sn;
    sw->y2 = y2n;
  }
}

// KKT pieces over the rows for the current iterate and the average:
// Σ max(0, μ_min − μ − σ)², Σ max(0, y − p)², Σ p σ, Σ y.
__global__ void __launch_bounds__(kLpThreads) k_lp_kkt_rows(LpVec v, int64_t n, double mu_min) {
  __shared__ double sh[32];
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)kLpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kLpThreads) {
    const double p = v.pen[i];
    double r = fmax(0.0, mu_min - v.mu[i] - v.sig[i]);
    double d = fmax(0.0, v.y1[i] - p);
    a[0] += r * r; a[1] += d * d; a[2] += p * v.sig[i]; a[3] += v.y1[i];
    r = fmax(0.0, mu_min - v.mu_avg[i] - v.sig_avg[i]);
    d = fmax(0.0, v.y_avg[i] - p);
    a[4] += r * r; a[5] += d * d; a[6] += p * v.sig_avg[i]; a[7] += v.y_avg[i];
  }
  for (int q = 0; q < 8; ++q) {
    const double s = block_sum(a[q], sh);
    if (threadIdx.x == 0) v.part[blockIdx.x * 8 + q] = s;
  }
}

// KKT pieces over this rank's columns: Σ max(0, (Aᵀy)_k − y_b − 1)² (current, average)
__global__ void __launch_bounds__(1024) k_lp_kkt_cols(LpVec v, int64_t k) {
  __shared__ double sh[32];
  const double y2 = v.sc->y2, y2a = v.sc->y2_avg;
  double a0 = 0.0, a1 = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double d0 = fmax(0.0, v.gT[j] - y2 - 1.0), d1 = fmax(0.0, v.gT_avg[j] - y2a - 1.0);
    a0 += d0 * d0;
    a1 += d1 * d1;
  }
  const double s0 = block_sum(a0, sh);
  const double s1 = block_sum(a1, sh);
  if (threadIdx.x == 0) { v.cols_out[0] = s0; v.cols_out[1] = s1; }
}

// restart movement: Σ(σ − σ_last)², Σ(y − y_last)² (rows) and Σ(t − t_last)² (cols)
__global__ void __launch_bounds__(kLpThreads) k_lp_move_rows(LpVec v, int64_t n, double eta) {
  __shared__ double sh[32];
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kLpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kLpThreads) {
    const double d0 = v.sig[i] - v.sig_last[i], d1 = v.y1[i] - v.y_last[i];
    a0 += d0 * d0 / eta;  // movement in the preconditioned space: ‖T^-½ Δx‖, ‖Σ^-½ Δy‖
    a1 += d1 * d1 / v.sig1[i];
  }
  const double s0 = block_sum(a0, sh);
  const double s1 = block_sum(a1, sh);
  if (threadIdx.x == 0) { v.part[blockIdx.x * 8] = s0; v.part[blockIdx.x * 8 + 1] = s1; }
}

__global__ void __launch_bounds__(1024) k_lp_move_cols(LpVec v, int64_t k) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double d = v.t[j] - v.t_last[j];
    a += d * d / v.tau[j];
  }
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.cols_out[2] = s;
}

// Σ_i Σ1_i (rows) and Σ_k T_k (cols): the initial primal weight in the preconditioned space
__global__ void __launch_bounds__(kLpThreads) k_lp_wsum_rows(LpVec v, int64_t n) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kLpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kLpThreads)
    a += v.sig1[i];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.part[blockIdx.x * 8] = s;
}

__global__ void __launch_bounds__(1024) k_lp_wsum_cols(LpVec v, int64_t k) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) a += v.tau[j];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.cols_out[3] = s;
}

// sum the per-block row partials in block order (q < nq quantities)
__global__ void k_lp_rows_final(LpVec v, int nq) {
  const int q = threadIdx.x;
  if (q >= nq) return;
  double s = 0.0;
  for (int b = 0; b < kLpBlocks; ++b) s += v.part[b * 8 + q];
  v.rows_out[q] = s;
}

// restart: optionally replace the iterate by the average; reset the average;
// set the anchors for the next movement measurement; set ω
__global__ void k_lp_restart_rows(LpVec v, int64_t n, int to_avg, int anchor) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (to_avg) { v.sig[i] = v.sig_avg[i]; v.y1[i] = v.y_avg[i]; v.mu[i] = v.mu_avg[i]; }
    if (anchor) { v.sig_last[i] = v.sig[i]; v.y_last[i] = v.y1[i]; }
  }
}

__global__ void k_lp_restart_cols(LpVec v, int64_t k, int to_avg, int anchor, double omega) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    if (to_avg) v.t[j] = v.t_avg[j];
    if (anchor) v.t_last[j] = v.t[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LpScal* s = v.sc;
    if (to_avg) { s->y2 = s->y2_avg; s->S = s->S_avg; }
    if (anchor) s->y2_last = s->y2;
    s->omega = omega;
    s->m = 0.0;
  }
}

// setup: preconditioners from the row/column sums of A (A ≥ 0), penalties, zero state
__global__ void k_lp_setup_rows(LpVec v, int64_t n, const double* __restrict__ rowsum, const double* pen_in,
                                double pen_scalar, double eta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    v.sig1[i] = eta / (rowsum[i] + 1.0);  // row i of K: Σ_k A_ik + 1 (σ_i)
    v.pen[i] = pen_in ? pen_in[i] : pen_scalar;
    v.sig[i] = 0.0; v.y1[i] = 0.0;
    v.sig_avg[i] = 0.0; v.mu_avg[i] = 0.0; v.y_avg[i] = 0.0;
  }
}

__global__ void k_lp_setup_cols(LpVec v, int64_t k, double eta) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    v.tau[j] = eta / (v.gT[j] + 1.0);  // column k of K: Σ_i A_ik + 1 (budget row)
    v.t_avg[j] = 0.0; v.gT_avg[j] = 0.0;
    v.t[j] = fmax(0.0, v.t[j]);
  }
}

__global__ void k_lp_init_scalars(LpVec v, int64_t n, double omega) {
  LpScal* s = v.sc;
  s->S = v.buf[n]; s->S_avg = 0.0; s->y2 = 0.0; s->y2_avg = 0.0; s->y2_last = 0.0;
  s->omega = omega; s->w = 1.0; s->m = 0.0;
}

__global__ void k_fill(double* x, int64_t n, double val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = val;
}

__global__ void k_sumsq_final(const double* __restrict__ x, int64_t n, double* out) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += x[i] * x[i];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(1024) k_lp_sum_t(LpVec v, int64_t k, int64_t n) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) a += v.t[j];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.buf[n] = s;
}

__global__ void k_lp_copy_mu(LpVec v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v.mu[i] = v.buf[i];
}

// S, y_b, S_avg, y_b avg, m, y_b anchor -> out[0..5]
__global__ void k_lp_scalars_out(LpVec v, double* out) {
  const LpScal* s = v.sc;
  out[0] = s->S; out[1] = s->y2; out[2] = s->S_avg; out[3] = s->y2_avg; out[4] = s->m; out[5] = s->y2_last;
}

}  // namespace uvd

using namespace uvd;

namespace {

struct HostKkt {
  double rp, rd, pobj, dobj, gap, rel_p, rel_d, rel_g, kkt_w;
};

HostKkt score(double rp2_rows, double rd2_rows, double psig, double sumy, double rd2_cols, double S, double y2,
              double mu_min, double t_max, double qn, double cn, double omega) {
  HostKkt h;
  const double over = std::max(0.0, S - t_max);
  h.rp = std::sqrt(rp2_rows + over * over);
  h.rd = std::sqrt(rd2_rows + rd2_cols);
  h.pobj = S + psig;
  h.dobj = mu_min * sumy - t_max * y2;
  h.gap = std::fabs(h.pobj - h.dobj);
  h.rel_p = h.rp / (1.0 + qn);
  h.rel_d = h.rd / (1.0 + cn);
  h.rel_g = h.gap / (1.0 + std::fabs(h.pobj) + std::fabs(h.dobj));
  h.kkt_w = std::sqrt(omega * h.rp * h.rp + h.rd * h.rd / omega + h.gap * h.gap);
  return h;
}

}  // namespace

extern "C" int uvd_lp_solve(const uvd_matrix_out* A, int64_t n, int64_t k, const uvd_lp_opts* o, double* t,
                            double* sigma, double* y, uvd_lp_result* res, void* stream) {
  clear_error();
  if (!A || !o || !res || n < 1 || k < 0 || !sigma || !y || (k > 0 && !t)) {
    set_error("uvd_lp_solve: bad argument (need A, opts, result, n >= 1, sigma, y and t when k > 0)");
    return UVD_ERR_INVALID;
  }
  if (!(o->mu_min > 0.0) || !(o->t_max > 0.0) || (!o->penalty && !(o->penalty_scalar > 0.0))) {
    set_error("uvd_lp_solve: need mu_min > 0, t_max > 0 and positive penalties");
    return UVD_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const double eps = o->eps > 0.0 ? o->eps : 1e-6;
  const int64_t max_iter = o->max_iter > 0 ? o->max_iter : 200000;
  const int M = o->check_every > 0 ? o->check_every : 64;
  const double eta = 0.999;  // strict: ‖Σ^½ K T^½‖ ≤ η < 1
  const bool multi = o->allreduce != nullptr;
  auto allreduce = [&](double* buf, int64_t cnt) -> int {
    if (!multi) return UVD_OK;
    const int rc = o->allreduce(buf, cnt, stream, o->allreduce_ctx);
    if (rc != 0) { set_error("uvd_lp_solve: allreduce callback failed (%d)", rc); return UVD_ERR_INVALID; }
    return UVD_OK;
  };

  // ---- workspace (one allocation; freed at the end) ----
  const int64_t kk = std::max<int64_t>(k, 1);
  const size_t nd = (size_t)5 * kk + (size_t)10 * n + 1 + (size_t)kLpBlocks * 8 + 8 + 4 + 2 * (size_t)n + 8;
  double* ws = nullptr;
  UVD_CUDA_TRY(cudaMalloc(&ws, nd * sizeof(double) + sizeof(LpScal) + 64));
  double* h = nullptr;  // pinned host mirror of the check results
  UVD_CUDA_TRY(cudaMallocHost(&h, 32 * sizeof(double)));
  LpVec v;
  double* p = ws;
  v.t = t;
  v.gT = p; p += kk;
  v.t_avg = p; p += kk;
  v.gT_avg = p; p += kk;
  v.t_last = p; p += kk;
  v.tau = p; p += kk;
  v.sig = sigma;
  v.y1 = y;
  v.mu = p; p += n;
  v.buf = p; p += n + 1;
  v.sig_avg = p; p += n;
  v.mu_avg = p; p += n;
  v.y_avg = p; p += n;
  v.sig_last = p; p += n;
  v.y_last = p; p += n;
  v.sig1 = p; p += n;
  v.pen = p; p += n;
  double* ones = p; p += std::max(n, kk);  // all-ones vector (setup only)
  v.part = p; p += kLpBlocks * 8;
  v.rows_out = p; p += 8;
  v.cols_out = p; p += 4;
  double* misc = p; p += 8;
  v.sc = reinterpret_cast<LpScal*>(p);

  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int rc = UVD_OK;
  auto finish = [&](int code) {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamSynchronize(st);
    cudaFree(ws);
    cudaFreeHost(h);
    return code;
  };
#define LP_TRY(expr)                 \
  do {                               \
    const int _r = (expr);           \
    if (_r != UVD_OK) return finish(_r); \
  } while (0)
#define LP_CUDA(expr)                                                                          \
  do {                                                                                         \
    const cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                                   \
      set_error("uvd_lp_solve: %s: %s", #expr, cudaGetErrorString(_e));                       \
      return finish(UVD_ERR_CUDA);                                                             \
    }                                                                                          \
  } while (0)

  const int nb_rows = (int)std::min<int64_t>((n + kLpThreads - 1) / kLpThreads, kLpBlocks);
  // ---- setup: preconditioners, ‖c‖, ‖q‖ ----
  k_fill<<<kLpBlocks, kLpThreads, 0, st>>>(ones, std::max(n, kk), 1.0);
  note_launch();
  LP_TRY(uvd_fluence(A, n, k, 1, ones, v.gT, stream));       // column sums Σ_i A_ik
  LP_TRY(uvd_fluence(A, n, k, 0, ones, v.buf, stream));      // partial row sums Σ_k A_ik
  LP_TRY(allreduce(v.buf, n));
  k_lp_setup_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, v.buf, o->penalty, o->penalty_scalar, eta);
  k_lp_setup_cols<<<kLpBlocks, kLpThreads, 0, st>>>(v, k, eta);
  k_sumsq_final<<<1, 1024, 0, st>>>(v.pen, n, misc);  // Σ p²
  note_launch(3);
  LP_CUDA(cudaMemcpyAsync(h, misc, sizeof(double), cudaMemcpyDeviceToHost, st));
  h[1] = (double)k;
  LP_CUDA(cudaStreamSynchronize(st));
  double sum_p2 = h[0];
  double k_tot = (double)k;
  if (multi) {  // global column count
    LP_CUDA(cudaMemcpyAsync(misc + 2, &h[1], sizeof(double), cudaMemcpyHostToDevice, st));
    LP_TRY(allreduce(misc + 2, 1));
    LP_CUDA(cudaMemcpyAsync(&h[2], misc + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    k_tot = h[2];
  }
  const double qn = std::sqrt((double)n * o->mu_min * o->mu_min + o->t_max * o->t_max);
  const double cn = std::sqrt(k_tot + sum_p2);
  const double sig2 = eta / std::max(k_tot, 1.0);  // budget row: Σ_k |−1| = K
  double omega = o->primal_weight;
  if (!(omega > 0.0)) {
    // PDLP's ω₀ = ‖c‖/‖q‖ measured in the preconditioned space (x̃ = T^-½x, ỹ = Σ^-½y):
    // ‖T^½ c‖² = Σ_k T_k + η Σ_i p_i²,  ‖Σ^½ q‖² = μ_min² Σ_i Σ1_i + Σ2 T_max²
    k_lp_wsum_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n);
    k_lp_rows_final<<<1, 32, 0, st>>>(v, 1);
    k_lp_wsum_cols<<<1, 1024, 0, st>>>(v, k);
    note_launch(3);
    LP_TRY(allreduce(v.cols_out + 3, 1));
    LP_CUDA(cudaMemcpyAsync(h, v.rows_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaMemcpyAsync(h + 1, v.cols_out + 3, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    const double cs = std::sqrt(h[1] + eta * sum_p2);
    const double qs = std::sqrt(o->mu_min * o->mu_min * h[0] + sig2 * o->t_max * o->t_max);
    omega = cs > 0.0 && qs > 0.0 ? cs / qs : 1.0;
  }

  // ---- initial point: μ = A t, S = Σ t, y = 0, σ = 0 ----
  LP_TRY(uvd_fluence(A, n, k, 0, t, v.buf, stream));
  k_lp_sum_t<<<1, 1024, 0, st>>>(v, k, n);
  note_launch();
  LP_TRY(allreduce(v.buf, n + 1));
  k_lp_copy_mu<<<kLpBlocks, kLpThreads, 0, st>>>(v, n);
  k_lp_init_scalars<<<1, 1, 0, st>>>(v, n, omega);
  k_lp_restart_cols<<<kLpBlocks, kLpThreads, 0, st>>>(v, k, 0, 1, omega);  // anchors t_last = t
  k_lp_restart_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, 0, 1);
  note_launch(4);
  LP_TRY(uvd_fluence(A, n, k, 1, v.y1, v.gT, stream));  // Aᵀy for the first iteration (y = 0)

  // one PDHG iteration: x-update, A·t⁺ (+ Σt⁺), [allreduce], y-update, Aᵀy⁺
  auto iteration = [&]() -> int {
    k_lp_primal<<<1, 1024, 0, st>>>(v, k, n);
    note_launch();
    UVD_TRY(uvd_fluence(A, n, k, 0, v.t, v.buf, stream));
    UVD_TRY(allreduce(v.buf, n + 1));
    k_lp_dual<<<nb_rows, kLpThreads, 0, st>>>(v, n, o->mu_min, o->t_max, sig2, eta);
    note_launch();
    UVD_TRY(uvd_fluence(A, n, k, 1, v.y1, v.gT, stream));
    return UVD_OK;
  };
  const bool graph_ok = o->use_graph && !multi && st != nullptr;
  if (graph_ok) {
    // warm the fluence scratch for this stream outside the capture
    LP_CUDA(cudaStreamSynchronize(st));
    LP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int crc = UVD_OK;
    for (int it = 0; it < M && crc == UVD_OK; ++it) crc = iteration();
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (crc != UVD_OK) return finish(crc);
    LP_CUDA(ce);
    LP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }

  // evaluate the KKT pieces of the current iterate and of the average
  auto evaluate = [&](HostKkt* cur, HostKkt* avg, double* S_out) -> int {
    k_lp_kkt_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, o->mu_min);
    k_lp_rows_final<<<1, 32, 0, st>>>(v, 8);
    k_lp_kkt_cols<<<1, 1024, 0, st>>>(v, k);
    note_launch(3);
    UVD_TRY(allreduce(v.cols_out, 2));
    k_lp_scalars_out<<<1, 1, 0, st>>>(v, misc);
    note_launch();
    UVD_CUDA_TRY(cudaMemcpyAsync(h, v.rows_out, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaMemcpyAsync(h + 8, v.cols_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaMemcpyAsync(h + 10, misc, 5 * sizeof(double), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    // misc: S, y2, S_avg, y2_avg, m
    *cur = score(h[0], h[1], h[2], h[3], h[8], h[10], h[11], o->mu_min, o->t_max, qn, cn, omega);
    *avg = score(h[4], h[5], h[6], h[7], h[9], h[12], h[13], o->mu_min, o->t_max, qn, cn, omega);
    if (h[14] < 0.5) *avg = *cur;  // no averaged iterate yet
    *S_out = h[10];
    return UVD_OK;
  };
  auto converged = [&](const HostKkt& c) { return c.rel_p <= eps && c.rel_d <= eps && c.rel_g <= eps; };

  HostKkt cur, avg;
  double S = 0.0;
  LP_TRY(evaluate(&cur, &avg, &S));
  double kkt_restart = cur.kkt_w, kkt_prev_cand = INFINITY;
  int64_t it = 0, it_restart = 0;
  int restarts = 0;
  bool done = converged(cur), use_avg = false;
  HostKkt fin = cur;
  while (!done && it < max_iter) {
    if (graph_ok) {
      LP_CUDA(cudaGraphLaunch(exec, st));
    } else {
      for (int q = 0; q < M; ++q) LP_TRY(iteration());
    }
    it += M;
    LP_TRY(evaluate(&cur, &avg, &S));
    if (converged(cur) || converged(avg)) {
      use_avg = !converged(cur);
      fin = use_avg ? avg : cur;
      done = true;
      break;
    }
    // restart decision (PDLP: β_sufficient 0.2, β_necessary 0.8, artificial 0.36)
    const bool avg_better = avg.kkt_w < cur.kkt_w;
    const double cand = avg_better ? avg.kkt_w : cur.kkt_w;
    const bool do_restart = cand <= 0.2 * kkt_restart ||
                            (cand <= 0.8 * kkt_restart && cand > kkt_prev_cand) ||
                            (double)(it - it_restart) >= 0.36 * (double)it;
    kkt_prev_cand = cand;
    if (do_restart) {
      if (avg_better) {  // the average becomes the iterate; its Aᵀy is recomputed
        k_lp_restart_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, 1, 0);
        k_lp_restart_cols<<<kLpBlocks, kLpThreads, 0, st>>>(v, k, 1, 0, omega);
        note_launch(2);
        LP_TRY(uvd_fluence(A, n, k, 1, v.y1, v.gT, stream));
      }
      // primal weight from the movement since the last restart (before the anchors move)
      k_lp_move_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, eta);
      k_lp_rows_final<<<1, 32, 0, st>>>(v, 2);
      k_lp_move_cols<<<1, 1024, 0, st>>>(v, k);
      k_lp_scalars_out<<<1, 1, 0, st>>>(v, misc);
      note_launch(4);
      LP_TRY(allreduce(v.cols_out + 2, 1));
      LP_CUDA(cudaMemcpyAsync(h, v.rows_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      LP_CUDA(cudaMemcpyAsync(h + 2, v.cols_out + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
      LP_CUDA(cudaMemcpyAsync(h + 3, misc, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
      LP_CUDA(cudaStreamSynchronize(st));
      const double dy2 = h[4] - h[8];  // y2 − y2_last
      const double dx = std::sqrt(h[2] + h[0]), dy = std::sqrt(h[1] + dy2 * dy2 / sig2);
      if (dx > 1e-10 && dy > 1e-10) omega = std::exp(0.5 * std::log(dy / dx) + 0.5 * std::log(omega));
      k_lp_restart_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, 0, 1);        // anchors = iterate
      k_lp_restart_cols<<<kLpBlocks, kLpThreads, 0, st>>>(v, k, 0, 1, omega);  // ω, m = 0
      note_launch(2);
      kkt_restart = cand;
      kkt_prev_cand = INFINITY;
      it_restart = it;
      ++restarts;
    }
  }
  if (use_avg) {  // hand back the average
    k_lp_restart_rows<<<kLpBlocks, kLpThreads, 0, st>>>(v, n, 1, 0);
    k_lp_restart_cols<<<kLpBlocks, kLpThreads, 0, st>>>(v, k, 1, 0, omega);
    note_launch(2);
  }
  if (!done) fin = cur;
  k_lp_scalars_out<<<1, 1, 0, st>>>(v, misc);
  note_launch();
  LP_CUDA(cudaMemcpyAsync(y + n, misc + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  LP_CUDA(cudaMemcpyAsync(h, misc, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  LP_CUDA(cudaStreamSynchronize(st));
  LP_CUDA(cudaGetLastError());
  res->status = done ? 0 : 1;
  res->restarts = restarts;
  res->iterations = it;
  res->primal_obj = fin.pobj;
  res->dual_obj = fin.dobj;
  res->rel_primal_res = fin.rel_p;
  res->rel_dual_res = fin.rel_d;
  res->rel_gap = fin.rel_g;
  res->sum_t = h[0];
  res->primal_weight = omega;
  res->averaged = use_avg ? 1 : 0;
  return finish(rc);
#undef LP_TRY
#undef LP_CUDA
}
