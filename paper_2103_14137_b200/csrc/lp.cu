// lp.cu — NEXT-1: the relaxed dwell-time LP of Eq. 9
// (P:262–272), the first stage of the paper's two-stage planner (§IV-D), solved
// on the GPU by a first-order primal–dual method instead of the paper's Gurobi
// interior point.
//
//   minimise Σ_k t_k + Σ_i p_i σ_i  s.t.  A t + σ ≥ μ_min 𝟙,  t ∈ Δ = {t ≥ 0, Σ t ≤ T_max},  σ ≥ 0
//
// Operator: PDHG (Chambolle & Pock 2011) on the saddle problem with the
// coverage rows dualised (y ≥ 0) and the budget kept as the simple set Δ:
//   t̂ = Π_Δ^T (t − (T/ω)(𝟙 − Aᵀy))          weighted projection onto Δ
//   σ̂ = max(0, σ − (η/ω)(p − y))
//   ŷ = max(0, y + (Σω)(μ_min − 2(A t̂ + σ̂) + (A t + σ)))
// with Chambolle–Pock's diagonal preconditioners for α = 1 (T_k = η/Σ_i A_ik,
// Σ_i = η/(Σ_k A_ik + 1), η = 0.999: ‖Σ^½ K T^½‖ < 1) and a primal weight ω.
// Π_Δ^T is the T⁻¹-weighted projection: t̂_k = max(0, v_k − λ T_k) with λ ≥ 0
// the root of Σ_k max(0, v_k − λT_k) = T_max (or λ = 0 if the cap is slack),
// found exactly by Newton's method from the left on this convex piecewise-
// linear function (finite; Michelot's simplex projection, weighted); ωλ is the
// budget's dual multiplier y_b.
//
// Outer method: reflected restarted Halpern iteration (Lu & Yang 2024):
//   z⁺ = w ((1+ρ) T(z) − ρ z) + (1 − w) z₀,   w = (k+1)/(k+2),  ρ = 1,
// restarted (z₀ ← T(z), k ← 0) when the fixed-point residual ‖z − T(z)‖_ω has
// decayed ×0.2 (sufficient), or ×0.8 and stalled (necessary), or after 36 % of
// the iterations (artificial); ω is then re-balanced from the primal and dual
// movement between restart points (PDLP's smoothed rule).  Because A·t and
// Aᵀ·y are linear, the mixed iterate's products are mixed the same way: every
// iteration costs one A·t̂ (k_nonzero + k_gemv_n: zero columns of the sparse t̂
// skipped) and one Aᵀ·ŷ (k_gemv_t) plus three fused fp64 vector kernels.
// Single-process solves replay `check_every` iterations as one CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "uvd_internal.cuh"

namespace uvd {

struct HpScal {   // device-resident scalars
  double omega;   // primal weight ω
  double w;       // Halpern weight of the current iteration
  double kc;      // iterations since the last restart
  double first;   // 1 in the first iteration after a restart
  double lam;     // budget multiplier λ of the last projection
  double rho;     // Halpern reflection ρ
  double pad[2];
};

struct HpVec {
  double *t, *gT, *t0, *gT0, *tT, *gTT, *tau;                             // [k]
  double *sig, *y, *mu, *sig0, *y0, *mu0, *sigT, *yT, *buf, *sig1, *pen;  // [n] (buf: A t̂, n+1)
  HpScal* sc;
  double* part;      // [kHpBlocks][8] row partials
  double* res;       // [kHpBlocks][4] row residual partials: last iteration (0,1), first after restart (2,3)
  double* cres;      // [8] column residual (0 last, 1 first), projection sums (2..4)
  double* rows_out;  // [8]
  double* cols_out;  // [8]
};

constexpr int kHpBlocks = 296;  // 2 x 148 SMs: fixed grid -> fixed reduction order
constexpr int kHpThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  // fixed-order block reduction (blockDim.x a multiple of 32, <= 1024); result in thread 0
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s += sh[i];
  return s;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = -INFINITY;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s = fmax(s, sh[i]);
  return s;
}

// t̂ = max(0, v − λT) (v stored in t̂), residual Σ(t̂ − t)²/T, Σ t̂, Halpern weight
__device__ void primal_finish(HpVec& v, int64_t k, int64_t n, double lam, double* sh, HpScal* s, double kc) {
  double r = 0.0, acc = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double tn = fmax(0.0, v.tT[j] - lam * v.tau[j]);
    const double d = tn - v.t[j];
    r += d * d / v.tau[j];
    acc += tn;
    v.tT[j] = tn;
  }
  const double rs = block_sum(r, sh);
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    v.cres[0] = rs;
    if (kc == 0.0) v.cres[1] = rs;
    v.buf[n] = tot;
    s->w = (kc + 1.0) / (kc + 2.0);
    s->first = kc == 0.0 ? 1.0 : 0.0;
    s->kc = kc + 1.0;
    s->lam = lam;
  }
}

// t-part of T(z), single process: v = t − (T/ω)(1 − Aᵀy), projection onto Δ
// inside the block (Newton from the left), then primal_finish
__global__ void __launch_bounds__(1024) k_hp_primal(HpVec v, int64_t k, int64_t n, double cap) {
  __shared__ double sh[32];
  __shared__ double bc[2];
  HpScal* s = v.sc;
  const double om = s->omega, kc = s->kc;
  double pos = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double val = v.t[j] - v.tau[j] / om * (1.0 - v.gT[j]);
    v.tT[j] = val;
    pos += fmax(0.0, val);
  }
  const double p0 = block_sum(pos, sh);
  if (threadIdx.x == 0) bc[0] = p0;
  __syncthreads();
  double lam = 0.0;
  if (bc[0] > cap) {
    double prev = -1.0;  // (meaningful in thread 0 only)
    for (int it = 0; it < 200; ++it) {  // finite and monotone
      double sv = 0.0, st = 0.0, cn = 0.0;
      for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
        const double val = v.tT[j], tj = v.tau[j];
        if (val > lam * tj) { sv += val; st += tj; cn += 1.0; }
      }
      const double SV = block_sum(sv, sh);
      const double ST = block_sum(st, sh);
      const double CN = block_sum(cn, sh);
      if (threadIdx.x == 0) { bc[0] = (SV - cap) / ST; bc[1] = CN == prev ? 1.0 : 0.0; prev = CN; }
      __syncthreads();
      lam = fmax(lam, bc[0]);
      const bool stop = bc[1] != 0.0;
      __syncthreads();
      if (stop) break;
    }
  }
  primal_finish(v, k, n, lam, sh, s, kc);
}

// multi-process projection: v and Σmax(0, v) (k_hp_primal_v), host-driven
// Newton steps over the ranks' summed (Σ v, Σ T, count) (k_hp_proj_sums), then
// k_hp_primal_fin
__global__ void __launch_bounds__(1024) k_hp_primal_v(HpVec v, int64_t k) {
  __shared__ double sh[32];
  const double om = v.sc->omega;
  double pos = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double val = v.t[j] - v.tau[j] / om * (1.0 - v.gT[j]);
    v.tT[j] = val;
    pos += fmax(0.0, val);
  }
  const double p0 = block_sum(pos, sh);
  if (threadIdx.x == 0) { v.cres[2] = p0; v.cres[3] = 0.0; v.cres[4] = 0.0; }
}

__global__ void __launch_bounds__(1024) k_hp_proj_sums(HpVec v, int64_t k, double lam) {
  __shared__ double sh[32];
  double sv = 0.0, st = 0.0, cn = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double val = v.tT[j], tj = v.tau[j];
    if (val > lam * tj) { sv += val; st += tj; cn += 1.0; }
  }
  const double SV = block_sum(sv, sh);
  const double ST = block_sum(st, sh);
  const double CN = block_sum(cn, sh);
  if (threadIdx.x == 0) { v.cres[2] = SV; v.cres[3] = ST; v.cres[4] = CN; }
}

__global__ void __launch_bounds__(1024) k_hp_primal_fin(HpVec v, int64_t k, int64_t n, double lam) {
  __shared__ double sh[32];
  primal_finish(v, k, n, lam, sh, v.sc, v.sc->kc);
}

// σ̂, ŷ of T(z), row residuals, then the Halpern mix of σ, y and A t
__global__ void __launch_bounds__(kHpThreads) k_hp_dual(HpVec v, int64_t n, double mu_min, double eta) {
  __shared__ double sh[32];
  const HpScal* s = v.sc;
  const double w = s->w, om = s->omega, rho = s->rho;
  const bool first = s->first != 0.0;
  double r0 = 0.0, r1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kHpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kHpThreads) {
    const double so = v.sig[i], yo = v.y[i], muo = v.mu[i], muh = v.buf[i];
    const double sn = fmax(0.0, so - eta / om * (v.pen[i] - yo));
    const double yh = fmax(0.0, yo + om * v.sig1[i] * (mu_min - 2.0 * (muh + sn) + (muo + so)));
    const double ds = sn - so, dy = yh - yo;
    r0 += ds * ds / eta;
    r1 += dy * dy / v.sig1[i];
    v.sigT[i] = sn;
    v.yT[i] = yh;
    v.sig[i] = w * ((1.0 + rho) * sn - rho * so) + (1.0 - w) * v.sig0[i];
    v.y[i] = w * ((1.0 + rho) * yh - rho * yo) + (1.0 - w) * v.y0[i];
    v.mu[i] = w * ((1.0 + rho) * muh - rho * muo) + (1.0 - w) * v.mu0[i];
  }
  const double a = block_sum(r0, sh);
  const double b = block_sum(r1, sh);
  if (threadIdx.x == 0) {
    v.res[blockIdx.x * 4 + 0] = a;
    v.res[blockIdx.x * 4 + 1] = b;
    if (first) { v.res[blockIdx.x * 4 + 2] = a; v.res[blockIdx.x * 4 + 3] = b; }
  }
}

// Halpern mix of t and Aᵀy
__global__ void k_hp_mix_cols(HpVec v, int64_t k) {
  const double w = v.sc->w, rho = v.sc->rho;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    v.t[j] = w * ((1.0 + rho) * v.tT[j] - rho * v.t[j]) + (1.0 - w) * v.t0[j];
    v.gT[j] = w * ((1.0 + rho) * v.gTT[j] - rho * v.gT[j]) + (1.0 - w) * v.gT0[j];
  }
}

// KKT pieces of T(z) over the rows: Σmax(0, μ_min − A t̂ − σ̂)², Σmax(0, ŷ − p)², Σ p σ̂, Σ ŷ
__global__ void __launch_bounds__(kHpThreads) k_hp_kkt_rows(HpVec v, int64_t n, double mu_min) {
  __shared__ double sh[32];
  double a[4] = {0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)kHpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kHpThreads) {
    const double p = v.pen[i];
    const double r = fmax(0.0, mu_min - v.buf[i] - v.sigT[i]);
    const double d = fmax(0.0, v.yT[i] - p);
    a[0] += r * r; a[1] += d * d; a[2] += p * v.sigT[i]; a[3] += v.yT[i];
  }
  for (int q = 0; q < 4; ++q) {
    const double s = block_sum(a[q], sh);
    if (threadIdx.x == 0) v.part[blockIdx.x * 8 + q] = s;
  }
}

// rows_out[0..nq) = row partial sums; [4..8) = residual partials (last, first after restart)
__global__ void k_hp_rows_final(HpVec v, int nq) {
  const int q = threadIdx.x;
  double s = 0.0;
  if (q < nq) {
    for (int b = 0; b < kHpBlocks; ++b) s += v.part[b * 8 + q];
    v.rows_out[q] = s;
  } else if (q >= 4 && q < 8) {
    for (int b = 0; b < kHpBlocks; ++b) s += v.res[b * 4 + (q - 4)];
    v.rows_out[q] = s;
  }
}

// cols_out = [Σmax(0, (Aᵀŷ)_k − ωλ − 1)², Σ t̂, col residual last, first | max_k (Aᵀŷ)_k, ωλ]
__global__ void __launch_bounds__(1024) k_hp_kkt_cols(HpVec v, int64_t k) {
  __shared__ double sh[32];
  const double yb = v.sc->omega * v.sc->lam;
  double a0 = 0.0, a1 = 0.0, mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double g = v.gTT[j];
    const double d = fmax(0.0, g - yb - 1.0);
    a0 += d * d;
    a1 += v.tT[j];
    mx = fmax(mx, g);
  }
  const double s0 = block_sum(a0, sh);
  const double s1 = block_sum(a1, sh);
  const double m = block_max(mx, sh);
  if (threadIdx.x == 0) {
    v.cols_out[0] = s0; v.cols_out[1] = s1; v.cols_out[2] = v.cres[0]; v.cols_out[3] = v.cres[1];
    v.cols_out[4] = m; v.cols_out[5] = yb;
  }
}

// movement between restart points (T(z) vs the anchor z₀), in the preconditioned norms
__global__ void __launch_bounds__(kHpThreads) k_hp_move_rows(HpVec v, int64_t n, double eta) {
  __shared__ double sh[32];
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kHpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kHpThreads) {
    const double d0 = v.sigT[i] - v.sig0[i], d1 = v.yT[i] - v.y0[i];
    a0 += d0 * d0 / eta;
    a1 += d1 * d1 / v.sig1[i];
  }
  const double s0 = block_sum(a0, sh);
  const double s1 = block_sum(a1, sh);
  if (threadIdx.x == 0) { v.part[blockIdx.x * 8] = s0; v.part[blockIdx.x * 8 + 1] = s1; }
}

__global__ void __launch_bounds__(1024) k_hp_move_cols(HpVec v, int64_t k) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double d = v.tT[j] - v.t0[j];
    a += d * d / v.tau[j];
  }
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.cols_out[6] = s;
}

// (re)start: z = z₀ = T(z) (from_T) or z₀ = z; products follow; ω set, k = 0
__global__ void k_hp_anchor_rows(HpVec v, int64_t n, int from_T) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (from_T) { v.sig[i] = v.sigT[i]; v.y[i] = v.yT[i]; v.mu[i] = v.buf[i]; }
    v.sig0[i] = v.sig[i]; v.y0[i] = v.y[i]; v.mu0[i] = v.mu[i];
  }
}

__global__ void k_hp_anchor_cols(HpVec v, int64_t k, int from_T, double omega, double rho) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    if (from_T) { v.t[j] = v.tT[j]; v.gT[j] = v.gTT[j]; }
    v.t0[j] = v.t[j]; v.gT0[j] = v.gT[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    v.sc->omega = omega;
    v.sc->rho = rho;
    v.sc->kc = 0.0;
    v.sc->w = 0.5;
    v.sc->first = 1.0;
  }
}

// setup: preconditioners from the row/column sums of A (A ≥ 0), penalties, state
__global__ void k_hp_setup_rows(HpVec v, int64_t n, const double* __restrict__ rowsum, const double* pen_in,
                                double pen_scalar, double eta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    v.sig1[i] = eta / (rowsum[i] + 1.0);  // row i of [A I]: Σ_k A_ik + 1
    v.pen[i] = pen_in ? pen_in[i] : pen_scalar;
    v.sig[i] = 0.0;
    v.y[i] = 0.0;
  }
}

__global__ void k_hp_setup_cols(HpVec v, int64_t k, double eta) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    v.tau[j] = eta / fmax(v.gT[j], 1e-6);  // column k of A: Σ_i A_ik (a dark column gets a large step)
    v.t[j] = fmax(0.0, v.t[j]);
  }
}

// Σ_i Σ1_i, Σ p_i² (rows) -> part; Σ_k T_k (cols) -> cols_out[7]
__global__ void __launch_bounds__(kHpThreads) k_hp_wsum_rows(HpVec v, int64_t n) {
  __shared__ double sh[32];
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kHpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kHpThreads) {
    a += v.sig1[i];
    b += v.pen[i] * v.pen[i];
  }
  const double s0 = block_sum(a, sh);
  const double s1 = block_sum(b, sh);
  if (threadIdx.x == 0) { v.part[blockIdx.x * 8] = s0; v.part[blockIdx.x * 8 + 1] = s1; }
}

__global__ void __launch_bounds__(1024) k_hp_wsum_cols(HpVec v, int64_t k) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) a += v.tau[j];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) v.cols_out[7] = s;
}

__global__ void k_fill(double* x, int64_t n, double val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = val;
}

__global__ void k_copy(double* dst, const double* src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace uvd

using namespace uvd;

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
  DeviceGuard dg(pointer_device(sigma));
  NvtxRange nvr("uvd_lp_solve");
  if (k > 0) UVD_TRY(fluence_check(A, n, k, sigma));  // an empty shard has no A to check
  cudaStream_t st = (cudaStream_t)stream;
  const double eps = o->eps > 0.0 ? o->eps : 1e-6;
  const int64_t max_iter = o->max_iter > 0 ? o->max_iter : 200000;
  const int M = o->check_every > 0 ? o->check_every : 64;
  const double eta = 0.999;
  const double mu_min = o->mu_min, t_max = o->t_max;
  // method constants (Lu & Yang 2024; PDLP): reflection, restart factors,
  // primal-weight smoothing; UVD_LP_* environment overrides are for tuning runs
  auto knob = [](const char* name, double def) {
    const char* e = getenv(name);
    return e ? atof(e) : def;
  };
  const double rho = knob("UVD_LP_RHO", 1.0), theta = knob("UVD_LP_THETA", 0.3);
  const double b_suff = knob("UVD_LP_SUFF", 0.2), b_nec = knob("UVD_LP_NEC", 0.8), b_art = knob("UVD_LP_ART", 0.36);
  const bool multi = o->allreduce != nullptr;
  auto allreduce = [&](double* buf, int64_t cnt, int op) -> int {
    if (!multi || cnt == 0) return UVD_OK;
    const int rc = o->allreduce(buf, cnt, op, stream, o->allreduce_ctx);
    if (rc != 0) { set_error("uvd_lp_solve: allreduce callback failed (%d)", rc); return UVD_ERR_INVALID; }
    return UVD_OK;
  };

  // ---- workspace ----
  const int64_t kk = std::max<int64_t>(k, 1);
  const size_t nd = (size_t)6 * kk + (size_t)9 * n + 1 + std::max<size_t>(n, kk) + (size_t)kHpBlocks * 12 + 32;
  int dev = 0;
  cudaGetDevice(&dev);
  // the whole workspace (iterates + the A·t scratch) from the matrix's allocator,
  // taken once: the iterations allocate nothing (they are captured in a graph)
  Alloc wal = matrix_alloc(A, dev, st);
  const size_t ws_main = (nd * sizeof(double) + sizeof(HpScal) + 64 + 255) & ~(size_t)255;
  const size_t ws_flu = fluence_ws_bytes(n, kk, A->format == UVD_CSC, dev);
  double* ws = (double*)wal.get(ws_main + ws_flu);
  if (!ws) { set_error("uvd_lp_solve: out of device memory (workspace)"); return UVD_ERR_NOMEM; }
  void* fws = (char*)ws + ws_main;
  double* h = nullptr;  // pinned host mirror of check results
  if (cudaMallocHost(&h, 64 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    wal.put(ws);
    set_error("uvd_lp_solve: pinned allocation failed");
    return UVD_ERR_NOMEM;
  }
  // a7 products on this stream with the preallocated scratch (an empty shard
  // contributes μ = 0 and no g)
  auto flu = [&](int transpose, const double* x, double* out) -> int {
    if (k == 0) {
      if (!transpose) UVD_CUDA_TRY(cudaMemsetAsync(out, 0, n * sizeof(double), st));
      return UVD_OK;
    }
    return fluence_run(A, n, k, transpose, x, out, st, fws);
  };
  HpVec v;
  double* p = ws;
  v.t = t;
  v.gT = p; p += kk;
  v.t0 = p; p += kk;
  v.gT0 = p; p += kk;
  v.tT = p; p += kk;
  v.gTT = p; p += kk;
  v.tau = p; p += kk;
  v.sig = sigma;
  v.y = y;
  v.mu = p; p += n;
  v.sig0 = p; p += n;
  v.y0 = p; p += n;
  v.mu0 = p; p += n;
  v.sigT = p; p += n;
  v.yT = p; p += n;
  v.buf = p; p += n + 1;
  v.sig1 = p; p += n;
  v.pen = p; p += n;
  double* ones = p; p += std::max(n, kk);
  v.part = p; p += (size_t)kHpBlocks * 8;
  v.res = p; p += (size_t)kHpBlocks * 4;
  v.cres = p; p += 8;
  v.rows_out = p; p += 8;
  v.cols_out = p; p += 8;
  v.sc = reinterpret_cast<HpScal*>(p);

  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  auto finish = [&](int code) {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamSynchronize(st);
    wal.put(ws);
    cudaFreeHost(h);
    return code;
  };
#define LP_TRY(expr)                       \
  do {                                     \
    const int _r = (expr);                 \
    if (_r != UVD_OK) return finish(_r);   \
  } while (0)
#define LP_CUDA(expr)                                                        \
  do {                                                                       \
    const cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) {                                                 \
      set_error("uvd_lp_solve: %s: %s", #expr, cudaGetErrorString(_e));     \
      return finish(UVD_ERR_CUDA);                                           \
    }                                                                        \
  } while (0)
  auto fetch = [&](double* dst, const double* src, int cnt) -> int {
    UVD_CUDA_TRY(cudaMemcpyAsync(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    return UVD_OK;
  };

  const int nb_rows = (int)std::min<int64_t>((n + kHpThreads - 1) / kHpThreads, kHpBlocks);
  LP_CUDA(cudaMemsetAsync(v.res, 0, (size_t)kHpBlocks * 4 * sizeof(double), st));  // blocks >= nb_rows stay 0
  // ---- setup: preconditioners, norms, ω₀ ----
  k_fill<<<kHpBlocks, kHpThreads, 0, st>>>(ones, std::max(n, kk), 1.0);
  note_launch();
  LP_TRY(flu(1, ones, v.gT));   // column sums Σ_i A_ik (local columns)
  LP_TRY(flu(0, ones, v.buf));  // row sums Σ_k A_ik (partial over ranks)
  LP_TRY(allreduce(v.buf, n, 0));
  k_hp_setup_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n, v.buf, o->penalty, o->penalty_scalar, eta);
  k_hp_setup_cols<<<kHpBlocks, kHpThreads, 0, st>>>(v, k, eta);
  k_hp_wsum_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n);
  k_hp_rows_final<<<1, 32, 0, st>>>(v, 2);
  k_hp_wsum_cols<<<1, 1024, 0, st>>>(v, k);
  note_launch(5);
  h[10] = (double)k;
  LP_CUDA(cudaMemcpyAsync(v.cols_out + 6, &h[10], sizeof(double), cudaMemcpyHostToDevice, st));
  LP_TRY(allreduce(v.cols_out + 6, 2, 0));  // [6] global column count, [7] Σ T_k
  LP_TRY(fetch(h, v.rows_out, 2));
  LP_TRY(fetch(h + 2, v.cols_out + 6, 2));
  LP_CUDA(cudaStreamSynchronize(st));
  const double sum_sig1 = h[0], sum_p2 = h[1], k_tot = h[2], sum_tau = h[3];
  const double qn = std::sqrt((double)n * mu_min * mu_min + t_max * t_max);
  const double cn = std::sqrt(k_tot + sum_p2);
  double omega = o->primal_weight;
  if (!(omega > 0.0)) {
    // PDLP's ω₀ = ‖c‖/‖q‖ in the preconditioned space: ‖T^½c‖² = Σ T_k + η Σ p², ‖Σ^½q‖² = μ_min² Σ Σ1_i
    const double cs = std::sqrt(sum_tau + eta * sum_p2), qs = std::sqrt(mu_min * mu_min * sum_sig1);
    omega = cs > 0.0 && qs > 0.0 ? cs / qs : 1.0;
  }

  // ---- initial point z = (t, 0, 0): A t, Aᵀy ----
  LP_TRY(flu(0, t, v.buf));
  LP_TRY(allreduce(v.buf, n, 0));
  k_copy<<<kHpBlocks, kHpThreads, 0, st>>>(v.mu, v.buf, n);
  note_launch();
  LP_TRY(flu(1, v.y, v.gT));
  k_hp_anchor_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n, 0);
  k_hp_anchor_cols<<<kHpBlocks, kHpThreads, 0, st>>>(v, k, 0, omega, rho);
  note_launch(2);

  // one iteration: T(z) (projection, A t̂, σ̂, ŷ, Aᵀŷ) and the Halpern mix
  auto project_multi = [&]() -> int {
    k_hp_primal_v<<<1, 1024, 0, st>>>(v, k);
    note_launch();
    UVD_TRY(allreduce(v.cres + 2, 1, 0));
    UVD_TRY(fetch(h + 20, v.cres + 2, 1));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    double lam = 0.0;
    if (h[20] > t_max) {
      double prev = -1.0;
      for (int it = 0; it < 200; ++it) {
        k_hp_proj_sums<<<1, 1024, 0, st>>>(v, k, lam);
        note_launch();
        UVD_TRY(allreduce(v.cres + 2, 3, 0));
        UVD_TRY(fetch(h + 20, v.cres + 2, 3));
        UVD_CUDA_TRY(cudaStreamSynchronize(st));
        lam = std::max(lam, (h[20] - t_max) / h[21]);
        if (h[22] == prev) break;
        prev = h[22];
      }
    }
    k_hp_primal_fin<<<1, 1024, 0, st>>>(v, k, n, lam);
    note_launch();
    return UVD_OK;
  };
  auto iteration = [&]() -> int {
    if (multi) {
      UVD_TRY(project_multi());
    } else {
      k_hp_primal<<<1, 1024, 0, st>>>(v, k, n, t_max);
      note_launch();
    }
    UVD_TRY(flu(0, v.tT, v.buf));
    UVD_TRY(allreduce(v.buf, n, 0));
    k_hp_dual<<<nb_rows, kHpThreads, 0, st>>>(v, n, mu_min, eta);
    note_launch();
    UVD_TRY(flu(1, v.yT, v.gTT));
    k_hp_mix_cols<<<kHpBlocks, kHpThreads, 0, st>>>(v, k);
    note_launch();
    return UVD_OK;
  };
  const bool graph_ok = o->use_graph && !multi && st != nullptr;
  if (graph_ok) {
    LP_CUDA(cudaStreamSynchronize(st));
    LP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int crc = UVD_OK;
    for (int q = 0; q < M && crc == UVD_OK; ++q) crc = iteration();
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (crc != UVD_OK) return finish(crc);
    LP_CUDA(ce);
    LP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }

  struct Kkt { double rel_p, rel_d, rel_g, pobj, dobj, yb, S; };
  double r_last = 0.0, r_first = 0.0;
  // KKT of T(z) (the last iteration's operator output) and the fixed-point residuals
  auto evaluate = [&](Kkt* out) -> int {
    k_hp_kkt_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n, mu_min);
    k_hp_rows_final<<<1, 32, 0, st>>>(v, 4);
    k_hp_kkt_cols<<<1, 1024, 0, st>>>(v, k);
    note_launch(3);
    UVD_TRY(allreduce(v.cols_out, 4, 0));
    UVD_TRY(allreduce(v.cols_out + 4, 1, 1));
    UVD_TRY(fetch(h, v.rows_out, 8));
    UVD_TRY(fetch(h + 8, v.cols_out, 6));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    const double S = h[9];
    const double over = std::max(0.0, S - t_max);
    const double rp = std::sqrt(h[0] + over * over);
    const double pobj = S + h[2];
    Kkt best{};
    double best_m = INFINITY;
    // two budget multipliers: the projection's ωλ, and the least y_b making every column dual feasible
    const double ybs[2] = {h[13], std::max(0.0, h[12] - 1.0)};
    const double dres[2] = {h[8], 0.0};
    for (int c = 0; c < 2; ++c) {
      const double rd = std::sqrt(h[1] + dres[c]);
      const double dobj = mu_min * h[3] - t_max * ybs[c];
      Kkt q{rp / (1.0 + qn), rd / (1.0 + cn), std::fabs(pobj - dobj) / (1.0 + std::fabs(pobj) + std::fabs(dobj)),
            pobj, dobj, ybs[c], S};
      const double m = std::max(q.rel_p, std::max(q.rel_d, q.rel_g));
      if (m < best_m) { best_m = m; best = q; }
    }
    *out = best;
    r_last = std::sqrt(omega * (h[10] + h[4]) + h[5] / omega);
    r_first = std::sqrt(omega * (h[11] + h[6]) + h[7] / omega);
    return UVD_OK;
  };
  auto converged = [&](const Kkt& c) { return c.rel_p <= eps && c.rel_d <= eps && c.rel_g <= eps; };

  Kkt cur{};
  int64_t it = 0, it_restart = 0;
  int restarts = 0;
  bool done = false;
  double r_prev = INFINITY;
  while (it < max_iter) {
    if (graph_ok) {
      LP_CUDA(cudaGraphLaunch(exec, st));
    } else {
      for (int q = 0; q < M; ++q) LP_TRY(iteration());
    }
    it += M;
    LP_TRY(evaluate(&cur));
    if (converged(cur)) { done = true; break; }
    const bool restart = r_last <= b_suff * r_first || (r_last <= b_nec * r_first && r_last > r_prev) ||
                         (double)(it - it_restart) >= b_art * (double)it;
    r_prev = r_last;
    if (restart) {
      // ω from the movement between restart points (before the anchors move)
      k_hp_move_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n, eta);
      k_hp_rows_final<<<1, 32, 0, st>>>(v, 2);
      k_hp_move_cols<<<1, 1024, 0, st>>>(v, k);
      note_launch(3);
      LP_TRY(allreduce(v.cols_out + 6, 1, 0));
      LP_TRY(fetch(h, v.rows_out, 2));
      LP_TRY(fetch(h + 2, v.cols_out + 6, 1));
      LP_CUDA(cudaStreamSynchronize(st));
      const double dx = std::sqrt(h[2] + h[0]), dy = std::sqrt(h[1]);
      if (dx > 1e-10 && dy > 1e-10) omega = std::exp(theta * std::log(dy / dx) + (1.0 - theta) * std::log(omega));
      k_hp_anchor_rows<<<kHpBlocks, kHpThreads, 0, st>>>(v, n, 1);
      k_hp_anchor_cols<<<kHpBlocks, kHpThreads, 0, st>>>(v, k, 1, omega, rho);
      note_launch(2);
      it_restart = it;
      r_prev = INFINITY;
      ++restarts;
    }
  }
  // hand back T(z) of the last iteration: t̂, σ̂, ŷ and the chosen y_b
  k_copy<<<kHpBlocks, kHpThreads, 0, st>>>(v.sig, v.sigT, n);
  k_copy<<<kHpBlocks, kHpThreads, 0, st>>>(v.y, v.yT, n);
  note_launch(2);
  if (k > 0) {
    k_copy<<<kHpBlocks, kHpThreads, 0, st>>>(v.t, v.tT, k);
    note_launch();
  }
  h[30] = cur.yb;
  LP_CUDA(cudaMemcpyAsync(y + n, &h[30], sizeof(double), cudaMemcpyHostToDevice, st));
  LP_CUDA(cudaStreamSynchronize(st));
  LP_CUDA(cudaGetLastError());
  res->status = done ? 0 : 1;
  res->restarts = restarts;
  res->iterations = it;
  res->primal_obj = cur.pobj;
  res->dual_obj = cur.dobj;
  res->rel_primal_res = cur.rel_p;
  res->rel_dual_res = cur.rel_d;
  res->rel_gap = cur.rel_g;
  res->sum_t = cur.S;
  res->primal_weight = omega;
  res->averaged = 0;
  return finish(UVD_OK);
#undef LP_TRY
#undef LP_CUDA
}
