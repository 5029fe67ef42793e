// cube.cu — NEXT-3: the paper's own irradiance pipeline, the
// "visibility cube", on the GPU — for a head-to-head
// comparison with the shadow-ray path of a4–a6 on the same scenes.
//
// Per lamp sample, 6 cube faces of R×R pixels around the lamp (six
// cameras; 512²).  Pixel (a,b) of face f looks along
//   +X (1,u,v)  −X (−1,u,v)  +Y (u,1,v)  −Y (u,−1,v)  +Z (u,v,1)  −Z (u,v,−1),
//   u = −1 + (2a+1)/R, v = −1 + (2b+1)/R,
// and carries the power e = (P/L)·Ω_px/(4π) of its exact solid angle (the
// precomputed emission texture E; Ω_px from G(u,v) = atan(uv/√(1+u²+v²))).
// The pixel's nearest surface (the Z-buffer) is the closest triangle the
// ray hits (per-lane BVH closest-hit: fp32 conservative boxes bounded by the
// current best t, fp32 filtered triangle test, fp64 Möller–Trumbore for the
// candidates, ties to the lower triangle index); its patch receives e when the
// hit is front-facing: F[i] += e by warp-aggregated fp64 atomics, then
// A[i,j] = F_i/|s_i| for the dense output.
//
//   k_cube_emission   E[R×R] (one face; the six are congruent)
//   k_cube_trace      one thread per pixel ray, 256 consecutive pixels per block
//   k_cube_finish     A = F/|s| for a chunk of columns
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

__device__ __forceinline__ double px_G(double u, double v) { return atan(u * v / sqrt(1.0 + u * u + v * v)); }

__global__ void k_cube_emission(int R, double* __restrict__ E) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= (int64_t)R * R) return;
  const int a = (int)(q % R), b = (int)(q / R);
  const double u0 = -1.0 + 2.0 * a / R, u1 = -1.0 + 2.0 * (a + 1) / R;
  const double v0 = -1.0 + 2.0 * b / R, v1 = -1.0 + 2.0 * (b + 1) / R;
  E[q] = px_G(u1, v1) - px_G(u0, v1) - px_G(u1, v0) + px_G(u0, v0);
}

struct CubeParams {
  const float4* __restrict__ tri;
  const Node* __restrict__ nodes;
  const Node* __restrict__ onodes;  // octant copies (nullptr: not built for this scene)
  int64_t n_nodes;
  uint32_t root;
  const float* __restrict__ lamps;
  int L;
  const int64_t* __restrict__ cols;  // device, nullptr = identity
  int64_t c0, nc;                    // column chunk [c0, c0 + nc)
  int R;
  const double* __restrict__ E;      // [R*R] pixel solid angles
  double scale;                      // (P/L)/(4π)
  int64_t N;
  double* __restrict__ F;            // [nc][N] flux of the chunk
  int32_t* __restrict__ hits;        // optional [n_cols][L][6][R][R]
  int* __restrict__ err;
};

constexpr int kCubeStack = 64;
constexpr int kCubeThreads = 256;

// closest front-or-back hit along O + t D, t > 0; returns the triangle position
// in leaf order (or -1), its facing, and its owner patch
template <bool OCT>
__device__ __forceinline__ int64_t cube_closest(const CubeParams& P, float ox, float oy, float oz, double dxd,
                                                double dyd, double dzd, bool* front, int* owner) {
  const float dx = (float)dxd, dy = (float)dyd, dz = (float)dzd;
  const float ix = safe_inv(dx), iy = safe_inv(dy), iz = safe_inv(dz);
  const float oix = ox * ix, oiy = oy * iy, oiz = oz * iz;
  const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const D3 O = d3(ox, oy, oz), D = d3(dxd, dyd, dzd);
  const double dd = ddot3(D, D);
  double best = INFINITY;
  int64_t bk = -1;
  int borig = 0x7fffffff;
  bool bfront = false;
  int bown = -1;
  float tmax = 3.0e38f;
  uint32_t stk[kCubeStack];
  int sp = 0;
  // the octant copy of the nodes for this ray (slabs stored entry, exit), as in k_assemble_lane
  const uint32_t oct = (__float_as_uint(ix) >> 31) | ((__float_as_uint(iy) >> 31) << 1) |
                       ((__float_as_uint(iz) >> 31) << 2);
  uint32_t ref = (!OCT || ref_is_leaf(P.root)) ? P.root : P.root + oct * (uint32_t)P.n_nodes;
  for (;;) {
    if (ref_is_leaf(ref)) {
      const uint32_t st = ref_start(ref), nt = ref_count(ref);
      for (uint32_t k = 0; k < nt; ++k) {
        const float4* t = P.tri + 3 * (int64_t)(st + k);
        const float4 a = __ldg(t), b = __ldg(t + 1), c = __ldg(t + 2);
        // fp32 filter on the segment t in (0, tmax): skip certain misses
        if (seg_tri_filter32(ox, oy, oz, dx, dy, dz, nD, 0.0f, tmax, a, b, c) == 0) continue;
        // exact: fp64 Möller–Trumbore (as the oracle), inclusive edges, t > 0
        const D3 V0 = f2d(a);
        const D3 E1 = dsub3(f2d(b), V0), E2 = dsub3(f2d(c), V0);
        const D3 Pv = dcross3(D, E2);
        const double det = ddot3(E1, Pv);
        const D3 Nv = dcross3(E1, E2);
        if (det * det <= kParallel * kParallel * dd * ddot3(Nv, Nv)) continue;
        const double inv = 1.0 / det;
        const D3 T = dsub3(O, V0);
        const double u = ddot3(T, Pv) * inv;
        const D3 Q = dcross3(T, E1);
        const double v = ddot3(D, Q) * inv;
        if (fmin(u, fmin(v, 1.0 - u - v)) < 0.0) continue;
        const double th = ddot3(E2, Q) * inv;
        if (!(th > 0.0)) continue;
        const int orig = __float_as_int(b.w);  // input triangle index (ties -> lower index)
        if (th < best || (th == best && orig < borig)) {
          best = th;
          bk = st + k;
          borig = orig;
          bfront = ddot3(D, Nv) < 0.0;
          bown = __float_as_int(a.w);
          tmax = __double2float_ru(best) * 1.000002f + 1e-7f;
        }
      }
      if (!sp) break;
      ref = stk[--sp];
      continue;
    }
    const Node* nd = (OCT ? P.onodes : P.nodes) + ref;
    const float4 na = __ldg(&nd->a), nb = __ldg(&nd->b), nc = __ldg(&nd->c);
    const uint2 ch = __ldg(reinterpret_cast<const uint2*>(&nd->d));
    // no widening per node: fl(1/d), fl(d) and the FFMA's rounding move a plane by
    // <= 2^-22 |b - o| + 2^-24 |o| <= 1e-5 m for |coords| <= 20 m, inside the box
    // padding (k_assemble_lane's argument, plus the fp32 rounding of the direction);
    // tmax keeps its widening above ru(best) (ties go to the lower input index)
    float an, af, bn, bf;
    if (OCT) {  // paired octant layout (bvh.cu k_octant_nodes): both children per FFMA2
      const float2 ex = ffma2(make_float2(na.x, na.y), make_float2(ix, ix), make_float2(-oix, -oix));
      const float2 xx = ffma2(make_float2(na.z, na.w), make_float2(ix, ix), make_float2(-oix, -oix));
      const float2 ey = ffma2(make_float2(nb.x, nb.y), make_float2(iy, iy), make_float2(-oiy, -oiy));
      const float2 xy = ffma2(make_float2(nb.z, nb.w), make_float2(iy, iy), make_float2(-oiy, -oiy));
      const float2 ez = ffma2(make_float2(nc.x, nc.y), make_float2(iz, iz), make_float2(-oiz, -oiz));
      const float2 xz = ffma2(make_float2(nc.z, nc.w), make_float2(iz, iz), make_float2(-oiz, -oiz));
      an = fmaxf(fmaxf(ex.x, ey.x), fmaxf(ez.x, 0.0f));
      af = fminf(fminf(xx.x, xy.x), fminf(xz.x, tmax));
      bn = fmaxf(fmaxf(ex.y, ey.y), fmaxf(ez.y, 0.0f));
      bf = fminf(fminf(xx.y, xy.y), fminf(xz.y, tmax));
    } else {
      const float ax0 = fmaf(na.x, ix, -oix), ax1 = fmaf(na.y, ix, -oix);
      const float ay0 = fmaf(na.z, iy, -oiy), ay1 = fmaf(na.w, iy, -oiy);
      const float az0 = fmaf(nc.x, iz, -oiz), az1 = fmaf(nc.y, iz, -oiz);
      const float bx0 = fmaf(nb.x, ix, -oix), bx1 = fmaf(nb.y, ix, -oix);
      const float by0 = fmaf(nb.z, iy, -oiy), by1 = fmaf(nb.w, iy, -oiy);
      const float bz0 = fmaf(nc.z, iz, -oiz), bz1 = fmaf(nc.w, iz, -oiz);
      an = fmaxf(fmaxf(fminf(ax0, ax1), fminf(ay0, ay1)), fmaxf(fminf(az0, az1), 0.0f));
      af = fminf(fminf(fmaxf(ax0, ax1), fmaxf(ay0, ay1)), fminf(fmaxf(az0, az1), tmax));
      bn = fmaxf(fmaxf(fminf(bx0, bx1), fminf(by0, by1)), fmaxf(fminf(bz0, bz1), 0.0f));
      bf = fminf(fminf(fmaxf(bx0, bx1), fmaxf(by0, by1)), fminf(fmaxf(bz0, bz1), tmax));
    }
    const bool h0 = an <= af;
    const bool h1 = bn <= bf;
    if (h0 && h1) {
      const bool swap = bn < an;  // near child first: the closest hit shrinks tmax early
      ref = swap ? ch.y : ch.x;
      if (sp < kCubeStack) stk[sp++] = swap ? ch.x : ch.y;
      else atomicExch(P.err, 2);
    } else if (h0 || h1) {
      ref = h0 ? ch.x : ch.y;
    } else {
      if (!sp) break;
      ref = stk[--sp];
    }
  }
  *front = bfront;
  *owner = bown;
  return bk;
}

#ifndef UVD_CUBE_MINB
#define UVD_CUBE_MINB 4
#endif
template <bool OCT>
__global__ void __launch_bounds__(kCubeThreads, UVD_CUBE_MINB) k_cube_trace(CubeParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t per_col = (int64_t)P.L * 6 * P.R * P.R;
  const int64_t total = P.nc * per_col;
  for (int64_t q = blockIdx.x * (int64_t)kCubeThreads + threadIdx.x; q - lane < total;
       q += (int64_t)gridDim.x * kCubeThreads) {
    const bool active = q < total;
    int key = -1;
    double e = 0.0;
    if (active) {
      const int64_t cl = q / per_col;
      int64_t rem = q - cl * per_col;
      const int l = (int)(rem / (6 * (int64_t)P.R * P.R));
      rem -= (int64_t)l * 6 * P.R * P.R;
      const int f = (int)(rem / ((int64_t)P.R * P.R));
      const int64_t px = rem - (int64_t)f * P.R * P.R;
      const int a = (int)(px % P.R), b = (int)(px / P.R);
      const int64_t c = P.c0 + cl;
      const int64_t j = P.cols ? P.cols[c] : c;
      const float* pl = P.lamps + 3 * (j * P.L + l);
      const double u = -1.0 + (2.0 * a + 1.0) / P.R, v = -1.0 + (2.0 * b + 1.0) / P.R;
      double dx, dy, dz;
      switch (f) {
        case 0: dx = 1.0; dy = u; dz = v; break;
        case 1: dx = -1.0; dy = u; dz = v; break;
        case 2: dx = u; dy = 1.0; dz = v; break;
        case 3: dx = u; dy = -1.0; dz = v; break;
        case 4: dx = u; dy = v; dz = 1.0; break;
        default: dx = u; dy = v; dz = -1.0; break;
      }
      bool front = false;
      int owner = -1;
      const int64_t k = cube_closest<OCT>(P, pl[0], pl[1], pl[2], dx, dy, dz, &front, &owner);
      if (P.hits) P.hits[c * per_col + (q - cl * per_col)] = k < 0 ? -1 : (front ? __float_as_int(P.tri[3 * k + 1].w) : -2);
      if (k >= 0 && front) {
        key = owner;
        e = P.scale * P.E[px];
      }
    }
    // warp-aggregated flux: lanes hitting the same patch of the same column add once
    const int64_t cl_lane = active ? q / per_col : -1;
    const unsigned long long gk = key >= 0 ? ((unsigned long long)cl_lane << 32) | (unsigned)key : ~0ull;
    const unsigned grp = __match_any_sync(0xffffffffu, gk);
    double sum = 0.0;
    for (int src = 0; src < 32; ++src) {
      const double w = __shfl_sync(0xffffffffu, e, src);
      if ((grp >> src) & 1u) sum += w;
    }
    if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(P.F + cl_lane * P.N + key, sum);
  }
}

__global__ void k_cube_finish(const double* __restrict__ F, const double* __restrict__ area, int64_t nc, int64_t N,
                              float* __restrict__ values, int64_t ld, int64_t c0) {
  const int64_t total = nc * ld;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cl = q / ld, r = q - cl * ld;
    values[(c0 + cl) * ld + r] = r < N ? (float)(F[cl * N + r] / area[r]) : 0.f;
  }
}

}  // namespace uvd

using namespace uvd;

extern "C" int uvd_cubemap_matrix(const uvd_scene* s, const float* lamp_xyz, int64_t k_total, const int64_t* cols,
                                  int64_t n_cols, const uvd_lamp* lamp, int32_t face_res, uvd_matrix_out* out,
                                  int32_t* hits, void* stream) {
  clear_error();
  if (!s || !lamp_xyz || !lamp || !out) { set_error("uvd_cubemap_matrix: null argument"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_cubemap_matrix");
  if (lamp->samples_per_config < 1 || !(lamp->power_w > 0.0) || face_res < 1 || face_res > 4096) {
    set_error("uvd_cubemap_matrix: need power_w > 0, samples_per_config >= 1, 1 <= face_res <= 4096");
    return UVD_ERR_INVALID;
  }
  if (!cols) n_cols = k_total;
  if (n_cols < 0 || k_total < 0) { set_error("uvd_cubemap_matrix: negative size"); return UVD_ERR_INVALID; }
  if (out->format != UVD_DENSE_COLMAJOR || !out->values || out->ld < s->N || out->ld % 32 != 0) {
    set_error("uvd_cubemap_matrix: dense output with ld >= N, ld %% 32 == 0");
    return UVD_ERR_INVALID;
  }
  if (cols)
    for (int64_t c = 0; c < n_cols; ++c)
      if (cols[c] < 0 || cols[c] >= k_total) { set_error("uvd_cubemap_matrix: column out of range"); return UVD_ERR_INVALID; }
  if (n_cols == 0) return UVD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch al(s->alloc, st);  // released at every exit
  const int R = face_res;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_cols, (int64_t)(256ll << 20) / (8 * std::max<int64_t>(s->N, 1))));
  double* E = (double*)al.get((size_t)R * R * sizeof(double));
  double* F = (double*)al.get((size_t)chunk * s->N * sizeof(double));
  int64_t* dcols = cols ? (int64_t*)al.get(n_cols * sizeof(int64_t)) : nullptr;
  if (!E || !F || (cols && !dcols)) { set_error("uvd_cubemap_matrix: out of device memory"); return UVD_ERR_NOMEM; }
  if (dcols) UVD_CUDA_TRY(cudaMemcpyAsync(dcols, cols, n_cols * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  k_cube_emission<<<(unsigned)(((int64_t)R * R + 255) / 256), 256, 0, st>>>(R, E);
  note_launch();
  const int dev = s->alloc.device, sms = sm_count(dev);
  CubeParams P;
  P.tri = s->tri;
  P.nodes = s->nodes;
  P.onodes = s->onodes;
  P.n_nodes = s->n_nodes;
  P.root = s->root;
  P.lamps = lamp_xyz;
  P.L = lamp->samples_per_config;
  P.cols = dcols;
  P.R = R;
  P.E = E;
  P.scale = lamp->power_w / (double)P.L / (4.0 * 3.14159265358979323846);
  P.N = s->N;
  P.F = F;
  P.hits = hits;
  P.err = s->err_flag;
  UVD_TRY(check_lamps(s, lamp_xyz, dcols, n_cols, P.L, st));  // the padding's lamp range (assemble.cu)
  for (int64_t c0 = 0; c0 < n_cols; c0 += chunk) {
    const int64_t nc = std::min(chunk, n_cols - c0);
    P.c0 = c0;
    P.nc = nc;
    UVD_CUDA_TRY(cudaMemsetAsync(F, 0, (size_t)nc * s->N * sizeof(double), st));
    const int64_t rays = nc * P.L * 6 * (int64_t)R * R;
    const unsigned g = (unsigned)std::min<int64_t>((rays + kCubeThreads - 1) / kCubeThreads, (int64_t)sms * 8);
    if (P.onodes) k_cube_trace<true><<<g, kCubeThreads, 0, st>>>(P);
    else k_cube_trace<false><<<g, kCubeThreads, 0, st>>>(P);
    k_cube_finish<<<(unsigned)std::min<int64_t>((nc * out->ld + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(
        F, s->area, nc, s->N, out->values, out->ld, c0);
    note_launch(2);
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}
