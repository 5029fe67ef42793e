// vantage.cu — uvd_vantage_sample ("uniform
// grid ... collision-free ... dilated by 5 cm").
//
//   k_grid_2d      DISC2D: floorplan distance to every wall, inside bounds,
//                  outside every obstacle polygon (crossing number)
//   k_grid_3d      FLOAT3D / TOWER / ARM-bases / ARM-lamps: BVH range query
//                  "any triangle closer than the clearance?" (fp64 distances),
//                  BVH closest-hit free-space test (Q20), ARM reach proxy
//   k_count/k_emit stable compaction in raw-grid order
// Grid coordinates are computed in fp64 with explicit rounding (no FMA) and
// stored as fp32: x = fl32(lo + (a + 1/2)·ρ) (Q9).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

struct Grid {
  double x0, y0, z0, rho;
  int64_t nx, ny, nz;
};

__device__ __forceinline__ float grid_coord(double lo, int64_t a, double rho) {
  return (float)__dadd_rn(lo, __dmul_rn((double)a + 0.5, rho));
}

__device__ __forceinline__ double pt_seg_dist2d(double px, double py, double ax, double ay, double bx,
                                                double by) {
  double ex = bx - ax, ey = by - ay;
  double t = ((px - ax) * ex + (py - ay) * ey) / (ex * ex + ey * ey);
  t = fmin(fmax(t, 0.0), 1.0);
  double qx = ax + t * ex - px, qy = ay + t * ey - py;
  return sqrt(qx * qx + qy * qy);
}

__global__ void k_grid_2d(Grid g, float lamp_z, double clearance, const Wall* __restrict__ walls,
                          int64_t n_walls, const float* __restrict__ poly_xy,
                          const int32_t* __restrict__ poly_off, int n_poly, float4 bounds,
                          float* __restrict__ pts, uint8_t* __restrict__ flag) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= g.nx * g.ny) return;
  int64_t a = q % g.nx, b = q / g.nx;
  float x = grid_coord(g.x0, a, g.rho), y = grid_coord(g.y0, b, g.rho);
  pts[3 * q] = x; pts[3 * q + 1] = y; pts[3 * q + 2] = lamp_z;
  double px = x, py = y;
  bool ok = x > bounds.x && x < bounds.z && y > bounds.y && y < bounds.w;
  for (int64_t w = 0; w < n_walls && ok; ++w) {
    Wall W = walls[w];
    if (pt_seg_dist2d(px, py, W.e0x, W.e0y, W.e1x, W.e1y) < clearance) ok = false;
  }
  for (int p = 0; p < n_poly && ok; ++p) {
    int k0 = poly_off[p], k1 = poly_off[p + 1], n = k1 - k0;
    bool in = false;
    for (int k = 0; k < n; ++k) {
      double ax = poly_xy[2 * (k0 + k)], ay = poly_xy[2 * (k0 + k) + 1];
      double bx = poly_xy[2 * (k0 + (k + 1) % n)], by = poly_xy[2 * (k0 + (k + 1) % n) + 1];
      if ((ay > py) != (by > py)) {
        double xi = ax + (py - ay) * (bx - ax) / (by - ay);
        if (xi > px) in = !in;
      }
    }
    if (in) ok = false;
  }
  flag[q] = ok;
}

// ---------------------------------------------------------------- 3D tests --
struct Scene3 {
  const float4* __restrict__ tri;
  const Node* __restrict__ nodes;
  uint32_t root;
};

// any triangle with fp64 distance < clr from p?
__device__ bool too_close(const Scene3& S, D3 p, double clr) {
  uint32_t stack[64];
  int sp = 0;
  stack[sp++] = S.root;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  const float lim = (float)clr + 1e-4f;
  const float lim2 = lim * lim;
  while (sp > 0) {
    uint32_t ref = stack[--sp];
    if (ref_is_leaf(ref)) {
      uint32_t st = ref_start(ref), cnt = ref_count(ref);
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4* t = S.tri + 3 * (int64_t)(st + k);
        if (point_tri_dist(p, t[0], t[1], t[2]) < clr) return true;
      }
    } else {
      Node nd = S.nodes[ref];
      if (box_dist2(px, py, pz, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.c.x, nd.c.y) <= lim2) {
        if (sp >= 64) return true;  // defensive: treat as infeasible
        stack[sp++] = nd.d.x;
      }
      if (box_dist2(px, py, pz, nd.b.x, nd.b.y, nd.b.z, nd.b.w, nd.c.z, nd.c.w) <= lim2) {
        if (sp >= 64) return true;
        stack[sp++] = nd.d.y;
      }
    }
  }
  return false;
}

// Q20: nearest hit along p + t w (t > 0) exists and is front-facing
__device__ bool is_free(const Scene3& S, D3 p) {
  const D3 w = d3(kFreeDirX, kFreeDirY, kFreeDirZ);
  const double ww = ddot3(w, w);
  Ray32 r = make_ray32((float)p.x, (float)p.y, (float)p.z, (float)w.x, (float)w.y, (float)w.z);
  double best = INFINITY;
  bool best_front = false;
  uint32_t stack[64];
  int sp = 0;
  stack[sp++] = S.root;
  while (sp > 0) {
    uint32_t ref = stack[--sp];
    if (ref_is_leaf(ref)) {
      uint32_t st = ref_start(ref), cnt = ref_count(ref);
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4* t = S.tri + 3 * (int64_t)(st + k);
        bool fr = false;
        double th = ray_tri_t(p, w, ww, t[0], t[1], t[2], &fr);
        // nearest hit; at an exactly equal t (a shared edge) a front face wins,
        // so the answer does not depend on the traversal order
        if (th > 0.0 && (th < best || (th == best && fr && !best_front))) { best = th; best_front = fr; }
      }
    } else {
      Node nd = S.nodes[ref];
      float tmax = best < 1e30 ? (float)best * 1.0001f + 1e-4f : 1e30f;
      if (slab(r, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.c.x, nd.c.y, tmax) && sp < 64) stack[sp++] = nd.d.x;
      if (slab(r, nd.b.x, nd.b.y, nd.b.z, nd.b.w, nd.c.z, nd.c.w, tmax) && sp < 64) stack[sp++] = nd.d.y;
    }
  }
  return best < INFINITY && best_front;
}

// mode: 0 = point grid (FLOAT3D / ARM lamps: xs × ys × zs), 1 = TOWER (floor
// grid × L samples), 2 = ARM bases (floor grid at base_z)
struct Grid3Args {
  Grid g;
  int mode;
  int L;
  double z0, z1;      // TOWER samples
  float base_z;       // ARM bases
  double clearance;
  // ARM reach
  const float* __restrict__ bases;
  const uint8_t* __restrict__ base_ok;
  int64_t n_bases;
  double reach;
};

__global__ void k_grid_3d(Scene3 S, Grid3Args A, float* __restrict__ pts, uint8_t* __restrict__ flag) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t R = A.g.nx * A.g.ny * A.g.nz;
  if (q >= R) return;
  int64_t a = q % A.g.nx, rest = q / A.g.nx;
  int64_t b = rest % A.g.ny, cz = rest / A.g.ny;
  float x = grid_coord(A.g.x0, a, A.g.rho), y = grid_coord(A.g.y0, b, A.g.rho);
  bool ok = true;
  if (A.mode == 1) {
    for (int l = 0; l < A.L; ++l) {
      float z = (float)__dadd_rn(A.z0, __ddiv_rn(__dmul_rn((double)l + 0.5, __dadd_rn(A.z1, -A.z0)),
                                                 (double)A.L));
      int64_t o = 3 * (q * A.L + l);
      pts[o] = x; pts[o + 1] = y; pts[o + 2] = z;
      if (ok && too_close(S, d3(x, y, z), A.clearance)) ok = false;
    }
    if (ok) ok = is_free(S, d3(pts[3 * q * A.L], pts[3 * q * A.L + 1], pts[3 * q * A.L + 2]));
  } else {
    float z = A.mode == 2 ? A.base_z : grid_coord(A.g.z0, cz, A.g.rho);
    pts[3 * q] = x; pts[3 * q + 1] = y; pts[3 * q + 2] = z;
    D3 p = d3(x, y, z);
    ok = !too_close(S, p, A.clearance) && is_free(S, p);
    if (ok && A.bases) {
      bool reach = false;
      for (int64_t k = 0; k < A.n_bases && !reach; ++k) {
        if (!A.base_ok[k]) continue;
        double dx = __dadd_rn(p.x, -(double)A.bases[3 * k]);
        double dy = __dadd_rn(p.y, -(double)A.bases[3 * k + 1]);
        double dz = __dadd_rn(p.z, -(double)A.bases[3 * k + 2]);
        double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        reach = dist <= A.reach;
      }
      ok = reach;
    }
  }
  flag[q] = ok;
}

// ------------------------------------------------------------- compaction --
__global__ void __launch_bounds__(1024) k_flag_scan(const uint8_t* __restrict__ flag, int64_t n,
                                                    int64_t* __restrict__ pos,
                                                    int64_t* __restrict__ total) {
  __shared__ int64_t part[1024];
  int64_t per = (n + 1023) / 1024;
  int64_t s = threadIdx.x * per, e = s + per < n ? s + per : n;
  int64_t c = 0;
  for (int64_t i = s; i < e; ++i) c += flag[i];
  part[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = s; i < e; ++i) {
    pos[i] = run;
    run += flag[i];
  }
  if (threadIdx.x == 1023) *total = part[1023];
}

__global__ void k_compact(const uint8_t* __restrict__ flag, const int64_t* __restrict__ pos,
                          int64_t n, const float* __restrict__ pts, int L, float* __restrict__ out,
                          int64_t* __restrict__ raw) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n || !flag[q]) return;
  int64_t k = pos[q];
  for (int e = 0; e < 3 * L; ++e) out[3 * L * k + e] = pts[3 * L * q + e];
  if (raw) raw[k] = q;
}

static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static Grid make_grid(float lo_x, float hi_x, float lo_y, float hi_y, float lo_z, float hi_z,
                      float rho, bool use_z) {
  Grid g;
  g.rho = (double)rho;
  g.x0 = lo_x; g.y0 = lo_y; g.z0 = lo_z;
  g.nx = (int64_t)std::floor(((double)hi_x - (double)lo_x) / g.rho);
  g.ny = (int64_t)std::floor(((double)hi_y - (double)lo_y) / g.rho);
  g.nz = use_z ? (int64_t)std::floor(((double)hi_z - (double)lo_z) / g.rho) : 1;
  if (g.nx < 0) g.nx = 0;
  if (g.ny < 0) g.ny = 0;
  if (g.nz < 0) g.nz = 0;
  return g;
}

}  // namespace uvd

using namespace uvd;

extern "C" int uvd_vantage_sample(const uvd_scene* s, const uvd_vantage_opts* o, float* lamp_xyz,
                                  int64_t* raw_index, int64_t cap, int64_t* out_k, void* stream) {
  clear_error();
  if (!s || !o || !out_k) { set_error("uvd_vantage_sample: null argument"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_vantage_sample");
  *out_k = 0;
  if (!(o->spacing > 0.f) || !(o->clearance >= 0.f) || !std::isfinite(o->spacing)) {
    set_error("uvd_vantage_sample: spacing must be > 0 and clearance >= 0");
    return UVD_ERR_INVALID;
  }
  const bool ext = s->kind == UVD_SCENE_EXTRUDED;
  if (ext != (o->robot == UVD_ROBOT_DISC2D)) {
    set_error("uvd_vantage_sample: DISC2D applies to EXTRUDED scenes, TOWER/FLOAT3D/ARM to TRIMESH");
    return UVD_ERR_INVALID;
  }
  if (o->robot < 0 || o->robot > 3) { set_error("uvd_vantage_sample: unknown robot %d", o->robot); return UVD_ERR_INVALID; }
  int L = o->robot == UVD_ROBOT_TOWER ? o->lamp_samples : 1;
  if (L < 1) { set_error("uvd_vantage_sample: TOWER needs lamp_samples >= 1"); return UVD_ERR_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch al(s->alloc, st);  // released at every exit
  Grid g;
  const float* bb = s->bbox;
  if (ext) g = make_grid(s->bounds[0], s->bounds[2], s->bounds[1], s->bounds[3], 0, 0, o->spacing, false);
  else if (o->robot == UVD_ROBOT_FLOAT3D) g = make_grid(bb[0], bb[3], bb[1], bb[4], bb[2], bb[5], o->spacing, true);
  else if (o->robot == UVD_ROBOT_ARM) g = make_grid(bb[0], bb[3], bb[1], bb[4], o->zmin, o->zmax, o->spacing, true);
  else g = make_grid(bb[0], bb[3], bb[1], bb[4], 0, 0, o->spacing, false);
  const int64_t R = g.nx * g.ny * g.nz;
  if (R <= 0) { set_error("uvd_vantage_sample: empty grid (S:303)"); return UVD_ERR_EMPTY; }
  float* pts = (float*)al.get(R * 3 * L * sizeof(float));
  uint8_t* flag = (uint8_t*)al.get(R);
  int64_t* pos = (int64_t*)al.get(R * sizeof(int64_t));
  int64_t* dtot = (int64_t*)al.get(sizeof(int64_t));
  float* bpts = nullptr;
  uint8_t* bflag = nullptr;
  if (!pts || !flag || !pos || !dtot) { set_error("uvd_vantage_sample: out of device memory"); return UVD_ERR_NOMEM; }
  Scene3 S3{s->tri, s->nodes, s->root};
  if (ext) {
    float4 bounds = make_float4(s->bounds[0], s->bounds[1], s->bounds[2], s->bounds[3]);
    k_grid_2d<<<blocks_for(R, 128), 128, 0, st>>>(g, o->lamp_z, (double)o->clearance, s->walls,
                                                  s->n_walls, s->poly_xy, s->poly_off, s->n_poly,
                                                  bounds, pts, flag);
    note_launch();
  } else {
    Grid3Args A{};
    A.g = g;
    A.clearance = (double)o->clearance;
    A.L = L;
    A.z0 = (double)o->lamp_z0;
    A.z1 = (double)o->lamp_z1;
    if (o->robot == UVD_ROBOT_TOWER) A.mode = 1;
    if (o->robot == UVD_ROBOT_ARM) {
      Grid3Args B = A;
      B.g = make_grid(bb[0], bb[3], bb[1], bb[4], 0, 0, o->spacing, false);
      B.mode = 2;
      B.base_z = o->base_z;
      B.clearance = (double)o->base_clearance;
      B.L = 1;
      int64_t RB = B.g.nx * B.g.ny;
      bpts = (float*)al.get(RB * 3 * sizeof(float));
      bflag = (uint8_t*)al.get(RB);
      if (!bpts || !bflag) { set_error("uvd_vantage_sample: out of device memory"); return UVD_ERR_NOMEM; }
      k_grid_3d<<<blocks_for(RB, 64), 64, 0, st>>>(S3, B, bpts, bflag);
      note_launch();
      A.bases = bpts;
      A.base_ok = bflag;
      A.n_bases = RB;
      A.reach = (double)o->reach;
    }
    k_grid_3d<<<blocks_for(R, 64), 64, 0, st>>>(S3, A, pts, flag);
    note_launch();
  }
  k_flag_scan<<<1, 1024, 0, st>>>(flag, R, pos, dtot);
  note_launch();
  int64_t K = 0;
  UVD_CUDA_TRY(cudaMemcpyAsync(&K, dtot, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  UVD_CUDA_TRY(cudaGetLastError());
  *out_k = K;
  int rc = UVD_OK;
  if (K == 0) { set_error("uvd_vantage_sample: zero feasible vantage points (S:303)"); rc = UVD_ERR_EMPTY; }
  else if (K > cap || !lamp_xyz) { set_error("uvd_vantage_sample: capacity %lld < K = %lld", (long long)cap, (long long)K); rc = UVD_ERR_CAPACITY; }
  else {
    k_compact<<<blocks_for(R, 256), 256, 0, st>>>(flag, pos, R, pts, L, lamp_xyz, raw_index);
    note_launch();
    UVD_CUDA_TRY(cudaGetLastError());
  }
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  return rc;
}
