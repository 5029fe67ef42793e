// free.cu — empty regions at the two ends of every shadow segment (a5).
//
// A segment p -> c_i can only meet a triangle where one exists.  Two radii,
// computed once, let the assembly walk skip the parts of a segment that lie in
// provably empty space — the box tests of k_assemble_lane are bounded to
// t in [t_min, t_max] instead of [0, t_hi] — without changing any decision:
//
//  * lamp radius r_L(p): the distance from the lamp sample p to the nearest
//    scene triangle.  Every point of the segment with t < r_L/|D| is within
//    r_L of p, so no triangle is hit there.
//  * front radius r_T(i): the distance from the centroid c_i to the nearest
//    triangle (other than patch i's own) having a vertex strictly in front of
//    the patch plane, n_i·(v − c_i) > 1e-7 m.  The segment's end arrives from
//    the front (n_i·(x − c_i) = (1 − t) n_i·(p − c_i) > 0), so the part with
//    t > 1 − r_T/|D| lies within r_T of c_i on the front side, where every
//    triangle either is farther than r_T or has no point (the t range keeps
//    the segment ≥ 1e-4 m·cosθ in front: the kernel applies r_T only when
//    cosθ ≥ 1e-2, so coplanar neighbours within 1e-7 m are never hit there).
//
// Both are exact fp64 point–triangle distances (closest point by region,
// point_tri_dist), found by a nearest-first BVH walk pruned with the fp32
// distance to the padded child boxes (a lower bound: the padding covers the
// rounding) and, for r_T, skipping boxes with no point in front of the patch
// plane; capped at kFreeCap (a valid lower bound when nothing is nearer).  The walk scales the radii by (1 ∓ 1e-6) and rounds the resulting
// t bounds outward, so the bounds stay conservative.
#include <cuda_runtime.h>

#include <cstdlib>

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

constexpr double kFreeCap = 0.1;     // m: radii beyond this are reported as 0.1 m (measured: most of the gain, ~1 ms per 1M patches)
constexpr double kLampCap = 2.0;     // m: the lamp radius search (K queries, cheap)
constexpr double kFrontEps = 1e-7;   // m: "strictly in front" of the patch plane
constexpr int kFreeStack = 64;

// max over the box of n·(x − p) (fp64 from the fp32 box corners: exact inputs,
// one rounding per operation, far below kFrontEps for scene-sized boxes)
__device__ __forceinline__ double box_front(const float* n, D3 p, float lx, float hx, float ly, float hy, float lz,
                                            float hz) {
  const double nx = n[0], ny = n[1], nz = n[2];
  return nx * ((nx > 0.0 ? (double)hx : (double)lx) - p.x) + ny * ((ny > 0.0 ? (double)hy : (double)ly) - p.y) +
         nz * ((nz > 0.0 ? (double)hz : (double)lz) - p.z);
}

// distance from p to the nearest triangle that is not owned by `own` and (with
// n != nullptr) has a vertex more than kFrontEps in front of the plane (n, p)
__device__ double nearest_tri(const Node* __restrict__ nodes, uint32_t root, const float4* __restrict__ tri, D3 p,
                              const float* n, int own, double cap) {
  uint32_t stk[kFreeStack];
  int sp = 0;
  double best = cap;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;  // p is an fp32 point: exact
  uint32_t ref = root;
  for (;;) {
    if (ref_is_leaf(ref)) {
      const uint32_t st = ref_start(ref), nt = ref_count(ref);
      for (uint32_t k = 0; k < nt; ++k) {
        const float4* t = tri + 3 * (int64_t)(st + k);
        const float4 a = t[0], b = t[1], c = t[2];
        if (__float_as_int(a.w) == own) continue;
        if (n) {
          const D3 nn = d3(n[0], n[1], n[2]);
          if (ddot3(dsub3(f2d(a), p), nn) <= kFrontEps && ddot3(dsub3(f2d(b), p), nn) <= kFrontEps &&
              ddot3(dsub3(f2d(c), p), nn) <= kFrontEps)
            continue;  // no point strictly in front of the patch
        }
        best = fmin(best, point_tri_dist(p, a, b, c));
      }
    } else {
      const Node nd = nodes[ref];
      float d0 = box_dist2(px, py, pz, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.c.x, nd.c.y);
      float d1 = box_dist2(px, py, pz, nd.b.x, nd.b.y, nd.b.z, nd.b.w, nd.c.z, nd.c.w);
      if (n) {  // a box with no point more than kFrontEps in front holds no front triangle
        if (box_front(n, p, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.c.x, nd.c.y) <= kFrontEps) d0 = INFINITY;
        if (box_front(n, p, nd.b.x, nd.b.y, nd.b.z, nd.b.w, nd.c.z, nd.c.w) <= kFrontEps) d1 = INFINITY;
      }
      uint32_t c0 = nd.d.x, c1 = nd.d.y;
      if (d1 < d0) {
        const float tf = d0; d0 = d1; d1 = tf;
        const uint32_t tu = c0; c0 = c1; c1 = tu;
      }
      const float lim = (float)(best * best);
      if (d1 < lim && sp < kFreeStack) stk[sp++] = c1;
      if (d0 < lim) {
        ref = c0;
        continue;
      }
    }
    if (!sp) break;
    ref = stk[--sp];
  }
  return best;
}

__global__ void k_front_radius(const Node* __restrict__ nodes, uint32_t root, const float4* __restrict__ tri,
                               const float* __restrict__ cen, const float* __restrict__ nrm, int64_t N,
                               double cap, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const D3 c = d3(cen[3 * i], cen[3 * i + 1], cen[3 * i + 2]);
  const double r = nearest_tri(nodes, root, tri, c, nrm + 3 * i, (int)i, cap);
  out[i] = __double2float_rd(r);  // rounded down: still a lower bound
}

__global__ void k_lamp_radius(const Node* __restrict__ nodes, uint32_t root, const float4* __restrict__ tri,
                              const float* __restrict__ lamps, int64_t n, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 p = d3(lamps[3 * i], lamps[3 * i + 1], lamps[3 * i + 2]);
  out[i] = __double2float_rd(nearest_tri(nodes, root, tri, p, nullptr, -1, kLampCap));
}

int front_radius(uvd_scene* s, cudaStream_t st) {
  if (s->front_free) s->alloc.put(s->front_free);
  s->front_free = (float*)s->alloc.get((size_t)std::max<int64_t>(s->N, 1) * sizeof(float));
  if (!s->front_free) { set_error("scene: out of device memory (front radii)"); return UVD_ERR_NOMEM; }
  double cap = kFreeCap;
  if (const char* e = getenv("UVD_FREE_CAP")) cap = atof(e);  // dev A/B
  k_front_radius<<<(unsigned)((s->N + 127) / 128), 128, 0, st>>>(s->nodes, s->root, s->tri, s->centroid, s->normal,
                                                                 s->N, cap, s->front_free);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

int lamp_radius(const uvd_scene* s, const float* lamps, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return UVD_OK;
  k_lamp_radius<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(s->nodes, s->root, s->tri, lamps, n, out);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

}  // namespace uvd
