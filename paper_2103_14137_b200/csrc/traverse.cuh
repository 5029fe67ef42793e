// traverse.cuh — device-side geometry primitives shared by the assembly and
// vantage kernels (CUDA path only).
//
// Precision scheme (SURVEY §8c "GPU numerics"):
//  * node boxes are tested in fp32 against an fp32 copy of the ray; the boxes
//    were padded outward at build time (1e-5 m + 1e-6 |x|) and the slab
//    interval is widened by 2e-6 relative, so a box is never culled when the
//    exact fp64 segment touches it;
//  * triangles are tested in fp64 from the exact fp32 vertices with
//    Möller–Trumbore (1997) in division-free form; margins are accepted down to
//    -1e-12 (watertight shared edges);
//  * irradiance arithmetic is fp64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "uvd_internal.cuh"

namespace uvd {

struct Ray32 {  // fp32 ray for slab tests: o + t*dir, t in [0, tmax]
  float ox, oy, oz;
  float ix, iy, iz;  // safe reciprocals of dir
};

// 1/d for slab tests: the hardware reciprocal (rcp.approx, relative error
// <= 2^-23, one instruction instead of the ~8 of an IEEE division).  With the
// FFMA's rounding a slab parameter is scaled by at most 1 + 1.5·2^-23, i.e. a
// plane moves by <= 7 µm over a 40 m scene — inside the >= 10 µm box padding.
__device__ __forceinline__ float safe_inv(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return fabsf(d) < 1e-30f ? copysignf(1e30f, d) : r;
}

// Blackwell's paired FP32 FMA (FFMA2: one instruction, two IEEE fmas with the
// same rounding as two FFMA); a scalar b / c is broadcast to both halves
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

__device__ __forceinline__ Ray32 make_ray32(float ox, float oy, float oz, float dx, float dy, float dz) {
  Ray32 r;
  r.ox = ox; r.oy = oy; r.oz = oz;
  r.ix = safe_inv(dx); r.iy = safe_inv(dy); r.iz = safe_inv(dz);
  return r;
}

// conservative slab test of the ray against [lo, hi] for t in [0, tmax]
__device__ __forceinline__ bool slab(const Ray32& r, float lx, float hx, float ly, float hy, float lz,
                                     float hz, float tmax) {
  float tx0 = (lx - r.ox) * r.ix, tx1 = (hx - r.ox) * r.ix;
  float ty0 = (ly - r.oy) * r.iy, ty1 = (hy - r.oy) * r.iy;
  float tz0 = (lz - r.oz) * r.iz, tz1 = (hz - r.oz) * r.iz;
  float tn = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
  float tf = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
  return tn <= tf * 1.000002f + 1e-7f;
}

struct D3 { double x, y, z; };
__device__ __forceinline__ D3 d3(double x, double y, double z) { D3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ D3 dsub3(D3 a, D3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double ddot3(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 dcross3(D3 a, D3 b) {
  return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ D3 f2d(float4 v) { return d3((double)v.x, (double)v.y, (double)v.z); }

// fp64 segment/triangle test: does O + t D, t in (t_lo, t_hi), meet the closed
// triangle (V0,V1,V2)?  Division-free Möller–Trumbore: with s = sign(det),
// a = |det|: u·a = s(T·P), v·a = s(D·Q), t·a = s(E2·Q).  Near-parallel
// (|det| <= 1e-12 |D||E1xE2|) never hits.
__device__ __forceinline__ bool seg_hits_tri(D3 O, D3 D, double dd /* D·D */, double t_lo,
                                             double t_hi, float4 a, float4 b, float4 c) {
  D3 V0 = f2d(a);
  D3 E1 = dsub3(f2d(b), V0), E2 = dsub3(f2d(c), V0);
  D3 P = dcross3(D, E2);
  double det = ddot3(E1, P);
  D3 Nv = dcross3(E1, E2);
  if (det * det <= kParallel * kParallel * dd * ddot3(Nv, Nv)) return false;
  double s = det > 0.0 ? 1.0 : -1.0;
  double A = fabs(det);
  double tol = kEdgeTol * A;
  D3 T = dsub3(O, V0);
  double U = s * ddot3(T, P);
  if (U < -tol) return false;
  D3 Q = dcross3(T, E1);
  double V = s * ddot3(D, Q);
  if (V < -tol || A - U - V < -tol) return false;
  double W = s * ddot3(E2, Q);
  return W - t_lo * A >= -tol && t_hi * A - W >= -tol;
}

// fp32 filtered segment/triangle test.  Same division-free Möller–Trumbore in
// fp32 from the exact fp32 vertices and lamp origin, with the fp32-rounded
// direction.  Forward error bound (u = 2^-24): the inputs D, T = O - V0,
// E1, E2 carry relative error <= u per component; a cross product component
// then errs by <= 4u x the sum of its |products|, and a dot product of such a
// vector with a u-perturbed vector by <= (4u + u + 3u) x the 1-norm product of
// the three factors, i.e. <= 8u |X|_1 |Y|_1 |Z|_1 for det, U, V and W alike.
// Each margin is therefore classified with K_ERR = 16u (2x the first-order
// bound) as a certain miss (< -err), a certain hit (> +err) or undecided.
// Returns 0 miss, 1 hit, 2 undecided (resolved in fp64 by the caller).
__device__ __forceinline__ int seg_tri_filter32(float ox, float oy, float oz, float dx, float dy,
                                                float dz, float nD, float t_lo, float t_hi,
                                                float4 a, float4 b, float4 c) {
  const float k = 16.0f * 5.9604645e-08f;
  float e1x = b.x - a.x, e1y = b.y - a.y, e1z = b.z - a.z;
  float e2x = c.x - a.x, e2y = c.y - a.y, e2z = c.z - a.z;
  float tx = ox - a.x, ty = oy - a.y, tz = oz - a.z;
  float px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
  float det = e1x * px + e1y * py + e1z * pz;
  float nE1 = fabsf(e1x) + fabsf(e1y) + fabsf(e1z);
  float nE2 = fabsf(e2x) + fabsf(e2y) + fabsf(e2z);
  float nT = fabsf(tx) + fabsf(ty) + fabsf(tz);
  float eDet = k * nE1 * nD * nE2;
  float A = fabsf(det);
  if (A <= eDet) return 2;
  float s = det > 0.f ? 1.f : -1.f;
  float U = s * (tx * px + ty * py + tz * pz);
  float eU = k * nT * nD * nE2;
  if (U < -eU) return 0;
  float qx = ty * e1z - tz * e1y, qy = tz * e1x - tx * e1z, qz = tx * e1y - ty * e1x;
  float V = s * (dx * qx + dy * qy + dz * qz);
  float eV = k * nD * nT * nE1;
  if (V < -eV) return 0;
  float Wm = A - U - V, eWm = eDet + eU + eV;
  if (Wm < -eWm) return 0;
  float W = s * (e2x * qx + e2y * qy + e2z * qz);
  float eW = k * nE2 * nT * nE1;
  float m0 = W - t_lo * A, e0 = eW + t_lo * eDet;
  float m1 = t_hi * A - W, e1 = eW + eDet;
  if (m0 < -e0 || m1 < -e1) return 0;
  if (U > eU && V > eV && Wm > eWm && m0 > e0 && m1 > e1) return 1;
  return 2;
}

// fp64 ray/triangle for the closest-hit free-space test (t > 0, no upper bound).
// Returns t (or a negative value for no hit) and the facing sign of the normal.
__device__ __forceinline__ double ray_tri_t(D3 O, D3 D, double dd, float4 a, float4 b, float4 c,
                                            bool* front) {
  D3 V0 = f2d(a);
  D3 E1 = dsub3(f2d(b), V0), E2 = dsub3(f2d(c), V0);
  D3 P = dcross3(D, E2);
  double det = ddot3(E1, P);
  D3 Nv = dcross3(E1, E2);
  if (det * det <= kParallel * kParallel * dd * ddot3(Nv, Nv)) return -1.0;
  double inv = 1.0 / det;
  D3 T = dsub3(O, V0);
  double u = ddot3(T, P) * inv;
  if (u < -kEdgeTol) return -1.0;
  D3 Q = dcross3(T, E1);
  double v = ddot3(D, Q) * inv;
  if (v < -kEdgeTol || 1.0 - u - v < -kEdgeTol) return -1.0;
  double t = ddot3(E2, Q) * inv;
  *front = ddot3(D, Nv) < 0.0;
  return t > 0.0 ? t : -1.0;
}

// fp64 point/triangle distance (closest point by barycentric region
// classification: vertex, edge or face region).
__device__ __forceinline__ double point_tri_dist(D3 p, float4 fa, float4 fb, float4 fc) {
  D3 a = f2d(fa), b = f2d(fb), c = f2d(fc);
  D3 ab = dsub3(b, a), ac = dsub3(c, a), ap = dsub3(p, a);
  double d1 = ddot3(ab, ap), d2 = ddot3(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return sqrt(ddot3(ap, ap));
  D3 bp = dsub3(p, b);
  double d3_ = ddot3(ab, bp), d4 = ddot3(ac, bp);
  if (d3_ >= 0.0 && d4 <= d3_) return sqrt(ddot3(bp, bp));
  double vc = d1 * d4 - d3_ * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) {
    double v = d1 / (d1 - d3_);
    D3 q = d3(a.x + v * ab.x - p.x, a.y + v * ab.y - p.y, a.z + v * ab.z - p.z);
    return sqrt(ddot3(q, q));
  }
  D3 cp = dsub3(p, c);
  double d5 = ddot3(ab, cp), d6 = ddot3(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return sqrt(ddot3(cp, cp));
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    D3 q = d3(a.x + w * ac.x - p.x, a.y + w * ac.y - p.y, a.z + w * ac.z - p.z);
    return sqrt(ddot3(q, q));
  }
  double va = d3_ * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3_) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3_) / ((d4 - d3_) + (d5 - d6));
    D3 q = d3(b.x + w * (c.x - b.x) - p.x, b.y + w * (c.y - b.y) - p.y, b.z + w * (c.z - b.z) - p.z);
    return sqrt(ddot3(q, q));
  }
  double den = 1.0 / (va + vb + vc);
  double v = vb * den, w = vc * den;
  D3 q = d3(a.x + ab.x * v + ac.x * w - p.x, a.y + ab.y * v + ac.y * w - p.y,
            a.z + ab.z * v + ac.z * w - p.z);
  return sqrt(ddot3(q, q));
}

// squared fp32 distance from point to box (boxes are padded, so this is a
// lower bound of the true distance to the contents up to rounding)
__device__ __forceinline__ float box_dist2(float px, float py, float pz, float lx, float hx, float ly,
                                           float hy, float lz, float hz) {
  float dx = fmaxf(fmaxf(lx - px, px - hx), 0.f);
  float dy = fmaxf(fmaxf(ly - py, py - hy), 0.f);
  float dz = fmaxf(fmaxf(lz - pz, pz - hz), 0.f);
  return dx * dx + dy * dy + dz * dz;
}

}  // namespace uvd
