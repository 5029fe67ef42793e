/* walkstats.c — traversal statistics of the assembly's per-lane BVH walk on
 * sampled work items (a development tool; not the oracle, not the product).
 *
 * Replays k_assemble_lane's walk on the CPU (fp32 slab tests bounded by the
 * segment's t range, near child first, any hit ends the ray, the fp32
 * triangle filter) on the scene's own BVH (dumped by tools/walkstats.py) and
 * reports, per node depth: visits per ray, and for each work item (one lamp,
 * 32 consecutive rows) the UNION of nodes its lanes visit — the work a
 * warp-shared (beam) traversal of that depth range could not avoid.
 *
 * usage: walkstats nodes.bin tri.bin cen.bin nrm.bin lamps.bin items.bin N M nn K root n_items
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct { float a[4], b[4], c[4]; uint32_t d[4]; } Node;
#define MAXD 96
#define STK 256
#ifndef MARCH
#define MARCH 24
#endif
#ifndef RT_CAP
#define RT_CAP 0.1
#endif
#ifndef DEFICIT
#define DEFICIT 0.0
#endif
#ifndef MARCH_EPS
#define MARCH_EPS 0.02
#endif

static void* slurp(const char* path, size_t* n) {
  FILE* f = fopen(path, "rb");
  if (!f) { perror(path); exit(1); }
  fseek(f, 0, SEEK_END);
  *n = (size_t)ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc(*n);
  if (fread(p, 1, *n, f) != *n) { perror("read"); exit(1); }
  fclose(f);
  return p;
}

static int is_leaf(uint32_t r) { return (r & 0x80000000u) != 0; }

/* fp32 filtered segment/triangle test as in traverse.cuh (0 miss, 1 hit, 2 undecided) */
static int tri32(float ox, float oy, float oz, float dx, float dy, float dz, float nD, float tlo, float thi,
                 const float* a, const float* b, const float* c) {
  const float k = 16.0f * 5.9604645e-08f;
  float e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  float e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  float tx = ox - a[0], ty = oy - a[1], tz = oz - a[2];
  float px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
  float det = e1x * px + e1y * py + e1z * pz;
  float nE1 = fabsf(e1x) + fabsf(e1y) + fabsf(e1z), nE2 = fabsf(e2x) + fabsf(e2y) + fabsf(e2z);
  float nT = fabsf(tx) + fabsf(ty) + fabsf(tz);
  float eDet = k * nE1 * nD * nE2, A = fabsf(det);
  if (A <= eDet) return 2;
  float s = det > 0.f ? 1.f : -1.f;
  float U = s * (tx * px + ty * py + tz * pz), eU = k * nT * nD * nE2;
  if (U < -eU) return 0;
  float qx = ty * e1z - tz * e1y, qy = tz * e1x - tx * e1z, qz = tx * e1y - ty * e1x;
  float V = s * (dx * qx + dy * qy + dz * qz), eV = k * nD * nT * nE1;
  if (V < -eV) return 0;
  float Wm = A - U - V, eWm = eDet + eU + eV;
  if (Wm < -eWm) return 0;
  float W = s * (e2x * qx + e2y * qy + e2z * qz), eW = k * nE2 * nT * nE1;
  float m0 = W - tlo * A, e0 = eW + tlo * eDet, m1 = thi * A - W, e1 = eW + eDet;
  if (m0 < -e0 || m1 < -e1) return 0;
  if (U > eU && V > eV && Wm > eWm && m0 > e0 && m1 > e1) return 1;
  return 2;
}

static float sinv(float d) { return fabsf(d) < 1e-30f ? copysignf(1e30f, d) : 1.0f / d; }

/* simple open-addressing set of node ids (per item) */
#define HSZ 65536
static uint32_t hkey[HSZ];
static uint16_t hstamp[HSZ];
static uint16_t cur_stamp = 0;
static int hset_add(uint32_t k) {  /* 1 if new */
  uint32_t h = (k * 2654435761u) & (HSZ - 1);
  while (hstamp[h] == cur_stamp) {
    if (hkey[h] == k) return 0;
    h = (h + 1) & (HSZ - 1);
  }
  hstamp[h] = cur_stamp;
  hkey[h] = k;
  return 1;
}



/* ---- free regions at the segment ends (what a shorter t range would save) ---- */
typedef struct { double x, y, z; } V3;
static V3 v3(double x, double y, double z) { V3 r = {x, y, z}; return r; }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V3 vld(const float* p) { return v3(p[0], p[1], p[2]); }
static V3 vmad(V3 a, V3 b, double s) { return v3(a.x + b.x * s, a.y + b.y * s, a.z + b.z * s); }
static double pt_tri(V3 p, V3 a, V3 b, V3 c) {  /* closest-point distance (Voronoi regions) */
  V3 ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
  double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return sqrt(vdot(ap, ap));
  V3 bp = vsub(p, b);
  double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return sqrt(vdot(bp, bp));
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) { V3 q = vsub(p, vmad(a, ab, d1 / (d1 - d3))); return sqrt(vdot(q, q)); }
  V3 cp = vsub(p, c);
  double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return sqrt(vdot(cp, cp));
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) { V3 q = vsub(p, vmad(a, ac, d2 / (d2 - d6))); return sqrt(vdot(q, q)); }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    V3 q = vsub(p, vmad(b, vsub(c, b), (d4 - d3) / ((d4 - d3) + (d5 - d6))));
    return sqrt(vdot(q, q));
  }
  double den = 1.0 / (va + vb + vc);
  V3 q = vsub(p, vmad(vmad(a, ab, vb * den), ac, vc * den));
  return sqrt(vdot(q, q));
}
static double box_d2(V3 p, float lx, float hx, float ly, float hy, float lz, float hz) {
  double dx = fmax(fmax(lx - p.x, p.x - hx), 0), dy = fmax(fmax(ly - p.y, p.y - hy), 0), dz = fmax(fmax(lz - p.z, p.z - hz), 0);
  return dx * dx + dy * dy + dz * dz;
}
/* distance from p to the nearest triangle (other than `own`) that has a vertex
   strictly in front of the plane (n, p) when n != NULL; all triangles otherwise */
static double nearest(const Node* nodes, const float* tri, uint32_t root, V3 p, const float* n, int own) {
  uint32_t stk[STK];
  int sp = 0;
  double best = 1e30;
  uint32_t ref = root;
  for (;;) {
    if (is_leaf(ref)) {
      const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float* tv = tri + 12 * (int64_t)(st + k);
        int o;
        memcpy(&o, tv + 3, 4);
        if (o == own) continue;
        V3 a = vld(tv), b = vld(tv + 4), c = vld(tv + 8);
        if (n) {
          V3 nn = v3(n[0], n[1], n[2]);
          const double e = 1e-6;
          if (vdot(vsub(a, p), nn) <= e && vdot(vsub(b, p), nn) <= e && vdot(vsub(c, p), nn) <= e) continue;
        }
        double d = pt_tri(p, a, b, c);
        if (d < best) best = d;
      }
    } else {
      const Node* nd = nodes + ref;
      double d0 = box_d2(p, nd->a[0], nd->a[1], nd->a[2], nd->a[3], nd->c[0], nd->c[1]);
      double d1 = box_d2(p, nd->b[0], nd->b[1], nd->b[2], nd->b[3], nd->c[2], nd->c[3]);
      uint32_t c0 = nd->d[0], c1 = nd->d[1];
      if (d1 < d0) { double t = d0; d0 = d1; d1 = t; uint32_t u = c0; c0 = c1; c1 = u; }
      if (d1 < best * best) stk[sp++] = c1;
      if (d0 < best * best) { ref = c0; continue; }
    }
    if (!sp) break;
    ref = stk[--sp];
  }
  return best;
}

/* the same walk with the box tests bounded to t in [tmin, thi] (a shorter segment); returns node visits */
static int replay(const Node* nodes, const float* tri, uint32_t root, float ox, float oy, float oz, float dx, float dy,
                  float dz, float tmin, float thi, float tlo, int own, double* ntri) {
  const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz), nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  uint32_t stk[STK];
  int sp = 0, nv = 0;
  uint32_t ref = root;
  for (;;) {
    while (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      ++nv;
      const float* bx[2] = {n->a, n->b};
      float an[2], af[2];
      for (int s = 0; s < 2; ++s) {
        float x0 = (bx[s][0] - ox) * ix, x1 = (bx[s][1] - ox) * ix;
        float y0 = (bx[s][2] - oy) * iy, y1 = (bx[s][3] - oy) * iy;
        float z0 = (n->c[2 * s] - oz) * iz, z1 = (n->c[2 * s + 1] - oz) * iz;
        an[s] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), tmin));
        af[s] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
      }
      const int h0 = an[0] <= af[0], h1 = an[1] <= af[1];
      if (h0 && h1) {
        const int sw = an[1] < an[0];
        ref = sw ? n->d[1] : n->d[0];
        stk[sp++] = sw ? n->d[0] : n->d[1];
      } else if (h0 || h1) {
        ref = h0 ? n->d[0] : n->d[1];
      } else {
        ref = sp ? stk[--sp] : 0xffffffffu;
      }
    }
    if (ref == 0xffffffffu) break;
    const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
    for (uint32_t k = 0; k < cnt; ++k) {
      const float* tv = tri + 12 * (int64_t)(st + k);
      int o;
      memcpy(&o, tv + 3, 4);
      if (o == own) continue;
      *ntri += 1;
      if (tri32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, tv, tv + 4, tv + 8) == 1) return nv;
    }
    ref = sp ? stk[--sp] : 0xffffffffu;
    if (ref == 0xffffffffu) break;
  }
  return nv;
}

/* any-hit walk returning the first certain-hit triangle (leaf order), -1 if none */
static int64_t walk_hit(const Node* nodes, const float* tri, uint32_t root, float ox, float oy, float oz, float dx,
                        float dy, float dz, int own) {
  const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz), nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const float tlo = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz), thi = 1.0f - tlo;
  uint32_t stk[STK];
  int sp = 0;
  uint32_t ref = root;
  for (;;) {
    while (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      const float* bx[2] = {n->a, n->b};
      float an[2], af[2];
      for (int s = 0; s < 2; ++s) {
        float x0 = (bx[s][0] - ox) * ix, x1 = (bx[s][1] - ox) * ix;
        float y0 = (bx[s][2] - oy) * iy, y1 = (bx[s][3] - oy) * iy;
        float z0 = (n->c[2 * s] - oz) * iz, z1 = (n->c[2 * s + 1] - oz) * iz;
        an[s] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.f));
        af[s] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
      }
      const int h0 = an[0] <= af[0], h1 = an[1] <= af[1];
      if (h0 && h1) {
        const int sw = an[1] < an[0];
        ref = sw ? n->d[1] : n->d[0];
        stk[sp++] = sw ? n->d[0] : n->d[1];
      } else if (h0 || h1) {
        ref = h0 ? n->d[0] : n->d[1];
      } else {
        ref = sp ? stk[--sp] : 0xffffffffu;
      }
    }
    if (ref == 0xffffffffu) return -1;
    const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
    for (uint32_t k = 0; k < cnt; ++k) {
      const float* tv = tri + 12 * (int64_t)(st + k);
      int o;
      memcpy(&o, tv + 3, 4);
      if (o == own) continue;
      if (tri32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, tv, tv + 4, tv + 8) == 1) return (int64_t)(st + k);
    }
    ref = sp ? stk[--sp] : 0xffffffffu;
    if (ref == 0xffffffffu) return -1;
  }
}

/* occluder hints: tiles processed for consecutive lamps; each patch remembers
   the last occluder found for it (lag = how many lamps earlier it was found) */
static void hint_sim(const Node* nodes, const float* tri, const float* cen, const float* nrm, const float* lamps,
                     int64_t N, int64_t K, uint32_t root, int n_tiles, int n_cols, int lag) {
  srand(12345);
  double occl = 0, hit_lag = 0, tested = 0, clear_tested = 0;
  for (int t = 0; t < n_tiles; ++t) {
    const int64_t tile = (int64_t)(((double)rand() / RAND_MAX) * ((N + 31) / 32 - 1));
    const int64_t c0 = (int64_t)(((double)rand() / RAND_MAX) * (K - n_cols - 1));
    int64_t hist[64][32];  /* occluder found for lamp c (ring of 64), lane */
    for (int a = 0; a < 64; ++a) for (int l = 0; l < 32; ++l) hist[a][l] = -1;
    for (int64_t c = c0; c < c0 + n_cols; ++c) {
      const float* p = lamps + 3 * c;
      const float ox = p[0], oy = p[1], oz = p[2];
      for (int l = 0; l < 32; ++l) {
        const int64_t r = tile * 32 + l;
        hist[c & 63][l] = -1;
        if (r >= N) continue;
        const float cx = cen[3 * r], cy = cen[3 * r + 1], cz = cen[3 * r + 2];
        const double Dx = (double)cx - ox, Dy = (double)cy - oy, Dz = (double)cz - oz;
        if (!(-(Dx * nrm[3 * r] + Dy * nrm[3 * r + 1] + Dz * nrm[3 * r + 2]) > 0.0)) continue;
        const float dx = cx - ox, dy = cy - oy, dz = cz - oz;
        const int64_t occ = walk_hit(nodes, tri, root, ox, oy, oz, dx, dy, dz, (int)r);
        /* the most recent hint at least `lag` lamps old */
        int64_t h = -1;
        for (int64_t q = c - lag; q >= c0 && q > c - 64; --q)
          if (hist[q & 63][l] >= 0) { h = hist[q & 63][l]; break; }
        if (h >= 0) {
          tested += 1;
          const float* tv = tri + 12 * h;
          const float tlo = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz), thi = 1.0f - tlo;
          const int cls = tri32(ox, oy, oz, dx, dy, dz, fabsf(dx) + fabsf(dy) + fabsf(dz), tlo, thi, tv, tv + 4, tv + 8);
          if (occ >= 0 && cls == 1) hit_lag += 1;
          if (occ < 0) clear_tested += 1;
        }
        if (occ >= 0) occl += 1;
        hist[c & 63][l] = occ;
      }
    }
  }
  printf(" \"hints_lag%d\": {\"occluded_rays\": %.0f, \"hint_hits\": %.0f, \"hint_hit_fraction_of_occluded\": %.4f, \"hint_tests\": %.0f, \"hint_tests_on_clear_rays\": %.0f},\n",
         lag, occl, hit_lag, hit_lag / occl, tested, clear_tested);
}

/* replay with a child ordering policy (for occluded rays the order decides how
   soon a hit ends the walk): 0 near child first, 1 larger subtree first,
   2 larger box surface area first, 3 far child first */
static int replay_order(const Node* nodes, const int* nsub, const float* tri, uint32_t root, float ox, float oy, float oz,
                        float dx, float dy, float dz, int own, int mode, int* hit_out) {
  const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz), nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const float tlo = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz), thi = 1.0f - tlo;
  uint32_t stk[STK];
  int sp = 0, nv = 0;
  uint32_t ref = root;
  *hit_out = 0;
  for (;;) {
    while (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      ++nv;
      const float* bx[2] = {n->a, n->b};
      float an[2], af[2], area[2];
      for (int s = 0; s < 2; ++s) {
        float x0 = (bx[s][0] - ox) * ix, x1 = (bx[s][1] - ox) * ix;
        float y0 = (bx[s][2] - oy) * iy, y1 = (bx[s][3] - oy) * iy;
        float z0 = (n->c[2 * s] - oz) * iz, z1 = (n->c[2 * s + 1] - oz) * iz;
        an[s] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.f));
        af[s] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
        const float ex = bx[s][1] - bx[s][0], ey = bx[s][3] - bx[s][2], ez = n->c[2 * s + 1] - n->c[2 * s];
        area[s] = ex * ey + ey * ez + ez * ex;
      }
      const int h0 = an[0] <= af[0], h1 = an[1] <= af[1];
      if (h0 && h1) {
        int sw;
        if (mode == 0) sw = an[1] < an[0];
        else if (mode == 1) {
          const int s0 = is_leaf(n->d[0]) ? (int)((n->d[0] & 7u) + 1u) : nsub[n->d[0]];
          const int s1 = is_leaf(n->d[1]) ? (int)((n->d[1] & 7u) + 1u) : nsub[n->d[1]];
          sw = s1 > s0;
        } else if (mode == 2) sw = area[1] > area[0];
        else sw = an[1] >= an[0];
        ref = sw ? n->d[1] : n->d[0];
        stk[sp++] = sw ? n->d[0] : n->d[1];
      } else if (h0 || h1) {
        ref = h0 ? n->d[0] : n->d[1];
      } else {
        ref = sp ? stk[--sp] : 0xffffffffu;
      }
    }
    if (ref == 0xffffffffu) break;
    const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
    for (uint32_t k = 0; k < cnt; ++k) {
      const float* tv = tri + 12 * (int64_t)(st + k);
      int o;
      memcpy(&o, tv + 3, 4);
      if (o == own) continue;
      if (tri32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, tv, tv + 4, tv + 8) == 1) { *hit_out = 1; return nv; }
    }
    ref = sp ? stk[--sp] : 0xffffffffu;
    if (ref == 0xffffffffu) break;
  }
  return nv;
}

/* Warp-packet replay of one work item: one DFS for all 32 lanes, each stack
 * entry carrying the mask of lanes whose segment enters that node; a node is
 * visited while some of its lanes are still undecided; at a leaf the lanes in
 * its mask test the triangles (a certain hit retires the lane).  Near child:
 * the one most of the lanes that hit both enter first. */
typedef struct { double node_steps, leaf_steps, tri_steps, lane_tri; } Pk;
static void packet_item(const Node* nodes, const float* tri, const float* cen, const float* nrm, int64_t N,
                        uint32_t root, float ox, float oy, float oz, int64_t tile, Pk* pk) {
  float ix[32], iy[32], iz[32], thi[32], tlo[32], dx[32], dy[32], dz[32], nD[32];
  uint32_t live = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t r = tile * 32 + l;
    if (r >= N) continue;
    const float cx = cen[3 * r], cy = cen[3 * r + 1], cz = cen[3 * r + 2];
    const double Dx = (double)cx - ox, Dy = (double)cy - oy, Dz = (double)cz - oz;
    if (!(-(Dx * nrm[3 * r] + Dy * nrm[3 * r + 1] + Dz * nrm[3 * r + 2]) > 0.0)) continue;
    dx[l] = cx - ox; dy[l] = cy - oy; dz[l] = cz - oz;
    ix[l] = sinv(dx[l]); iy[l] = sinv(dy[l]); iz[l] = sinv(dz[l]);
    tlo[l] = 1e-4f / sqrtf(dx[l] * dx[l] + dy[l] * dy[l] + dz[l] * dz[l]);
    thi[l] = 1.0f - tlo[l];
    nD[l] = fabsf(dx[l]) + fabsf(dy[l]) + fabsf(dz[l]);
    live |= 1u << l;
  }
  if (!live) return;
  uint32_t sref[STK], smask[STK];
  int sp = 0;
  uint32_t ref = root, mask = live, done = 0;
  for (;;) {
    const uint32_t act = mask & ~done;
    if (act) {
      if (!is_leaf(ref)) {
        const Node* n = nodes + ref;
        pk->node_steps += 1;
        uint32_t m0 = 0, m1 = 0, nearer1 = 0;
        for (int l = 0; l < 32; ++l) {
          if (!((act >> l) & 1)) continue;
          const float* bx[2] = {n->a, n->b};
          float an[2], af[2];
          for (int s2 = 0; s2 < 2; ++s2) {
            float x0 = (bx[s2][0] - ox) * ix[l], x1 = (bx[s2][1] - ox) * ix[l];
            float y0 = (bx[s2][2] - oy) * iy[l], y1 = (bx[s2][3] - oy) * iy[l];
            float z0 = (n->c[2 * s2] - oz) * iz[l], z1 = (n->c[2 * s2 + 1] - oz) * iz[l];
            an[s2] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.f));
            af[s2] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi[l]));
          }
          if (an[0] <= af[0]) m0 |= 1u << l;
          if (an[1] <= af[1]) m1 |= 1u << l;
          if (an[0] <= af[0] && an[1] <= af[1] && an[1] < an[0]) nearer1 |= 1u << l;
        }
        if (m0 && m1) {
          const int both = __builtin_popcount(m0 & m1);
          const int sw = 2 * __builtin_popcount(nearer1) > both;
          sref[sp] = sw ? n->d[0] : n->d[1];
          smask[sp++] = sw ? m0 : m1;
          ref = sw ? n->d[1] : n->d[0];
          mask = sw ? m1 : m0;
          continue;
        } else if (m0 || m1) {
          ref = m0 ? n->d[0] : n->d[1];
          mask = m0 ? m0 : m1;
          continue;
        }
      } else {
        pk->leaf_steps += 1;
        const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
        for (uint32_t k = 0; k < cnt; ++k) {
          const float* tv = tri + 12 * (int64_t)(st + k);
          int own;
          memcpy(&own, tv + 3, 4);
          const uint32_t a2 = mask & ~done;
          if (!a2) break;
          pk->tri_steps += 1;
          for (int l = 0; l < 32; ++l) {
            if (!((a2 >> l) & 1)) continue;
            if (own == (int)(tile * 32 + l)) continue;
            pk->lane_tri += 1;
            if (tri32(ox, oy, oz, dx[l], dy[l], dz[l], nD[l], tlo[l], thi[l], tv, tv + 4, tv + 8) == 1)
              done |= 1u << l;
          }
        }
      }
    }
    if (!sp) break;
    ref = sref[--sp];
    mask = smask[sp];
  }
}


/* ---- beam (frustum) replay: one conservative pyramid per work item (apex at
 * the lamp, side planes bounding the 32 target directions, near/far caps from
 * the trimmed segment ends); a DFS of the BVH against it collects candidate
 * leaves; then every lane slab-tests its own segment against the candidate
 * leaf boxes (near first) and tests the triangles of the leaves it enters. */
typedef struct { double items, fallback, fr_nodes, cand_leaves, lane_box, lane_tri, lanes, cand_hist[8]; } Bm;
static double lin_min(const double w[3], double c, const float lo[3], const float hi[3], V3 L) {
  /* min over the box of w·(x − L) − c */
  double m = -c;
  const double l[3] = {lo[0] - L.x, lo[1] - L.y, lo[2] - L.z}, h[3] = {hi[0] - L.x, hi[1] - L.y, hi[2] - L.z};
  for (int k = 0; k < 3; ++k) m += fmin(w[k] * l[k], w[k] * h[k]);
  return m;
}
static void beam_item(const Node* nodes, const float* tri, const float* cen, const float* nrm, int64_t N, uint32_t root,
                      float ox, float oy, float oz, double rL, int64_t tile, Bm* bm) {
  double D[32][3], tmn[32], tmx[32];
  int live[32], nl = 0;
  V3 L = v3(ox, oy, oz);
  double ax[3] = {0, 0, 0};
  for (int l = 0; l < 32; ++l) {
    live[l] = 0;
    const int64_t r = tile * 32 + l;
    if (r >= N) continue;
    const double Dx = (double)cen[3 * r] - ox, Dy = (double)cen[3 * r + 1] - oy, Dz = (double)cen[3 * r + 2] - oz;
    if (!(-(Dx * nrm[3 * r] + Dy * nrm[3 * r + 1] + Dz * nrm[3 * r + 2]) > 0.0)) continue;
    const double len = sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
    const double rT = fmin(nearest(nodes, tri, root, v3(cen[3 * r], cen[3 * r + 1], cen[3 * r + 2]), nrm + 3 * r, (int)r), RT_CAP);
    D[l][0] = Dx; D[l][1] = Dy; D[l][2] = Dz;
    tmn[l] = fmin(rL, 2.0) / len * 0.999;
    tmx[l] = fmin(1.0 - 1e-4 / len, 1.0 - rT / len * 0.999);
    ax[0] += Dx / len; ax[1] += Dy / len; ax[2] += Dz / len;
    live[l] = 1;
    ++nl;
  }
  if (!nl) return;
  bm->items += 1;
  double an = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
  for (int k = 0; k < 3; ++k) ax[k] /= an;
  /* e1, e2 perpendicular to the axis */
  double e1[3], e2[3];
  { double t[3] = {fabs(ax[0]) < 0.9 ? 1.0 : 0.0, fabs(ax[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    double d = t[0] * ax[0] + t[1] * ax[1] + t[2] * ax[2];
    for (int k = 0; k < 3; ++k) e1[k] = t[k] - d * ax[k];
    double n1 = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
    for (int k = 0; k < 3; ++k) e1[k] /= n1;
    e2[0] = ax[1] * e1[2] - ax[2] * e1[1]; e2[1] = ax[2] * e1[0] - ax[0] * e1[2]; e2[2] = ax[0] * e1[1] - ax[1] * e1[0]; }
  double s1lo = 1e300, s1hi = -1e300, s2lo = 1e300, s2hi = -1e300, hlo = 1e300, hhi = -1e300;
  int bad = 0;
  for (int l = 0; l < 32; ++l) {
    if (!live[l]) continue;
    const double h = D[l][0] * ax[0] + D[l][1] * ax[1] + D[l][2] * ax[2];
    if (h <= 1e-3 * sqrt(D[l][0] * D[l][0] + D[l][1] * D[l][1] + D[l][2] * D[l][2])) { bad = 1; break; }
    const double p1 = (D[l][0] * e1[0] + D[l][1] * e1[1] + D[l][2] * e1[2]) / h;
    const double p2 = (D[l][0] * e2[0] + D[l][1] * e2[1] + D[l][2] * e2[2]) / h;
    s1lo = fmin(s1lo, p1); s1hi = fmax(s1hi, p1); s2lo = fmin(s2lo, p2); s2hi = fmax(s2hi, p2);
    hlo = fmin(hlo, h * tmn[l]); hhi = fmax(hhi, h * tmx[l]);
  }
  if (bad || s1hi - s1lo > 4.0 || s2hi - s2lo > 4.0) { bm->fallback += 1; return; }
  bm->lanes += nl;
  const double pad = 1e-4;
  /* half-spaces w·y <= c (y = x − L): p1 − s1hi h <= 0, s1lo h − p1 <= 0, same for 2, h <= hhi, −h <= −hlo */
  double W[6][3], C[6];
  for (int k = 0; k < 3; ++k) {
    W[0][k] = e1[k] - s1hi * ax[k]; W[1][k] = s1lo * ax[k] - e1[k];
    W[2][k] = e2[k] - s2hi * ax[k]; W[3][k] = s2lo * ax[k] - e2[k];
    W[4][k] = ax[k]; W[5][k] = -ax[k];
  }
  for (int q = 0; q < 4; ++q) { double n = sqrt(W[q][0] * W[q][0] + W[q][1] * W[q][1] + W[q][2] * W[q][2]); for (int k = 0; k < 3; ++k) W[q][k] /= n; C[q] = pad; }
  C[4] = hhi + pad; C[5] = -hlo + pad;
  /* DFS */
  uint32_t stk[STK];
  float cl[4096][6];
  uint32_t cr[4096];
  double ch[4096];
  int nc = 0, sp = 0;
  uint32_t ref = root;
  for (;;) {
    if (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      bm->fr_nodes += 1;
      for (int s = 0; s < 2; ++s) {
        const float lo[3] = {s ? n->b[0] : n->a[0], s ? n->b[2] : n->a[2], n->c[2 * s]};
        const float hi[3] = {s ? n->b[1] : n->a[1], s ? n->b[3] : n->a[3], n->c[2 * s + 1]};
        if (lo[0] > hi[0]) continue;
        int out = 0;
        for (int q = 0; q < 6 && !out; ++q) out = lin_min(W[q], C[q], lo, hi, L) > 0;
        if (out) continue;
        const uint32_t c = n->d[s];
        if (is_leaf(c)) {
          if (nc < 4096) {
            for (int k = 0; k < 3; ++k) { cl[nc][2 * k] = lo[k]; cl[nc][2 * k + 1] = hi[k]; }
            cr[nc] = c;
            ch[nc] = ((lo[0] + hi[0]) * 0.5 - ox) * ax[0] + ((lo[1] + hi[1]) * 0.5 - oy) * ax[1] + ((lo[2] + hi[2]) * 0.5 - oz) * ax[2];
            ++nc;
          }
        } else {
          stk[sp++] = c;
        }
      }
    }
    if (!sp) break;
    ref = stk[--sp];
  }
  bm->cand_leaves += nc;
  { int b = nc < 4 ? 0 : nc < 8 ? 1 : nc < 16 ? 2 : nc < 32 ? 3 : nc < 64 ? 4 : nc < 128 ? 5 : nc < 256 ? 6 : 7; bm->cand_hist[b] += 1; }
  /* sort candidates near first (insertion sort) */
  int ord[4096];
  for (int i = 0; i < nc; ++i) ord[i] = i;
  for (int i = 1; i < nc; ++i) { int v = ord[i], j = i - 1; while (j >= 0 && ch[ord[j]] > ch[v]) { ord[j + 1] = ord[j]; --j; } ord[j + 1] = v; }
  for (int l = 0; l < 32; ++l) {
    if (!live[l]) continue;
    const int64_t r = tile * 32 + l;
    const float dx = (float)D[l][0], dy = (float)D[l][1], dz = (float)D[l][2];
    const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz), nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
    const float tlo = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz), thi = (float)tmx[l], tmin = (float)tmn[l];
    for (int q = 0; q < nc; ++q) {
      const float* b = cl[ord[q]];
      bm->lane_box += 1;
      float x0 = (b[0] - ox) * ix, x1 = (b[1] - ox) * ix, y0 = (b[2] - oy) * iy, y1 = (b[3] - oy) * iy;
      float z0 = (b[4] - oz) * iz, z1 = (b[5] - oz) * iz;
      float a0 = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), tmin));
      float a1 = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
      if (a0 > a1) continue;
      const uint32_t c = cr[ord[q]], st = (c & 0x7fffffffu) >> 3, cnt = (c & 7u) + 1u;
      int hit = 0;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float* tv = tri + 12 * (int64_t)(st + k);
        int own;
        memcpy(&own, tv + 3, 4);
        if (own == (int)r) continue;
        bm->lane_tri += 1;
        if (tri32(ox, oy, oz, dx, dy, dz, nD, tlo, 1.0f - tlo, tv, tv + 4, tv + 8) == 1) { hit = 1; break; }
      }
      if (hit) break;
    }
  }
}

/* ---- beam over the TOP of the tree only: the item's pyramid culls the BVH
 * down to depth D (subtree roots at depth D and leaves above it become the
 * item's candidate list, near first); each lane then slab-tests its own
 * segment against the candidate boxes (a shared list: no dependent node
 * fetches) and walks only the subtrees it enters. */
typedef struct { double items, cands, beam_tests, lane_cand_tests, lane_visits, lane_tri, lanes, warp_steps, cur_steps, max_front, levels; } Bm2;
static int walk_sub(const Node* nodes, const float* tri, uint32_t root, float ox, float oy, float oz, float dx, float dy,
                    float dz, float tmin, float thi, float tlo, float thi_tri, int own, double* ntri, int* hit) {
  const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz), nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  uint32_t stk[STK];
  int sp = 0, nv = 0;
  uint32_t ref = root;
  *hit = 0;
  for (;;) {
    while (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      ++nv;
      const float* bx[2] = {n->a, n->b};
      float an[2], af[2];
      for (int s = 0; s < 2; ++s) {
        float x0 = (bx[s][0] - ox) * ix, x1 = (bx[s][1] - ox) * ix;
        float y0 = (bx[s][2] - oy) * iy, y1 = (bx[s][3] - oy) * iy;
        float z0 = (n->c[2 * s] - oz) * iz, z1 = (n->c[2 * s + 1] - oz) * iz;
        an[s] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), tmin));
        af[s] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
      }
      const int h0 = an[0] <= af[0], h1 = an[1] <= af[1];
      if (h0 && h1) {
        const int sw = an[1] < an[0];
        ref = sw ? n->d[1] : n->d[0];
        stk[sp++] = sw ? n->d[0] : n->d[1];
      } else if (h0 || h1) {
        ref = h0 ? n->d[0] : n->d[1];
      } else {
        ref = sp ? stk[--sp] : 0xffffffffu;
      }
    }
    if (ref == 0xffffffffu) break;
    const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
    for (uint32_t k = 0; k < cnt; ++k) {
      const float* tv = tri + 12 * (int64_t)(st + k);
      int o;
      memcpy(&o, tv + 3, 4);
      if (o == own) continue;
      *ntri += 1;
      if (tri32(ox, oy, oz, dx, dy, dz, nD, tlo, thi_tri, tv, tv + 4, tv + 8) == 1) { *hit = 1; return nv; }
    }
    ref = sp ? stk[--sp] : 0xffffffffu;
    if (ref == 0xffffffffu) break;
  }
  return nv;
}

static int g_ia = 0;  /* 1: interval-arithmetic bundle test instead of the pyramid */
static void beam2_item(const Node* nodes, const int* depth, const float* tri, const float* cen, const float* nrm,
                       int64_t N, uint32_t root, float ox, float oy, float oz, double rL, int64_t tile, int D, Bm2* bm) {
  double Dv[32][3], tmn[32], tmx[32];
  int live[32], nl = 0;
  V3 L = v3(ox, oy, oz);
  double ax[3] = {0, 0, 0};
  for (int l = 0; l < 32; ++l) {
    live[l] = 0;
    const int64_t r = tile * 32 + l;
    if (r >= N) continue;
    const double Dx = (double)cen[3 * r] - ox, Dy = (double)cen[3 * r + 1] - oy, Dz = (double)cen[3 * r + 2] - oz;
    if (!(-(Dx * nrm[3 * r] + Dy * nrm[3 * r + 1] + Dz * nrm[3 * r + 2]) > 0.0)) continue;
    const double len = sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
    const double rT = fmin(nearest(nodes, tri, root, v3(cen[3 * r], cen[3 * r + 1], cen[3 * r + 2]), nrm + 3 * r, (int)r), RT_CAP);
    Dv[l][0] = Dx; Dv[l][1] = Dy; Dv[l][2] = Dz;
    tmn[l] = fmin(rL, 2.0) / len * 0.999;
    tmx[l] = fmin(1.0 - 1e-4 / len, 1.0 - rT / len * 0.999);
    ax[0] += Dx / len; ax[1] += Dy / len; ax[2] += Dz / len;
    live[l] = 1;
    ++nl;
  }
  if (!nl) return;
  double an = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
  for (int k = 0; k < 3; ++k) ax[k] /= an;
  double e1[3], e2[3];
  { double t[3] = {fabs(ax[0]) < 0.9 ? 1.0 : 0.0, fabs(ax[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    double d = t[0] * ax[0] + t[1] * ax[1] + t[2] * ax[2];
    for (int k = 0; k < 3; ++k) e1[k] = t[k] - d * ax[k];
    double n1 = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
    for (int k = 0; k < 3; ++k) e1[k] /= n1;
    e2[0] = ax[1] * e1[2] - ax[2] * e1[1]; e2[1] = ax[2] * e1[0] - ax[0] * e1[2]; e2[2] = ax[0] * e1[1] - ax[1] * e1[0]; }
  double s1lo = 1e300, s1hi = -1e300, s2lo = 1e300, s2hi = -1e300, hlo = 1e300, hhi = -1e300;
  int bad = 0;
  for (int l = 0; l < 32; ++l) {
    if (!live[l]) continue;
    const double h = Dv[l][0] * ax[0] + Dv[l][1] * ax[1] + Dv[l][2] * ax[2];
    if (h <= 1e-3 * sqrt(Dv[l][0] * Dv[l][0] + Dv[l][1] * Dv[l][1] + Dv[l][2] * Dv[l][2])) { bad = 1; break; }
    const double p1 = (Dv[l][0] * e1[0] + Dv[l][1] * e1[1] + Dv[l][2] * e1[2]) / h;
    const double p2 = (Dv[l][0] * e2[0] + Dv[l][1] * e2[1] + Dv[l][2] * e2[2]) / h;
    s1lo = fmin(s1lo, p1); s1hi = fmax(s1hi, p1); s2lo = fmin(s2lo, p2); s2hi = fmax(s2hi, p2);
    hlo = fmin(hlo, h * tmn[l]); hhi = fmax(hhi, h * tmx[l]);
  }
  if (bad || s1hi - s1lo > 4.0 || s2hi - s2lo > 4.0) return;
  bm->items += 1;
  bm->lanes += nl;
  float ia_lo[3] = {1e30f, 1e30f, 1e30f}, ia_hi[3] = {-1e30f, -1e30f, -1e30f}, ia_tmin = 1e30f, ia_tmax = -1e30f;
  for (int l = 0; l < 32; ++l) {
    if (!live[l]) continue;
    for (int a = 0; a < 3; ++a) {
      const float iv = sinv((float)Dv[l][a]);
      ia_lo[a] = fminf(ia_lo[a], iv); ia_hi[a] = fmaxf(ia_hi[a], iv);
    }
    ia_tmin = fminf(ia_tmin, (float)tmn[l]); ia_tmax = fmaxf(ia_tmax, (float)tmx[l]);
  }
  const double pad = 1e-4;
  double W[6][3], C[6];
  for (int k = 0; k < 3; ++k) {
    W[0][k] = e1[k] - s1hi * ax[k]; W[1][k] = s1lo * ax[k] - e1[k];
    W[2][k] = e2[k] - s2hi * ax[k]; W[3][k] = s2lo * ax[k] - e2[k];
    W[4][k] = ax[k]; W[5][k] = -ax[k];
  }
  for (int q = 0; q < 4; ++q) { double n = sqrt(W[q][0] * W[q][0] + W[q][1] * W[q][1] + W[q][2] * W[q][2]); for (int k = 0; k < 3; ++k) W[q][k] /= n; C[q] = pad; }
  C[4] = hhi + pad; C[5] = -hlo + pad;
  uint32_t stk[STK];
  static float cl[8192][6];
  static uint32_t cr[8192];
  static double ch[8192];
  int nc = 0, sp = 0;
  uint32_t ref = root;
  for (;;) {
    if (!is_leaf(ref)) {
      const Node* n = nodes + ref;
      bm->beam_tests += 1;
      for (int s = 0; s < 2; ++s) {
        const float lo[3] = {s ? n->b[0] : n->a[0], s ? n->b[2] : n->a[2], n->c[2 * s]};
        const float hi[3] = {s ? n->b[1] : n->a[1], s ? n->b[3] : n->a[3], n->c[2 * s + 1]};
        if (lo[0] > hi[0]) continue;
        int out = 0;
        if (g_ia) {
          /* interval slab test of the bundle: t = (b - L)·i, i in [imin, imax] per axis */
          float ten = ia_tmin, tex = ia_tmax;
          for (int a = 0; a < 3; ++a) {
            const float bl = lo[a] - (a == 0 ? ox : a == 1 ? oy : oz), bh = hi[a] - (a == 0 ? ox : a == 1 ? oy : oz);
            const float i0 = ia_lo[a], i1 = ia_hi[a];
            if (i0 <= 0.f && i1 >= 0.f && !(i0 == 0.f && i1 == 0.f)) {
              /* sign change: unbounded on this axis unless L is outside the slab */
              continue;
            }
            const float p0 = bl * i0, p1 = bl * i1, p2 = bh * i0, p3 = bh * i1;
            const float mn = fminf(fminf(p0, p1), fminf(p2, p3)), mx = fmaxf(fmaxf(p0, p1), fmaxf(p2, p3));
            ten = fmaxf(ten, mn);
            tex = fminf(tex, mx);
          }
          out = ten > tex * 1.00001f + 1e-6f;
        } else {
          for (int q = 0; q < 6 && !out; ++q) out = lin_min(W[q], C[q], lo, hi, L) > 0;
        }
        if (out) continue;
        const uint32_t c = n->d[s];
        if (is_leaf(c) || depth[c] >= D) {
          if (nc < 8192) {
            for (int k = 0; k < 3; ++k) { cl[nc][2 * k] = lo[k]; cl[nc][2 * k + 1] = hi[k]; }
            cr[nc] = c;
            ch[nc] = ((lo[0] - ox) * ax[0] + (lo[1] - oy) * ax[1] + (lo[2] - oz) * ax[2]);  /* near corner along the axis, roughly */
            ++nc;
          }
        } else {
          stk[sp++] = c;
        }
      }
    }
    if (!sp) break;
    ref = stk[--sp];
  }
  bm->cands += nc;
  int ord[8192];
  for (int i = 0; i < nc; ++i) ord[i] = i;
  for (int i = 1; i < nc; ++i) { int v = ord[i], j = i - 1; while (j >= 0 && ch[ord[j]] > ch[v]) { ord[j + 1] = ord[j]; --j; } ord[j + 1] = v; }
  int done[32] = {0};
  float lix[32], liy[32], liz[32], ltlo[32], lthi[32], ltmin[32];
  for (int l = 0; l < 32; ++l) {
    if (!live[l]) continue;
    const float dx = (float)Dv[l][0], dy = (float)Dv[l][1], dz = (float)Dv[l][2];
    lix[l] = sinv(dx); liy[l] = sinv(dy); liz[l] = sinv(dz);
    ltlo[l] = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz); lthi[l] = (float)tmx[l]; ltmin[l] = (float)tmn[l];
  }
  /* current design's warp cost for this item: max over lanes of the full walk's visits (free regions) */
  { int mx = 0;
    for (int l = 0; l < 32; ++l) {
      if (!live[l]) continue;
      double nt = 0;
      const int v = replay(nodes, tri, root, ox, oy, oz, (float)Dv[l][0], (float)Dv[l][1], (float)Dv[l][2], ltmin[l], lthi[l], ltlo[l], (int)(tile * 32 + l), &nt);
      if (v > mx) mx = v;
    }
    bm->cur_steps += mx; }
  double wsteps = D;  /* BFS levels */
  for (int q = 0; q < nc; ++q) {
    int mx = 0, any = 0;
    for (int l = 0; l < 32; ++l) {
      if (!live[l] || done[l]) continue;
      any = 1;
      const int64_t r = tile * 32 + l;
      const float dx = (float)Dv[l][0], dy = (float)Dv[l][1], dz = (float)Dv[l][2];
      const float* b = cl[ord[q]];
      bm->lane_cand_tests += 1;
      float x0 = (b[0] - ox) * lix[l], x1 = (b[1] - ox) * lix[l], y0 = (b[2] - oy) * liy[l], y1 = (b[3] - oy) * liy[l];
      float z0 = (b[4] - oz) * liz[l], z1 = (b[5] - oz) * liz[l];
      float a0 = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), ltmin[l]));
      float a1 = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), lthi[l]));
      if (a0 > a1) continue;
      int hit = 0;
      const int v = walk_sub(nodes, tri, cr[ord[q]], ox, oy, oz, dx, dy, dz, ltmin[l], lthi[l], ltlo[l], 1.0f - ltlo[l], (int)r,
                             &bm->lane_tri, &hit);
      bm->lane_visits += v;
      if (v > mx) mx = v;
      if (hit) done[l] = 1;
    }
    if (!any) break;
    wsteps += 1 + mx;
  }
  bm->warp_steps += wsteps;
}

int main(int argc, char** argv) {
  if (argc < 13) { fprintf(stderr, "usage\n"); return 1; }
  size_t sz;
  const Node* nodes = (const Node*)slurp(argv[1], &sz);
  const float* tri = (const float*)slurp(argv[2], &sz);
  const float* cen = (const float*)slurp(argv[3], &sz);
  const float* nrm = (const float*)slurp(argv[4], &sz);
  const float* lamps = (const float*)slurp(argv[5], &sz);
  const int64_t* items = (const int64_t*)slurp(argv[6], &sz);
  const int64_t N = atoll(argv[7]), nn = atoll(argv[9]);
  const uint32_t root = (uint32_t)strtoul(argv[11], 0, 10);
  const int64_t n_items = atoll(argv[12]);
  (void)argv[8];
  /* node depths (preorder: parents before children) */
  int* depth = (int*)calloc((size_t)nn, sizeof(int));
  for (int64_t i = 0; i < nn; ++i)
    for (int s = 0; s < 2; ++s)
      if (!is_leaf(nodes[i].d[s])) depth[nodes[i].d[s]] = depth[i] + 1;
  int* nsub = (int*)calloc((size_t)nn, sizeof(int));
  for (int64_t i = nn - 1; i >= 0; --i)
    for (int s2 = 0; s2 < 2; ++s2) {
      const uint32_t c = nodes[i].d[s2];
      nsub[i] += is_leaf(c) ? (int)((c & 7u) + 1u) : nsub[c];
    }
  double ord_v[4][2] = {{0}}, ord_n[2] = {0, 0};
  double uni_d[MAXD] = {0}, lanes_d[MAXD] = {0};
  double rays[2] = {0, 0}, tri_tests[2] = {0, 0}, n_it = 0, und = 0;
  double maxlane_sum = 0, nv_res[2] = {0, 0}, leaf_lane = 0;
  Pk pk = {0, 0, 0, 0};
  Bm bm;
  memset(&bm, 0, sizeof(bm));
  static const int kDs[4] = {6, 9, 12, 15};
  Bm2 bm2[4], bm3[4];
  memset(bm2, 0, sizeof(bm2));
  memset(bm3, 0, sizeof(bm3));
  double nv_free = 0, tri_free = 0, free_t_lo = 0, free_t_hi = 0, march_steps = 0, march_free = 0, march_free_clear = 0, nv_march = 0, tri_march = 0;
  double uni_leaf = 0;
  for (int64_t it = 0; it < n_items; ++it) {
    const int64_t c = items[2 * it], tile = items[2 * it + 1];
    const float* p = lamps + 3 * c;
    const float ox = p[0], oy = p[1], oz = p[2];
    const double rL = nearest(nodes, tri, root, v3(ox, oy, oz), NULL, -1);
    ++cur_stamp;
    if (cur_stamp == 0) { memset(hstamp, 0, sizeof(hstamp)); cur_stamp = 1; }
    double item_vis[MAXD] = {0};
    int any = 0, maxlane = 0;
    packet_item(nodes, tri, cen, nrm, N, root, ox, oy, oz, tile, &pk);
    beam_item(nodes, tri, cen, nrm, N, root, ox, oy, oz, rL, tile, &bm);
    for (int q = 0; q < 4; ++q) beam2_item(nodes, depth, tri, cen, nrm, N, root, ox, oy, oz, rL, tile, kDs[q], &bm2[q]);
    g_ia = 1;
    for (int q = 0; q < 4; ++q) beam2_item(nodes, depth, tri, cen, nrm, N, root, ox, oy, oz, rL, tile, kDs[q], &bm3[q]);
    g_ia = 0;
    for (int lane = 0; lane < 32; ++lane) {
      const int64_t r = tile * 32 + lane;
      if (r >= N) continue;
      const float cx = cen[3 * r], cy = cen[3 * r + 1], cz = cen[3 * r + 2];
      const double Dx = (double)cx - ox, Dy = (double)cy - oy, Dz = (double)cz - oz;
      const double cosd = -(Dx * nrm[3 * r] + Dy * nrm[3 * r + 1] + Dz * nrm[3 * r + 2]);
      if (!(cosd > 0.0)) continue;
      any = 1;
      const float dx = cx - ox, dy = cy - oy, dz = cz - oz;
      const float ix = sinv(dx), iy = sinv(dy), iz = sinv(dz);
      const float tlo = 1e-4f / sqrtf(dx * dx + dy * dy + dz * dz), thi = 1.0f - tlo;
      /* free regions: no triangle within rL of the lamp; none strictly in front of the target within rT */
      {
        const double len = sqrt((double)dx * dx + (double)dy * dy + (double)dz * dz);
        const double rT = nearest(nodes, tri, root, v3(cx, cy, cz), nrm + 3 * r, (int)r);
        free_t_lo += fmin(rL / len, 0.5);
        free_t_hi += fmin(rT / len, 0.5);
        const float tmin2 = (float)fmax(0.0, rL / len * 0.999), thi2 = (float)fmin(thi, 1.0 - rT / len * 0.999);
        nv_free += replay(nodes, tri, root, ox, oy, oz, dx, dy, dz, tmin2, thi2, tlo, (int)r, &tri_free);
      }
      const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
      uint32_t stk[STK];
      int sp = 0, res = 0, undec = 0, nv = 0, ntri = 0;
      uint32_t ref = root;
      for (;;) {
        while (!is_leaf(ref)) {
          const Node* n = nodes + ref;
          const int dep = depth[ref] < MAXD ? depth[ref] : MAXD - 1;
          item_vis[dep] += 1;
          if (hset_add(ref)) uni_d[dep] += 1;
          ++nv;
          const float* bx[2] = {n->a, n->b};
          float an[2], af[2];
          for (int s = 0; s < 2; ++s) {
            float x0 = (bx[s][0] - ox) * ix, x1 = (bx[s][1] - ox) * ix;
            float y0 = (bx[s][2] - oy) * iy, y1 = (bx[s][3] - oy) * iy;
            float z0 = (n->c[2 * s] - oz) * iz, z1 = (n->c[2 * s + 1] - oz) * iz;
            an[s] = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.f));
            af[s] = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), thi));
          }
          const int h0 = an[0] <= af[0], h1 = an[1] <= af[1];
          if (h0 && h1) {
            const int sw = an[1] < an[0];
            ref = sw ? n->d[1] : n->d[0];
            stk[sp++] = sw ? n->d[0] : n->d[1];
          } else if (h0 || h1) {
            ref = h0 ? n->d[0] : n->d[1];
          } else {
            ref = sp ? stk[--sp] : 0xffffffffu;
          }
        }
        if (ref == 0xffffffffu) break;
        const uint32_t st = (ref & 0x7fffffffu) >> 3, cnt = (ref & 7u) + 1u;
        int hit = 0;
        leaf_lane += 1;
        if (hset_add(ref)) uni_leaf += 1;
        for (uint32_t k = 0; k < cnt; ++k) {
          const float* tv = tri + 12 * (int64_t)(st + k);
          int own;
          memcpy(&own, tv + 3, 4);
          if (own == (int)r) continue;
          ++ntri;
          const int cls = tri32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, tv, tv + 4, tv + 8);
          if (cls == 1) { hit = 1; break; }
          if (cls == 2) undec = 1;
        }
        if (hit) { res = 1; break; }
        ref = sp ? stk[--sp] : 0xffffffffu;
        if (ref == 0xffffffffu) break;
      }
      rays[res] += 1;
      tri_tests[res] += ntri;
      for (int mo = 0; mo < 4; ++mo) {
        int h = 0;
        ord_v[mo][res] += replay_order(nodes, nsub, tri, root, ox, oy, oz, dx, dy, dz, (int)r, mo, &h);
      }
      ord_n[res] += 1;
      /* sphere tracing from the lamp with exact distances (upper bound of a distance-field march) */
      {
        const double len = sqrt((double)dx * dx + (double)dy * dy + (double)dz * dz);
        const double rT2 = nearest(nodes, tri, root, v3(cx, cy, cz), nrm + 3 * r, (int)r);
        double t = rL / len * 0.999;
        const double tend = fmin((double)thi, 1.0 - fmin(rT2, RT_CAP) / len * 0.999);
        int k = 0;
        for (; k < MARCH && t < tend; ++k) {
          const V3 x = v3(ox + t * dx, oy + t * dy, oz + t * dz);
          const double dist = nearest(nodes, tri, root, x, NULL, -1) - DEFICIT;
          if (dist < MARCH_EPS) break;
          t += (dist - 1e-5) / len;
        }
        march_steps += k;
        if (t >= tend) march_free += 1;
        if (t >= tend && res == 0) march_free_clear += 1;
        const float tm = (float)fmin(t, tend);
        const float thi3 = (float)tend;
        nv_march += t >= tend ? 0 : replay(nodes, tri, root, ox, oy, oz, dx, dy, dz, tm, thi3, tlo, (int)r, &tri_march);
      }
      nv_res[res] += nv;
      und += undec;
      if (nv > maxlane) maxlane = nv;
    }
    if (any) {
      n_it += 1;
      maxlane_sum += maxlane;
      for (int d = 0; d < MAXD; ++d) lanes_d[d] += item_vis[d];
    }
  }
  const double R = rays[0] + rays[1];
  printf("{\"items\": %.0f, \"rays\": %.0f, \"occluded_fraction\": %.5f, \"undecided_fraction\": %.6f,\n", n_it, R,
         rays[1] / R, und / R);
  printf(" \"tri_tests_per_ray\": %.3f, \"max_lane_visits_per_item\": %.3f,\n", (tri_tests[0] + tri_tests[1]) / R,
         maxlane_sum / n_it);
  double tot = 0, totu = 0;
  for (int d = 0; d < MAXD; ++d) { tot += lanes_d[d]; totu += uni_d[d]; }
  printf(" \"visits_per_ray\": %.3f, \"visits_per_clear_ray\": %.3f, \"visits_per_occluded_ray\": %.3f, \"union_visits_per_item\": %.3f,\n",
         tot / R, nv_res[0] / rays[0], nv_res[1] / rays[1], totu / n_it);
  printf(" \"leaf_visits_per_ray\": %.3f, \"union_leaves_per_item\": %.3f,\n", leaf_lane / R, uni_leaf / n_it);
  printf(" \"packet\": {\"node_steps_per_item\": %.3f, \"leaf_steps_per_item\": %.3f, \"tri_steps_per_item\": %.3f, \"lane_tri_tests_per_ray\": %.3f},\n",
         pk.node_steps / n_it, pk.leaf_steps / n_it, pk.tri_steps / n_it, pk.lane_tri / R);
  printf(" \"lanes_per_item\": %.3f,\n", R / n_it);
  for (int q = 0; q < 4; ++q)
    printf(" \"beam_top_D%d\": {\"items\": %.0f, \"cands_per_item\": %.2f, \"beam_node_tests_per_item\": %.2f, \"lane_cand_tests_per_ray\": %.2f, \"lane_visits_per_ray\": %.2f, \"lane_tri_per_ray\": %.3f, \"warp_steps_per_item\": %.2f, \"current_max_lane_visits_per_item\": %.2f},\n",
           kDs[q], bm2[q].items, bm2[q].cands / bm2[q].items, bm2[q].beam_tests / bm2[q].items, bm2[q].lane_cand_tests / bm2[q].lanes,
           bm2[q].lane_visits / bm2[q].lanes, bm2[q].lane_tri / bm2[q].lanes, bm2[q].warp_steps / bm2[q].items, bm2[q].cur_steps / bm2[q].items);
  for (int q = 0; q < 4; ++q)
    printf(" \"beam_ia_D%d\": {\"items\": %.0f, \"cands_per_item\": %.2f, \"beam_node_tests_per_item\": %.2f, \"lane_cand_tests_per_ray\": %.2f, \"lane_visits_per_ray\": %.2f, \"lane_tri_per_ray\": %.3f, \"warp_steps_per_item\": %.2f, \"current_max_lane_visits_per_item\": %.2f},\n",
           kDs[q], bm3[q].items, bm3[q].cands / bm3[q].items, bm3[q].beam_tests / bm3[q].items, bm3[q].lane_cand_tests / bm3[q].lanes,
           bm3[q].lane_visits / bm3[q].lanes, bm3[q].lane_tri / bm3[q].lanes, bm3[q].warp_steps / bm3[q].items, bm3[q].cur_steps / bm3[q].items);
  printf(" \"beam\": {\"items\": %.0f, \"fallback_items\": %.0f, \"frustum_nodes_per_item\": %.2f, \"cand_leaves_per_item\": %.2f, \"lane_leaf_box_tests_per_ray\": %.2f, \"lane_tri_tests_per_ray\": %.3f, \"cand_hist_lt4_8_16_32_64_128_256_more\": [%.0f, %.0f, %.0f, %.0f, %.0f, %.0f, %.0f, %.0f]},\n",
         bm.items, bm.fallback, bm.fr_nodes / (bm.items - bm.fallback), bm.cand_leaves / (bm.items - bm.fallback),
         bm.lane_box / bm.lanes, bm.lane_tri / bm.lanes, bm.cand_hist[0], bm.cand_hist[1], bm.cand_hist[2], bm.cand_hist[3],
         bm.cand_hist[4], bm.cand_hist[5], bm.cand_hist[6], bm.cand_hist[7]);
  printf(" \"order_visits\": {\"near_first\": [%.2f, %.2f], \"larger_subtree\": [%.2f, %.2f], \"larger_area\": [%.2f, %.2f], \"far_first\": [%.2f, %.2f]},\n",
         ord_v[0][0] / ord_n[0], ord_v[0][1] / ord_n[1], ord_v[1][0] / ord_n[0], ord_v[1][1] / ord_n[1],
         ord_v[2][0] / ord_n[0], ord_v[2][1] / ord_n[1], ord_v[3][0] / ord_n[0], ord_v[3][1] / ord_n[1]);
  printf(" \"march\": {\"max_steps\": %d, \"eps\": %.3f, \"steps_per_ray\": %.3f, \"fully_free_rays\": %.4f, \"fully_free_of_clear\": %.4f, \"visits_per_ray_after\": %.3f, \"tri_per_ray_after\": %.3f},\n",
         MARCH, MARCH_EPS, march_steps / R, march_free / R, march_free_clear / rays[0], nv_march / R, tri_march / R);
  {
    const int64_t K = atoll(argv[10]);
    hint_sim(nodes, tri, cen, nrm, lamps, N, K, root, 300, 48, 1);
    hint_sim(nodes, tri, cen, nrm, lamps, N, K, root, 300, 48, 9);
  }
  printf(" \"free_regions\": {\"visits_per_ray\": %.3f, \"tri_tests_per_ray\": %.3f, \"mean_t_cut_lamp\": %.4f, \"mean_t_cut_target\": %.4f},\n",
         nv_free / R, tri_free / R, free_t_lo / R, free_t_hi / R);
  printf(" \"by_depth\": [");
  for (int d = 0, first = 1; d < MAXD; ++d) {
    if (lanes_d[d] == 0) continue;
    printf("%s[%d, %.4f, %.4f]", first ? "" : ", ", d, lanes_d[d] / R, uni_d[d] / n_it);
    first = 0;
  }
  printf("]}\n");
  return 0;
}
