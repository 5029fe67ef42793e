/*
 * uvd_oracle.c — plain, slow, obviously correct fp64 CPU oracle for the
 * irradiance-matrix hot path of arXiv 2103.14137 ("Optimized Coverage Planning
 * for UV Surface Disinfection").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2103_14137_b200/csrc/ and never includes include/uvd.h.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, Q# = readings
 * listed in DESIGN.md §Readings.
 *
 * What it computes (SURVEY §8(a) rows a1, a3, a4–a6; a7/a8 are in oracle.py):
 *   a1  canonical patch attributes (2.5D extruded walls; 3D triangles)
 *   a3  vantage feasibility (grid, clearance, free-space test, reach proxy)
 *   a4  front-face cull, a5 occlusion by brute force (every ray against every
 *       triangle), a6 point-source irradiance Eq. 7 summed over lamp samples.
 *   plus an independent 2D floorplan occlusion oracle for extruded worlds
 *   ("visibility graph amongst vantage points and segment midpoints").
 *
 * Arithmetic: IEEE fp64, built with -O2 -ffp-contract=off (no fused
 * multiply-add, no fast-math) so every rounding is the plain one written.
 * Parity pins: see tests/test_oracle_*.py (closed forms, symmetry, hand-built
 * occlusion, 2D-vs-3D agreement, brute force on tiny scenes).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORC_EPS_SELF 1e-4   /* Q6: ignore occluders within 0.1 mm of either end */
#define ORC_DEG 1e-6        /* Q8: degenerate band on margins and on cos(theta)  */
#define ORC_PAR 1e-12       /* near-parallel threshold |det| <= 1e-12 |D||E1xE2| */
#define ORC_DMIN 1e-9       /* lamp–surface distance below 1e-9 m is a domain error */

/* ------------------------------------------------------------------------ */
/* small fp64 vector helpers                                                 */
/* ------------------------------------------------------------------------ */
typedef struct { double x, y, z; } v3;
static v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 ld3(const float* p) { return mk((double)p[0], (double)p[1], (double)p[2]); }
static v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double norm(v3 a) { return sqrt(dot(a, a)); }
static double dmin(double a, double b) { return a < b ? a : b; }
static double dmax(double a, double b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------ */
/* thread pool: run f(i, ctx) for i in [0, n) over n_threads workers          */
/* ------------------------------------------------------------------------ */
typedef void (*orc_task)(int64_t i, void* ctx);
typedef struct { orc_task f; void* ctx; int64_t n; int64_t next; pthread_mutex_t mu; } orc_pool;
static void* orc_worker(void* arg) {
  orc_pool* p = (orc_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int64_t i0 = p->next;
    p->next += 16;
    pthread_mutex_unlock(&p->mu);
    if (i0 >= p->n) break;
    int64_t i1 = i0 + 16 < p->n ? i0 + 16 : p->n;
    for (int64_t i = i0; i < i1; ++i) p->f(i, p->ctx);
  }
  return NULL;
}
int orc_default_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}
static void orc_parallel_for(int64_t n, int n_threads, orc_task f, void* ctx) {
  if (n_threads <= 0) n_threads = orc_default_threads();
  if (n_threads > 256) n_threads = 256;
  orc_pool p;
  p.f = f; p.ctx = ctx; p.n = n; p.next = 0;
  pthread_mutex_init(&p.mu, NULL);
  pthread_t th[256];
  for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, orc_worker, &p);
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&p.mu);
}

/* ======================================================================== */
/* a1 — canonical patch attributes                                           */
/* ======================================================================== */

/* 2.5D walls ("each wall is subdivided into fixed-length subsegments";
 * S:71 "walls are split into ceil(len/res) equal-width patches").
 * Wall list = room boundary (bounds traversed CCW: (x0,y0)->(x1,y0)->(x1,y1)->
 * (x0,y1)) then each obstacle polygon's edges v_k -> v_{k+1 mod n} in order.
 * Normals (Q2/Q14): boundary edges point into the room, (-dy, dx)/len;
 * obstacle edges point out of the obstacle, (dy, -dx)/len. */
static int64_t n_walls(int n_poly, const int* poly_n) {
  int64_t n = 4;
  for (int p = 0; p < n_poly; ++p) n += poly_n[p];
  return n;
}
/* wall w -> endpoints (fp32 inputs) and orientation sign (+1 boundary, -1 obstacle) */
static void wall_ends(const float* bounds, const float* poly_xy, const int* poly_n, int n_poly,
                      int64_t w, float e0[2], float e1[2], int* boundary) {
  if (w < 4) {
    float cx[4] = {bounds[0], bounds[2], bounds[2], bounds[0]};
    float cy[4] = {bounds[1], bounds[1], bounds[3], bounds[3]};
    e0[0] = cx[w]; e0[1] = cy[w];
    e1[0] = cx[(w + 1) % 4]; e1[1] = cy[(w + 1) % 4];
    *boundary = 1;
    return;
  }
  int64_t k = w - 4, off = 0;
  for (int p = 0; p < n_poly; ++p) {
    if (k < poly_n[p]) {
      const float* v = poly_xy + 2 * (off + k);
      const float* u = poly_xy + 2 * (off + (k + 1) % poly_n[p]);
      e0[0] = v[0]; e0[1] = v[1]; e1[0] = u[0]; e1[1] = u[1];
      *boundary = 0;
      return;
    }
    k -= poly_n[p];
    off += poly_n[p];
  }
}
static int64_t wall_nseg(const float e0[2], const float e1[2], float res) {
  double dx = (double)e1[0] - (double)e0[0], dy = (double)e1[1] - (double)e0[1];
  double len = sqrt(dx * dx + dy * dy);
  return (int64_t)ceil(len / (double)res);
}

int64_t orc_extruded_count(const float* bounds, const float* poly_xy, const int* poly_n,
                           int n_poly, float res) {
  int64_t N = 0, W = n_walls(n_poly, poly_n);
  for (int64_t w = 0; w < W; ++w) {
    float e0[2], e1[2]; int b;
    wall_ends(bounds, poly_xy, poly_n, n_poly, w, e0, e1, &b);
    N += wall_nseg(e0, e1, res);
  }
  return N;
}

/* Outputs (N = orc_extruded_count):
 *   seg[N*4]      fp32 q_s.xy, q_{s+1}.xy (the 2D floorplan segment of patch i)
 *   centroid[N*3] fp32 ((q_s+q_{s+1})/2, h/2)
 *   normal[N*3]   fp32 horizontal unit normal
 *   area[N]       fp64 |q_{s+1}-q_s| * h
 *   tri[2N*9]     fp32 the patch quad as 2 triangles, wound so (b-a)x(c-a) ~ n
 *   tri_patch[2N] owner patch id of each triangle                              */
void orc_extruded_patches(const float* bounds, float h, const float* poly_xy, const int* poly_n,
                          int n_poly, float res, float* seg, float* centroid, float* normal,
                          double* area, float* tri, int32_t* tri_patch) {
  int64_t W = n_walls(n_poly, poly_n), i = 0;
  for (int64_t w = 0; w < W; ++w) {
    float e0[2], e1[2]; int boundary;
    wall_ends(bounds, poly_xy, poly_n, n_poly, w, e0, e1, &boundary);
    int64_t ns = wall_nseg(e0, e1, res);
    double ex = (double)e1[0] - (double)e0[0], ey = (double)e1[1] - (double)e0[1];
    for (int64_t s = 0; s < ns; ++s, ++i) {
      /* q_s = fl32(e0 + ((e1 - e0) * s) / n_seg) */
      float qa[2], qb[2];
      qa[0] = (float)((double)e0[0] + (ex * (double)s) / (double)ns);
      qa[1] = (float)((double)e0[1] + (ey * (double)s) / (double)ns);
      qb[0] = (float)((double)e0[0] + (ex * (double)(s + 1)) / (double)ns);
      qb[1] = (float)((double)e0[1] + (ey * (double)(s + 1)) / (double)ns);
      if (s + 1 == ns) { qb[0] = e1[0]; qb[1] = e1[1]; }
      seg[4 * i + 0] = qa[0]; seg[4 * i + 1] = qa[1];
      seg[4 * i + 2] = qb[0]; seg[4 * i + 3] = qb[1];
      double dx = (double)qb[0] - (double)qa[0], dy = (double)qb[1] - (double)qa[1];
      double len = sqrt(dx * dx + dy * dy);
      centroid[3 * i + 0] = (float)(((double)qa[0] + (double)qb[0]) / 2.0);
      centroid[3 * i + 1] = (float)(((double)qa[1] + (double)qb[1]) / 2.0);
      centroid[3 * i + 2] = (float)((double)h / 2.0);
      double nx = boundary ? -dy / len : dy / len;
      double ny = boundary ? dx / len : -dx / len;
      normal[3 * i + 0] = (float)nx;
      normal[3 * i + 1] = (float)ny;
      normal[3 * i + 2] = 0.0f;
      area[i] = len * (double)h;
      /* quad corners A=(qa,0) B=(qb,0) C=(qb,h) D=(qa,h); diagonal A–C.
       * (B-A)x(C-A) ~ (dy,-dx,0): obstacle orientation.  Boundary walls use the
       * reversed winding so the right-hand normal points into the room. */
      float A[3] = {qa[0], qa[1], 0.0f}, B[3] = {qb[0], qb[1], 0.0f};
      float C[3] = {qb[0], qb[1], h}, D[3] = {qa[0], qa[1], h};
      const float* t0[3]; const float* t1[3];
      if (!boundary) { t0[0] = A; t0[1] = B; t0[2] = C; t1[0] = A; t1[1] = C; t1[2] = D; }
      else           { t0[0] = A; t0[1] = C; t0[2] = B; t1[0] = A; t1[1] = D; t1[2] = C; }
      for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) {
          tri[(2 * i) * 9 + 3 * c + k] = t0[c][k];
          tri[(2 * i + 1) * 9 + 3 * c + k] = t1[c][k];
        }
      tri_patch[2 * i] = (int32_t)i;
      tri_patch[2 * i + 1] = (int32_t)i;
    }
  }
}

/* 3D: patch = triangle ("simplicial complex with N triangles").
 * centroid = fl32((a+b+c)/3), normal = fl32(cross(b-a, c-a)/|.|) (right-hand,
 * outward by the scene's winding, Q14), area = |cross|/2 (fp64).
 * Returns the index of the first zero-area triangle, or -1. */
int64_t orc_trimesh_patches(const float* V, int64_t nv, const int32_t* F, int64_t nt,
                            float* centroid, float* normal, double* area) {
  (void)nv;
  for (int64_t i = 0; i < nt; ++i) {
    v3 a = ld3(V + 3 * (int64_t)F[3 * i]), b = ld3(V + 3 * (int64_t)F[3 * i + 1]),
       c = ld3(V + 3 * (int64_t)F[3 * i + 2]);
    centroid[3 * i + 0] = (float)(((a.x + b.x) + c.x) / 3.0);
    centroid[3 * i + 1] = (float)(((a.y + b.y) + c.y) / 3.0);
    centroid[3 * i + 2] = (float)(((a.z + b.z) + c.z) / 3.0);
    v3 n = cross(sub(b, a), sub(c, a));
    double len = sqrt(n.x * n.x + n.y * n.y + n.z * n.z);
    if (!(len > 0.0)) return i;
    normal[3 * i + 0] = (float)(n.x / len);
    normal[3 * i + 1] = (float)(n.y / len);
    normal[3 * i + 2] = (float)(n.z / len);
    area[i] = len / 2.0;
  }
  return -1;
}

/* ======================================================================== */
/* a5 — occlusion margins                                                    */
/* ======================================================================== */

/* 2D helpers for the coplanar special case */
static double cross2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }
static int seg_seg_2d_touch(double px, double py, double qx, double qy,
                            double ax, double ay, double bx, double by) {
  /* closed segments pq and ab intersect (including touching / collinear overlap) */
  double d1 = cross2(bx - ax, by - ay, px - ax, py - ay);
  double d2 = cross2(bx - ax, by - ay, qx - ax, qy - ay);
  double d3 = cross2(qx - px, qy - py, ax - px, ay - py);
  double d4 = cross2(qx - px, qy - py, bx - px, by - py);
  if (((d1 > 0 && d2 < 0) || (d1 < 0 && d2 > 0)) && ((d3 > 0 && d4 < 0) || (d3 < 0 && d4 > 0)))
    return 1;
  /* collinear / endpoint cases: bounding-box overlap along the shared line */
  if (d1 == 0 && dmin(ax, bx) <= px && px <= dmax(ax, bx) && dmin(ay, by) <= py && py <= dmax(ay, by)) return 1;
  if (d2 == 0 && dmin(ax, bx) <= qx && qx <= dmax(ax, bx) && dmin(ay, by) <= qy && qy <= dmax(ay, by)) return 1;
  if (d3 == 0 && dmin(px, qx) <= ax && ax <= dmax(px, qx) && dmin(py, qy) <= ay && ay <= dmax(py, qy)) return 1;
  if (d4 == 0 && dmin(px, qx) <= bx && bx <= dmax(px, qx) && dmin(py, qy) <= by && by <= dmax(py, qy)) return 1;
  return 0;
}
static int pt_in_tri_2d(double px, double py, const double* t /* 6 */) {
  double c0 = cross2(t[2] - t[0], t[3] - t[1], px - t[0], py - t[1]);
  double c1 = cross2(t[4] - t[2], t[5] - t[3], px - t[2], py - t[3]);
  double c2 = cross2(t[0] - t[4], t[1] - t[5], px - t[4], py - t[5]);
  return (c0 >= 0 && c1 >= 0 && c2 >= 0) || (c0 <= 0 && c1 <= 0 && c2 <= 0);
}

/* Signed margin of the open segment O + t D, t in (t_lo, t_hi), against the
 * closed triangle (V0,V1,V2), by Möller–Trumbore (1997):
 *   E1 = V1-V0, E2 = V2-V0, P = D x E2, det = E1·P, T = O-V0,
 *   u = T·P/det, Q = T x E1, v = D·Q/det, t = E2·Q/det,
 *   margin = min(u, v, 1-u-v, t - t_lo, t_hi - t).
 * margin >= 0  <=>  the segment meets the triangle (inclusive edges).
 * Near-parallel (|det| <= 1e-12 |D||E1xE2|): -inf, unless the segment lies
 * within 1e-6 m of the triangle's plane and overlaps it, then 0 (degenerate). */
double orc_tri_margin(v3 O, v3 D, double dlen, v3 V0, v3 V1, v3 V2) {
  v3 E1 = sub(V1, V0), E2 = sub(V2, V0);
  v3 P = cross(D, E2);
  double det = dot(E1, P);
  v3 Nrm = cross(E1, E2);
  double nlen = norm(Nrm);
  if (fabs(det) <= ORC_PAR * dlen * nlen) {
    double d0 = dot(sub(O, V0), Nrm) / nlen;
    double d1 = dot(sub(add(O, D), V0), Nrm) / nlen;
    if (fabs(d0) > ORC_DEG || fabs(d1) > ORC_DEG) return -INFINITY;
    /* coplanar: project onto the dominant axis plane and test overlap */
    int ax = 0;
    double m = fabs(Nrm.x);
    if (fabs(Nrm.y) > m) { ax = 1; m = fabs(Nrm.y); }
    if (fabs(Nrm.z) > m) ax = 2;
    double o[3] = {O.x, O.y, O.z}, e[3] = {O.x + D.x, O.y + D.y, O.z + D.z};
    double a[3] = {V0.x, V0.y, V0.z}, b[3] = {V1.x, V1.y, V1.z}, c[3] = {V2.x, V2.y, V2.z};
    int i0 = ax == 0 ? 1 : 0, i1 = ax == 2 ? 1 : 2;
    double t2[6] = {a[i0], a[i1], b[i0], b[i1], c[i0], c[i1]};
    if (pt_in_tri_2d(o[i0], o[i1], t2) || pt_in_tri_2d(e[i0], e[i1], t2)) return 0.0;
    for (int k = 0; k < 3; ++k) {
      int k1 = (k + 1) % 3;
      if (seg_seg_2d_touch(o[i0], o[i1], e[i0], e[i1], t2[2 * k], t2[2 * k + 1], t2[2 * k1],
                           t2[2 * k1 + 1]))
        return 0.0;
    }
    return -INFINITY;
  }
  double inv = 1.0 / det;
  v3 T = sub(O, V0);
  double u = dot(T, P) * inv;
  v3 Q = cross(T, E1);
  double v = dot(D, Q) * inv;
  double t = dot(E2, Q) * inv;
  double t_lo = ORC_EPS_SELF / dlen, t_hi = 1.0 - ORC_EPS_SELF / dlen;
  double s = u;
  s = dmin(s, v);
  s = dmin(s, 1.0 - u - v);
  s = dmin(s, t - t_lo);
  s = dmin(s, t_hi - t);
  return s;
}

/* 2D floorplan margin of the open ray p -> c (parameter t along the ray, the
 * same t as in 3D since the projection is affine) against wall segment a–b
 * (parameter s in [0,1]):  margin = min(s, 1-s, t - t_lo, t_hi - t).
 * Parallel (|cross| <= 1e-12 |d||e|): 0 if collinear within 1e-6 m and
 * overlapping, else -inf.  t_lo/t_hi use the 3D length dlen (Q6). */
static double seg_margin_2d(double px, double py, double dx, double dy, double dlen,
                            double ax, double ay, double bx, double by) {
  double ex = bx - ax, ey = by - ay;
  double den = cross2(dx, dy, ex, ey);
  double dl2 = sqrt(dx * dx + dy * dy), el = sqrt(ex * ex + ey * ey);
  if (fabs(den) <= ORC_PAR * dl2 * el) {
    double off = cross2(ex, ey, px - ax, py - ay) / el;
    if (fabs(off) > ORC_DEG) return -INFINITY;
    return seg_seg_2d_touch(px, py, px + dx, py + dy, ax, ay, bx, by) ? 0.0 : -INFINITY;
  }
  double wx = ax - px, wy = ay - py;
  double t = cross2(wx, wy, ex, ey) / den;
  double s = cross2(wx, wy, dx, dy) / den;
  double t_lo = ORC_EPS_SELF / dlen, t_hi = 1.0 - ORC_EPS_SELF / dlen;
  double m = s;
  m = dmin(m, 1.0 - s);
  m = dmin(m, t - t_lo);
  m = dmin(m, t_hi - t);
  return m;
}

/* ======================================================================== */
/* a4–a6 — irradiance entries for a list of (patch i, column j) pairs        */
/* ======================================================================== */
typedef struct {
  /* geometry */
  const float* tri; const int32_t* tri_patch; int64_t M;   /* 3D occluders */
  const float* seg; int64_t n_seg;                           /* 2D occluders (= patches) */
  const float* centroid; const float* normal; int64_t N;
  const float* lamps; int64_t K; int L; double P;
  const int64_t* pi; const int64_t* pj;
  int mode;           /* 0 = 3D triangles, 1 = 2D floorplan */
  int early_exit;     /* 1: stop scanning once S >= 1e-6 (result provably unchanged) */
  /* outputs */
  double* A; uint8_t* vis; uint8_t* deg; double* S_out; int32_t* err;
} irr_ctx;

static void irr_pair(int64_t q, void* vctx) {
  irr_ctx* c = (irr_ctx*)vctx;
  int64_t i = c->pi[q], j = c->pj[q];
  v3 C = ld3(c->centroid + 3 * i);
  v3 n = ld3(c->normal + 3 * i);
  double acc = 0.0;
  for (int l = 0; l < c->L; ++l) {
    v3 p = ld3(c->lamps + 3 * (j * c->L + l));
    v3 D = sub(C, p);                       /* ray p -> c (exact in fp64)   */
    double d = norm(D);
    int64_t o = q * c->L + l;
    if (d < ORC_DMIN) { c->err[0] = 1; c->vis[o] = 0; c->deg[o] = 1; if (c->S_out) c->S_out[o] = NAN; continue; }
    double cosd = dot(sub(p, C), n);        /* cos(theta) * d, Q2: <x_k - s, n> */
    double cos_t = cosd / d;
    double S = -INFINITY;
    if (cos_t > 0.0) {                      /* visible only if <.,n> > 0 */
      if (c->mode == 0) {
        for (int64_t m = 0; m < c->M; ++m) {
          if (c->tri_patch[m] == (int32_t)i) continue;   /* Q15: own triangles */
          const float* t = c->tri + 9 * m;
          double s = orc_tri_margin(p, D, d, ld3(t), ld3(t + 3), ld3(t + 6));
          if (s > S) S = s;
          if (c->early_exit && S >= ORC_DEG) break;
        }
      } else {
        for (int64_t m = 0; m < c->n_seg; ++m) {
          if (m == i) continue;
          const float* sg = c->seg + 4 * m;
          double s = seg_margin_2d(p.x, p.y, D.x, D.y, d, sg[0], sg[1], sg[2], sg[3]);
          if (s > S) S = s;
          if (c->early_exit && S >= ORC_DEG) break;
        }
      }
    }
    int visible = cos_t > 0.0 && S < 0.0;   /* occluded iff S >= 0 */
    c->vis[o] = (uint8_t)visible;
    c->deg[o] = (uint8_t)((cos_t > 0.0 && fabs(S) < ORC_DEG) || fabs(cos_t) < ORC_DEG);
    if (c->S_out) c->S_out[o] = cos_t > 0.0 ? S : NAN;
    if (visible)                            /* Eq. 7 with the Q1/Q2 reading, power P/L */
      acc += (c->P / (double)c->L) * cosd / (4.0 * M_PI * d * d * d);
  }
  c->A[q] = acc;
}

/* 3D brute force.  Outputs per pair q: A[q]; per (q, l): vis, deg, S (optional).
 * Returns 0, or -2 if some lamp–centroid distance was < 1e-9 m. */
int orc_irradiance_3d(const float* tri, const int32_t* tri_patch, int64_t M,
                      const float* centroid, const float* normal, int64_t N,
                      const float* lamps, int64_t K, int L, double P,
                      const int64_t* pi, const int64_t* pj, int64_t n_pairs,
                      double* A, uint8_t* vis, uint8_t* deg, double* S_out,
                      int early_exit, int n_threads) {
  int32_t err = 0;
  irr_ctx c = {tri, tri_patch, M, NULL, 0, centroid, normal, N, lamps, K, L, P, pi, pj,
               0, early_exit, A, vis, deg, S_out, &err};
  orc_parallel_for(n_pairs, n_threads, irr_pair, &c);
  return err ? -2 : 0;
}

/* 2D floorplan oracle for extruded worlds.  seg[N*4] are the
 * patch segments from orc_extruded_patches (every patch is an occluder except
 * the target itself); lamps must lie strictly between floor and wall top. */
int orc_irradiance_2d(const float* seg, const float* centroid, const float* normal, int64_t N,
                      const float* lamps, int64_t K, int L, double P,
                      const int64_t* pi, const int64_t* pj, int64_t n_pairs,
                      double* A, uint8_t* vis, uint8_t* deg, double* S_out,
                      int early_exit, int n_threads) {
  int32_t err = 0;
  irr_ctx c = {NULL, NULL, 0, seg, N, centroid, normal, N, lamps, K, L, P, pi, pj,
               1, early_exit, A, vis, deg, S_out, &err};
  orc_parallel_for(n_pairs, n_threads, irr_pair, &c);
  return err ? -2 : 0;
}

/* ======================================================================== */
/* a3 — vantage feasibility                                                  */
/* ======================================================================== */

/* Closest point on triangle abc to p (Ericson, "Real-Time Collision
 * Detection", §5.1.5, Voronoi-region method); returns the fp64 distance. */
double orc_point_tri_dist(v3 p, v3 a, v3 b, v3 c) {
  v3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return norm(ap);
  v3 bp = sub(p, b);
  double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return norm(bp);
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = d1 / (d1 - d3);
    return norm(sub(p, add(a, scl(ab, v))));
  }
  v3 cp = sub(p, c);
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return norm(cp);
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    return norm(sub(p, add(a, scl(ac, w))));
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return norm(sub(p, add(b, scl(sub(c, b), w))));
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom, w = vc * denom;
  return norm(sub(p, add(a, add(scl(ab, v), scl(ac, w)))));
}

/* 2D closest distance from point to segment */
static double pt_seg_dist_2d(double px, double py, double ax, double ay, double bx, double by) {
  double ex = bx - ax, ey = by - ay;
  double l2 = ex * ex + ey * ey;
  double t = ((px - ax) * ex + (py - ay) * ey) / l2;
  if (t < 0.0) t = 0.0;
  if (t > 1.0) t = 1.0;
  double qx = ax + t * ex - px, qy = ay + t * ey - py;
  return sqrt(qx * qx + qy * qy);
}

typedef struct {
  const float* tri; int64_t M;
  const float* pts; int64_t n_pts; int n_sub;   /* n_sub points per candidate (Towerbot samples) */
  double clearance;
  int check_free;                               /* free-space test of the first sub-point */
  uint8_t* feasible; uint8_t* ambiguous; double* min_dist;
} v3_ctx;

/* Free-space test (Q20): cast the ray p + t·w, t > 0, with the fixed
 * slightly tilted direction w = (0.0123, 0.0371, 1) (tilted so that axis-aligned
 * tessellations do not put grid-aligned rays exactly on edges), find the
 * nearest triangle hit; p is free iff a hit exists and it is front-facing
 * (direction·normal < 0).  Closed outward-wound solids + an inward shell make
 * this "first hit is a back face <=> inside a solid / outside the room". */
static void free_test(const float* tri, int64_t M, v3 p, int* is_free, int* amb) {
  v3 dir = mk(0.0123, 0.0371, 1.0);
  double wlen = norm(dir);
  double best = INFINITY, second = INFINITY;
  int best_front = 0, second_front = 0;
  double best_margin = 0.0, best_cos = 1.0;
  for (int64_t m = 0; m < M; ++m) {
    const float* t = tri + 9 * m;
    v3 V0 = ld3(t), V1 = ld3(t + 3), V2 = ld3(t + 6);
    v3 E1 = sub(V1, V0), E2 = sub(V2, V0);
    v3 P = cross(dir, E2);
    double det = dot(E1, P);
    v3 Nrm = cross(E1, E2);
    double nlen = norm(Nrm);
    if (fabs(det) <= ORC_PAR * wlen * nlen) continue;   /* parallel to w: no crossing */
    double inv = 1.0 / det;
    v3 T = sub(p, V0);
    double u = dot(T, P) * inv;
    v3 Q = cross(T, E1);
    double v = dot(dir, Q) * inv;
    double tt = dot(E2, Q) * inv;
    double marg = dmin(dmin(u, v), 1.0 - u - v);
    if (marg < -ORC_DEG || tt <= 0.0) continue;
    /* candidates within the degenerate band are kept so ambiguity is reported */
    int front = dot(dir, Nrm) < 0.0;
    if (tt < best) {
      second = best; second_front = best_front;
      best = tt; best_front = front; best_margin = marg; best_cos = dot(dir, Nrm) / (wlen * nlen);
    } else if (tt < second) {
      second = tt; second_front = front;
    }
  }
  *is_free = best < INFINITY && best_front && best_margin >= 0.0;
  *amb = 0;
  if (best < INFINITY && (fabs(best_margin) < ORC_DEG || fabs(best_cos) < ORC_DEG)) *amb = 1;
  if (second < INFINITY && second - best < ORC_DEG && second_front != best_front) *amb = 1;
}

static void v3_point(int64_t q, void* vctx) {
  v3_ctx* c = (v3_ctx*)vctx;
  double dmin_all = INFINITY;
  for (int s = 0; s < c->n_sub; ++s) {
    v3 p = ld3(c->pts + 3 * (q * c->n_sub + s));
    for (int64_t m = 0; m < c->M; ++m) {
      const float* t = c->tri + 9 * m;
      double dd = orc_point_tri_dist(p, ld3(t), ld3(t + 3), ld3(t + 6));
      if (dd < dmin_all) dmin_all = dd;
    }
  }
  int ok = dmin_all >= c->clearance;
  int amb = fabs(dmin_all - c->clearance) < ORC_DEG;
  if (c->check_free) {
    int fr = 0, famb = 0;
    free_test(c->tri, c->M, ld3(c->pts + 3 * (q * c->n_sub)), &fr, &famb);
    ok = ok && fr;
    amb = amb || famb;
  }
  c->feasible[q] = (uint8_t)ok;
  c->ambiguous[q] = (uint8_t)amb;
  if (c->min_dist) c->min_dist[q] = dmin_all;
}

/* Feasibility of candidate points against a triangle scene: every one of the
 * n_sub sub-points of candidate q must be >= clearance from every triangle
 * ("collision-free ... dilated by 5 cm"), and (check_free) the first
 * sub-point must be in free space. */
void orc_vantage_eval_3d(const float* tri, int64_t M, const float* pts, int64_t n_pts, int n_sub,
                         double clearance, int check_free, uint8_t* feasible, uint8_t* ambiguous,
                         double* min_dist, int n_threads) {
  v3_ctx c = {tri, M, pts, n_pts, n_sub, clearance, check_free, feasible, ambiguous, min_dist};
  orc_parallel_for(n_pts, n_threads, v3_point, &c);
}

/* Floorplan feasibility for the planar disc robot in a 2.5D world (P:290,
 * S:299–307): inside the bounds, 2D distance to every wall (boundary and
 * obstacle edges) >= clearance, and outside every obstacle polygon (crossing
 * number along +x; ambiguous if a vertex lies within 1e-6 of the ray's y). */
void orc_vantage_eval_2d(const float* bounds, const float* poly_xy, const int* poly_n, int n_poly,
                         const float* pts, int64_t n_pts, double clearance,
                         uint8_t* feasible, uint8_t* ambiguous) {
  int64_t W = n_walls(n_poly, poly_n);
  for (int64_t q = 0; q < n_pts; ++q) {
    double px = pts[3 * q], py = pts[3 * q + 1];
    double dm = INFINITY;
    for (int64_t w = 0; w < W; ++w) {
      float e0[2], e1[2]; int b;
      wall_ends(bounds, poly_xy, poly_n, n_poly, w, e0, e1, &b);
      double dd = pt_seg_dist_2d(px, py, e0[0], e0[1], e1[0], e1[1]);
      if (dd < dm) dm = dd;
    }
    int inside_room = px > bounds[0] && px < bounds[2] && py > bounds[1] && py < bounds[3];
    int in_obst = 0, amb = fabs(dm - clearance) < ORC_DEG;
    int64_t off = 0;
    for (int p = 0; p < n_poly; ++p) {
      int cross_n = 0;
      for (int k = 0; k < poly_n[p]; ++k) {
        const float* a = poly_xy + 2 * (off + k);
        const float* b = poly_xy + 2 * (off + (k + 1) % poly_n[p]);
        double ay = a[1], by = b[1], ax = a[0], bx = b[0];
        if (fabs(ay - py) < ORC_DEG) amb = 1;
        if ((ay > py) != (by > py)) {
          double xi = ax + (py - ay) * (bx - ax) / (by - ay);
          if (xi > px) cross_n ^= 1;
        }
      }
      if (cross_n) in_obst = 1;
      off += poly_n[p];
    }
    feasible[q] = (uint8_t)(inside_room && dm >= clearance && !in_obst);
    ambiguous[q] = (uint8_t)amb;
  }
}

/* ======================================================================== */
/* NEXT-2 — area-integrated irradiance (Eq. 4 as written)                    */
/* ======================================================================== */
/* Eq. 4 integrates the point-source irradiance over the patch and
 * §IV-C divides the flux by the patch area ("mean irradiance
 * I_i(x_k) = F[i]/|s_i|").  Reading Q23:
 *   A[i,j] = (1/|s_i|) Σ_l (P/L)/(4π) Σ_s vis(p_l → c_s) · Ω(p_l, s)
 * s ranges over the 4^m sub-triangles of each of patch i's triangles (edge
 * midpoints, recursively, fp64); Ω = the solid angle of sub-triangle s seen
 * from p_l (Van Oosterom & Strackee 1983, the closed form behind Mosher 1999);
 * c_s = fl32 of the sub-triangle's centroid is the visibility target (the same
 * open-segment test as a5, own triangles excluded); the front-facing test is the
 * patch's (same as a4).  For an unoccluded patch Σ_s Ω_s = Ω of the patch
 * exactly, so A is then exact; occlusion is resolved at 4^m samples per
 * triangle. */
static double solid_angle(v3 p, v3 a, v3 b, v3 c) {
  v3 r1 = sub(a, p), r2 = sub(b, p), r3 = sub(c, p);
  double l1 = norm(r1), l2 = norm(r2), l3 = norm(r3);
  double num = fabs(dot(r1, cross(r2, r3)));
  double den = l1 * l2 * l3 + dot(r1, r2) * l3 + dot(r1, r3) * l2 + dot(r2, r3) * l1;
  return 2.0 * atan2(num, den);
}

typedef struct {
  const float* tri; const int32_t* tri_patch; int64_t M;   /* 3D occluders */
  const float* seg; int64_t n_seg;                           /* 2D occluders */
  const float* ptri; const int64_t* pfirst; const int32_t* pcount;  /* patch triangles */
  const float* centroid; const float* normal; const double* area;
  const float* lamps; int L; double P; int m;
  const int64_t* pi; const int64_t* pj;
  int mode;
  double* A; uint8_t* deg; int32_t* nvis; int32_t* nsub; int32_t* err;
} area_ctx;

/* max margin of the open segment p -> x against every occluder of patch i */
static double max_margin(const area_ctx* c, int64_t i, v3 p, v3 x) {
  v3 D = sub(x, p);
  double d = norm(D);
  double S = -INFINITY;
  if (c->mode == 0) {
    for (int64_t k = 0; k < c->M; ++k) {
      if (c->tri_patch[k] == (int32_t)i) continue;
      const float* t = c->tri + 9 * k;
      double s = orc_tri_margin(p, D, d, ld3(t), ld3(t + 3), ld3(t + 6));
      if (s > S) S = s;
    }
  } else {
    for (int64_t k = 0; k < c->n_seg; ++k) {
      if (k == i) continue;
      const float* sg = c->seg + 4 * k;
      double s = seg_margin_2d(p.x, p.y, D.x, D.y, d, sg[0], sg[1], sg[2], sg[3]);
      if (s > S) S = s;
    }
  }
  return S;
}

typedef struct { double acc; int nvis, nsub, deg, err; } area_acc;

static void area_sub(const area_ctx* c, int64_t i, v3 p, v3 a, v3 b, v3 cc, int level, area_acc* r) {
  if (level > 0) {
    v3 ab = scl(add(a, b), 0.5), bc = scl(add(b, cc), 0.5), ca = scl(add(cc, a), 0.5);
    area_sub(c, i, p, a, ab, ca, level - 1, r);
    area_sub(c, i, p, ab, b, bc, level - 1, r);
    area_sub(c, i, p, ca, bc, cc, level - 1, r);
    area_sub(c, i, p, ab, bc, ca, level - 1, r);
    return;
  }
  /* visibility target: the sub-triangle centroid rounded to fp32 */
  float xf[3] = {(float)(((a.x + b.x) + cc.x) / 3.0), (float)(((a.y + b.y) + cc.y) / 3.0),
                 (float)(((a.z + b.z) + cc.z) / 3.0)};
  v3 x = ld3(xf);
  r->nsub += 1;
  if (norm(sub(x, p)) < ORC_DMIN) { r->err = 1; return; }
  double S = max_margin(c, i, p, x);
  if (fabs(S) < ORC_DEG) r->deg = 1;
  if (S < 0.0) {
    r->acc += solid_angle(p, a, b, cc);
    r->nvis += 1;
  }
}

static void area_pair(int64_t q, void* vctx) {
  area_ctx* c = (area_ctx*)vctx;
  int64_t i = c->pi[q], j = c->pj[q];
  v3 C = ld3(c->centroid + 3 * i), n = ld3(c->normal + 3 * i);
  double total = 0.0;
  int deg = 0, nvis = 0, nsub = 0;
  for (int l = 0; l < c->L; ++l) {
    v3 p = ld3(c->lamps + 3 * (j * c->L + l));
    v3 D = sub(C, p);
    double d = norm(D);
    if (d < ORC_DMIN) { c->err[0] = 1; deg = 1; continue; }
    double cos_t = dot(sub(p, C), n) / d;
    if (fabs(cos_t) < ORC_DEG) deg = 1;
    if (!(cos_t > 0.0)) continue;           /* the patch faces away */
    area_acc r = {0.0, 0, 0, 0, 0};
    for (int32_t k = 0; k < c->pcount[i]; ++k) {
      const float* t = c->ptri + 9 * (c->pfirst[i] + k);
      area_sub(c, i, p, ld3(t), ld3(t + 3), ld3(t + 6), c->m, &r);
    }
    if (r.err) c->err[0] = 1;
    deg |= r.deg;
    nvis += r.nvis;
    nsub += r.nsub;
    total += (c->P / (double)c->L) / (4.0 * M_PI) * r.acc;
  }
  c->A[q] = total / c->area[i];
  c->deg[q] = (uint8_t)deg;
  c->nvis[q] = nvis;
  c->nsub[q] = nsub;
}

/* mode 0: 3D occluders (tri, tri_patch, M); mode 1: 2D floorplan (seg, n_seg).
 * Patch i's triangles: ptri[9 * (pfirst[i] + k)], k < pcount[i].  Per pair q:
 * A[q], deg[q] (any sub-ray with |margin| < 1e-6 or |cosθ| < 1e-6), nvis[q] /
 * nsub[q] visible / traced sub-rays (all lamp samples).  Returns 0 or -2. */
int orc_irradiance_area(int mode, const float* tri, const int32_t* tri_patch, int64_t M,
                        const float* seg, int64_t n_seg, const float* ptri, const int64_t* pfirst,
                        const int32_t* pcount, const float* centroid, const float* normal,
                        const double* area, const float* lamps, int L, double P, int m,
                        const int64_t* pi, const int64_t* pj, int64_t n_pairs, double* A,
                        uint8_t* deg, int32_t* nvis, int32_t* nsub, int n_threads) {
  int32_t err = 0;
  area_ctx c = {tri, tri_patch, M, seg, n_seg, ptri, pfirst, pcount, centroid, normal, area,
                lamps, L, P, m, pi, pj, mode, A, deg, nvis, nsub, &err};
  orc_parallel_for(n_pairs, n_threads, area_pair, &c);
  return err ? -2 : 0;
}

/* Solid angle of triangle (a, b, c) seen from p (exported for the pins). */
double orc_solid_angle(const double* p, const double* a, const double* b, const double* c) {
  return solid_angle(mk(p[0], p[1], p[2]), mk(a[0], a[1], a[2]), mk(b[0], b[1], b[2]), mk(c[0], c[1], c[2]));
}

/* ======================================================================== */
/* NEXT-3 — the paper's visibility-cube method                   */
/* ======================================================================== */
/* Per lamp sample the scene is "rendered" into 6 cube faces of R×R pixels
 * ("six ... cameras": 512²).  Face f has the ray directions
 *   +X (1,u,v)  −X (−1,u,v)  +Y (u,1,v)  −Y (u,−1,v)  +Z (u,v,1)  −Z (u,v,−1)
 * with pixel (a,b) centre u = −1 + (2a+1)/R, v = −1 + (2b+1)/R.  Each pixel
 * carries the power e = (P/L)·Ω_px/(4π) of its exact solid angle (the paper's
 * precomputed emission texture E):
 *   Ω_px = G(u1,v1) − G(u0,v1) − G(u1,v0) + G(u0,v0),  G(u,v) = atan(uv/√(1+u²+v²)),
 * so each face holds P/(6L).  The pixel's nearest surface (the Z-buffer)
 * is the closest triangle hit by the ray (fp64 Möller–Trumbore, t > 0, inclusive
 * edges, ties to the lower triangle index); its patch receives e when the hit
 * is front-facing, and A[i,j] = F_i/|s_i|.  A pixel is flagged
 * degenerate when the winner's barycentric margin is < 1e-6 or the runner-up
 * hit is within 1e-9·t of it. */
static double px_G(double u, double v) { return atan(u * v / sqrt(1.0 + u * u + v * v)); }

double orc_pixel_solid_angle(int R, int a, int b) {
  double u0 = -1.0 + 2.0 * a / R, u1 = -1.0 + 2.0 * (a + 1) / R;
  double v0 = -1.0 + 2.0 * b / R, v1 = -1.0 + 2.0 * (b + 1) / R;
  return px_G(u1, v1) - px_G(u0, v1) - px_G(u1, v0) + px_G(u0, v0);
}

static v3 px_dir(int f, int R, int a, int b) {
  double u = -1.0 + (2.0 * a + 1.0) / R, v = -1.0 + (2.0 * b + 1.0) / R;
  switch (f) {
    case 0: return mk(1.0, u, v);
    case 1: return mk(-1.0, u, v);
    case 2: return mk(u, 1.0, v);
    case 3: return mk(u, -1.0, v);
    case 4: return mk(u, v, 1.0);
    default: return mk(u, v, -1.0);
  }
}

/* the ray O + t D against triangle V0V1V2: returns t of the plane crossing
 * (or -1 when parallel or t <= 0) with the barycentric margin min(u, v, 1-u-v)
 * (a hit iff margin >= 0) and the facing */
static double ray_hit(v3 O, v3 D, v3 V0, v3 V1, v3 V2, double* margin, int* front) {
  v3 E1 = sub(V1, V0), E2 = sub(V2, V0);
  v3 P = cross(D, E2);
  double det = dot(E1, P);
  v3 Nrm = cross(E1, E2);
  if (fabs(det) <= ORC_PAR * norm(D) * norm(Nrm)) return -1.0;
  double inv = 1.0 / det;
  v3 T = sub(O, V0);
  double u = dot(T, P) * inv;
  v3 Q = cross(T, E1);
  double v = dot(D, Q) * inv;
  double t = dot(E2, Q) * inv;
  if (!(t > 0.0)) return -1.0;
  *margin = dmin(u, dmin(v, 1.0 - u - v));
  *front = dot(D, Nrm) < 0.0;
  return t;
}

typedef struct {
  const float* tri; const int32_t* tri_patch; int64_t M; int64_t N;
  const float* lamps; int L; double P; int R;
  const int64_t* cols; int64_t n_cols;
  double* F;          /* [n_cols][N] flux */
  int32_t* hit;       /* optional [n_cols][L][6][R][R] winning triangle (-1 none, -2 back-facing) */
  uint8_t* deg;       /* optional, same shape */
  double* deg_e;      /* [n_cols] energy on degenerate pixels */
} cube_ctx;

/* one task = one (column, lamp sample, face) */
static void cube_task(int64_t q, void* vctx) {
  cube_ctx* c = (cube_ctx*)vctx;
  int64_t cl = q / (6 * (int64_t)c->L);
  int l = (int)((q / 6) % c->L), f = (int)(q % 6);
  int64_t j = c->cols[cl];
  v3 O = ld3(c->lamps + 3 * (j * c->L + l));
  for (int b = 0; b < c->R; ++b)
    for (int a = 0; a < c->R; ++a) {
      v3 D = px_dir(f, c->R, a, b);
      double best = INFINITY, second = INFINITY, bm = 0.0, near_t = INFINITY;
      int64_t bk = -1;
      int bfront = 0;
      for (int64_t k = 0; k < c->M; ++k) {
        const float* t = c->tri + 9 * k;
        double m; int fr;
        double th = ray_hit(O, D, ld3(t), ld3(t + 3), ld3(t + 6), &m, &fr);
        if (th < 0.0) continue;
        if (m < 0.0) {                      /* a miss; remember misses by less than 1e-6 */
          if (m > -ORC_DEG && th < near_t) near_t = th;
          continue;
        }
        if (th < best) { second = best; best = th; bk = k; bm = m; bfront = fr; }
        else if (th < second) second = th;
      }
      double e = (c->P / c->L) * orc_pixel_solid_angle(c->R, a, b) / (4.0 * M_PI);
      int64_t o = (((cl * c->L + l) * 6 + f) * c->R + b) * (int64_t)c->R + a;
      /* degenerate: the winner within 1e-6 of an edge, a runner-up within
       * 1e-9·t, or a near miss (within 1e-6 of an edge) at or before the winner
       * (e.g. a ray through a shared edge that both triangles miss by rounding) */
      int dg = (bk >= 0 && (bm < ORC_DEG || second - best <= 1e-9 * best)) || (near_t < INFINITY && near_t <= best * (1.0 + 1e-9));
      if (c->hit) c->hit[o] = bk < 0 ? -1 : (bfront ? (int32_t)bk : -2);
      if (c->deg) c->deg[o] = (uint8_t)dg;
      if (bk >= 0 && bfront) {
        int64_t i = c->tri_patch[bk];
        /* faces of one column run as concurrent tasks: atomic fp64 add */
        double* dst = c->F + cl * c->N + i;
        double old = *dst, nw;
        do { nw = old + e; } while (!__atomic_compare_exchange(dst, &old, &nw, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED));
        if (dg) {
          double* de = c->deg_e + cl;
          double o2 = *de, n2;
          do { n2 = o2 + e; } while (!__atomic_compare_exchange(de, &o2, &n2, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED));
        }
      }
    }
}

/* F[n_cols][N] (zeroed by the caller) gets the flux of every column; hit/deg
 * optional per-pixel outputs.  Summation order across faces is not fixed
 * (parallel tasks): F is exact up to fp64 rounding order. */
void orc_cubemap(const float* tri, const int32_t* tri_patch, int64_t M, int64_t N, const float* lamps, int L,
                 double P, int R, const int64_t* cols, int64_t n_cols, double* F, int32_t* hit, uint8_t* deg,
                 double* deg_e, int n_threads) {
  cube_ctx c = {tri, tri_patch, M, N, lamps, L, P, R, cols, n_cols, F, hit, deg, deg_e};
  orc_parallel_for(n_cols * L * 6, n_threads, cube_task, &c);
}
