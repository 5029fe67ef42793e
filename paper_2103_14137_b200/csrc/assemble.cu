// assemble.cu — irradiance-matrix assembly (SURVEY §8(a) rows a4–a6, the
// dominant kernel): for every local column c (configuration j = cols[c]) and
// every patch i,
//   A[i,j] = Σ_l vis_ijl (P/L) <p_jl - c_i, n_i> / (4π |p_jl - c_i|³)
// (Eq. 7, P:234–242 with the Q1/Q2 reading; P:252 for L samples; P:248 mean
// irradiance units), vis = front-facing and no other scene triangle on the open
// segment p_jl -> c_i (Q5–Q8, Q15).
//
// k_assemble: persistent warps; a work item is (column, 32-patch tile).  The
// 32 lanes hold 32 consecutive patches (spatially coherent: 3D rows are in
// Morton order), all rays share the lamp origin, and the warp walks ONE shared
// stack through the BVH: every node is fetched once for the warp (broadcast)
// and tested by all active lanes, children are descended when any lane hits
// (ballot).  Occluded lanes drop out (any-hit); the walk ends when no lane is
// left.  The column tile is written with one coalesced 128-B store per warp,
// plus the ballot word of the visibility mask.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

constexpr int kAsmWarps = 8;
constexpr int kAsmThreads = kAsmWarps * 32;
#ifndef UVD_ASM_MINB
#define UVD_ASM_MINB 4
#endif
constexpr int kAsmMinBlocks = UVD_ASM_MINB;  // <= 85 registers: 24 warps per SM to hide node-fetch latency

struct AsmParams {
  const float4* __restrict__ tri;
  const Node4* __restrict__ nodes4;
  const Node* __restrict__ nodes;  // BVH2 (per-lane traversal)
  uint32_t root;
  const float* __restrict__ centroid;
  const float* __restrict__ normal;
  int64_t N;
  const float* __restrict__ lamps;
  int L;
  double scale;  // P / (4π L)
  const int64_t* __restrict__ cols;  // device, nullptr = identity
  int64_t n_cols;
  int64_t tiles;  // ld / 32 (dense) or ceil(N/32)
  int64_t words;  // ceil(N/32)
  float* __restrict__ values;  // dense [n_cols][ld] or nullptr
  int64_t ld;
  uint32_t* __restrict__ vis_bits;  // [n_cols][L][words] or nullptr
  double* __restrict__ col_sumsq;
  unsigned long long* __restrict__ counters;  // [6] or nullptr (instrumented kernel)
  uint32_t* __restrict__ pending;  // [n_cols][words] entries left undecided in fp32
  int* __restrict__ err;
};

// rare path (fp32 filter ambiguous): exact fp64 re-test of segment p -> c from
// the fp32 inputs.  Kept out of line so its fp64 registers do not count
// against the traversal loop's occupancy.
__device__ __forceinline__ int exact_retest(float px, float py, float pz, float cx, float cy, float cz,
                                         float4 a, float4 b, float4 c) {
  D3 O = d3(px, py, pz);
  D3 D = d3((double)cx - O.x, (double)cy - O.y, (double)cz - O.z);
  double dd = ddot3(D, D);
  double t_lo = kSelfEps / sqrt(dd);
  return seg_hits_tri(O, D, dd, t_lo, 1.0 - t_lo, a, b, c) ? 1 : 0;
}

// Per-warp shared state of the pair-parallel walk.
constexpr int kAmbCap = 32 + 4 * 32;  // deferred fp64 re-tests per warp: < 32 pending + one leaf (<= 4 rounds x 32)
struct WarpSmem {
  uint2 stack[kStackDepth];  // (node ref, ray mask)
  uint32_t list[32];         // compaction: k-th ray of the current mask -> lane
  float4 ray[32][3];         // per ray: (1/d, -), (d, t_lo), (t_hi, owner, |d|_1, -)
  uint2 amb[kAmbCap];        // (ray lane, triangle index) pairs the fp32 filter left open
};

// Warp-cooperative, pair-parallel any-hit walk over the BVH4.
//
// The 32 rays of a warp share the lamp origin o.  The warp keeps ONE current
// node and a stack of (ref, ray mask) entries; the mask holds the rays whose
// segment entered that node's box.  Work on a node or leaf is spread over
// (ray, child) PAIRS rather than over rays: lane l takes child/triangle l&3 of
// the (q·8 + l>>2)-th ray of the mask (compaction list in shared memory), so a
// node needed by n rays costs ceil(n/8) slab rounds instead of 4 tests per
// lane, and a 4-triangle leaf ceil(n/8) triangle rounds instead of 4.  Per-child
// ray masks are rebuilt with warp OR-reductions; the fullest child is descended
// next, the others pushed; entries whose rays have all been occluded meanwhile
// are dropped unfetched.  Returns the warp's mask of occluded rays.
template <bool COUNT>
__device__ __forceinline__ uint32_t warp_trace_pairs(const AsmParams& P, WarpSmem& W, uint32_t live,
                                                     float ox, float oy, float oz,
                                                     unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const int k = lane & 3;          // child / triangle slot of this lane
  const int sub = lane >> 2;       // ray slot within a round of 8
  uint32_t occ = 0;
  uint32_t ref = P.root, mask = live;
  int sp = 0;
  bool done = false;
  for (;;) {
    int n_amb = 0;
    // ---- walk until done or until >= 32 fp64 re-tests are pending ----
    while (!done && n_amb < 32) {
      // compaction list of the rays in `mask`
      const int n = __popc(mask);
      if ((mask >> lane) & 1u) W.list[__popc(mask & ((1u << lane) - 1u))] = (uint32_t)lane;
      __syncwarp();
      bool pop = false;
      if (!ref_is_leaf(ref)) {
        const Node4* nd = P.nodes4 + ref;
        const float4 lo = __ldg(&nd->c[2 * k]), hi = __ldg(&nd->c[2 * k + 1]);
        const uint32_t cref = __float_as_uint(lo.w);
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
        for (int q = 0; q * 8 < n; ++q) {
          const int s = q * 8 + sub;
          uint32_t val = 0;
          if (s < n && cref != kEmptyRef) {
            const uint32_t r = W.list[s];
            const float4 iv = W.ray[r][0];
            const float tx0 = (lo.x - ox) * iv.x, tx1 = (hi.x - ox) * iv.x;
            const float ty0 = (lo.y - oy) * iv.y, ty1 = (hi.y - oy) * iv.y;
            const float tz0 = (lo.z - oz) * iv.z, tz1 = (hi.z - oz) * iv.z;
            const float tn = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
            const float tf = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), 1.0f));
            if (tn <= tf * 1.000002f + 1e-7f) val = 1u << r;
          }
          m0 |= __reduce_or_sync(0xffffffffu, k == 0 ? val : 0u);
          m1 |= __reduce_or_sync(0xffffffffu, k == 1 ? val : 0u);
          m2 |= __reduce_or_sync(0xffffffffu, k == 2 ? val : 0u);
          m3 |= __reduce_or_sync(0xffffffffu, k == 3 ? val : 0u);
        }
        if (COUNT) {
          cnt[1] += (unsigned long long)n * __popc(__ballot_sync(0xffffffffu, lane < 4 && cref != kEmptyRef));
          cnt[3] += 1;
        }
        const int p0 = __popc(m0), p1 = __popc(m1), p2 = __popc(m2), p3 = __popc(m3);
        int best = 0, pb = p0;
        if (p1 > pb) { best = 1; pb = p1; }
        if (p2 > pb) { best = 2; pb = p2; }
        if (p3 > pb) { best = 3; pb = p3; }
        if (pb == 0) {
          pop = true;
        } else {
          const bool q0 = p0 && best != 0, q1 = p1 && best != 1, q2 = p2 && best != 2, q3 = p3 && best != 3;
          const uint32_t mk = k == 0 ? m0 : k == 1 ? m1 : k == 2 ? m2 : m3;
          const bool mine = lane < 4 && (k == 0 ? q0 : k == 1 ? q1 : k == 2 ? q2 : q3);
          if (mine) {
            const int slot = sp + (k > 0 && q0) + (k > 1 && q1) + (k > 2 && q2);
            W.stack[slot] = make_uint2(cref, mk);
          }
          sp += (int)q0 + (int)q1 + (int)q2 + (int)q3;
          ref = __shfl_sync(0xffffffffu, cref, best);
          mask = best == 0 ? m0 : best == 1 ? m1 : best == 2 ? m2 : m3;
          if (sp > kStackDepth - 4) {  // cannot happen for depth < 40; fail loudly
            if (lane == 0) atomicExch(P.err, 2);
            return occ;
          }
        }
      } else {
        const uint32_t st = ref_start(ref), nt = ref_count(ref);
        const bool have = (uint32_t)k < nt;
        const uint32_t ti = st + (uint32_t)k;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a;
        if (have) {
          const float4* t = P.tri + 3 * (int64_t)ti;
          a = __ldg(t); b = __ldg(t + 1); c = __ldg(t + 2);
        }
        uint32_t hits = 0;
        for (int q = 0; q * 8 < n; ++q) {
          const int s = q * 8 + sub;
          uint32_t val = 0;
          bool test = false, amb = false;
          uint32_t r = 0;
          if (s < n && have) {
            r = W.list[s];
            test = __float_as_int(a.w) != __float_as_int(W.ray[r][2].y);  // not the target's own
          }
          if (COUNT) cnt[2] += __popc(__ballot_sync(0xffffffffu, test));
          if (test) {
            const float4 d = W.ray[r][1], e = W.ray[r][2];
            const int cls = seg_tri_filter32(ox, oy, oz, d.x, d.y, d.z, e.z, d.w, e.x, a, b, c);
            if (cls == 1) val = 1u << r;
            amb = cls == 2;
          }
          hits |= __reduce_or_sync(0xffffffffu, val);
          // defer fp64 re-tests (queue; flushed outside this loop)
          const uint32_t am = __ballot_sync(0xffffffffu, amb);
          if (amb) W.amb[n_amb + __popc(am & ((1u << lane) - 1u))] = make_uint2(r, ti);
          n_amb += __popc(am);
        }
        occ |= hits;
        live &= ~hits;
        pop = true;
      }
      if (pop) {
        for (;;) {
          if (sp == 0 || !live) { done = true; break; }
          const uint2 e = W.stack[--sp];
          ref = e.x;
          mask = e.y & live;
          if (mask) break;
        }
      }
      __syncwarp();
    }
    // ---- exact fp64 re-tests of the pending ambiguous pairs ----
    if (n_amb) {
      __syncwarp();
      uint32_t hits = 0;
      for (int e0 = 0; e0 < n_amb; e0 += 32) {
        uint32_t val = 0;
        const int e = e0 + lane;
        if (e < n_amb) {
          const uint2 q = W.amb[e];
          if ((live >> q.x) & 1u) {
            const int row = __float_as_int(W.ray[q.x][2].y);
            const float4* t = P.tri + 3 * (int64_t)q.y;
            if (exact_retest(ox, oy, oz, P.centroid[3 * row], P.centroid[3 * row + 1],
                             P.centroid[3 * row + 2], __ldg(t), __ldg(t + 1), __ldg(t + 2)))
              val = 1u << q.x;
          }
        }
        hits |= __reduce_or_sync(0xffffffffu, val);
      }
      occ |= hits;
      live &= ~hits;
      __syncwarp();
      if (!live) done = true;
      if (!done && !mask) {  // the current entry lost all its rays: pop
        for (;;) {
          if (sp == 0) { done = true; break; }
          const uint2 e = W.stack[--sp];
          ref = e.x;
          mask = e.y & live;
          if (mask) break;
        }
      }
    }
    if (done) return occ;
    mask &= live;
  }
}

template <bool COUNT>
__global__ void __launch_bounds__(kAsmThreads, kAsmMinBlocks) k_assemble(AsmParams P) {
  __shared__ WarpSmem s_w[kAsmWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};  // warp-uniform tallies (COUNT only)
  const int64_t total = P.n_cols * P.tiles;
  for (int64_t item = (int64_t)blockIdx.x * kAsmWarps + warp; item < total;
       item += (int64_t)gridDim.x * kAsmWarps) {
    const int64_t c = item / P.tiles, tile = item - c * P.tiles;
    const int64_t j = P.cols ? P.cols[c] : c;
    const int64_t r = tile * 32 + lane;
    const bool valid = r < P.N;
    double acc = 0.0;
    for (int l = 0; l < P.L; ++l) {
      const float* pl = P.lamps + 3 * (j * P.L + l);
      // a4: ray p -> c in fp64 (exact differences of fp32 inputs), front-face cull
      bool front = false;
      float ox, oy, oz;
      {
        ox = pl[0]; oy = pl[1]; oz = pl[2];
        float fdx = 0.f, fdy = 0.f, fdz = 0.f, tlo32 = 0.f, thi32 = 0.f;
        if (valid) {
          const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
          const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
          D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
          double dd = ddot3(D, D);
          double d = sqrt(dd);
          double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);  // <p - c, n>
          front = cosd > 0.0;
          if (d < kMinDist) {
            atomicExch(P.err, 1);
            front = false;
          }
          const double t_lo = kSelfEps / d;
          fdx = (float)D.x; fdy = (float)D.y; fdz = (float)D.z;
          tlo32 = (float)t_lo;
          thi32 = (float)(1.0 - t_lo);
        }
        WarpSmem& W = s_w[warp];
        W.ray[lane][0] = make_float4(safe_inv(fdx), safe_inv(fdy), safe_inv(fdz), 0.f);
        W.ray[lane][1] = make_float4(fdx, fdy, fdz, tlo32);
        W.ray[lane][2] = make_float4(thi32, __int_as_float((int)r), fabsf(fdx) + fabsf(fdy) + fabsf(fdz), 0.f);
      }
      uint32_t fm = __ballot_sync(0xffffffffu, front);
      if (COUNT) cnt[0] += __popc(fm);
      uint32_t vm = fm;
      if (fm) {
        // a5: occlusion of the open segment, t in (1e-4/d, 1 - 1e-4/d)
        __syncwarp();
        vm &= ~warp_trace_pairs<COUNT>(P, s_w[warp], fm, ox, oy, oz, cnt);
        __syncwarp();
      }
      if (P.vis_bits && lane == 0 && tile < P.words)
        P.vis_bits[(c * P.L + l) * P.words + tile] = vm;
      if ((vm >> lane) & 1u) {  // a6: Eq. 7 in fp64 (recomputed from the fp32 inputs)
        const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
        const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
        D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
        double dd = ddot3(D, D);
        double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);
        acc += cosd / (dd * sqrt(dd));
      }
    }
    const float a = (float)(acc * P.scale);
    if (P.values) P.values[c * P.ld + r] = a;
  }
  if (COUNT && lane == 0)
    for (int k = 0; k < 4; ++k)
      if (cnt[k]) atomicAdd(P.counters + k, cnt[k]);
}

// ---------------------------------------------------------------------------
// Per-lane traversal (Aila & Laine 2009 "while-while"): every lane walks its
// own shadow ray through the BVH2 with a private stack (local memory, L1
// resident at the top), near child first; triangles are tested with the fp32
// filter and ambiguous cases re-tested exactly in fp64; any hit ends the ray.
// The 32 rays of a warp share the lamp origin and end on 32 Morton-adjacent
// patches, so the lanes fetch mostly the same nodes (L1 broadcast) and
// diverge little.
constexpr int kLaneStack = 64;
constexpr uint32_t kDone = 0xffffffffu;

enum { kClear = 0, kBlocked = 1, kUndecided = 2 };

// One lane's any-hit walk with fp32 decisions only.  Returns kBlocked on a
// certain hit, kClear when every triangle the segment may meet was a certain
// miss, kUndecided when no certain hit was found but the fp32 filter could not
// decide some triangle (the caller flags the entry for exact re-tracing).
template <bool COUNT>
__device__ __forceinline__ int lane_walk32(const AsmParams& P, float ox, float oy, float oz,
                                           float dx, float dy, float dz, int owner,
                                           unsigned long long* cnt) {
  uint32_t stk[kLaneStack];
  int sp = 0;
  bool undecided = false;
  const float ix = safe_inv(dx), iy = safe_inv(dy), iz = safe_inv(dz);
  const float oix = ox * ix, oiy = oy * iy, oiz = oz * iz;
  // the segment's own extent t in (t_lo, t_hi) also bounds the box tests: boxes
  // the segment only enters within 0.1 mm of the target (e.g. the target's own
  // flat leaf and its flat ancestors) are never visited
  const float tlo = (float)kSelfEps * rsqrtf(dx * dx + dy * dy + dz * dz);
  const float thi = 1.0f - tlo;
  uint32_t ref = P.root;
  for (;;) {
    // ---- inner nodes until this lane holds a leaf (or is done) ----
    while (!ref_is_leaf(ref)) {
      const Node* nd = P.nodes + ref;
      const float4 na = __ldg(&nd->a), nb = __ldg(&nd->b), nc = __ldg(&nd->c);
      const uint2 ch = __ldg(reinterpret_cast<const uint2*>(&nd->d));
      if (COUNT) { cnt[1] += 2; cnt[3] += 1; }
      // t = b/d - o/d as one FFMA per plane: fma(b, 1/d, -fl(o/d)) is the exact
      // slab parameter of the plane b shifted by at most eps|o| (<= 1.2e-6 m for
      // |o| <= 20 m), which the build-time box padding (>= 1e-5 m + 4 eps x the
      // scene's largest coordinate) absorbs; the final rounding is covered by
      // the 2e-6 relative widening
      const float ax0 = fmaf(na.x, ix, -oix), ax1 = fmaf(na.y, ix, -oix);
      const float ay0 = fmaf(na.z, iy, -oiy), ay1 = fmaf(na.w, iy, -oiy);
      const float az0 = fmaf(nc.x, iz, -oiz), az1 = fmaf(nc.y, iz, -oiz);
      const float bx0 = fmaf(nb.x, ix, -oix), bx1 = fmaf(nb.y, ix, -oix);
      const float by0 = fmaf(nb.z, iy, -oiy), by1 = fmaf(nb.w, iy, -oiy);
      const float bz0 = fmaf(nc.z, iz, -oiz), bz1 = fmaf(nc.w, iz, -oiz);
      const float an = fmaxf(fmaxf(fminf(ax0, ax1), fminf(ay0, ay1)), fmaxf(fminf(az0, az1), 0.0f));
      const float af = fminf(fminf(fmaxf(ax0, ax1), fmaxf(ay0, ay1)), fminf(fmaxf(az0, az1), thi));
      const float bn = fmaxf(fmaxf(fminf(bx0, bx1), fminf(by0, by1)), fmaxf(fminf(bz0, bz1), 0.0f));
      const float bf = fminf(fminf(fmaxf(bx0, bx1), fmaxf(by0, by1)), fminf(fmaxf(bz0, bz1), thi));
      const bool h0 = an <= fmaf(af, 1.000002f, 1e-7f);
      const bool h1 = bn <= fmaf(bf, 1.000002f, 1e-7f);
      if (h0 && h1) {
        const bool swap = bn < an;  // near child first
        ref = swap ? ch.y : ch.x;
        if (sp < kLaneStack) stk[sp++] = swap ? ch.x : ch.y;
        else atomicExch(P.err, 2);  // cannot happen for depth < 64; fail loudly
      } else if (h0 || h1) {
        ref = h0 ? ch.x : ch.y;
      } else {
        ref = sp ? stk[--sp] : kDone;
      }
    }
    if (ref == kDone) return undecided ? kUndecided : kClear;
    // ---- leaf: up to 4 triangles ----
    const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
    const uint32_t st = ref_start(ref), nt = ref_count(ref);
    for (uint32_t k = 0; k < nt; ++k) {
      const float4* t = P.tri + 3 * (int64_t)(st + k);
      const float4 a = __ldg(t);
      if (__float_as_int(a.w) == owner) continue;  // the target's own triangles
      const float4 b = __ldg(t + 1), c = __ldg(t + 2);
      if (COUNT) cnt[2] += 1;
      const int cls = seg_tri_filter32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, a, b, c);
      if (cls == 1) return kBlocked;
      undecided |= cls == 2;
    }
    ref = sp ? stk[--sp] : kDone;
    if (ref == kDone) return undecided ? kUndecided : kClear;
  }
}

template <bool COUNT>
__global__ void __launch_bounds__(kAsmThreads, kAsmMinBlocks) k_assemble_lane(AsmParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};  // per-lane tallies (COUNT only)
  const int64_t total = P.n_cols * P.tiles;
  for (int64_t item = (int64_t)blockIdx.x * kAsmWarps + warp; item < total;
       item += (int64_t)gridDim.x * kAsmWarps) {
    const int64_t c = item / P.tiles, tile = item - c * P.tiles;
    const int64_t j = P.cols ? P.cols[c] : c;
    const int r = (int)(tile * 32 + lane);
    const bool valid = r < P.N;
    double acc = 0.0;
    bool pend = false;
    for (int l = 0; l < P.L; ++l) {
      const float* pl = P.lamps + 3 * (j * P.L + l);
      const float ox = pl[0], oy = pl[1], oz = pl[2];
      bool vis = false;
      if (valid) {
        const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
        const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
        // a4: ray p -> c in fp64 (exact differences of fp32 inputs), front-face cull
        const D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
        const double dd = ddot3(D, D);
        const double d = sqrt(dd);
        const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);  // <p - c, n>
        bool front = cosd > 0.0;
        if (d < kMinDist) {
          atomicExch(P.err, 1);
          front = false;
        }
        if (front) {
          if (COUNT) cnt[0] += 1;
          // a5: occlusion of the open segment, t in (1e-4/d, 1 - 1e-4/d), fp32 decisions
          const int res = lane_walk32<COUNT>(P, ox, oy, oz, cx - ox, cy - oy, cz - oz, r, cnt);
          vis = res == kClear;
          pend |= res == kUndecided;
          if (vis) acc += cosd / (dd * d);  // a6: Eq. 7 in fp64
        }
      }
      const uint32_t vm = __ballot_sync(0xffffffffu, vis);
      if (P.vis_bits && lane == 0 && tile < P.words) __stcs(P.vis_bits + (c * P.L + l) * P.words + tile, vm);
    }
    // entries with an undecided ray are re-traced exactly by k_fixup
    const uint32_t pm = __ballot_sync(0xffffffffu, pend);
    if (lane == 0 && tile < P.words) __stcs(P.pending + c * P.words + tile, pm);
    if (COUNT) cnt[4] += pend;
    const float a = (float)(acc * P.scale);
    if (P.values) __stcs(P.values + c * P.ld + r, a);  // streaming: keep the BVH in L2
  }
  if (COUNT)
    for (int k = 0; k < 6; ++k) {
      unsigned long long v = cnt[k];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(P.counters + k, v);
    }
}

// ---------------------------------------------------------------------------
// Persistent per-lane traversal with dynamic ray refill (Aila & Laine 2009,
// "replacing terminated rays").  A warp owns a chunk of kChunkRows consecutive
// patches of one column; a lane whose ray ends (certain hit, stack exhausted)
// or whose sample is back-facing immediately takes the next sample / the next
// row of the chunk, so lanes do not idle while the slowest ray of a fixed tile
// finishes.  Visibility and pending bits are OR-ed into the chunk's words,
// which the warp clears first (chunks are word-aligned and owned by one warp).
constexpr int kChunkRows = 256;

template <bool COUNT>
__global__ void __launch_bounds__(kAsmThreads, kAsmMinBlocks) k_assemble_dyn(AsmParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  const int ld = (int)P.ld, N = (int)P.N, words = (int)P.words;
  const int64_t cpc = (P.ld + kChunkRows - 1) / kChunkRows;  // chunks per column
  const int64_t total = P.n_cols * cpc;
  uint32_t stk[kLaneStack];
  for (int64_t item = (int64_t)blockIdx.x * kAsmWarps + warp; item < total;
       item += (int64_t)gridDim.x * kAsmWarps) {
    const int64_t c = item / cpc;
    const int rb0 = (int)(item - c * cpc) * kChunkRows;
    const int rb1 = min(rb0 + kChunkRows, ld);
    const int64_t j = P.cols ? P.cols[c] : c;
    const float* lamp = P.lamps + 3 * j * P.L;
    {  // clear the chunk's bit words
      const int w0 = rb0 >> 5, w1 = min((rb1 + 31) >> 5, words);
      for (int w = w0 + lane; w < w1; w += 32) {
        P.pending[c * words + w] = 0u;
        if (P.vis_bits)
          for (int l = 0; l < P.L; ++l) P.vis_bits[(c * P.L + l) * words + w] = 0u;
      }
      __syncwarp();
    }
    int cursor = rb0;
    bool busy = false, has_row = false, pend = false, und = false;
    int r = 0, l = 0, sp = 0;
    double acc = 0.0;
    float ox = 0.f, oy = 0.f, oz = 0.f, ix = 0.f, iy = 0.f, iz = 0.f, oix = 0.f, oiy = 0.f, oiz = 0.f;
    float dx = 0.f, dy = 0.f, dz = 0.f;
    uint32_t ref = kDone;
    for (;;) {
      // ---- idle lanes: claim rows / start the next front-facing sample ----
      for (;;) {
        const uint32_t want = __ballot_sync(0xffffffffu, !busy && !has_row);
        if (want && cursor < rb1) {
          const int row = cursor + __popc(want & lt);
          if (!busy && !has_row && row < rb1) {
            has_row = true; r = row; l = 0; acc = 0.0; pend = false;
          }
          cursor = min(cursor + __popc(want), rb1);
        }
        if (!busy && has_row) {
          if (l < P.L && r < N) {
            const float* pl = lamp + 3 * l;
            ox = pl[0]; oy = pl[1]; oz = pl[2];
            const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
            const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
            // a4: front-face cull in fp64 (exact differences of fp32 inputs)
            const double Dx = (double)cx - (double)ox, Dy = (double)cy - (double)oy, Dz = (double)cz - (double)oz;
            const double dd = Dx * Dx + Dy * Dy + Dz * Dz;
            const double cosd = -(Dx * (double)nx + Dy * (double)ny + Dz * (double)nz);
            bool front = cosd > 0.0;
            if (sqrt(dd) < kMinDist) { atomicExch(P.err, 1); front = false; }
            if (front) {
              if (COUNT) cnt[0] += 1;
              dx = cx - ox; dy = cy - oy; dz = cz - oz;  // == fl32 of the exact difference
              ix = safe_inv(dx); iy = safe_inv(dy); iz = safe_inv(dz);
              oix = ox * ix; oiy = oy * iy; oiz = oz * iz;
              ref = P.root; sp = 0; und = false;
              busy = true;
            } else {
              ++l;  // back-facing sample: contributes 0, visibility bit stays 0
            }
          } else {  // row finished: store the entry (rows >= N are the zero padding)
            if (P.values) P.values[c * P.ld + r] = (float)(acc * P.scale);
            if (pend) atomicOr(P.pending + c * words + (r >> 5), 1u << (r & 31));
            if (COUNT) cnt[4] += pend;
            has_row = false;
          }
        }
        if (!__ballot_sync(0xffffffffu, !busy && (has_row || cursor < rb1))) break;
      }
      if (!__any_sync(0xffffffffu, busy)) break;  // chunk done
      if (!busy) continue;
      // ---- a5: inner nodes until a leaf, then that leaf ----
      int res = -1;
      while (!ref_is_leaf(ref)) {
        const Node* nd = P.nodes + ref;
        const float4 na = __ldg(&nd->a), nb = __ldg(&nd->b), nc = __ldg(&nd->c);
        const uint2 ch = __ldg(reinterpret_cast<const uint2*>(&nd->d));
        if (COUNT) { cnt[1] += 2; cnt[3] += 1; }
        const float ax0 = fmaf(na.x, ix, -oix), ax1 = fmaf(na.y, ix, -oix);
        const float ay0 = fmaf(na.z, iy, -oiy), ay1 = fmaf(na.w, iy, -oiy);
        const float az0 = fmaf(nc.x, iz, -oiz), az1 = fmaf(nc.y, iz, -oiz);
        const float bx0 = fmaf(nb.x, ix, -oix), bx1 = fmaf(nb.y, ix, -oix);
        const float by0 = fmaf(nb.z, iy, -oiy), by1 = fmaf(nb.w, iy, -oiy);
        const float bz0 = fmaf(nc.z, iz, -oiz), bz1 = fmaf(nc.w, iz, -oiz);
        const float an = fmaxf(fmaxf(fminf(ax0, ax1), fminf(ay0, ay1)), fmaxf(fminf(az0, az1), 0.0f));
        const float af = fminf(fminf(fmaxf(ax0, ax1), fmaxf(ay0, ay1)), fminf(fmaxf(az0, az1), 1.0f));
        const float bn = fmaxf(fmaxf(fminf(bx0, bx1), fminf(by0, by1)), fmaxf(fminf(bz0, bz1), 0.0f));
        const float bf = fminf(fminf(fmaxf(bx0, bx1), fmaxf(by0, by1)), fminf(fmaxf(bz0, bz1), 1.0f));
        const bool h0 = an <= fmaf(af, 1.000002f, 1e-7f);
        const bool h1 = bn <= fmaf(bf, 1.000002f, 1e-7f);
        if (h0 && h1) {
          const bool swap = bn < an;  // near child first
          ref = swap ? ch.y : ch.x;
          if (sp < kLaneStack) stk[sp++] = swap ? ch.x : ch.y;
          else atomicExch(P.err, 2);  // cannot happen for depth < 64; fail loudly
        } else if (h0 || h1) {
          ref = h0 ? ch.x : ch.y;
        } else {
          ref = sp ? stk[--sp] : kDone;
        }
      }
      if (ref == kDone) {
        res = und ? kUndecided : kClear;
      } else {  // leaf: up to 4 triangles (fp32 filter)
        const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
        const float tlo = (float)kSelfEps * rsqrtf(dx * dx + dy * dy + dz * dz);
        const float thi = 1.0f - tlo;
        const uint32_t st = ref_start(ref), nt = ref_count(ref);
        for (uint32_t k = 0; k < nt && res < 0; ++k) {
          const float4* t = P.tri + 3 * (int64_t)(st + k);
          const float4 a = __ldg(t);
          if (__float_as_int(a.w) == r) continue;  // the target's own triangles
          const float4 b = __ldg(t + 1), cc = __ldg(t + 2);
          if (COUNT) cnt[2] += 1;
          const int cls = seg_tri_filter32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, a, b, cc);
          if (cls == 1) res = kBlocked;
          und |= cls == 2;
        }
        if (res < 0) {
          ref = sp ? stk[--sp] : kDone;
          if (ref == kDone) res = und ? kUndecided : kClear;
        }
      }
      if (res >= 0) {  // sample l decided
        if (res == kClear) {  // a6: Eq. 7 in fp64
          const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
          const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
          const double Dx = (double)cx - (double)ox, Dy = (double)cy - (double)oy, Dz = (double)cz - (double)oz;
          const double dd = Dx * Dx + Dy * Dy + Dz * Dz;
          const double cosd = -(Dx * (double)nx + Dy * (double)ny + Dz * (double)nz);
          acc += cosd / (dd * sqrt(dd));
          if (P.vis_bits) atomicOr(P.vis_bits + (c * P.L + l) * words + (r >> 5), 1u << (r & 31));
        }
        pend |= res == kUndecided;
        ++l;
        busy = false;
      }
    }
  }
  if (COUNT)
    for (int k = 0; k < 6; ++k) {
      unsigned long long v = cnt[k];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(P.counters + k, v);
    }
}

// Exact (fp64 triangle tests) any-hit walk for one ray, used by k_fixup.
__device__ bool lane_clear_exact(const AsmParams& P, float ox, float oy, float oz, float cx, float cy,
                                 float cz, int owner) {
  uint32_t stk[kLaneStack];
  int sp = 0;
  const D3 O = d3(ox, oy, oz);
  const D3 D = d3((double)cx - O.x, (double)cy - O.y, (double)cz - O.z);
  const double dd = ddot3(D, D);
  const double t_lo = kSelfEps / sqrt(dd);
  const Ray32 r32 = make_ray32(ox, oy, oz, (float)D.x, (float)D.y, (float)D.z);
  uint32_t ref = P.root;
  for (;;) {
    if (ref_is_leaf(ref)) {
      const uint32_t st = ref_start(ref), nt = ref_count(ref);
      for (uint32_t k = 0; k < nt; ++k) {
        const float4* t = P.tri + 3 * (int64_t)(st + k);
        if (__float_as_int(t[0].w) == owner) continue;
        if (seg_hits_tri(O, D, dd, t_lo, 1.0 - t_lo, t[0], t[1], t[2])) return false;
      }
      if (!sp) return true;
      ref = stk[--sp];
    } else {
      const Node nd = P.nodes[ref];
      const bool h0 = slab(r32, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.c.x, nd.c.y, 1.0f);
      const bool h1 = slab(r32, nd.b.x, nd.b.y, nd.b.z, nd.b.w, nd.c.z, nd.c.w, 1.0f);
      if (h0 && h1) {
        ref = nd.d.x;
        if (sp < kLaneStack) stk[sp++] = nd.d.y;
        else atomicExch(P.err, 2);
      } else if (h0 || h1) {
        ref = h0 ? nd.d.x : nd.d.y;
      } else {
        if (!sp) return true;
        ref = stk[--sp];
      }
    }
  }
}

// Re-trace, with exact fp64 triangle tests, every entry flagged by
// k_assemble_lane and rewrite its value and visibility bits.
__global__ void k_fixup(AsmParams P) {
  const int64_t nwords = P.n_cols * P.words;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = P.pending[w];
    if (!bits) continue;
    const int64_t c = w / P.words, word = w - c * P.words;
    const int64_t j = P.cols ? P.cols[c] : c;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int r = (int)(word * 32 + b);
      const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
      const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
      double acc = 0.0;
      for (int l = 0; l < P.L; ++l) {
        const float* pl = P.lamps + 3 * (j * P.L + l);
        const float ox = pl[0], oy = pl[1], oz = pl[2];
        const D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
        const double dd = ddot3(D, D);
        const double d = sqrt(dd);
        const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);
        const bool vis = cosd > 0.0 && d >= kMinDist && lane_clear_exact(P, ox, oy, oz, cx, cy, cz, r);
        if (vis) acc += cosd / (dd * d);
        if (P.vis_bits) {
          uint32_t* vw = P.vis_bits + (c * P.L + l) * P.words + word;
          if (vis) atomicOr(vw, 1u << b);
          else atomicAnd(vw, ~(1u << b));
        }
      }
      if (P.values) P.values[c * P.ld + r] = (float)(acc * P.scale);
    }
  }
}

// ‖A‖_F by-product: per-column Σ A² (fp64, fixed order within a column tile)
__global__ void k_col_sumsq(const AsmParams P, double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < P.N; r += blockDim.x) {
    const double a = P.values[c * P.ld + r];
    s += a * a;
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

template <bool COUNT>
static int grid_size_assemble(int algo) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (algo == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assemble<COUNT>, kAsmThreads, 0);
  else if (algo == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assemble_lane<COUNT>, kAsmThreads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assemble_dyn<COUNT>, kAsmThreads, 0);
  return std::max(1, sms * std::max(per, 1));
}

}  // namespace uvd

using namespace uvd;

extern "C" int uvd_irradiance_matrix(const uvd_scene* s, const float* lamp_xyz, int64_t k_total,
                                     const int64_t* cols, int64_t n_cols, const uvd_lamp* lamp,
                                     uvd_matrix_out* out, void* stream) {
  clear_error();
  if (!s || !lamp_xyz || !lamp || !out) {
    set_error("uvd_irradiance_matrix: null argument");
    return UVD_ERR_INVALID;
  }
  if (lamp->samples_per_config < 1 || !(lamp->power_w > 0.0)) {
    set_error("uvd_irradiance_matrix: need power_w > 0 and samples_per_config >= 1");
    return UVD_ERR_INVALID;
  }
  if (!cols) n_cols = k_total;
  if (n_cols < 0 || k_total < 0) { set_error("uvd_irradiance_matrix: negative size"); return UVD_ERR_INVALID; }
  if (cols)
    for (int64_t c = 0; c < n_cols; ++c)
      if (cols[c] < 0 || cols[c] >= k_total) {
        set_error("uvd_irradiance_matrix: cols[%lld] = %lld out of range", (long long)c, (long long)cols[c]);
        return UVD_ERR_INVALID;
      }
  if (out->format != UVD_DENSE_COLMAJOR) {
    set_error("uvd_irradiance_matrix: format %d not supported yet", out->format);
    return UVD_ERR_INVALID;
  }
  if (!out->values || out->ld < s->N || out->ld % 32 != 0) {
    set_error("uvd_irradiance_matrix: dense output needs values and ld >= N, ld %% 32 == 0");
    return UVD_ERR_INVALID;
  }
  if (n_cols == 0) return UVD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Alloc al = s->alloc;
  al.stream = st;
  int64_t* dcols = nullptr;
  if (cols) {
    dcols = (int64_t*)al.get(n_cols * sizeof(int64_t));
    if (!dcols) { set_error("uvd_irradiance_matrix: out of device memory"); return UVD_ERR_NOMEM; }
    UVD_CUDA_TRY(cudaMemcpyAsync(dcols, cols, n_cols * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  AsmParams P;
  P.tri = s->tri;
  P.nodes4 = s->nodes4;
  P.nodes = s->nodes;
  P.root = s->root;
  P.centroid = s->centroid;
  P.normal = s->normal;
  P.N = s->N;
  P.lamps = lamp_xyz;
  P.L = lamp->samples_per_config;
  P.scale = lamp->power_w / (4.0 * 3.14159265358979323846 * (double)P.L);
  P.cols = dcols;
  P.n_cols = n_cols;
  P.words = (s->N + 31) / 32;
  P.tiles = out->ld / 32;
  P.values = out->values;
  P.ld = out->ld;
  P.vis_bits = out->vis_bits;
  P.col_sumsq = out->col_sumsq;
  P.counters = out->counters;
  P.err = s->err_flag;
  P.pending = (uint32_t*)al.get((size_t)n_cols * P.words * sizeof(uint32_t));
  if (!P.pending) { set_error("uvd_irradiance_matrix: out of device memory"); return UVD_ERR_NOMEM; }
  // algorithm: 0 = per-lane while-while over the BVH2 with dynamic ray refill
  // (default), 2 = the same per fixed 32-row tile, 1 = warp pair-parallel
  // packets over the BVH4 (UVD_ASM_ALGO=1/2 kept for comparison)
  static int algo = -1;
  if (algo < 0) {
    const char* e = getenv("UVD_ASM_ALGO");
    algo = e ? atoi(e) : 2;
  }
  if (algo == 1)  // the packet kernel resolves undecided tests inline
    UVD_CUDA_TRY(cudaMemsetAsync(P.pending, 0, (size_t)n_cols * P.words * sizeof(uint32_t), st));
  static int grid_c = 0, grid = 0;
  if (P.counters) {
    if (!grid_c) grid_c = grid_size_assemble<true>(algo);
    if (algo == 1) k_assemble<true><<<grid_c, kAsmThreads, 0, st>>>(P);
    else if (algo == 2) k_assemble_lane<true><<<grid_c, kAsmThreads, 0, st>>>(P);
    else k_assemble_dyn<true><<<grid_c, kAsmThreads, 0, st>>>(P);
  } else {
    if (!grid) grid = grid_size_assemble<false>(algo);
    if (algo == 1) k_assemble<false><<<grid, kAsmThreads, 0, st>>>(P);
    else if (algo == 2) k_assemble_lane<false><<<grid, kAsmThreads, 0, st>>>(P);
    else k_assemble_dyn<false><<<grid, kAsmThreads, 0, st>>>(P);
  }
  note_launch();
  {  // exact fp64 re-trace of the (rare) entries the fp32 pass left undecided
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nwords = n_cols * P.words;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nwords + 255) / 256, 4 * sms));
    k_fixup<<<g, 256, 0, st>>>(P);
    note_launch();
  }
  if (P.col_sumsq) {
    k_col_sumsq<<<(unsigned)n_cols, 256, 0, st>>>(P, P.col_sumsq);
    note_launch();
  }
  al.put(P.pending);
  UVD_CUDA_TRY(cudaGetLastError());
  if (dcols) al.put(dcols);
  return UVD_OK;
}
