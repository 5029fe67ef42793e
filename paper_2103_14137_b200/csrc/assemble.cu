// assemble.cu — irradiance-matrix assembly (SURVEY §8(a) rows a4–a6, the
// dominant kernel): for every local column c (configuration j = cols[c]) and
// every patch i,
//   A[i,j] = Σ_l vis_ijl (P/L) <p_jl - c_i, n_i> / (4π |p_jl - c_i|³)
// (Eq. 7, P:234–242 with the Q1/Q2 reading; P:252 for L samples; P:248 mean
// irradiance units), vis = front-facing and no other scene triangle on the open
// segment p_jl -> c_i (Q5–Q8, Q15).
//
//   k_assemble_lane  one warp per (column, 32 adjacent patches in the BVH's
//                    leaf order); every lane walks its own shadow ray through the
//                    BVH2 (Aila & Laine 2009 while-while, near child first,
//                    private stack): the top six levels from fp16 H nodes
//                    (hnodes.cu, HFMA2), below that the octant node copies in
//                    the paired layout (one FFMA2 per plane pair), box tests
//                    bounded by the segment's part outside its empty end
//                    regions (free.cu), triangles decided by an fp32 filter with
//                    forward error bounds; super-tiles of 2048 tiles per column
//                    sweep when the BVH exceeds the L2
//   k_fixup          exact fp64 re-trace of the rare entries the fp32 pass left
//                    undecided (~1e-3 of entries), rewriting value and bits
//   k_csc_count/fill compressed-sparse-column output from the visibility bits
//   k_col_sumsq      per-column Σ A² (‖A‖_F for the LP penalty)
//
// Designs measured and dropped: warp-cooperative packet
// traversal of a BVH2 and of a BVH4 with pair-parallel lanes (2.4 G entries/s
// on C5 vs 6.6 for this kernel: 10x more instructions per ray-node), dynamic
// per-lane ray refill (-20 %), speculative leaf postponing (-10 %).
#include <cuda_runtime.h>

#include <cassert>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

#ifndef UVD_ASM_WARPS
#define UVD_ASM_WARPS 32
#endif
constexpr int kAsmWarps = UVD_ASM_WARPS;
constexpr int kAsmThreads = kAsmWarps * 32;
#ifndef UVD_ASM_MINB
#define UVD_ASM_MINB 1
#endif
constexpr int kAsmMinBlocks = UVD_ASM_MINB;  // 1024-thread blocks x 1 per SM: <= 64 registers, 32 warps per SM

struct AsmParams {
  const float4* __restrict__ tri;
  const Node* __restrict__ nodes;
  const Node* __restrict__ onodes;  // 8 octant copies of nodes (near, far slab order)
  int64_t n_nodes;
  uint32_t root;
  const float* __restrict__ centroid;
  const float* __restrict__ normal;
  int64_t N;
  const float* __restrict__ lamps;
  const float* __restrict__ lampc;  // [n_cols][L][3] lamps gathered per column (k_assemble_lane)
  const float* __restrict__ lamp_free;   // [n_cols][L] lamp radius r_L (free.cu), or nullptr
  const float* __restrict__ front_free;  // [N] front radius r_T (free.cu), or nullptr
  int64_t n_tris;                        // leaf-ordered triangles (UVD_CHECKED bounds)
  const HNode* __restrict__ hnodes;      // 8 octant copies of the H nodes (hnodes.cu), or nullptr
  int32_t n_h;
  float hcx, hcy, hcz, hex, hey, hez;    // H coordinate origin and the scene's half extents
  int L;
  double scale;  // P / (4π L)
  const int64_t* __restrict__ cols;  // device, nullptr = identity
  int64_t n_cols;
  int64_t tiles;  // ceil(rows / 32): ld/32 (dense) or words (CSC)
  bool items32;  // n_cols * tiles < 2^32: 32-bit work-item arithmetic
  int super_log2;  // work order: < 0 column-major, else 2^super_log2 tiles per super-tile (item_to_tile)
  int64_t words;  // ceil(N/32)
  float* __restrict__ values;  // dense [n_cols][ld] or nullptr
  int64_t ld;
  uint32_t* __restrict__ vis_bits;  // [n_cols][L][words] or nullptr
  unsigned long long* __restrict__ counters;  // [6] or nullptr (instrumented kernel)
  uint32_t* __restrict__ pending;  // [n_cols][words] entries left undecided in fp32
  int* __restrict__ err;
  // NEXT-2 area model (area_m >= 0): patch areas, patch-ordered wall triangles
  // (extruded scenes; 3D patch r is the leaf-ordered triangle r), subdivision level
  const double* __restrict__ area;
  const float4* __restrict__ ptri;
  int area_m;  // < 0: the centroid model (a4–a6)
};

// ---------------------------------------------------------------------------
// Per-lane traversal (Aila & Laine 2009 "while-while"): every lane walks its
// own shadow ray through the BVH2 with a private stack (local memory, L1
// resident at the top), near child first; triangles are tested with the fp32
// filter and ambiguous cases re-tested exactly in fp64; any hit ends the ray.
// The 32 rays of a warp share the lamp origin and end on 32 Morton-adjacent
// patches, so the lanes fetch mostly the same nodes (L1 broadcast) and
// diverge little.
constexpr int kLaneStack = 64;
// UVD_CHECKED=1 (test builds: the sanitizer is closed on the GPU pool): device
// asserts on every node / triangle index, stack access and output index
#ifndef UVD_CHECKED
#define UVD_CHECKED 0
#endif
#if UVD_CHECKED
#define UVD_CHECK(c) assert(c)
#else
#define UVD_CHECK(c) ((void)0)
#endif
constexpr uint32_t kDone = 0xffffffffu;

enum { kClear = 0, kBlocked = 1, kUndecided = 2 };

// One lane's any-hit walk with fp32 decisions only.  Returns kBlocked on a
// certain hit, kClear when every triangle the segment may meet was a certain
// miss, kUndecided when no certain hit was found but the fp32 filter could not
// decide some triangle (the caller flags the entry for exact re-tracing).
template <bool COUNT, bool OCT>
__device__ __forceinline__ int lane_walk32(const AsmParams& P, float ox, float oy, float oz,
                                           float dx, float dy, float dz, int owner, float rl, float rt,
                                           unsigned long long* cnt) {
  uint32_t stk[kLaneStack];
  int sp = 0;
  bool undecided = false;
  const float ix = safe_inv(dx), iy = safe_inv(dy), iz = safe_inv(dz);
  const float oix = ox * ix, oiy = oy * iy, oiz = oz * iz;
  // the segment's own extent t in (t_lo, t_hi) also bounds the box tests: boxes
  // the segment only enters within 0.1 mm of the target (e.g. the target's own
  // flat leaf and its flat ancestors) are never visited
  const float inv_len = rsqrtf(dx * dx + dy * dy + dz * dz);
  const float tlo = (float)kSelfEps * inv_len;
  const float thi = 1.0f - tlo;
  // and by the empty regions at its ends (free.cu): nothing within r_L of the
  // lamp, nothing in front of the patch within r_T; the box range shrinks to
  // [tmin, tmax] (factors 1 - 1e-5 and the 2e-7 slack cover rsqrtf's and the
  // products' rounding, so the bounds stay outside the true ones)
  const float tmin = rl * inv_len * 0.99999f;
  const float tmax = fminf(thi, 1.0f - fmaxf(rt * inv_len * 0.99999f - 2e-7f, 0.0f));
  // start in the copy of the nodes whose slabs are stored (near, far) for this
  // ray's octant; child refs stay inside that copy
  const uint32_t oct = (__float_as_uint(ix) >> 31) | ((__float_as_uint(iy) >> 31) << 1) |
                       ((__float_as_uint(iz) >> 31) << 2);
  // OCT = false: the scene has no octant copies (memory cap), one array, min/max per slab
  uint32_t ref = (!OCT || ref_is_leaf(P.root)) ? P.root : P.root + oct * (uint32_t)P.n_nodes;
  // the top of the tree in fp16 (hnodes.cu) when this segment is in fp16 range:
  // |1/d| <= 2048 per axis, the lamp inside the scene box; constants packed in
  // half2 pairs (the HFMA2 operands select their halves)
  __half2 hA = __float2half2_rn(0.f), hB = hA, hC = hA, hT = hA;
  if (OCT && P.hnodes && fmaxf(fabsf(ix), fmaxf(fabsf(iy), fabsf(iz))) <= 2048.0f) {
    const float orx = ox - P.hcx, ory = oy - P.hcy, orz = oz - P.hcz;
    if (fabsf(orx) <= P.hex && fabsf(ory) <= P.hey && fabsf(orz) <= P.hez) {
      const __half hix = __float2half_rn(ix), hiy = __float2half_rn(iy), hiz = __float2half_rn(iz);
      hA = __halves2half2(hix, hiy);
      hB = __halves2half2(hiz, __float2half_rn(-orx * __half2float(hix)));
      hC = __halves2half2(__float2half_rn(-ory * __half2float(hiy)), __float2half_rn(-orz * __half2float(hiz)));
      hT = __halves2half2(__float2half_rd(tmin), __float2half_ru(tmax));
      ref = kHalfRef | (oct * (uint32_t)P.n_h);  // H root: H node 0 of this octant's copy
    }
  }
  for (;;) {
    // ---- inner nodes until this lane holds a leaf (or is done) ----
    while (!ref_is_leaf(ref)) {
      if (OCT && (ref & kHalfRef)) {
        // ---- H node: 32 bytes, both children per HFMA2 (hnodes.cu) ----
        UVD_CHECK((ref & ~kHalfRef) < 8u * (uint32_t)P.n_h);
        const uint4* hq = reinterpret_cast<const uint4*>(P.hnodes + (ref & ~kHalfRef));
        const uint4 q0 = __ldg(hq), q1 = __ldg(hq + 1);
        if (COUNT) { cnt[1] += 2; cnt[3] += 1; cnt[5] += 1; }
        const __half2 tex = __hfma2(*reinterpret_cast<const __half2*>(&q0.x), __low2half2(hA), __high2half2(hB));
        const __half2 txx = __hfma2(*reinterpret_cast<const __half2*>(&q0.y), __low2half2(hA), __high2half2(hB));
        const __half2 tey = __hfma2(*reinterpret_cast<const __half2*>(&q0.z), __high2half2(hA), __low2half2(hC));
        const __half2 txy = __hfma2(*reinterpret_cast<const __half2*>(&q0.w), __high2half2(hA), __low2half2(hC));
        const __half2 tez = __hfma2(*reinterpret_cast<const __half2*>(&q1.x), __low2half2(hB), __high2half2(hC));
        const __half2 txz = __hfma2(*reinterpret_cast<const __half2*>(&q1.y), __low2half2(hB), __high2half2(hC));
        const __half2 en = __hmax2(__hmax2(tex, tey), __hmax2(tez, __low2half2(hT)));
        const __half2 ex = __hmin2(__hmin2(txx, txy), __hmin2(txz, __high2half2(hT)));
        const bool h0 = __hle(__low2half(en), __low2half(ex));
        const bool h1 = __hle(__high2half(en), __high2half(ex));
        if (h0 && h1) {
          const bool swap = __hlt(__high2half(en), __low2half(en));  // near child first
          ref = swap ? q1.w : q1.z;
          if (sp < kLaneStack) stk[sp++] = swap ? q1.z : q1.w;
          else atomicExch(P.err, 2);
        } else if (h0 || h1) {
          ref = h0 ? q1.z : q1.w;
        } else {
          ref = sp ? stk[--sp] : kDone;
        }
        continue;
      }
      UVD_CHECK((int64_t)ref < (OCT ? 8 : 1) * P.n_nodes);
      const Node* nd = (OCT ? P.onodes : P.nodes) + ref;
      const float4 na = __ldg(&nd->a), nb = __ldg(&nd->b), nc = __ldg(&nd->c);
      const uint2 ch = __ldg(reinterpret_cast<const uint2*>(&nd->d));
      if (COUNT) { cnt[1] += 2; cnt[3] += 1; }
      // t = b/d - o/d as one FFMA per plane: fma(b, 1/d, -fl(o/d)) is the exact
      // slab parameter of the plane b shifted by at most eps|o| (<= 1.2e-6 m for
      // |o| <= 20 m), which the build-time box padding (>= 1e-5 m + 4 eps x the
      // scene's largest coordinate) absorbs; the final rounding is covered by
      // the padding as well: the FFMA's one rounding and fl(1/d) scale each t by
      // at most (1 + 2^-23), i.e. move a plane by <= 2^-23 |b - o| <= 5e-6 m, under
      // the >= 1e-5 m padding, so a box the exact segment meets passes an <= af
      // with no widening.  In this octant's copy the first plane of each slab is
      // the entry (t rounds monotonically: entry <= exit).
      float an, af, bn, bf;
      if (OCT) {
        // paired layout (k_octant_nodes): one FFMA2 per (entry or exit, axis) gives
        // both children's parameters, each rounded exactly as one FFMA
        const float2 ex = ffma2(make_float2(na.x, na.y), make_float2(ix, ix), make_float2(-oix, -oix));
        const float2 xx = ffma2(make_float2(na.z, na.w), make_float2(ix, ix), make_float2(-oix, -oix));
        const float2 ey = ffma2(make_float2(nb.x, nb.y), make_float2(iy, iy), make_float2(-oiy, -oiy));
        const float2 xy = ffma2(make_float2(nb.z, nb.w), make_float2(iy, iy), make_float2(-oiy, -oiy));
        const float2 ez = ffma2(make_float2(nc.x, nc.y), make_float2(iz, iz), make_float2(-oiz, -oiz));
        const float2 xz = ffma2(make_float2(nc.z, nc.w), make_float2(iz, iz), make_float2(-oiz, -oiz));
        an = fmaxf(fmaxf(ex.x, ey.x), fmaxf(ez.x, tmin));
        af = fminf(fminf(xx.x, xy.x), fminf(xz.x, tmax));
        bn = fmaxf(fmaxf(ex.y, ey.y), fmaxf(ez.y, tmin));
        bf = fminf(fminf(xx.y, xy.y), fminf(xz.y, tmax));
      } else {
        const float ax0 = fmaf(na.x, ix, -oix), ax1 = fmaf(na.y, ix, -oix);
        const float ay0 = fmaf(na.z, iy, -oiy), ay1 = fmaf(na.w, iy, -oiy);
        const float az0 = fmaf(nc.x, iz, -oiz), az1 = fmaf(nc.y, iz, -oiz);
        const float bx0 = fmaf(nb.x, ix, -oix), bx1 = fmaf(nb.y, ix, -oix);
        const float by0 = fmaf(nb.z, iy, -oiy), by1 = fmaf(nb.w, iy, -oiy);
        const float bz0 = fmaf(nc.z, iz, -oiz), bz1 = fmaf(nc.w, iz, -oiz);
        an = fmaxf(fmaxf(fminf(ax0, ax1), fminf(ay0, ay1)), fmaxf(fminf(az0, az1), tmin));
        af = fminf(fminf(fmaxf(ax0, ax1), fmaxf(ay0, ay1)), fminf(fmaxf(az0, az1), tmax));
        bn = fmaxf(fmaxf(fminf(bx0, bx1), fminf(by0, by1)), fmaxf(fminf(bz0, bz1), tmin));
        bf = fminf(fminf(fmaxf(bx0, bx1), fmaxf(by0, by1)), fminf(fmaxf(bz0, bz1), tmax));
      }
      const bool h0 = an <= af;
      const bool h1 = bn <= bf;
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
    // ---- leaf: up to kLeafMax triangles ----
    const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
    const uint32_t st = ref_start(ref), nt = ref_count(ref);
    for (uint32_t k = 0; k < nt; ++k) {
      UVD_CHECK((int64_t)(st + k) < P.n_tris);
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

// work item -> (column, tile).  P.super_log2 < 0: column-major (all SMs sweep
// one column's tiles: rays from one or two lamps in flight); > 0: super-tiles of
// that many tiles, every column of a super-tile before the next one (default
// 2048 tiles: rays from ~2–3 lamps to the same 64 K patches in flight), chosen
// when the BVH is several times the L2: the paths near the patches are then
// shared across lamps (2^8 / 2^9 / 2^10 / 2^11 / 2^12 / 2^13 tiles measured on
// C5: 904 / 905 / 895 / 892 / 898 / 903 ms).
__device__ __forceinline__ void item_to_unit(const AsmParams& P, int64_t units, int super_log2, int64_t item,
                                             int64_t& c, int64_t& tile) {
  if (super_log2 < 0) {
    if (P.items32) {  // 32-bit division (a 64-bit one is a ~70-instruction sequence)
      const uint32_t cc = (uint32_t)item / (uint32_t)units;
      c = cc;
      tile = (int64_t)((uint32_t)item - cc * (uint32_t)units);
    } else {
      c = item / units;
      tile = item - c * units;
    }
    return;
  }
  // super-tiles of T = 2^super_log2 units; items < 2^32 (checked on the host)
  const uint32_t sh = (uint32_t)super_log2, T = 1u << sh, it = (uint32_t)item;
  const uint32_t full = (uint32_t)units >> sh, per = (uint32_t)P.n_cols << sh, base = full * per;
  if (it < base) {
    const uint32_t s = it / per, rem = it - s * per;
    c = rem >> sh;
    tile = (int64_t)((s << sh) + (rem & (T - 1u)));
  } else {
    const uint32_t rem = it - base, tl = (uint32_t)units - (full << sh);
    const uint32_t cc = rem / tl;
    c = cc;
    tile = (int64_t)((full << sh) + rem - cc * tl);
  }
}
__device__ __forceinline__ void item_to_tile(const AsmParams& P, int64_t item, int64_t& c, int64_t& tile) {
  item_to_unit(P, P.tiles, P.super_log2, item, c, tile);
}

template <bool COUNT, bool OCT>
__global__ void __launch_bounds__(kAsmThreads, kAsmMinBlocks) k_assemble_lane(AsmParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};  // per-lane tallies (COUNT only)
  const int64_t total = P.n_cols * P.tiles;
  // static stride: warp w of block b takes items b·W + w, + G·W, ... (a per-block
  // dynamic schedule keeping an SM's warps on one lamp was measured slower)
  for (int64_t item = (int64_t)blockIdx.x * kAsmWarps + warp; item < total;
       item += (int64_t)gridDim.x * kAsmWarps) {
    // tile fastest: concurrent warps trace adjacent patches from the same lamp
    int64_t c, tile;
    item_to_tile(P, item, c, tile);
    const int r = (int)(tile * 32 + lane);
    const bool valid = r < P.N;
    double acc = 0.0;
    bool pend = false;
    for (int l = 0; l < P.L; ++l) {
      const float* pl = P.lampc + 3 * (c * P.L + l);  // one load, no cols[c] -> lamps[j] chain
      const float ox = pl[0], oy = pl[1], oz = pl[2];
      bool vis = false, front = false;
      float cx = 0.f, cy = 0.f, cz = 0.f;
      double w = 0.0, cosr = 0.0;
      if (valid) {
        cx = P.centroid[3 * r]; cy = P.centroid[3 * r + 1]; cz = P.centroid[3 * r + 2];
        const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
        // a4: ray p -> c in fp64 (exact differences of fp32 inputs), front-face cull
        const D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
        const double dd = ddot3(D, D);
        const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);  // <p - c, n>
        front = cosd > 0.0;
        if (dd < kMinDist * kMinDist) {
          atomicExch(P.err, 1);
          front = false;
        }
        const double ri = rsqrt(dd);  // 1/d (fp64, ~1 ulp): one square root instead of sqrt + division
        w = cosd * (ri * ri * ri);    // a6: Eq. 7 in fp64, added if the ray is clear
        cosr = cosd * ri >= 1e-2 ? 1.0 : 0.0;  // cos θ ≥ 1e-2
      }
      const float dx = cx - ox, dy = cy - oy, dz = cz - oz;
      if (front) {
        if (COUNT) cnt[0] += 1;
        // empty end regions (free.cu); the front one only away from grazing (cos θ ≥ 1e-2)
        const float rl = P.lamp_free ? P.lamp_free[c * P.L + l] : 0.0f;
        const float rt = P.front_free && cosr >= 1e-2 ? P.front_free[r] : 0.0f;
        // a5: occlusion of the open segment, t in (1e-4/d, 1 - 1e-4/d), fp32 decisions
        const int res = lane_walk32<COUNT, OCT>(P, ox, oy, oz, dx, dy, dz, r, rl, rt, cnt);
        vis = res == kClear;
        pend |= res == kUndecided;
        if (vis) acc += w;
      }
      const uint32_t vm = __ballot_sync(0xffffffffu, vis);
      if (P.vis_bits && lane == 0 && tile < P.words) __stcs(P.vis_bits + (c * P.L + l) * P.words + tile, vm);
    }
    // entries with an undecided ray are re-traced exactly by k_fixup
    const uint32_t pm = __ballot_sync(0xffffffffu, pend);
    if (lane == 0 && tile < P.words) __stcs(P.pending + c * P.words + tile, pm);
    if (COUNT) cnt[4] += pend;
    const float a = (float)(acc * P.scale);
    UVD_CHECK(c < P.n_cols && (int64_t)r < P.ld);
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
// NEXT-2: area-integrated irradiance (Eq. 4 as written, P:159–162, P:248;
// reading Q23).  Each triangle of patch r is split m times at its edge
// midpoints (fp64, exact); sub-triangle s contributes its exact solid angle
// (Van Oosterom & Strackee 1983) when the open segment from the lamp sample to
// its centroid (rounded to fp32, the same target the oracle uses) is clear:
//   A[r,j] = (P/L)/(4π|s_r|) Σ_l Σ_s vis_ls Ω_ls.
// Same warp/tile mapping and traversal as k_assemble_lane; sub-rays of a lane
// run back to back (the lanes of a warp trace the same sub-index of adjacent
// patches, so they stay coherent).
struct DTri { D3 a, b, c; };

__device__ __forceinline__ D3 dmid(D3 u, D3 v) {  // exact midpoint of fp64 points from fp32 data
  return d3(__dmul_rn(__dadd_rn(u.x, v.x), 0.5), __dmul_rn(__dadd_rn(u.y, v.y), 0.5),
            __dmul_rn(__dadd_rn(u.z, v.z), 0.5));
}

// sub-triangle s of t after m midpoint subdivisions; base-4 digits of s, most
// significant first, pick the child: 0 (a,ab,ca), 1 (ab,b,bc), 2 (ca,bc,c), 3 (ab,bc,ca)
__device__ __forceinline__ DTri sub_tri(DTri t, uint32_t s, int m) {
  for (int lv = m - 1; lv >= 0; --lv) {
    const uint32_t dgt = (s >> (2 * lv)) & 3u;
    const D3 ab = dmid(t.a, t.b), bc = dmid(t.b, t.c), ca = dmid(t.c, t.a);
    DTri n;
    if (dgt == 0) { n.a = t.a; n.b = ab; n.c = ca; }
    else if (dgt == 1) { n.a = ab; n.b = t.b; n.c = bc; }
    else if (dgt == 2) { n.a = ca; n.b = bc; n.c = t.c; }
    else { n.a = ab; n.b = bc; n.c = ca; }
    t = n;
  }
  return t;
}

__device__ __forceinline__ double tri_solid_angle(D3 p, const DTri& t) {
  const D3 r1 = dsub3(t.a, p), r2 = dsub3(t.b, p), r3 = dsub3(t.c, p);
  const double l1 = sqrt(ddot3(r1, r1)), l2 = sqrt(ddot3(r2, r2)), l3 = sqrt(ddot3(r3, r3));
  const double num = fabs(ddot3(r1, dcross3(r2, r3)));
  const double den = l1 * l2 * l3 + ddot3(r1, r2) * l3 + ddot3(r1, r3) * l2 + ddot3(r2, r3) * l1;
  return 2.0 * atan2(num, den);
}

__device__ __forceinline__ float3 sub_target(const DTri& t) {  // fl32(((a+b)+c)/3), no contraction
  return make_float3(__double2float_rn(__ddiv_rn(__dadd_rn(__dadd_rn(t.a.x, t.b.x), t.c.x), 3.0)),
                     __double2float_rn(__ddiv_rn(__dadd_rn(__dadd_rn(t.a.y, t.b.y), t.c.y), 3.0)),
                     __double2float_rn(__ddiv_rn(__dadd_rn(__dadd_rn(t.a.z, t.b.z), t.c.z), 3.0)));
}

__device__ __forceinline__ DTri patch_tri(const AsmParams& P, int r, int k) {
  const float4* tv = P.ptri ? P.ptri + 3 * (2 * (int64_t)r + k) : P.tri + 3 * (int64_t)r;
  DTri t;
  t.a = f2d(tv[0]); t.b = f2d(tv[1]); t.c = f2d(tv[2]);
  return t;
}

#ifndef UVD_AREA_THREADS
#define UVD_AREA_THREADS 1024
#endif
#ifndef UVD_AREA_MINB
#define UVD_AREA_MINB 1
#endif
constexpr int kAreaThreads = UVD_AREA_THREADS;

template <bool COUNT, bool OCT>
__global__ void __launch_bounds__(kAreaThreads, UVD_AREA_MINB) k_assemble_area(AsmParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kAreaThreads / 32;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  const int64_t total = P.n_cols * P.tiles;
  const int ntri = P.ptri ? 2 : 1;
  const uint32_t nsub = 1u << (2 * P.area_m);
  for (int64_t item = (int64_t)blockIdx.x * nw + warp; item < total; item += (int64_t)gridDim.x * nw) {
    const int64_t c = item / P.tiles, tile = item - c * P.tiles;
    const int64_t j = P.cols ? P.cols[c] : c;
    const int r = (int)(tile * 32 + lane);
    const bool valid = r < P.N;
    double acc = 0.0;
    bool pend = false;
    for (int l = 0; l < P.L; ++l) {
      const float* pl = P.lamps + 3 * (j * P.L + l);
      const float ox = pl[0], oy = pl[1], oz = pl[2];
      bool anyvis = false, front = false;
      if (valid) {
        const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
        const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
        const D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
        const double d = sqrt(ddot3(D, D));
        const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);
        front = cosd > 0.0;  // P:242, the patch's facing (as a4)
        if (d < kMinDist) { atomicExch(P.err, 1); front = false; }
      }
      {  // the walks are entered from one reconvergence point (as k_assemble_lane)
        if (front) {
          for (int k = 0; k < ntri; ++k) {
            for (uint32_t s = 0; s < nsub; ++s) {
              // the sub-triangle is rebuilt after the walk rather than kept live
              // across it (the traversal needs the registers)
              const float3 x = sub_target(sub_tri(patch_tri(P, r, k), s, P.area_m));
              const float dx = x.x - ox, dy = x.y - oy, dz = x.z - oz;
              if ((double)dx * dx + (double)dy * dy + (double)dz * dz < kMinDist * kMinDist) {
                atomicExch(P.err, 1);
                continue;
              }
              if (COUNT) cnt[0] += 1;
              const int res = lane_walk32<COUNT, OCT>(P, ox, oy, oz, dx, dy, dz, r, 0.0f, 0.0f, cnt);
              if (COUNT && res == kBlocked) cnt[5] += 1;
              pend |= res == kUndecided;
              if (res == kClear) {
                asm volatile("" ::: "memory");
                acc += tri_solid_angle(d3(ox, oy, oz), sub_tri(patch_tri(P, r, k), s, P.area_m));
                anyvis = true;
              }
            }
          }
        }
      }
      const uint32_t vm = __ballot_sync(0xffffffffu, anyvis);
      if (P.vis_bits && lane == 0 && tile < P.words) __stcs(P.vis_bits + (c * P.L + l) * P.words + tile, vm);
    }
    const uint32_t pm = __ballot_sync(0xffffffffu, pend);
    if (lane == 0 && tile < P.words) __stcs(P.pending + c * P.words + tile, pm);
    if (COUNT) cnt[4] += pend;
    const float a = valid ? (float)(acc * P.scale / P.area[r]) : 0.f;
    if (P.values) __stcs(P.values + c * P.ld + r, a);
  }
  if (COUNT)
    for (int k = 0; k < 6; ++k) {
      unsigned long long v = cnt[k];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(P.counters + k, v);
    }
}

// ------------------------------------------------------------------ CSC --
// Entry (c, i) is nonzero iff some lamp sample sees patch i (Eq. 7 > 0 when
// visible and front-facing).  count: one block per column, popcount of the OR
// of the L visibility words; fill: block-wide exclusive scan of the per-word
// counts gives each word's slot, rows ascending within the column.
constexpr int kCscThreads = 256;

__global__ void __launch_bounds__(kCscThreads) k_csc_count(const AsmParams P, int64_t* __restrict__ colcnt) {
  const int64_t c = blockIdx.x;
  int64_t s = 0;
  for (int64_t w = threadIdx.x; w < P.words; w += kCscThreads) {
    uint32_t m = 0;
    for (int l = 0; l < P.L; ++l) m |= P.vis_bits[(c * P.L + l) * P.words + w];
    s += __popc(m);
  }
  __shared__ int64_t red[kCscThreads];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kCscThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) colcnt[c] = red[0];
}

// exclusive scan of n int64 counts into colptr[0..n] (one block)
__global__ void __launch_bounds__(1024) k_csc_colptr(const int64_t* __restrict__ cnt, int64_t n,
                                                     int64_t* __restrict__ colptr) {
  __shared__ int64_t part[1024];
  const int64_t per = (n + 1023) / 1024;
  const int64_t s = threadIdx.x * per, e = s + per < n ? s + per : n;
  int64_t sum = 0;
  for (int64_t i = s; i < e; ++i) sum += cnt[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = s; i < e; ++i) { colptr[i] = run; run += cnt[i]; }
  if (threadIdx.x == 1023) colptr[n] = part[1023];
}

__global__ void __launch_bounds__(kCscThreads) k_csc_fill(const AsmParams P, const int64_t* __restrict__ colptr,
                                                          int32_t* __restrict__ rowidx, float* __restrict__ vals) {
  const int64_t c = blockIdx.x;
  const int64_t j = P.cols ? P.cols[c] : c;
  __shared__ int32_t sc[kCscThreads];
  __shared__ int64_t base;
  if (threadIdx.x == 0) base = colptr[c];
  __syncthreads();
  for (int64_t w0 = 0; w0 < P.words; w0 += kCscThreads) {
    const int64_t w = w0 + threadIdx.x;
    uint32_t m = 0;
    if (w < P.words)
      for (int l = 0; l < P.L; ++l) m |= P.vis_bits[(c * P.L + l) * P.words + w];
    const int cntw = __popc(m);
    sc[threadIdx.x] = cntw;
    __syncthreads();
    for (int off = 1; off < kCscThreads; off <<= 1) {  // inclusive scan
      int v = threadIdx.x >= off ? sc[threadIdx.x - off] : 0;
      __syncthreads();
      sc[threadIdx.x] += v;
      __syncthreads();
    }
    int64_t o = base + sc[threadIdx.x] - cntw;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int r = (int)(w * 32 + b);
      const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
      const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
      double acc = 0.0;
      for (int l = 0; l < P.L; ++l) {
        if (!((P.vis_bits[(c * P.L + l) * P.words + w] >> b) & 1u)) continue;
        const float* pl = P.lamps + 3 * (j * P.L + l);
        const D3 D = d3((double)cx - (double)pl[0], (double)cy - (double)pl[1], (double)cz - (double)pl[2]);
        const double dd = ddot3(D, D);
        const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);
        const double ri = rsqrt(dd);  // Eq. 7 exactly as k_assemble_lane computes it
        acc += cosd * (ri * ri * ri);
      }
      rowidx[o] = r;
      vals[o] = (float)(acc * P.scale);
      ++o;
    }
    __syncthreads();
    if (threadIdx.x == kCscThreads - 1) base += sc[kCscThreads - 1];
    __syncthreads();
  }
}

// Exact any-hit walk for one ray, used by k_fixup: the same fp32 boxes and
// fp32 triangle filter as the hot kernel, with every undecided triangle
// re-tested at once in fp64 (no register pressure concern in this kernel).
__device__ bool lane_clear_exact(const AsmParams& P, float ox, float oy, float oz, float cx, float cy,
                                 float cz, int owner, float rl = 0.0f, float rt = 0.0f) {
  uint32_t stk[kLaneStack];
  int sp = 0;
  const float dx = cx - ox, dy = cy - oy, dz = cz - oz;
  const float ix = safe_inv(dx), iy = safe_inv(dy), iz = safe_inv(dz);
  const float oix = ox * ix, oiy = oy * iy, oiz = oz * iz;
  const float nD = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const float inv_len = rsqrtf(dx * dx + dy * dy + dz * dz);
  const float tlo = (float)kSelfEps * inv_len;
  const float thi = 1.0f - tlo;
  // the box tests use the segment's part outside its empty end regions, exactly
  // as k_assemble_lane (free.cu; the triangle tests keep the full range)
  const float tmin = rl * inv_len * 0.99999f;
  const float tmax = fminf(thi, 1.0f - fmaxf(rt * inv_len * 0.99999f - 2e-7f, 0.0f));
  const D3 O = d3(ox, oy, oz);
  const D3 D = d3((double)cx - O.x, (double)cy - O.y, (double)cz - O.z);
  const double dd = ddot3(D, D);
  const double t_lo = kSelfEps / sqrt(dd);
  uint32_t ref = P.root;
  for (;;) {
    if (ref_is_leaf(ref)) {
      const uint32_t st = ref_start(ref), nt = ref_count(ref);
      for (uint32_t k = 0; k < nt; ++k) {
        UVD_CHECK((int64_t)(st + k) < P.n_tris);
        const float4* t = P.tri + 3 * (int64_t)(st + k);
        const float4 a = t[0], b = t[1], c = t[2];
        if (__float_as_int(a.w) == owner) continue;
        int cls = seg_tri_filter32(ox, oy, oz, dx, dy, dz, nD, tlo, thi, a, b, c);
        if (cls == 2) cls = seg_hits_tri(O, D, dd, t_lo, 1.0 - t_lo, a, b, c) ? 1 : 0;
        if (cls == 1) return false;
      }
      if (!sp) return true;
      ref = stk[--sp];
    } else {
      UVD_CHECK((int64_t)ref < P.n_nodes);
      const Node nd = P.nodes[ref];
      const float ax0 = fmaf(nd.a.x, ix, -oix), ax1 = fmaf(nd.a.y, ix, -oix);
      const float ay0 = fmaf(nd.a.z, iy, -oiy), ay1 = fmaf(nd.a.w, iy, -oiy);
      const float az0 = fmaf(nd.c.x, iz, -oiz), az1 = fmaf(nd.c.y, iz, -oiz);
      const float bx0 = fmaf(nd.b.x, ix, -oix), bx1 = fmaf(nd.b.y, ix, -oix);
      const float by0 = fmaf(nd.b.z, iy, -oiy), by1 = fmaf(nd.b.w, iy, -oiy);
      const float bz0 = fmaf(nd.c.z, iz, -oiz), bz1 = fmaf(nd.c.w, iz, -oiz);
      const float an = fmaxf(fmaxf(fminf(ax0, ax1), fminf(ay0, ay1)), fmaxf(fminf(az0, az1), tmin));
      const float af = fminf(fminf(fmaxf(ax0, ax1), fmaxf(ay0, ay1)), fminf(fmaxf(az0, az1), tmax));
      const float bn = fmaxf(fmaxf(fminf(bx0, bx1), fminf(by0, by1)), fmaxf(fminf(bz0, bz1), tmin));
      const float bf = fminf(fminf(fmaxf(bx0, bx1), fmaxf(by0, by1)), fminf(fmaxf(bz0, bz1), tmax));
      const bool h0 = an <= fmaf(af, 1.000002f, 1e-7f);
      const bool h1 = bn <= fmaf(bf, 1.000002f, 1e-7f);
      if (h0 && h1) {
        const bool swap = bn < an;  // near child first: an occluder ends the walk sooner
        ref = swap ? nd.d.y : nd.d.x;
        if (sp < kLaneStack) stk[sp++] = swap ? nd.d.x : nd.d.y;
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
// k_assemble_lane and rewrite its value and visibility bits.  The flagged
// entries (~1e-3 of all) are first compacted into a list (warp-aggregated
// atomics) so the re-trace runs with full warps; entries beyond the list's
// capacity are re-traced in place by the collecting thread.
__device__ void fixup_entry(const AsmParams& P, int64_t c, int r) {
  const int64_t j = P.cols ? P.cols[c] : c;
  const int64_t word = r >> 5;
  const int b = r & 31;
  const float cx = P.centroid[3 * r], cy = P.centroid[3 * r + 1], cz = P.centroid[3 * r + 2];
  const float nx = P.normal[3 * r], ny = P.normal[3 * r + 1], nz = P.normal[3 * r + 2];
  double acc = 0.0;
  for (int l = 0; l < P.L; ++l) {
    const float* pl = P.lamps + 3 * (j * P.L + l);
    const float ox = pl[0], oy = pl[1], oz = pl[2];
    const D3 D = d3((double)cx - (double)ox, (double)cy - (double)oy, (double)cz - (double)oz);
    const double dd = ddot3(D, D);
    const double d = sqrt(dd);
    const double ri = rsqrt(dd);  // Eq. 7 as in k_assemble_lane: cosd · (1/d)³
    const double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);
    bool vis;
    if (P.area_m >= 0) {  // NEXT-2: every sub-triangle re-traced exactly
      vis = false;
      if (cosd > 0.0 && d >= kMinDist) {
        const D3 po = d3(ox, oy, oz);
        const uint32_t nsub = 1u << (2 * P.area_m);
        for (int k = 0; k < (P.ptri ? 2 : 1); ++k) {
          const DTri base = patch_tri(P, r, k);
          for (uint32_t s = 0; s < nsub; ++s) {
            const DTri t = sub_tri(base, s, P.area_m);
            const float3 x = sub_target(t);
            const float ex = x.x - ox, ey = x.y - oy, ez = x.z - oz;
            if ((double)ex * ex + (double)ey * ey + (double)ez * ez < kMinDist * kMinDist) continue;
            if (lane_clear_exact(P, ox, oy, oz, x.x, x.y, x.z, r)) {
              acc += tri_solid_angle(po, t);
              vis = true;
            }
          }
        }
      }
    } else {
      // the empty end regions of k_assemble_lane (lamp radius of this call's column, front radius
      // when cos θ >= 1e-2, the same expressions)
      const float rl = P.lamp_free ? P.lamp_free[c * P.L + l] : 0.0f;
      const float rt = P.front_free && cosd * ri >= 1e-2 ? P.front_free[r] : 0.0f;
      vis = cosd > 0.0 && dd >= kMinDist * kMinDist && lane_clear_exact(P, ox, oy, oz, cx, cy, cz, r, rl, rt);
      if (vis) acc += cosd * (ri * ri * ri);
    }
    if (P.vis_bits) {
      uint32_t* vw = P.vis_bits + (c * P.L + l) * P.words + word;
      if (vis) atomicOr(vw, 1u << b);
      else atomicAnd(vw, ~(1u << b));
    }
  }
  if (P.values) P.values[c * P.ld + r] = (float)(P.area_m >= 0 ? acc * P.scale / P.area[r] : acc * P.scale);
}

// Compaction of the pending bits into (column, row) entries: each thread owns 4
// consecutive words, blocks with no pending bit (almost all) leave after one
// __syncthreads_or; otherwise one atomic per block reserves the slots.
constexpr int kCollectThreads = 256, kCollectWords = 16;  // 64 B per thread: 4 x 16-B loads in flight
__global__ void __launch_bounds__(kCollectThreads) k_fixup_collect(AsmParams P, uint64_t* __restrict__ list,
                                                                    int64_t cap,
                                                                    unsigned long long* __restrict__ count) {
  __shared__ int s_warp[kCollectThreads / 32];
  __shared__ unsigned long long s_base;
  const int64_t nwords = P.n_cols * P.words;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int64_t kPer = (int64_t)kCollectThreads * kCollectWords;
  for (int64_t w0 = blockIdx.x * kPer; w0 < nwords; w0 += (int64_t)gridDim.x * kPer) {
    const int64_t w = w0 + (int64_t)threadIdx.x * kCollectWords;
    uint32_t bits[kCollectWords];
    int n = 0;
    if (w + kCollectWords <= nwords) {  // the buffer and w are 64-B aligned
      const uint4* p4 = reinterpret_cast<const uint4*>(P.pending + w);
#pragma unroll
      for (int k = 0; k < kCollectWords / 4; ++k) {
        const uint4 v = __ldcs(p4 + k);
        bits[4 * k] = v.x; bits[4 * k + 1] = v.y; bits[4 * k + 2] = v.z; bits[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kCollectWords; ++k) bits[k] = w + k < nwords ? P.pending[w + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kCollectWords; ++k) n += __popc(bits[k]);
    if (!__syncthreads_or(n)) continue;
    int incl = n;  // block exclusive scan of the counts
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kCollectThreads / 32; ++k) {
      const int v = s_warp[k];
      before += k < wid ? v : 0;
      total += v;
    }
    if (threadIdx.x == 0) s_base = atomicAdd(count, (unsigned long long)total);
    __syncthreads();
    int64_t slot = (int64_t)s_base + before + incl - n;
    __syncthreads();  // s_warp / s_base are rewritten by the next iteration
#pragma unroll
    for (int k = 0; k < kCollectWords; ++k) {
      uint32_t b = bits[k];
      if (!b) continue;
      const int64_t wk = w + k, c = wk / P.words, word = wk - c * P.words;
      uint32_t keep = 0;  // entries beyond the list's capacity stay pending for k_fixup_overflow
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        if (slot < cap) list[slot] = ((uint64_t)c << 32) | (uint32_t)(word * 32 + bit);
        else keep |= 1u << bit;
        ++slot;
      }
      P.pending[wk] = keep;
    }
  }
}

// Entries the list had no room for (count > cap): re-traced here, found by
// their pending bits (k_fixup_collect cleared the listed ones).
__global__ void k_fixup_overflow(AsmParams P, int64_t cap, const unsigned long long* __restrict__ count) {
  if ((int64_t)*count <= cap) return;
  const int64_t nwords = P.n_cols * P.words;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = P.pending[w];
    const int64_t c = w / P.words, word = w - c * P.words;
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      fixup_entry(P, c, (int)(word * 32 + bit));
    }
  }
}

#ifndef UVD_FIX_MINB
#define UVD_FIX_MINB 8  // 64 registers: 8.6 ms per C5 launch (12 blocks / 40 registers: 9.8, 6: 9.4, 4: 10.1, 16: 17.6)
#endif
__global__ void __launch_bounds__(128, UVD_FIX_MINB) k_fixup_run(AsmParams P, const uint64_t* __restrict__ list, int64_t cap,
                            const unsigned long long* __restrict__ count) {
  const int64_t n = min((int64_t)*count, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = list[i];
    fixup_entry(P, (int64_t)(e >> 32), (int)(uint32_t)e);
  }
}

// ‖A‖_F by-product: per-column Σ A² in fp64, fixed reduction order
__global__ void k_col_sumsq(const AsmParams P, const int64_t* __restrict__ colptr,
                            const float* __restrict__ cvals, double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  double s = 0.0;
  if (colptr) {
    for (int64_t e = colptr[c] + threadIdx.x; e < colptr[c + 1]; e += blockDim.x) {
      const double a = cvals[e];
      s += a * a;
    }
  } else {
    for (int64_t r = threadIdx.x; r < P.N; r += blockDim.x) {
      const double a = P.values[c * P.ld + r];
      s += a * a;
    }
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

// lamps of each output column, gathered once per call: k_assemble_lane's item
// prelude then loads its lamp directly instead of cols[c] -> lamps[cols[c]]
__global__ void k_gather_lamps(const AsmParams P, float* __restrict__ out) {
  const int64_t per = 3 * (int64_t)P.L, n = P.n_cols * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / per, q = i - c * per;
    const int64_t j = P.cols ? P.cols[c] : c;
    out[i] = P.lamps[j * per + q];
  }
}

// The walk's conservativeness rests on the box padding (bvh.cu pad_lo/hi:
// 1e-5 m + 1e-6|x| + 4·2^-24·max|scene coordinate|) covering the slab
// rounding, which grows with |lamp| (plane shift <= 1.5·2^-23 |o| beyond the
// scene's own terms): valid for lamp coordinates within the scene's largest
// |coordinate| + 50 m.  Lamps outside that (or non-finite) raise flag 3, which
// uvd_sync_status reports as UVD_ERR_INVALID — the matrix is not trusted then.
__global__ void k_check_lamps(const float* __restrict__ lamps, const int64_t* __restrict__ cols, int64_t n_cols,
                              int L, float bound, int* __restrict__ err) {
  const int64_t per = 3 * (int64_t)L, n = n_cols * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / per, q = i - c * per;
    const float v = lamps[(cols ? cols[c] : c) * per + q];
    if (!(fabsf(v) <= bound)) atomicExch(err, 3);
  }
}

int check_lamps(const uvd_scene* s, const float* lamps, const int64_t* dcols, int64_t n_cols, int L, cudaStream_t st) {
  float maxc = 0.f;
  for (int k = 0; k < 6; ++k) maxc = std::max(maxc, std::fabs(s->bbox[k]));
  const int64_t n = n_cols * L * 3;
  if (n <= 0) return UVD_OK;
  k_check_lamps<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1024)), 256, 0, st>>>(
      lamps, dcols, n_cols, L, maxc + 50.0f, s->err_flag);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

// persistent grids (occupancy x SMs), cached per device and kernel
template <typename K>
static int persistent_grid(K kernel, int threads, int dev, int* cache) {
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (!cache[dev]) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
    cache[dev] = std::max(1, sm_count(dev) * std::max(per, 1));
  }
  return cache[dev];
}

__global__ void k_take_fixups(const uint64_t* __restrict__ list, const unsigned long long* __restrict__ count,
                              int64_t cap, uint64_t* __restrict__ out, int64_t out_cap, int64_t* __restrict__ n_out) {
  const int64_t n = (int64_t)*count;
  const int64_t m = min(min(n, cap), out_cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = list[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = n;
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
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_irradiance_matrix");
  if (lamp->samples_per_config < 1 || !(lamp->power_w > 0.0)) {
    set_error("uvd_irradiance_matrix: need power_w > 0 and samples_per_config >= 1");
    return UVD_ERR_INVALID;
  }
  const bool area_model = lamp->model == UVD_MODEL_AREA;
  if ((lamp->model != UVD_MODEL_CENTROID && !area_model) ||
      (area_model && (lamp->subdiv < 0 || lamp->subdiv > 6))) {
    set_error("uvd_irradiance_matrix: model must be CENTROID or AREA with 0 <= subdiv <= 6");
    return UVD_ERR_INVALID;
  }
  if (area_model && (out->format == UVD_CSC || (s->kind == UVD_SCENE_EXTRUDED && !s->ptri) || !UVD_ROWS_DFS)) {
    set_error("uvd_irradiance_matrix: the AREA model needs dense output");
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
  const bool csc = out->format == UVD_CSC;
  if (!csc && out->format != UVD_DENSE_COLMAJOR) {
    set_error("uvd_irradiance_matrix: unknown format %d", out->format);
    return UVD_ERR_INVALID;
  }
  if ((out->fixup_list && (!out->fixup_count || out->fixup_cap < 0)) || (out->fixup_count && !out->fixup_list)) {
    set_error("uvd_irradiance_matrix: fixup_list needs fixup_count and fixup_cap >= 0");
    return UVD_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (n_cols == 0) {
    if (csc && out->colptr) UVD_CUDA_TRY(cudaMemsetAsync(out->colptr, 0, sizeof(int64_t), st));
    if (out->fixup_count) UVD_CUDA_TRY(cudaMemsetAsync(out->fixup_count, 0, sizeof(int64_t), st));
    return UVD_OK;
  }
  if (!csc && (!out->values || out->ld < s->N || out->ld % 32 != 0)) {
    set_error("uvd_irradiance_matrix: dense output needs values and ld >= N, ld %% 32 == 0");
    return UVD_ERR_INVALID;
  }
  if (csc && (!out->colptr || out->nnz_cap < 0 || (out->nnz_cap > 0 && (!out->rowidx || !out->values)))) {
    set_error("uvd_irradiance_matrix: CSC output needs colptr (and rowidx/values when nnz_cap > 0)");
    return UVD_ERR_INVALID;
  }
  const int dev = s->alloc.device;
  const int sms = sm_count(dev);
  Scratch sc(s->alloc, st);  // every scratch buffer below goes back at every exit
  AsmParams P;
  P.tri = s->tri;
  P.nodes = s->nodes;
  P.onodes = s->onodes;
  P.n_nodes = s->n_nodes;
  P.root = s->root;
  P.centroid = s->centroid;
  P.normal = s->normal;
  P.N = s->N;
  P.lamps = lamp_xyz;
  P.L = lamp->samples_per_config;
  P.scale = lamp->power_w / (4.0 * 3.14159265358979323846 * (double)P.L);
  P.n_cols = n_cols;
  P.words = (s->N + 31) / 32;
  P.tiles = csc ? P.words : out->ld / 32;
  {  // work order (item_to_tile): super-tiles of 2048 tiles when the traversal data is > 2x the L2
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const double bvh_bytes = 8.0 * (double)s->n_nodes * sizeof(Node) + 48.0 * (double)s->M;
    P.super_log2 = bvh_bytes > 2.0 * (double)l2 ? 11 : -1;
    if (const char* e = getenv("UVD_ASM_SUPER")) P.super_log2 = atoi(e);  // dev override (log2, < 0 off)
    P.items32 = n_cols * P.tiles < ((int64_t)1 << 32);
    if (P.super_log2 > 30 || !P.items32 ||
        (P.super_log2 >= 0 && (n_cols << P.super_log2) >= ((int64_t)1 << 32)))
      P.super_log2 = -1;
  }
  P.values = csc ? nullptr : out->values;
  P.ld = csc ? P.words * 32 : out->ld;
  P.counters = out->counters;
  P.err = s->err_flag;
  P.area = s->area;
  P.ptri = s->kind == UVD_SCENE_EXTRUDED ? s->ptri : nullptr;
  P.area_m = area_model ? lamp->subdiv : -1;
  // scratch: column ids, undecided-entry bits, visibility bits for CSC
  int64_t* dcols = cols ? (int64_t*)sc.get(n_cols * sizeof(int64_t)) : nullptr;
  P.pending = (uint32_t*)sc.get((size_t)n_cols * P.words * sizeof(uint32_t));
  uint32_t* vis_scratch =
      csc && !out->vis_bits ? (uint32_t*)sc.get((size_t)n_cols * P.L * P.words * sizeof(uint32_t)) : nullptr;
  int64_t* colcnt = csc ? (int64_t*)sc.get(n_cols * sizeof(int64_t)) : nullptr;
  if ((cols && !dcols) || !P.pending || (csc && !out->vis_bits && !vis_scratch) || (csc && !colcnt)) {
    set_error("uvd_irradiance_matrix: out of device memory");
    return UVD_ERR_NOMEM;
  }
  if ((uintptr_t)P.pending & 15u) {  // k_fixup_collect reads it with 16-B loads
    set_error("uvd_irradiance_matrix: allocator returned a buffer not 16-B aligned");
    return UVD_ERR_INVALID;
  }
  if (dcols) UVD_CUDA_TRY(cudaMemcpyAsync(dcols, cols, n_cols * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  P.cols = dcols;
  P.vis_bits = out->vis_bits ? out->vis_bits : vis_scratch;
  P.lampc = nullptr;
  P.lamp_free = nullptr;
  P.hnodes = s->hnodes;
  P.n_h = s->n_h;
  P.n_tris = s->M;
  if (const char* e = getenv("UVD_HNODES")) if (atoi(e) == 0) P.hnodes = nullptr;  // dev A/B
  P.hcx = s->hcenter[0]; P.hcy = s->hcenter[1]; P.hcz = s->hcenter[2];
  P.hex = 0.5f * (s->bbox[3] - s->bbox[0]); P.hey = 0.5f * (s->bbox[4] - s->bbox[1]);
  P.hez = 0.5f * (s->bbox[5] - s->bbox[2]);
  P.front_free = s->front_free;
  if (const char* e = getenv("UVD_FREE")) if (atoi(e) == 0) P.front_free = nullptr;  // dev A/B
  UVD_TRY(check_lamps(s, lamp_xyz, dcols, n_cols, P.L, st));  // lamps inside the range the box padding covers
  if (!area_model) {
    float* lampc = (float*)sc.get((size_t)n_cols * P.L * 3 * sizeof(float));
    if (!lampc) { set_error("uvd_irradiance_matrix: out of device memory"); return UVD_ERR_NOMEM; }
    const int64_t n = n_cols * P.L * 3;
    k_gather_lamps<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(P, lampc);
    note_launch();
    P.lampc = lampc;
    float* lfree = (float*)sc.get((size_t)n_cols * P.L * sizeof(float));
    if (!lfree) { set_error("uvd_irradiance_matrix: out of device memory"); return UVD_ERR_NOMEM; }
    UVD_TRY(lamp_radius(s, lampc, n_cols * P.L, lfree, st));
    P.lamp_free = P.front_free ? lfree : nullptr;
  }
  static int g_lane[4][kMaxDevices], g_area[4][kMaxDevices];  // [COUNT * 2 + OCT][device]
  const int gi = (P.counters ? 2 : 0) + (P.onodes ? 1 : 0);
  // octant node copies when the scene has them (bvh.cu caps their memory)
  if (area_model) {
    auto kern = P.counters ? (P.onodes ? k_assemble_area<true, true> : k_assemble_area<true, false>)
                           : (P.onodes ? k_assemble_area<false, true> : k_assemble_area<false, false>);
    kern<<<persistent_grid(kern, kAreaThreads, dev, g_area[gi]), kAreaThreads, 0, st>>>(P);
  } else {
    auto kern = P.counters ? (P.onodes ? k_assemble_lane<true, true> : k_assemble_lane<true, false>)
                           : (P.onodes ? k_assemble_lane<false, true> : k_assemble_lane<false, false>);
    kern<<<persistent_grid(kern, kAsmThreads, dev, g_lane[gi]), kAsmThreads, 0, st>>>(P);
  }
  note_launch();
  {  // exact fp64 re-trace of the (rare) entries the fp32 pass left undecided
    const int64_t nwords = n_cols * P.words;
    // room for 2^24 entries (128 MB): C5 flags ~6.6 M; beyond it k_fixup_overflow re-traces the rest
    int64_t cap = std::min<int64_t>(nwords * 32, (int64_t)1 << 24);
    if (const char* e = getenv("UVD_FIXUP_CAP")) cap = std::max<int64_t>(1, std::min<int64_t>(cap, atoll(e)));  // tests
    uint64_t* list = (uint64_t*)sc.get((size_t)cap * sizeof(uint64_t) + 256);
    if (!list) { set_error("uvd_irradiance_matrix: out of device memory"); return UVD_ERR_NOMEM; }
    unsigned long long* count = (unsigned long long*)((char*)list + (size_t)cap * sizeof(uint64_t));
    UVD_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned long long), st));
    const int64_t per = (int64_t)kCollectThreads * kCollectWords;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nwords + per - 1) / per, 8 * sms));
    k_fixup_collect<<<g, kCollectThreads, 0, st>>>(P, list, cap, count);
    if (out->fixup_list) {  // debug/parity export, before the re-trace (the list itself is unchanged by it)
      k_take_fixups<<<(unsigned)std::max(1, 2 * sms), 256, 0, st>>>(list, count, cap, out->fixup_list, out->fixup_cap,
                                                                    out->fixup_count);
      note_launch();
    }
    k_fixup_run<<<UVD_FIX_MINB * sms, 128, 0, st>>>(P, list, cap, count);
    k_fixup_overflow<<<2 * sms, 256, 0, st>>>(P, cap, count);
    note_launch(3);
  }
  int rc = UVD_OK;
  if (csc) {
    k_csc_count<<<(unsigned)n_cols, kCscThreads, 0, st>>>(P, colcnt);
    k_csc_colptr<<<1, 1024, 0, st>>>(colcnt, n_cols, out->colptr);
    note_launch(2);
    int64_t nnz = 0;
    UVD_CUDA_TRY(cudaMemcpyAsync(&nnz, out->colptr + n_cols, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    if (nnz > out->nnz_cap) {
      set_error("uvd_irradiance_matrix: CSC needs nnz = %lld > nnz_cap = %lld", (long long)nnz,
                (long long)out->nnz_cap);
      rc = UVD_ERR_CAPACITY;
    } else {
      k_csc_fill<<<(unsigned)n_cols, kCscThreads, 0, st>>>(P, out->colptr, out->rowidx, out->values);
      note_launch();
    }
  }
  if (out->col_sumsq && rc == UVD_OK) {
    k_col_sumsq<<<(unsigned)n_cols, 256, 0, st>>>(P, csc ? out->colptr : nullptr, csc ? out->values : nullptr,
                                                   out->col_sumsq);
    note_launch();
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return rc;
}
