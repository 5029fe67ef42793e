// bvh.cu — GPU LBVH build (BASELINE north_star "GPU LBVH
// build (Morton codes, radix sort, Karras hierarchy)").
//
//   k_morton    63-bit Morton code of each triangle centroid in the scene bbox
//   radix sort  hand-written LSD sort of (u64 key, u32 value), 8-bit digits,
//               stable block-local ranking with warp match/ballot
//   PLOC        (default) agglomerative clustering of the Morton-ordered
//               triangles (Meister & Bittner 2018): nearest neighbours within
//               a +-16 window merge when mutual; DFS leaf order afterwards
//   k_karras    (UVD_BVH=karras) internal-node topology from longest common
//               prefixes (Karras 2012; equal keys broken by index) + k_refit,
//               bottom-up AABBs with atomic arrival counters
//   k_emit      BVH2 nodes holding both child boxes (64 B), subtrees of
//               <= kLeafMax triangles collapsed into leaf ranges, boxes padded
//               outward so fp32 slab tests are conservative for the fp64 ray.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <cmath>

#include "uvd_internal.cuh"

namespace uvd {

// ----------------------------------------------------------------- morton --
__device__ __forceinline__ uint64_t spread21(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__global__ void k_morton(const float4* __restrict__ tri_in, int64_t M, float3 lo, float3 inv_ext,
                         uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= M) return;
  float4 a = tri_in[3 * t], b = tri_in[3 * t + 1], c = tri_in[3 * t + 2];
  float cx = (a.x + b.x + c.x) * (1.0f / 3.0f);
  float cy = (a.y + b.y + c.y) * (1.0f / 3.0f);
  float cz = (a.z + b.z + c.z) * (1.0f / 3.0f);
  const float scale = 2097151.0f;  // 2^21 - 1
  uint32_t ix = (uint32_t)fminf(fmaxf((cx - lo.x) * inv_ext.x * scale, 0.f), scale);
  uint32_t iy = (uint32_t)fminf(fmaxf((cy - lo.y) * inv_ext.y * scale, 0.f), scale);
  uint32_t iz = (uint32_t)fminf(fmaxf((cz - lo.z) * inv_ext.z * scale, 0.f), scale);
  keys[t] = (spread21(ix) << 2) | (spread21(iy) << 1) | spread21(iz);
  vals[t] = (uint32_t)t;
}

// ------------------------------------------------------------- radix sort --
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kSortWarps = kSortThreads / 32;

__global__ void __launch_bounds__(kSortThreads) k_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                       int shift, uint32_t* __restrict__ counts,
                                                       int nblocks) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortItems; ++r) {
    int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of `n` uint32 in place, one block of 1024 threads
__global__ void __launch_bounds__(1024) k_scan_excl(uint32_t* __restrict__ a, int64_t n) {
  __shared__ uint32_t part[1024];
  int64_t per = (n + 1023) / 1024;
  int64_t s = threadIdx.x * per, e = s + per < n ? s + per : n;
  uint32_t sum = 0;
  for (int64_t i = s; i < e; ++i) sum += a[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    uint32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = s; i < e; ++i) {
    uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kSortThreads) k_scatter(const uint64_t* __restrict__ kin,
                                                          const uint32_t* __restrict__ vin,
                                                          uint64_t* __restrict__ kout,
                                                          uint32_t* __restrict__ vout, int64_t n,
                                                          int shift,
                                                          const uint32_t* __restrict__ offsets,
                                                          int nblocks) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[kSortWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  base[threadIdx.x] = offsets[(int64_t)threadIdx.x * nblocks + blockIdx.x];
  for (int w = 0; w < kSortWarps; ++w) wcnt[w][threadIdx.x] = 0;
  __syncthreads();
  const uint32_t lt_mask = (1u << lane) - 1u;
  int64_t tile = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortItems; ++r) {
    int64_t i = tile + r * kSortThreads + threadIdx.x;
    bool valid = i < n;
    uint64_t k = valid ? kin[i] : 0;
    uint32_t v = valid ? vin[i] : 0;
    uint32_t dg = valid ? (uint32_t)((k >> shift) & 255u) : 256u + lane;
    uint32_t peers = __match_any_sync(0xffffffffu, dg);
    uint32_t rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    {  // per-digit prefix over warps (thread = digit)
      uint32_t run = base[threadIdx.x];
      for (int w = 0; w < kSortWarps; ++w) {
        uint32_t c = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = run;
        run += c;
      }
      base[threadIdx.x] = run;
    }
    __syncthreads();
    if (valid) {
      uint32_t pos = wcnt[warp][dg] + rank;
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    for (int w = 0; w < kSortWarps; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
  }
}

int sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, Alloc& al, cudaStream_t st) {
  if (n <= 1) return UVD_OK;
  int nblocks = (int)((n + kSortTile - 1) / kSortTile);
  uint64_t* k2 = (uint64_t*)al.get(n * sizeof(uint64_t));
  uint32_t* v2 = (uint32_t*)al.get(n * sizeof(uint32_t));
  uint32_t* cnt = (uint32_t*)al.get((size_t)256 * nblocks * sizeof(uint32_t));
  if (!k2 || !v2 || !cnt) {
    set_error("sort: out of device memory (n=%lld)", (long long)n);
    return UVD_ERR_NOMEM;
  }
  uint64_t *ka = keys, *kb = k2;
  uint32_t *va = vals, *vb = v2;
  for (int pass = 0; pass < 8; ++pass) {   // 8 x 8 bits covers the 63-bit codes
    int shift = pass * 8;
    k_hist<<<nblocks, kSortThreads, 0, st>>>(ka, n, shift, cnt, nblocks);
    note_launch();
    k_scan_excl<<<1, 1024, 0, st>>>(cnt, (int64_t)256 * nblocks);
    note_launch();
    k_scatter<<<nblocks, kSortThreads, 0, st>>>(ka, va, kb, vb, n, shift, cnt, nblocks);
    note_launch();
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  // 8 passes: the result is back in (keys, vals)
  UVD_CUDA_TRY(cudaGetLastError());
  al.put(k2);
  al.put(v2);
  al.put(cnt);
  return UVD_OK;
}

// ----------------------------------------------------------------- karras --
__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int64_t n, int64_t i, int64_t j) {
  if (j < 0 || j >= n) return -1;
  uint64_t a = k[i], b = k[j];
  if (a == b) return 64 + __clzll((unsigned long long)(i ^ j));
  return __clzll((unsigned long long)(a ^ b));
}

// internal node i in [0, n-2]: range [first,last], children as refs into
// (internal: idx, leaf: 0x80000000|idx) -> int32 arrays
__global__ void k_karras(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ left,
                         int32_t* __restrict__ right, int32_t* __restrict__ rfirst,
                         int32_t* __restrict__ rlast, int32_t* __restrict__ parent_int,
                         int32_t* __restrict__ parent_leaf) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1) >= 0 ? 1 : -1;
  int dmin = delta(keys, n, i, i - d);
  int64_t lmax = 2;
  while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int64_t l = 0;
  for (int64_t t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
  int64_t j = i + l * d;
  int dnode = delta(keys, n, i, j);
  int64_t s = 0;
  int64_t len = l;
  // binary search for the split: largest s with delta(i, i+s*d) > dnode
  int64_t t = len;
  do {
    t = (t + 1) >> 1;
    if (s + t < len + 1 && delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
  int64_t first = d > 0 ? i : j, last = d > 0 ? j : i;
  int32_t lc, rc;
  if (first == gamma) { lc = (int32_t)(0x80000000u | (uint32_t)gamma); parent_leaf[gamma] = (int32_t)i; }
  else { lc = (int32_t)gamma; parent_int[gamma] = (int32_t)i; }
  if (last == gamma + 1) { rc = (int32_t)(0x80000000u | (uint32_t)(gamma + 1)); parent_leaf[gamma + 1] = (int32_t)i; }
  else { rc = (int32_t)(gamma + 1); parent_int[gamma + 1] = (int32_t)i; }
  left[i] = lc;
  right[i] = rc;
  rfirst[i] = (int32_t)first;
  rlast[i] = (int32_t)last;
}

struct Box { float lx, ly, lz, hx, hy, hz; };

__device__ __forceinline__ Box tri_box(const float4* __restrict__ tri, int64_t r) {
  float4 a = tri[3 * r], b = tri[3 * r + 1], c = tri[3 * r + 2];
  Box x;
  x.lx = fminf(a.x, fminf(b.x, c.x)); x.hx = fmaxf(a.x, fmaxf(b.x, c.x));
  x.ly = fminf(a.y, fminf(b.y, c.y)); x.hy = fmaxf(a.y, fmaxf(b.y, c.y));
  x.lz = fminf(a.z, fminf(b.z, c.z)); x.hz = fmaxf(a.z, fmaxf(b.z, c.z));
  return x;
}
__device__ __forceinline__ Box join(Box a, Box b) {
  Box x;
  x.lx = fminf(a.lx, b.lx); x.ly = fminf(a.ly, b.ly); x.lz = fminf(a.lz, b.lz);
  x.hx = fmaxf(a.hx, b.hx); x.hy = fmaxf(a.hy, b.hy); x.hz = fmaxf(a.hz, b.hz);
  return x;
}

__device__ __forceinline__ Box load_box(const float* __restrict__ bx, int64_t i) {
  const volatile float* p = bx + 6 * i;
  Box x;
  x.lx = p[0]; x.ly = p[1]; x.lz = p[2]; x.hx = p[3]; x.hy = p[4]; x.hz = p[5];
  return x;
}
__device__ __forceinline__ void store_box(float* bx, int64_t i, Box x) {
  volatile float* p = bx + 6 * i;
  p[0] = x.lx; p[1] = x.ly; p[2] = x.lz; p[3] = x.hx; p[4] = x.hy; p[5] = x.hz;
}

__global__ void k_refit(const float4* __restrict__ tri, int64_t n, const int32_t* __restrict__ left,
                        const int32_t* __restrict__ right, const int32_t* __restrict__ parent_int,
                        const int32_t* __restrict__ parent_leaf, float* __restrict__ ibox,
                        int* __restrict__ arrive) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t p = parent_leaf[r];
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(&arrive[p], 1) == 0) return;  // first child to arrive stops
    __threadfence();
    int32_t lc = left[p], rc = right[p];
    Box bl = lc < 0 ? tri_box(tri, (int64_t)(lc & 0x7fffffff)) : load_box(ibox, lc);
    Box br = rc < 0 ? tri_box(tri, (int64_t)(rc & 0x7fffffff)) : load_box(ibox, rc);
    store_box(ibox, p, join(bl, br));
    p = p == 0 ? -1 : parent_int[p];
  }
}

// Outward box padding: 1e-5 m + 1e-6 |x| + c_pad, where c_pad = 4 eps32 x the
// scene's largest |coordinate| (set per build) covers the rounding of the
// traversal's fp32 ray (its direction is fl32 of the exact one) and of the
// FFMA-form slab parameters (plane shift <= eps |origin|).
__device__ __forceinline__ float pad_lo(float x, float cp) { return x - (1e-5f + 1e-6f * fabsf(x) + cp); }
__device__ __forceinline__ float pad_hi(float x, float cp) { return x + (1e-5f + 1e-6f * fabsf(x) + cp); }

__device__ __forceinline__ void child_info(const float4* __restrict__ tri, const float* __restrict__ ibox,
                                           const int32_t* __restrict__ rfirst,
                                           const int32_t* __restrict__ rlast, int32_t c, Box* b,
                                           uint32_t* ref) {
  if (c < 0) {
    int64_t r = c & 0x7fffffff;
    *b = tri_box(tri, r);
    *ref = make_leaf((uint32_t)r, 1u);
  } else {
    *b = load_box(ibox, c);
    int32_t f = rfirst[c], l = rlast[c];
    int32_t cnt = l - f + 1;
    *ref = cnt <= kLeafMax ? make_leaf((uint32_t)f, (uint32_t)cnt) : (uint32_t)c;
  }
}

// depth-first preorder position of every internal node (root 0, left child =
// parent + 1, right child = parent + 1 + internal nodes of the left subtree), by
// walking up from the node: a node and its first child share a 128-B line half
// of the time, and subtrees are contiguous in memory
__global__ void k_preorder(const int32_t* __restrict__ left, const int32_t* __restrict__ parent_int,
                           const int32_t* __restrict__ rfirst, const int32_t* __restrict__ rlast,
                           int64_t n_int, int32_t* __restrict__ pre) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_int) return;
  int32_t acc = 0, c = (int32_t)v;
  while (c != 0) {
    const int32_t p = parent_int[c];
    const int32_t l = left[p];
    acc += 1;
    if (l != c && l >= 0) acc += rlast[l] - rfirst[l];  // internal nodes of the left subtree
    c = p;
  }
  pre[v] = acc;
}

__global__ void k_emit(const float4* __restrict__ tri, int64_t n, const int32_t* __restrict__ left,
                       const int32_t* __restrict__ right, const int32_t* __restrict__ rfirst,
                       const int32_t* __restrict__ rlast, const float* __restrict__ ibox,
                       const int32_t* __restrict__ pre, Node* __restrict__ nodes, float cp) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  Box b0, b1;
  uint32_t r0, r1;
  child_info(tri, ibox, rfirst, rlast, left[i], &b0, &r0);
  child_info(tri, ibox, rfirst, rlast, right[i], &b1, &r1);
  if (!ref_is_leaf(r0)) r0 = (uint32_t)pre[r0];
  if (!ref_is_leaf(r1)) r1 = (uint32_t)pre[r1];
  Node nd;
  nd.a = make_float4(pad_lo(b0.lx, cp), pad_hi(b0.hx, cp), pad_lo(b0.ly, cp), pad_hi(b0.hy, cp));
  nd.b = make_float4(pad_lo(b1.lx, cp), pad_hi(b1.hx, cp), pad_lo(b1.ly, cp), pad_hi(b1.hy, cp));
  nd.c = make_float4(pad_lo(b0.lz, cp), pad_hi(b0.hz, cp), pad_lo(b1.lz, cp), pad_hi(b1.hz, cp));
  nd.d = make_uint4(r0, r1, 0u, 0u);
  nodes[pre[i]] = nd;
}

// Octant copies of the nodes: copy o (bit 0/1/2 = the ray's 1/d is negative in
// x/y/z) stores every child box slab as (near plane, far plane) for rays of that
// octant, so the traversal takes the slab entry and exit without a min/max per
// axis, and pairs the two children's planes for the paired FMA (FFMA2):
//   a = (x entry c0, x entry c1, x exit c0, x exit c1), b = the same for y,
//   c = for z, d = child refs.
// Same boxes; internal child refs point into the same copy (+ o x nn).
__global__ void k_octant_nodes(const Node* __restrict__ nodes, int64_t nn, Node* __restrict__ onodes) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 8 * nn) return;
  const int o = (int)(i / nn);
  const Node nd = nodes[i - o * nn];
  Node on;
  const bool nx = o & 1, ny = o & 2, nz = o & 4;
  on.a = nx ? make_float4(nd.a.y, nd.b.y, nd.a.x, nd.b.x) : make_float4(nd.a.x, nd.b.x, nd.a.y, nd.b.y);
  on.b = ny ? make_float4(nd.a.w, nd.b.w, nd.a.z, nd.b.z) : make_float4(nd.a.z, nd.b.z, nd.a.w, nd.b.w);
  on.c = nz ? make_float4(nd.c.y, nd.c.w, nd.c.x, nd.c.z) : make_float4(nd.c.x, nd.c.z, nd.c.y, nd.c.w);
  on.d = nd.d;
  if (!ref_is_leaf(on.d.x)) on.d.x += (uint32_t)(o * nn);
  if (!ref_is_leaf(on.d.y)) on.d.y += (uint32_t)(o * nn);
  onodes[i] = on;
}

// single-leaf scene (M <= kLeafMax): a root node with one leaf child and an
// empty second child
__global__ void k_emit_small(const float4* __restrict__ tri, int64_t n, Node* nodes, float cp) {
  Box b = tri_box(tri, 0);
  for (int64_t r = 1; r < n; ++r) b = join(b, tri_box(tri, r));
  Node nd;
  nd.a = make_float4(pad_lo(b.lx, cp), pad_hi(b.hx, cp), pad_lo(b.ly, cp), pad_hi(b.hy, cp));
  nd.b = make_float4(1.f, -1.f, 1.f, -1.f);  // empty box: never hit
  nd.c = make_float4(pad_lo(b.lz, cp), pad_hi(b.hz, cp), 1.f, -1.f);
  nd.d = make_uint4(make_leaf(0u, (uint32_t)n), make_leaf(0u, 1u), 0u, 0u);
  nodes[0] = nd;
}

// ------------------------------------------------------------------ PLOC --
// Parallel Locally-Ordered Clustering (Meister & Bittner 2018): start from one
// cluster per triangle in Morton order; every round each cluster finds its
// nearest neighbour (smallest surface area of the union box) within a window
// of +-kPlocRadius positions, mutual nearest neighbours merge into a new
// internal node, and the surviving clusters are compacted in order.  Yields a
// tree of markedly better SAH quality than the Karras LBVH (fewer node visits
// per shadow ray), in the same (left, right, range, box) arrays.

#ifndef UVD_PLOC_RADIUS
#define UVD_PLOC_RADIUS 24
#endif
constexpr int kPlocRadius = UVD_PLOC_RADIUS;

__device__ __forceinline__ float union_area(const float* __restrict__ a, const float* __restrict__ b) {
  float dx = fmaxf(a[3], b[3]) - fminf(a[0], b[0]);
  float dy = fmaxf(a[4], b[4]) - fminf(a[1], b[1]);
  float dz = fmaxf(a[5], b[5]) - fminf(a[2], b[2]);
  return dx * dy + dy * dz + dz * dx;
}

// cluster k: box cbox[6k..6k+5], node id cid[k] (< 0: leaf triangle ~cid)
__global__ void k_ploc_init(const float4* __restrict__ tri, int64_t n, float* __restrict__ cbox,
                            int32_t* __restrict__ cid) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Box x = tri_box(tri, i);
  float* o = cbox + 6 * i;
  o[0] = x.lx; o[1] = x.ly; o[2] = x.lz; o[3] = x.hx; o[4] = x.hy; o[5] = x.hz;
  cid[i] = (int32_t)(0x80000000u | (uint32_t)i);
}

__global__ void k_ploc_nn(const float* __restrict__ cbox, const int* __restrict__ n_ptr,
                          int32_t* __restrict__ nn) {
  const int n = *n_ptr;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* bi = cbox + 6 * i;
  float best = INFINITY;
  int bj = -1;
  const int lo = max(0, i - kPlocRadius), hi = min(n - 1, i + kPlocRadius);
  for (int j = lo; j <= hi; ++j) {
    if (j == i) continue;
    float d = union_area(bi, cbox + 6 * j);
    if (d < best || (d == best && j < bj)) { best = d; bj = j; }
  }
  nn[i] = bj;
}

// flag[i] = 1 if cluster i survives (merge leader or unmerged); merges[i] = 1
// if i leads a merge
__global__ void k_ploc_flags(const int32_t* __restrict__ nn, const int* __restrict__ n_ptr,
                             int32_t* __restrict__ keep, int32_t* __restrict__ lead) {
  const int n = *n_ptr;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = nn[i];
  const bool mutual = j >= 0 && nn[j] == i;
  lead[i] = mutual && i < j;
  keep[i] = !mutual || i < j;
}

// inclusive scans of two int32 arrays (<= 2^31) in one block
__global__ void __launch_bounds__(1024) k_scan2_incl(int32_t* __restrict__ a, int32_t* __restrict__ b,
                                                     const int* __restrict__ n_ptr) {
  __shared__ int32_t pa[1024], pb[1024];
  const int n = *n_ptr;
  const int per = (n + 1023) / 1024;
  const int s = threadIdx.x * per, e = min(s + per, n);
  int32_t sa = 0, sb = 0;
  for (int i = s; i < e; ++i) { sa += a[i]; sb += b[i]; }
  pa[threadIdx.x] = sa;
  pb[threadIdx.x] = sb;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int32_t va = threadIdx.x >= off ? pa[threadIdx.x - off] : 0;
    int32_t vb = threadIdx.x >= off ? pb[threadIdx.x - off] : 0;
    __syncthreads();
    pa[threadIdx.x] += va;
    pb[threadIdx.x] += vb;
    __syncthreads();
  }
  int32_t ra = threadIdx.x ? pa[threadIdx.x - 1] : 0, rb = threadIdx.x ? pb[threadIdx.x - 1] : 0;
  for (int i = s; i < e; ++i) { ra += a[i]; a[i] = ra; rb += b[i]; b[i] = rb; }
}

// merge leaders create node (node_base + lead_rank); survivors compact into
// the output arrays in order; the new cluster count is written to n_out
__global__ void k_ploc_merge(const float* __restrict__ cbox, const int32_t* __restrict__ cid,
                             const int32_t* __restrict__ nn, const int32_t* __restrict__ keep_incl,
                             const int32_t* __restrict__ lead_incl, const int* __restrict__ n_ptr,
                             const int* __restrict__ node_base, float* __restrict__ cbox_out,
                             int32_t* __restrict__ cid_out, int32_t* __restrict__ left,
                             int32_t* __restrict__ right, float* __restrict__ ibox,
                             int32_t* __restrict__ parent_int, int32_t* __restrict__ parent_leaf,
                             int* __restrict__ n_out, int* __restrict__ node_base_out) {
  const int n = *n_ptr;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    *n_out = keep_incl[n - 1];
    *node_base_out = *node_base - lead_incl[n - 1];
  }
  if (i >= n) return;
  const int kept = keep_incl[i] - (i ? keep_incl[i - 1] : 0);
  if (!kept) return;
  const int o = keep_incl[i] - 1;
  const int j = nn[i];
  const bool lead = (lead_incl[i] - (i ? lead_incl[i - 1] : 0)) != 0;
  float* bo = cbox_out + 6 * o;
  if (!lead) {
    for (int k = 0; k < 6; ++k) bo[k] = cbox[6 * i + k];
    cid_out[o] = cid[i];
    return;
  }
  // internal nodes are numbered downwards from n_tris - 2 so the last merge is the root (0)
  const int node = *node_base - lead_incl[i];
  const float* a = cbox + 6 * i;
  const float* b = cbox + 6 * j;
  float u[6] = {fminf(a[0], b[0]), fminf(a[1], b[1]), fminf(a[2], b[2]),
                fmaxf(a[3], b[3]), fmaxf(a[4], b[4]), fmaxf(a[5], b[5])};
  for (int k = 0; k < 6; ++k) { bo[k] = u[k]; ibox[6 * node + k] = u[k]; }
  const int32_t ci = cid[i], cj = cid[j];
  left[node] = ci;
  right[node] = cj;
  if (ci < 0) parent_leaf[ci & 0x7fffffff] = node; else parent_int[ci] = node;
  if (cj < 0) parent_leaf[cj & 0x7fffffff] = node; else parent_int[cj] = node;
  cid_out[o] = node;
}

// subtree sizes bottom-up (arrival counters, like the refit)
__global__ void k_subtree_size(const int32_t* __restrict__ parent_leaf, const int32_t* __restrict__ parent_int,
                               const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                               int64_t n, int32_t* __restrict__ size, int* __restrict__ arrive) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int32_t p = parent_leaf[r];
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(&arrive[p], 1) == 0) return;
    __threadfence();
    const int32_t l = left[p], q = right[p];
    const int32_t sl = l < 0 ? 1 : ((volatile int32_t*)size)[l];
    const int32_t sr = q < 0 ? 1 : ((volatile int32_t*)size)[q];
    ((volatile int32_t*)size)[p] = sl + sr;
    p = p == 0 ? -1 : parent_int[p];
  }
}

// DFS leaf order: first[node] = number of leaves left of the subtree, found by
// walking up from each node; each triangle's new position is first of its leaf
__global__ void k_dfs_first(const int32_t* __restrict__ parent_int, const int32_t* __restrict__ left,
                            const int32_t* __restrict__ size, int64_t n_int, int32_t* __restrict__ first) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_int) return;
  int32_t off = 0, c = (int32_t)v;
  while (c != 0) {
    const int32_t p = parent_int[c];
    if (left[p] != c) {  // c is the right child: everything under the left sibling precedes it
      const int32_t l = left[p];
      off += l < 0 ? 1 : size[l];
    }
    c = p;
  }
  first[v] = off;
}

__global__ void k_leaf_pos(const int32_t* __restrict__ parent_leaf, const int32_t* __restrict__ left,
                           const int32_t* __restrict__ right, const int32_t* __restrict__ size,
                           const int32_t* __restrict__ first, int64_t n, int32_t* __restrict__ pos) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t p = parent_leaf[r];
  const int32_t me = (int32_t)(0x80000000u | (uint32_t)r);
  if (left[p] == me) pos[r] = first[p];
  else pos[r] = first[p] + (left[p] < 0 ? 1 : size[left[p]]);
}

// rewrite leaf refs to DFS positions and compute node ranges
__global__ void k_ploc_finish(int32_t* __restrict__ left, int32_t* __restrict__ right,
                              const int32_t* __restrict__ size, const int32_t* __restrict__ first,
                              const int32_t* __restrict__ pos, int64_t n_int, int32_t* __restrict__ rfirst,
                              int32_t* __restrict__ rlast) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_int) return;
  int32_t l = left[v], r = right[v];
  if (l < 0) left[v] = (int32_t)(0x80000000u | (uint32_t)pos[l & 0x7fffffff]);
  if (r < 0) right[v] = (int32_t)(0x80000000u | (uint32_t)pos[r & 0x7fffffff]);
  rfirst[v] = first[v];
  rlast[v] = first[v] + size[v] - 1;
}

__global__ void k_scatter_tri(const float4* __restrict__ in, const int32_t* __restrict__ pos, int64_t n,
                              float4* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t d = pos[r];
  out[3 * d] = in[3 * r];
  out[3 * d + 1] = in[3 * r + 1];
  out[3 * d + 2] = in[3 * r + 2];
}

__global__ void k_scatter_u32(const uint32_t* __restrict__ in, const int32_t* __restrict__ pos, int64_t n,
                              uint32_t* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) out[pos[r]] = in[r];
}

// 3D scenes: the owner (row) of the triangle at Morton position r is r
__global__ void k_set_owner(float4* __restrict__ tri, int64_t n) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) tri[3 * r].w = __int_as_float((int)r);
}

// gather input-order triangles into sorted (leaf) order
__global__ void k_gather_tri(const float4* __restrict__ tri_in, const uint32_t* __restrict__ order,
                             int64_t M, float4* __restrict__ tri) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= M) return;
  int64_t t = order[r];
  tri[3 * r] = tri_in[3 * t];
  tri[3 * r + 1] = tri_in[3 * t + 1];
  tri[3 * r + 2] = tri_in[3 * t + 2];
}

static inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// PLOC driver: clusters -> binary tree (left/right/ibox/parents), then DFS
// leaf order (triangles reordered so every subtree is a contiguous range).
static int build_ploc(uvd_scene* s, int64_t M, int32_t* left, int32_t* right, int32_t* rf, int32_t* rl,
                      int32_t* pint, int32_t* pleaf, float* ibox, int* arrive, uint32_t* order,
                      cudaStream_t st) {
  Scratch al(s->alloc, st);  // released at every exit
  float* cbA = (float*)al.get(M * 6 * sizeof(float));
  float* cbB = (float*)al.get(M * 6 * sizeof(float));
  int32_t* idA = (int32_t*)al.get(M * 4);
  int32_t* idB = (int32_t*)al.get(M * 4);
  int32_t* nn = (int32_t*)al.get(M * 4);
  int32_t* keep = (int32_t*)al.get(M * 4);
  int32_t* lead = (int32_t*)al.get(M * 4);
  int* ctr = (int*)al.get(4 * sizeof(int));  // nA, baseA, nB, baseB
  float4* tri2 = (float4*)al.get(3 * M * sizeof(float4));
  if (!cbA || !cbB || !idA || !idB || !nn || !keep || !lead || !ctr || !tri2) {
    set_error("scene: out of device memory (PLOC scratch)");
    return UVD_ERR_NOMEM;
  }
  k_ploc_init<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M, cbA, idA);
  note_launch();
  int h[4] = {(int)M, (int)(M - 1), 0, 0};
  UVD_CUDA_TRY(cudaMemcpyAsync(ctr, h, 4 * sizeof(int), cudaMemcpyHostToDevice, st));
  int n_host = (int)M, iters = 0;
  while (n_host > 1) {
    for (int sub = 0; sub < 4; ++sub, ++iters) {
      const unsigned g = grid_for(n_host, 256);
      k_ploc_nn<<<g, 256, 0, st>>>(cbA, ctr + 0, nn);
      k_ploc_flags<<<g, 256, 0, st>>>(nn, ctr + 0, keep, lead);
      k_scan2_incl<<<1, 1024, 0, st>>>(keep, lead, ctr + 0);
      k_ploc_merge<<<g, 256, 0, st>>>(cbA, idA, nn, keep, lead, ctr + 0, ctr + 1, cbB, idB, left, right,
                                      ibox, pint, pleaf, ctr + 2, ctr + 3);
      note_launch(4);
      UVD_CUDA_TRY(cudaMemcpyAsync(ctr, ctr + 2, 2 * sizeof(int), cudaMemcpyDeviceToDevice, st));
      std::swap(cbA, cbB);
      std::swap(idA, idB);
    }
    UVD_CUDA_TRY(cudaMemcpyAsync(h, ctr, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    n_host = h[0];
    if (iters > 8192) { set_error("scene: PLOC did not converge"); return UVD_ERR_CUDA; }
  }
  // subtree sizes, DFS positions, reorder triangles, leaf refs -> positions
  const int64_t ni = M - 1;
  int32_t* size = keep;   // reuse scratch (sizes of internal nodes)
  int32_t* first = lead;
  int32_t* pos = nn;
  k_subtree_size<<<grid_for(M, 256), 256, 0, st>>>(pleaf, pint, left, right, M, size, arrive);
  k_dfs_first<<<grid_for(ni, 256), 256, 0, st>>>(pint, left, size, ni, first);
  k_leaf_pos<<<grid_for(M, 256), 256, 0, st>>>(pleaf, left, right, size, first, M, pos);
  k_scatter_tri<<<grid_for(M, 256), 256, 0, st>>>(s->tri, pos, M, tri2);
  k_ploc_finish<<<grid_for(ni, 256), 256, 0, st>>>(left, right, size, first, pos, ni, rf, rl);
  note_launch(5);
  UVD_CUDA_TRY(cudaMemcpyAsync(s->tri, tri2, 3 * M * sizeof(float4), cudaMemcpyDeviceToDevice, st));
#if UVD_ROWS_DFS
  if (s->kind == UVD_SCENE_TRIMESH) {
    // 3D rows follow the BVH leaf (DFS) order: adjacent rows are adjacent leaves
    uint32_t* ord2 = (uint32_t*)tri2;  // reuse the scratch (>= 4 B per triangle)
    k_scatter_u32<<<grid_for(M, 256), 256, 0, st>>>(order, pos, M, ord2);
    k_set_owner<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M);
    note_launch(2);
    UVD_CUDA_TRY(cudaMemcpyAsync(order, ord2, M * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
#endif
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

// ---------------------------------------------------------------------------
// Top-down binned-SAH builder (UVD_BVH=sah): level-synchronous, one CTA per
// node of the level; the CTA bins its triangles' box centres (16 bins per
// axis; bin boxes kept exact with ordered-int shared-memory atomics), sweeps
// the bins for the split of least SAH cost, partitions its range stably (left
// first, so every subtree is a contiguous DFS range), and creates its children
// (a single triangle is a leaf reference).  Node boxes come from k_refit.
#ifndef UVD_SAH_BINS
#define UVD_SAH_BINS 32
#endif
constexpr int kSahBins = UVD_SAH_BINS;
constexpr int kSahBig = 8192;     // nodes above this many triangles get 1024-thread CTAs
constexpr int kSahHuge = 65536;   // ... and above this, several CTAs (chunks of kSahChunk)
constexpr int kSahChunk = 32768;

__device__ __forceinline__ int f2o(float f) {  // order-preserving float -> int
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// half the box surface; explicit roundings (no contraction) so every sweep of
// the builder computes the same cost bits for the same bins
__device__ __forceinline__ float sah_area(float lx, float ly, float lz, float hx, float hy, float hz) {
  const float dx = __fsub_rn(hx, lx), dy = __fsub_rn(hy, ly), dz = __fsub_rn(hz, lz);
  return __fadd_rn(__fadd_rn(__fmul_rn(dx, dy), __fmul_rn(dy, dz)), __fmul_rn(dz, dx));
}
__device__ __forceinline__ float sah_cost(float area_l, int n_l, float area_r, int n_r) {
  return __fadd_rn(__fmul_rn(area_l, (float)n_l), __fmul_rn(area_r, (float)n_r));
}

// children of a split node: a single triangle is a leaf reference, larger
// ranges become internal nodes routed to the next level's small / big / huge list
__device__ void sah_children(int node, int first, int last, int nl, int32_t* rf, int32_t* rl, int32_t* left,
                             int32_t* right, int32_t* pint, int32_t* pleaf, int* ctr, int32_t* next,
                             int32_t* next_big, int32_t* next_huge, int huge) {
  const int lo[2] = {first, first + nl}, hi[2] = {first + nl - 1, last};
  int32_t ref[2];
  for (int s = 0; s < 2; ++s) {
    if (hi[s] == lo[s]) {
      ref[s] = (int32_t)(0x80000000u | (uint32_t)lo[s]);
      pleaf[lo[s]] = node;
      continue;
    }
    const int id = atomicAdd(&ctr[0], 1);
    rf[id] = lo[s]; rl[id] = hi[s]; pint[id] = node;
    const int n = hi[s] - lo[s] + 1;
    if (n > huge) next_huge[atomicAdd(&ctr[3], 1)] = id;
    else if (n > kSahBig) next_big[atomicAdd(&ctr[2], 1)] = id;
    else next[atomicAdd(&ctr[1], 1)] = id;
    ref[s] = id;
  }
  left[node] = ref[0];
  right[node] = ref[1];
}

template <int kSahThreads>
__global__ void __launch_bounds__(kSahThreads) k_sah_split(const float4* __restrict__ tri, int32_t* __restrict__ perm,
                                                           int32_t* __restrict__ tmp, const int32_t* __restrict__ list,
                                                           int32_t* __restrict__ rf, int32_t* __restrict__ rl,
                                                           int32_t* __restrict__ left, int32_t* __restrict__ right,
                                                           int32_t* __restrict__ pint, int32_t* __restrict__ pleaf,
                                                           int* __restrict__ ctr, int32_t* __restrict__ next,
                                                           int32_t* __restrict__ next_big, int32_t* __restrict__ next_huge, int huge) {
  __shared__ int s_cnt[3][kSahBins];
  __shared__ int s_lo[3][kSahBins][3], s_hi[3][kSahBins][3];
  __shared__ int s_cb[6];      // centre bounds (ordered ints)
  __shared__ int s_split[3];  // axis, bin, n_left
  __shared__ int s_scan[kSahThreads / 32];
  __shared__ float s_cost[3];
  __shared__ int s_bin[3], s_nl[3];
  static_assert(kSahBins == 32 && kSahThreads >= 96, "the sweep maps one warp per axis, one lane per bin");
  const int node = list[blockIdx.x];
  const int first = rf[node], last = rl[node], n = last - first + 1;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // 1. bounds of the box centres
  float cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int p = first + tid; p <= last; p += kSahThreads) {
    const Box b = tri_box(tri, perm[p]);
    const float c[3] = {0.5f * (b.lx + b.hx), 0.5f * (b.ly + b.hy), 0.5f * (b.lz + b.hz)};
    for (int a = 0; a < 3; ++a) { cl[a] = fminf(cl[a], c[a]); ch[a] = fmaxf(ch[a], c[a]); }
  }
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      cl[a] = fminf(cl[a], __shfl_xor_sync(0xffffffffu, cl[a], o));
      ch[a] = fmaxf(ch[a], __shfl_xor_sync(0xffffffffu, ch[a], o));
    }
  // bins cleared; centre bounds reduced across warps as ordered ints
  for (int q = tid; q < 3 * kSahBins; q += kSahThreads) {
    const int a = q / kSahBins, b = q % kSahBins;
    s_cnt[a][b] = 0;
    for (int k = 0; k < 3; ++k) { s_lo[a][b][k] = 0x7fffffff; s_hi[a][b][k] = (int)0x80000000; }
  }
  if (tid < 6) s_cb[tid] = tid < 3 ? 0x7fffffff : (int)0x80000000;
  __syncthreads();
  if (lane == 0)
    for (int a = 0; a < 3; ++a) {
      atomicMin(&s_cb[a], f2o(cl[a]));
      atomicMax(&s_cb[3 + a], f2o(ch[a]));
    }
  __syncthreads();
  float cmin[3], cscale[3];
  for (int a = 0; a < 3; ++a) {
    const float lo = o2f(s_cb[a]), hi = o2f(s_cb[3 + a]);
    cmin[a] = lo;
    cscale[a] = hi > lo ? (float)kSahBins / (hi - lo) : 0.f;
  }
  // 2. bins (skipped for n == 2: split at the middle)
  if (n > 2) {
    // each thread bins a contiguous run: the input is Morton-ordered, so lanes
    // striding by one would all hit the same few bins (serialised atomics)
    const int per = (n + kSahThreads - 1) / kSahThreads;
    const int p_end = min(first + (tid + 1) * per, last + 1);
    for (int p = first + tid * per; p < p_end; ++p) {
      const Box b = tri_box(tri, perm[p]);
      const float c[3] = {0.5f * (b.lx + b.hx), 0.5f * (b.ly + b.hy), 0.5f * (b.lz + b.hz)};
      const int lo[3] = {f2o(b.lx), f2o(b.ly), f2o(b.lz)}, hi[3] = {f2o(b.hx), f2o(b.hy), f2o(b.hz)};
      for (int a = 0; a < 3; ++a) {
        if (cscale[a] == 0.f) continue;
        const int bin = min(kSahBins - 1, max(0, (int)((c[a] - cmin[a]) * cscale[a])));
        atomicAdd(&s_cnt[a][bin], 1);
        for (int k = 0; k < 3; ++k) { atomicMin(&s_lo[a][bin][k], lo[k]); atomicMax(&s_hi[a][bin][k], hi[k]); }
      }
    }
  }
  __syncthreads();
  // 3. sweep: least SAH cost split among the 3 x (B-1) bin planes; warp a scans
  // axis a (lane = bin: prefix / suffix boxes by shuffles), ties to the lowest
  // (axis, bin) as a sequential sweep would take them
  if (wid < 3) {
    const int ax = wid, b = lane;
    const bool on = n > 2 && cscale[ax] != 0.f;
    int c = 0;
    float l0 = INFINITY, l1 = INFINITY, l2 = INFINITY, h0 = -INFINITY, h1 = -INFINITY, h2 = -INFINITY;
    if (on && s_cnt[ax][b]) {
      c = s_cnt[ax][b];
      l0 = o2f(s_lo[ax][b][0]); l1 = o2f(s_lo[ax][b][1]); l2 = o2f(s_lo[ax][b][2]);
      h0 = o2f(s_hi[ax][b][0]); h1 = o2f(s_hi[ax][b][1]); h2 = o2f(s_hi[ax][b][2]);
    }
    float pl0 = l0, pl1 = l1, pl2 = l2, ph0 = h0, ph1 = h1, ph2 = h2;  // bins <= b
    float ql0 = l0, ql1 = l1, ql2 = l2, qh0 = h0, qh1 = h1, qh2 = h2;  // bins >= b
    int pc = c, qc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const float u0 = __shfl_up_sync(0xffffffffu, pl0, o), u1 = __shfl_up_sync(0xffffffffu, pl1, o);
      const float u2 = __shfl_up_sync(0xffffffffu, pl2, o), v0 = __shfl_up_sync(0xffffffffu, ph0, o);
      const float v1 = __shfl_up_sync(0xffffffffu, ph1, o), v2 = __shfl_up_sync(0xffffffffu, ph2, o);
      const int uc = __shfl_up_sync(0xffffffffu, pc, o);
      if (lane >= o) {
        pl0 = fminf(pl0, u0); pl1 = fminf(pl1, u1); pl2 = fminf(pl2, u2);
        ph0 = fmaxf(ph0, v0); ph1 = fmaxf(ph1, v1); ph2 = fmaxf(ph2, v2);
        pc += uc;
      }
      const float w0 = __shfl_down_sync(0xffffffffu, ql0, o), w1 = __shfl_down_sync(0xffffffffu, ql1, o);
      const float w2 = __shfl_down_sync(0xffffffffu, ql2, o), x0 = __shfl_down_sync(0xffffffffu, qh0, o);
      const float x1 = __shfl_down_sync(0xffffffffu, qh1, o), x2 = __shfl_down_sync(0xffffffffu, qh2, o);
      const int wc = __shfl_down_sync(0xffffffffu, qc, o);
      if (lane + o < 32) {
        ql0 = fminf(ql0, w0); ql1 = fminf(ql1, w1); ql2 = fminf(ql2, w2);
        qh0 = fmaxf(qh0, x0); qh1 = fmaxf(qh1, x1); qh2 = fmaxf(qh2, x2);
        qc += wc;
      }
    }
    // the right side of the plane after bin b is the suffix from bin b + 1
    const float r0 = __shfl_down_sync(0xffffffffu, ql0, 1), r1 = __shfl_down_sync(0xffffffffu, ql1, 1);
    const float r2 = __shfl_down_sync(0xffffffffu, ql2, 1), s0 = __shfl_down_sync(0xffffffffu, qh0, 1);
    const float s1 = __shfl_down_sync(0xffffffffu, qh1, 1), s2 = __shfl_down_sync(0xffffffffu, qh2, 1);
    const int rc = __shfl_down_sync(0xffffffffu, qc, 1);
    float cost = INFINITY;
    if (on && b < kSahBins - 1 && pc > 0 && rc > 0)
      cost = sah_cost(sah_area(pl0, pl1, pl2, ph0, ph1, ph2), pc, sah_area(r0, r1, r2, s0, s1, s2), rc);
    // warp argmin (cost, bin)
    float bc = cost;
    int bbin = cost < INFINITY ? b : kSahBins, bnl = pc;
    for (int o = 16; o > 0; o >>= 1) {
      const float oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bbin, o), onl = __shfl_xor_sync(0xffffffffu, bnl, o);
      if (oc < bc || (oc == bc && ob < bbin)) { bc = oc; bbin = ob; bnl = onl; }
    }
    if (lane == 0) { s_cost[ax] = bc; s_bin[ax] = bbin; s_nl[ax] = bnl; }
  }
  __syncthreads();
  if (tid == 0) {
    int ba = -1, bb = -1, bnl = 0;
    float best = INFINITY;
    for (int ax = 0; ax < 3; ++ax)
      if (s_bin[ax] < kSahBins && s_cost[ax] < best) { best = s_cost[ax]; ba = ax; bb = s_bin[ax]; bnl = s_nl[ax]; }
    s_split[0] = ba;  // -1: median split by position
    s_split[1] = bb;
    s_split[2] = ba < 0 ? n / 2 : bnl;
  }
  __syncthreads();
  const int sa = s_split[0], sb = s_split[1], nl = s_split[2];
  // 4. stable partition of the range (left first) through tmp
  if (sa >= 0) {
    int base_l = 0, base_r = 0;
    for (int p0 = first; p0 <= last; p0 += kSahThreads) {
      const int p = p0 + tid;
      int flag = 0, t = 0;
      if (p <= last) {
        t = perm[p];
        const Box b = tri_box(tri, t);
        const float c = sa == 0 ? 0.5f * (b.lx + b.hx) : sa == 1 ? 0.5f * (b.ly + b.hy) : 0.5f * (b.lz + b.hz);
        const int bin = min(kSahBins - 1, max(0, (int)((c - cmin[sa]) * cscale[sa])));
        flag = bin <= sb;
      }
      // block exclusive scan of flag
      const unsigned bal = __ballot_sync(0xffffffffu, flag);
      const int in_warp = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) s_scan[wid] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int w = 0; w < kSahThreads / 32; ++w) {
        const int v = s_scan[w];
        if (w < wid) before += v;
        total += v;
      }
      if (p <= last) {
        const int rank_l = base_l + before + in_warp;
        const int idx = p - p0;
        const int rank_r = base_r + (idx - (before + in_warp));
        tmp[flag ? first + rank_l : first + nl + rank_r] = t;
      }
      const int chunk = min(kSahThreads, last - p0 + 1);
      base_l += total;
      base_r += chunk - total;
      __syncthreads();
    }
    __syncthreads();
    for (int p = first + tid; p <= last; p += kSahThreads) perm[p] = tmp[p];
  }
  // 5. children
  if (tid == 0) sah_children(node, first, last, nl, rf, rl, left, right, pint, pleaf, ctr, next, next_big, next_huge, huge);
}

// ---- huge nodes: several CTAs per node, one per chunk of kSahChunk positions ----
struct SahChunks {
  const int32_t* node;   // [n_chunks] node id
  const int32_t* hidx;   // [n_chunks] index of the node in this level's huge list
  const int32_t* cbeg;   // [n_chunks] first position
  const int32_t* cend;   // [n_chunks] last position + 1
  const int32_t* hfirst; // [n_huge + 1] first chunk of each huge node
  int* cb;               // [n_huge][6] centre bounds (ordered ints)
  int* bcnt;             // [n_huge][3][B] bin counts
  int* blo;              // [n_huge][3][B][3] bin box lows (ordered ints)
  int* bhi;              // [n_huge][3][B][3]
  int* ccnt;             // [n_chunks][3][B] per-chunk bin counts
  int* split;            // [n_huge][3] axis, bin, n_left
  int* off;              // [n_chunks][2] left / right offsets of each chunk within its node
};

constexpr int kHugeThreads = 1024;
static_assert(3 * kSahBins <= kHugeThreads, "the huge-node kernels clear / merge one bin per thread");

__global__ void __launch_bounds__(kHugeThreads) k_sah_huge_bounds(const float4* __restrict__ tri,
                                                                   const int32_t* __restrict__ perm, SahChunks C) {
  const int c = blockIdx.x, h = C.hidx[c];
  float cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int p = C.cbeg[c] + threadIdx.x; p < C.cend[c]; p += kHugeThreads) {
    const Box b = tri_box(tri, perm[p]);
    const float x[3] = {0.5f * (b.lx + b.hx), 0.5f * (b.ly + b.hy), 0.5f * (b.lz + b.hz)};
    for (int a = 0; a < 3; ++a) { cl[a] = fminf(cl[a], x[a]); ch[a] = fmaxf(ch[a], x[a]); }
  }
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      cl[a] = fminf(cl[a], __shfl_xor_sync(0xffffffffu, cl[a], o));
      ch[a] = fmaxf(ch[a], __shfl_xor_sync(0xffffffffu, ch[a], o));
    }
  if ((threadIdx.x & 31) == 0)
    for (int a = 0; a < 3; ++a) { atomicMin(&C.cb[6 * h + a], f2o(cl[a])); atomicMax(&C.cb[6 * h + 3 + a], f2o(ch[a])); }
}

__device__ __forceinline__ void huge_scale(const SahChunks& C, int h, float* cmin, float* cscale) {
  for (int a = 0; a < 3; ++a) {
    const float lo = o2f(C.cb[6 * h + a]), hi = o2f(C.cb[6 * h + 3 + a]);
    cmin[a] = lo;
    cscale[a] = hi > lo ? (float)kSahBins / (hi - lo) : 0.f;
  }
}

__global__ void __launch_bounds__(kHugeThreads) k_sah_huge_bins(const float4* __restrict__ tri,
                                                                 const int32_t* __restrict__ perm, SahChunks C) {
  __shared__ int s_cnt[3][kSahBins];
  __shared__ int s_lo[3][kSahBins][3], s_hi[3][kSahBins][3];
  const int c = blockIdx.x, h = C.hidx[c], tid = threadIdx.x;
  if (tid < 3 * kSahBins) {
    const int a = tid / kSahBins, b = tid % kSahBins;
    s_cnt[a][b] = 0;
    for (int k = 0; k < 3; ++k) { s_lo[a][b][k] = 0x7fffffff; s_hi[a][b][k] = (int)0x80000000; }
  }
  __syncthreads();
  float cmin[3], cscale[3];
  huge_scale(C, h, cmin, cscale);
  const int beg = C.cbeg[c], n = C.cend[c] - beg;
  const int per = (n + kHugeThreads - 1) / kHugeThreads;
  const int p_end = min(beg + (tid + 1) * per, beg + n);
  for (int p = beg + tid * per; p < p_end; ++p) {
    const Box b = tri_box(tri, perm[p]);
    const float x[3] = {0.5f * (b.lx + b.hx), 0.5f * (b.ly + b.hy), 0.5f * (b.lz + b.hz)};
    const int lo[3] = {f2o(b.lx), f2o(b.ly), f2o(b.lz)}, hi[3] = {f2o(b.hx), f2o(b.hy), f2o(b.hz)};
    for (int a = 0; a < 3; ++a) {
      if (cscale[a] == 0.f) continue;
      const int bin = min(kSahBins - 1, max(0, (int)((x[a] - cmin[a]) * cscale[a])));
      atomicAdd(&s_cnt[a][bin], 1);
      for (int k = 0; k < 3; ++k) { atomicMin(&s_lo[a][bin][k], lo[k]); atomicMax(&s_hi[a][bin][k], hi[k]); }
    }
  }
  __syncthreads();
  if (tid < 3 * kSahBins) {
    const int a = tid / kSahBins, b = tid % kSahBins, cnt = s_cnt[a][b];
    C.ccnt[(c * 3 + a) * kSahBins + b] = cnt;
    if (cnt) {
      atomicAdd(&C.bcnt[(h * 3 + a) * kSahBins + b], cnt);
      for (int k = 0; k < 3; ++k) {
        atomicMin(&C.blo[((h * 3 + a) * kSahBins + b) * 3 + k], s_lo[a][b][k]);
        atomicMax(&C.bhi[((h * 3 + a) * kSahBins + b) * 3 + k], s_hi[a][b][k]);
      }
    }
  }
}

// one thread per huge node: the split, the chunks' partition offsets, the children
__global__ void k_sah_huge_decide(const int32_t* __restrict__ list, int n_huge, SahChunks C, int32_t* rf, int32_t* rl,
                                  int32_t* left, int32_t* right, int32_t* pint, int32_t* pleaf, int* ctr,
                                  int32_t* next, int32_t* next_big, int32_t* next_huge, int huge) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_huge) return;
  const int node = list[h], first = rf[node], last = rl[node], n = last - first + 1;
  float cmin[3], cscale[3];
  huge_scale(C, h, cmin, cscale);
  float best = INFINITY;
  int ba = -1, bb = -1, bnl = 0;
  for (int a = 0; a < 3; ++a) {
    if (cscale[a] == 0.f) continue;
    const int* cnt = C.bcnt + (h * 3 + a) * kSahBins;
    const int* blo = C.blo + (h * 3 + a) * kSahBins * 3;
    const int* bhi = C.bhi + (h * 3 + a) * kSahBins * 3;
    float rarea[kSahBins];
    int rcnt[kSahBins];
    float lx = INFINITY, ly = INFINITY, lz = INFINITY, hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
    int c = 0;
    for (int b = kSahBins - 1; b >= 0; --b) {
      if (cnt[b]) {
        lx = fminf(lx, o2f(blo[3 * b])); ly = fminf(ly, o2f(blo[3 * b + 1])); lz = fminf(lz, o2f(blo[3 * b + 2]));
        hx = fmaxf(hx, o2f(bhi[3 * b])); hy = fmaxf(hy, o2f(bhi[3 * b + 1])); hz = fmaxf(hz, o2f(bhi[3 * b + 2]));
        c += cnt[b];
      }
      rarea[b] = c ? sah_area(lx, ly, lz, hx, hy, hz) : 0.f;
      rcnt[b] = c;
    }
    lx = ly = lz = INFINITY; hx = hy = hz = -INFINITY;
    c = 0;
    for (int b = 0; b < kSahBins - 1; ++b) {
      if (cnt[b]) {
        lx = fminf(lx, o2f(blo[3 * b])); ly = fminf(ly, o2f(blo[3 * b + 1])); lz = fminf(lz, o2f(blo[3 * b + 2]));
        hx = fmaxf(hx, o2f(bhi[3 * b])); hy = fmaxf(hy, o2f(bhi[3 * b + 1])); hz = fmaxf(hz, o2f(bhi[3 * b + 2]));
        c += cnt[b];
      }
      if (c == 0 || rcnt[b + 1] == 0) continue;
      const float cost = sah_cost(sah_area(lx, ly, lz, hx, hy, hz), c, rarea[b + 1], rcnt[b + 1]);
      if (cost < best) { best = cost; ba = a; bb = b; bnl = c; }
    }
  }
  const int nl = ba < 0 ? n / 2 : bnl;
  C.split[3 * h] = ba; C.split[3 * h + 1] = bb; C.split[3 * h + 2] = nl;
  // stable partition offsets of each chunk (chunks are in position order)
  int before_l = 0, before = 0;
  for (int cc = C.hfirst[h]; cc < C.hfirst[h + 1]; ++cc) {
    int l = 0;
    if (ba >= 0)
      for (int b = 0; b <= bb; ++b) l += C.ccnt[(cc * 3 + ba) * kSahBins + b];
    C.off[2 * cc] = before_l;
    C.off[2 * cc + 1] = before - before_l;
    before_l += l;
    before += C.cend[cc] - C.cbeg[cc];
  }
  sah_children(node, first, last, nl, rf, rl, left, right, pint, pleaf, ctr, next, next_big, next_huge, huge);
}

__global__ void __launch_bounds__(kHugeThreads) k_sah_huge_partition(const float4* __restrict__ tri,
                                                                      const int32_t* __restrict__ perm,
                                                                      int32_t* __restrict__ tmp, const int32_t* __restrict__ rf,
                                                                      SahChunks C) {
  __shared__ int s_scan[kHugeThreads / 32];
  const int c = blockIdx.x, h = C.hidx[c], tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int sa = C.split[3 * h], sb = C.split[3 * h + 1], nl = C.split[3 * h + 2];
  const int first = rf[C.node[c]], beg = C.cbeg[c], end = C.cend[c];
  if (sa < 0) {  // median split by position: the order is kept
    for (int p = beg + tid; p < end; p += kHugeThreads) tmp[p] = perm[p];
    return;
  }
  float cmin[3], cscale[3];
  huge_scale(C, h, cmin, cscale);
  int base_l = C.off[2 * c], base_r = C.off[2 * c + 1];
  for (int p0 = beg; p0 < end; p0 += kHugeThreads) {
    const int p = p0 + tid;
    int flag = 0, t = 0;
    if (p < end) {
      t = perm[p];
      const Box b = tri_box(tri, t);
      const float x = sa == 0 ? 0.5f * (b.lx + b.hx) : sa == 1 ? 0.5f * (b.ly + b.hy) : 0.5f * (b.lz + b.hz);
      flag = min(kSahBins - 1, max(0, (int)((x - cmin[sa]) * cscale[sa]))) <= sb;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_scan[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < kHugeThreads / 32; ++w) {
      const int v = s_scan[w];
      if (w < wid) before += v;
      total += v;
    }
    if (p < end) {
      const int rank_l = base_l + before + in_warp;
      const int rank_r = base_r + (p - p0 - (before + in_warp));
      tmp[flag ? first + rank_l : first + nl + rank_r] = t;
    }
    base_l += total;
    base_r += min(kHugeThreads, end - p0) - total;
    __syncthreads();
  }
}

__global__ void k_sah_huge_copy(int32_t* __restrict__ perm, const int32_t* __restrict__ tmp, SahChunks C) {
  const int c = blockIdx.x;
  for (int p = C.cbeg[c] + threadIdx.x; p < C.cend[c]; p += blockDim.x) perm[p] = tmp[p];
}

__global__ void k_iota32(int32_t* __restrict__ x, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}

__global__ void k_gather_tri_i32(const float4* __restrict__ in, const int32_t* __restrict__ perm, int64_t n,
                                 float4* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t t = perm[r];
  out[3 * r] = in[3 * t]; out[3 * r + 1] = in[3 * t + 1]; out[3 * r + 2] = in[3 * t + 2];
}

__global__ void k_gather_u32(const uint32_t* __restrict__ in, const int32_t* __restrict__ perm, int64_t n,
                             uint32_t* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) out[r] = in[perm[r]];
}

static int build_sah(uvd_scene* s, int64_t M, int32_t* left, int32_t* right, int32_t* rf, int32_t* rl,
                     int32_t* pint, int32_t* pleaf, float* ibox, int* arrive, uint32_t* order, cudaStream_t st) {
  Scratch al(s->alloc, st);  // released at every exit
  // thresholds of the multi-CTA path; UVD_SAH_HUGE / UVD_SAH_CHUNK override them (tests
  // force the chunked path on small scenes with them)
  auto env_pos = [](const char* name, int dflt) {
    const char* e = getenv(name);
    const int v = e ? atoi(e) : 0;
    return v >= 2 ? v : dflt;
  };
  const int huge = std::max(env_pos("UVD_SAH_HUGE", kSahHuge), 2), chunk = env_pos("UVD_SAH_CHUNK", kSahChunk);
  int32_t* perm = (int32_t*)al.get(M * 4);
  int32_t* tmp = (int32_t*)al.get(M * 4);
  int32_t* la = (int32_t*)al.get(M * 4);   // small-node lists (this level, next level)
  int32_t* lb = (int32_t*)al.get(M * 4);
  int32_t* ba = (int32_t*)al.get(M * 4);   // big-node lists
  int32_t* bb = (int32_t*)al.get(M * 4);
  const int64_t max_huge = M / huge + 2, max_chunks = M / chunk + 2 * max_huge + 2;
  int32_t* ha = (int32_t*)al.get(max_huge * 4);  // huge-node lists
  int32_t* hb = (int32_t*)al.get(max_huge * 4);
  // chunk tables and per-huge-node bins (one block of scratch)
  const size_t huge_ints = (size_t)max_chunks * (4 + 3 * kSahBins + 2) + (size_t)(max_huge + 1) +
                           (size_t)max_huge * (6 + 3 * kSahBins * 7 + 3);
  int* hs = (int*)al.get(huge_ints * sizeof(int));
  int* ctr = (int*)al.get(4 * sizeof(int));
  float4* tri2 = (float4*)al.get(3 * M * sizeof(float4));
  if (!perm || !tmp || !la || !lb || !ba || !bb || !ha || !hb || !hs || !ctr || !tri2) {
    set_error("scene: out of device memory (SAH scratch)");
    return UVD_ERR_NOMEM;
  }
  SahChunks C;
  {
    int* q = hs;
    C.node = q; q += max_chunks;
    C.hidx = q; q += max_chunks;
    C.cbeg = q; q += max_chunks;
    C.cend = q; q += max_chunks;
    C.ccnt = q; q += (size_t)max_chunks * 3 * kSahBins;
    C.off = q; q += (size_t)max_chunks * 2;
    C.hfirst = q; q += max_huge + 1;
    C.cb = q; q += (size_t)max_huge * 6;
    C.bcnt = q; q += (size_t)max_huge * 3 * kSahBins;
    C.blo = q; q += (size_t)max_huge * 3 * kSahBins * 3;
    C.bhi = q; q += (size_t)max_huge * 3 * kSahBins * 3;
    C.split = q; q += (size_t)max_huge * 3;
  }
  std::vector<int32_t> h_list, h_rf, h_rl, t_node, t_hidx, t_beg, t_end, t_first;
  std::vector<int> h_init;
  k_iota32<<<grid_for(M, 256), 256, 0, st>>>(perm, M);
  note_launch();
  int h[4] = {1, 0, 0, 0};  // next internal node id, next-level small / big / huge list lengths
  int32_t zero = 0, last = (int32_t)(M - 1);
  UVD_CUDA_TRY(cudaMemcpyAsync(rf, &zero, 4, cudaMemcpyHostToDevice, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(rl, &last, 4, cudaMemcpyHostToDevice, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(M > huge ? ha : M > kSahBig ? ba : la, &zero, 4, cudaMemcpyHostToDevice, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(pint, &zero, 4, cudaMemcpyHostToDevice, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(ctr, h, sizeof(int), cudaMemcpyHostToDevice, st));  // node id 1 next
  int n_small = M <= kSahBig && M <= huge, n_big = M > kSahBig && M <= huge, n_huge = M > huge, levels = 0;
  while (n_small + n_big + n_huge > 0) {
    UVD_CUDA_TRY(cudaMemsetAsync(ctr + 1, 0, 3 * sizeof(int), st));  // next level's list lengths
    if (n_huge) {
      // chunk table of this level's huge nodes (few: host-built)
      h_list.resize(n_huge); h_rf.resize(n_huge); h_rl.resize(n_huge);
      UVD_CUDA_TRY(cudaMemcpyAsync(h_list.data(), ha, n_huge * 4, cudaMemcpyDeviceToHost, st));
      UVD_CUDA_TRY(cudaStreamSynchronize(st));
      for (int k = 0; k < n_huge; ++k) {
        UVD_CUDA_TRY(cudaMemcpyAsync(&h_rf[k], rf + h_list[k], 4, cudaMemcpyDeviceToHost, st));
        UVD_CUDA_TRY(cudaMemcpyAsync(&h_rl[k], rl + h_list[k], 4, cudaMemcpyDeviceToHost, st));
      }
      UVD_CUDA_TRY(cudaStreamSynchronize(st));
      t_node.clear(); t_hidx.clear(); t_beg.clear(); t_end.clear(); t_first.assign(1, 0);
      for (int k = 0; k < n_huge; ++k) {
        for (int p = h_rf[k]; p <= h_rl[k]; p += chunk) {
          t_node.push_back(h_list[k]); t_hidx.push_back(k);
          t_beg.push_back(p); t_end.push_back(std::min(p + chunk, h_rl[k] + 1));
        }
        t_first.push_back((int32_t)t_node.size());
      }
      const int nch = (int)t_node.size();
      if (nch > max_chunks) { set_error("scene: SAH chunk table overflow"); return UVD_ERR_CUDA; }
      UVD_CUDA_TRY(cudaMemcpyAsync((void*)C.node, t_node.data(), nch * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync((void*)C.hidx, t_hidx.data(), nch * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync((void*)C.cbeg, t_beg.data(), nch * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync((void*)C.cend, t_end.data(), nch * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync((void*)C.hfirst, t_first.data(), (n_huge + 1) * 4, cudaMemcpyHostToDevice, st));
      // per-node bounds / bins reset: ordered-int "+inf" lows, "-inf" highs, zero counts
      h_init.assign((size_t)n_huge * (6 + 3 * kSahBins * 7), 0);
      for (int k = 0; k < n_huge; ++k)
        for (int a = 0; a < 6; ++a) h_init[6 * k + a] = a < 3 ? 0x7fffffff : (int)0x80000000;
      int* bcnt0 = h_init.data() + 6 * n_huge;
      int* blo0 = bcnt0 + (size_t)n_huge * 3 * kSahBins;
      int* bhi0 = blo0 + (size_t)n_huge * 3 * kSahBins * 3;
      for (size_t q = 0; q < (size_t)n_huge * 3 * kSahBins * 3; ++q) { blo0[q] = 0x7fffffff; bhi0[q] = (int)0x80000000; }
      UVD_CUDA_TRY(cudaMemcpyAsync(C.cb, h_init.data(), (size_t)n_huge * 6 * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync(C.bcnt, bcnt0, (size_t)n_huge * 3 * kSahBins * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync(C.blo, blo0, (size_t)n_huge * 3 * kSahBins * 3 * 4, cudaMemcpyHostToDevice, st));
      UVD_CUDA_TRY(cudaMemcpyAsync(C.bhi, bhi0, (size_t)n_huge * 3 * kSahBins * 3 * 4, cudaMemcpyHostToDevice, st));
      k_sah_huge_bounds<<<nch, kHugeThreads, 0, st>>>(s->tri, perm, C);
      k_sah_huge_bins<<<nch, kHugeThreads, 0, st>>>(s->tri, perm, C);
      k_sah_huge_decide<<<(n_huge + 31) / 32, 32, 0, st>>>(ha, n_huge, C, rf, rl, left, right, pint, pleaf, ctr, lb,
                                                            bb, hb, huge);
      k_sah_huge_partition<<<nch, kHugeThreads, 0, st>>>(s->tri, perm, tmp, rf, C);
      k_sah_huge_copy<<<nch, 1024, 0, st>>>(perm, tmp, C);
      note_launch(5);
      UVD_CUDA_TRY(cudaStreamSynchronize(st));  // the host vectors above are reused next level
    }
    if (n_big)
      k_sah_split<1024><<<n_big, 1024, 0, st>>>(s->tri, perm, tmp, ba, rf, rl, left, right, pint, pleaf, ctr, lb, bb, hb, huge);
    if (n_small)
      k_sah_split<128><<<n_small, 128, 0, st>>>(s->tri, perm, tmp, la, rf, rl, left, right, pint, pleaf, ctr, lb, bb, hb, huge);
    note_launch((n_big > 0) + (n_small > 0));
    UVD_CUDA_TRY(cudaMemcpyAsync(h, ctr, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    n_small = h[1];
    n_big = h[2];
    n_huge = h[3];
    std::swap(la, lb);
    std::swap(ba, bb);
    std::swap(ha, hb);
    if (++levels > 4096) { set_error("scene: SAH build did not terminate"); return UVD_ERR_CUDA; }
  }
  if (h[0] != M - 1) { set_error("scene: SAH build made %d internal nodes, expected %lld", h[0], (long long)(M - 1)); return UVD_ERR_CUDA; }
  // triangles (and the sorted -> input map) into the DFS leaf order of the tree
  k_gather_tri_i32<<<grid_for(M, 256), 256, 0, st>>>(s->tri, perm, M, tri2);
  note_launch();
  UVD_CUDA_TRY(cudaMemcpyAsync(s->tri, tri2, 3 * M * sizeof(float4), cudaMemcpyDeviceToDevice, st));
  if (order) {
    uint32_t* o2 = (uint32_t*)tri2;
    k_gather_u32<<<grid_for(M, 256), 256, 0, st>>>(order, perm, M, o2);
    note_launch();
    UVD_CUDA_TRY(cudaMemcpyAsync(order, o2, M * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  if (s->kind == UVD_SCENE_TRIMESH) {  // rows follow the leaf order
    k_set_owner<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M);
    note_launch();
  }
  k_refit<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M, left, right, pint, pleaf, ibox, arrive);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

// deepest leaf (an upper bound of the traversal stack depth), via parent links
__global__ void k_max_depth(const int32_t* __restrict__ parent_leaf, const int32_t* __restrict__ parent_int,
                            int64_t n, int* __restrict__ depth) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int d = 1;
  for (int32_t p = parent_leaf[r]; p != 0 && d < 4096; p = parent_int[p]) ++d;
  atomicMax(depth, d);
}

// Octant copies of the nodes (k_octant_nodes) unless they would take > 1/16 of
// the device memory or UVD_OCT=0: the traversal then reads the one array
// (min/max per slab).  Also used by uvd_scene_import (the copies are rebuilt
// locally, not shipped).
int build_octants(uvd_scene* s, cudaStream_t st) {
  Alloc& al = s->alloc;
  const int64_t nn = std::max<int64_t>(s->M - 1, 1);
  if (s->onodes) al.put(s->onodes);
  s->onodes = nullptr;
  s->n_nodes = nn;
  const size_t total_b = device_total_mem(al.device);
  const char* e = getenv("UVD_OCT");
  const bool want = !(e && atoi(e) == 0) && 8 * nn < ((int64_t)1 << 31) &&
                    (double)(8 * nn * (int64_t)sizeof(Node)) <= (double)total_b / 16.0;
  if (want) s->onodes = (Node*)al.get(8 * nn * sizeof(Node));  // nullptr (no memory): one array
  if (s->onodes) {
    k_octant_nodes<<<grid_for(8 * nn, 256), 256, 0, st>>>(s->nodes, nn, s->onodes);
    note_launch();
  }
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

#ifndef UVD_BVH_DEFAULT
#define UVD_BVH_DEFAULT 2  // binned SAH; UVD_BVH=ploc / karras select the others
#endif
// Morton-sort the triangles (tri_in, input order) and build the BVH over them.
// On return s->tri is leaf-ordered and `order` (if non-null) receives the
// sorted -> input permutation (caller frees).
int build_bvh(uvd_scene* s, float4* tri_in, uint32_t** order_out, cudaStream_t st) {
  Alloc& al = s->alloc;     // scene-owned buffers (freed with the scene)
  Scratch sc(al, st);       // this build's temporaries, released at every exit
  const int64_t M = s->M;
  uint64_t* keys = (uint64_t*)sc.get(M * sizeof(uint64_t));
  uint32_t* vals = (uint32_t*)sc.get(M * sizeof(uint32_t));
  s->tri = (float4*)al.get(3 * M * sizeof(float4));
  s->nodes = (Node*)al.get(std::max<int64_t>(M - 1, 1) * sizeof(Node));
  if (!keys || !vals || !s->tri || !s->nodes) {
    set_error("scene: out of device memory building the BVH (M=%lld)", (long long)M);
    return UVD_ERR_NOMEM;
  }
  float cp = 0.f;  // padding term 4 eps32 x the scene's largest |coordinate|
  for (int k = 0; k < 6; ++k) cp = std::max(cp, std::fabs(s->bbox[k]));
  cp *= 4.0f * 5.9604645e-08f;
  float3 lo = make_float3(s->bbox[0], s->bbox[1], s->bbox[2]);
  float ex = s->bbox[3] - s->bbox[0], ey = s->bbox[4] - s->bbox[1], ez = s->bbox[5] - s->bbox[2];
  float3 inv = make_float3(ex > 0 ? 1.f / ex : 0.f, ey > 0 ? 1.f / ey : 0.f, ez > 0 ? 1.f / ez : 0.f);
  k_morton<<<grid_for(M, 256), 256, 0, st>>>(tri_in, M, lo, inv, keys, vals);
  note_launch();
  HostTrace::mark("bvh: morton");
  UVD_TRY(sort_pairs_u64(keys, vals, M, al, st));
  HostTrace::mark("bvh: sort");
  k_gather_tri<<<grid_for(M, 256), 256, 0, st>>>(tri_in, vals, M, s->tri);
  note_launch();
  if (s->kind == UVD_SCENE_TRIMESH) {  // row (patch) of the triangle at Morton position r is r
    k_set_owner<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M);
    note_launch();
  }
  if (M <= kLeafMax) {
    k_emit_small<<<1, 1, 0, st>>>(s->tri, M, s->nodes, cp);
    note_launch();
    s->root = 0;
  } else {
    int64_t ni = M - 1;
    int32_t* left = (int32_t*)sc.get(ni * 4);
    int32_t* right = (int32_t*)sc.get(ni * 4);
    int32_t* rf = (int32_t*)sc.get(ni * 4);
    int32_t* rl = (int32_t*)sc.get(ni * 4);
    int32_t* pint = (int32_t*)sc.get(ni * 4);
    int32_t* pleaf = (int32_t*)sc.get(M * 4);
    float* ibox = (float*)sc.get(ni * 6 * sizeof(float));
    int* arrive = (int*)sc.get(ni * sizeof(int));
    if (!left || !right || !rf || !rl || !pint || !pleaf || !ibox || !arrive) {
      set_error("scene: out of device memory (BVH scratch)");
      return UVD_ERR_NOMEM;
    }
    UVD_CUDA_TRY(cudaMemsetAsync(arrive, 0, ni * sizeof(int), st));
    // 0 PLOC, 1 Karras LBVH, 2 binned SAH (default); read per build
    const char* e = getenv("UVD_BVH");
    const std::string v = e ? e : "";
    const int builder = v == "ploc" ? 0 : v == "karras" ? 1 : v == "sah" ? 2 : UVD_BVH_DEFAULT;
    if (builder == 2) {  // top-down binned SAH (level-synchronous, one CTA per node)
      UVD_TRY(build_sah(s, M, left, right, rf, rl, pint, pleaf, ibox, arrive,
                        s->kind == UVD_SCENE_TRIMESH ? vals : nullptr, st));
    } else if (builder == 1) {  // Karras 2012 LBVH + bottom-up refit
      k_karras<<<grid_for(ni, 256), 256, 0, st>>>(keys, M, left, right, rf, rl, pint, pleaf);
      note_launch();
      k_refit<<<grid_for(M, 256), 256, 0, st>>>(s->tri, M, left, right, pint, pleaf, ibox, arrive);
      note_launch();
    } else {  // PLOC (default): agglomerative clustering over the Morton order
      UVD_TRY(build_ploc(s, M, left, right, rf, rl, pint, pleaf, ibox, arrive, vals, st));
    }
    HostTrace::mark("bvh: builder");
    {  // the traversal stacks hold 64 entries: refuse deeper trees loudly
      int* dd = (int*)sc.get(sizeof(int));
      if (!dd) { set_error("scene: out of device memory"); return UVD_ERR_NOMEM; }
      UVD_CUDA_TRY(cudaMemsetAsync(dd, 0, sizeof(int), st));
      k_max_depth<<<grid_for(M, 256), 256, 0, st>>>(pleaf, pint, M, dd);
      note_launch();
      int hd = 0;
      UVD_CUDA_TRY(cudaMemcpyAsync(&hd, dd, sizeof(int), cudaMemcpyDeviceToHost, st));
      UVD_CUDA_TRY(cudaStreamSynchronize(st));
      sc.release(dd);
      if (hd > 62) {
        set_error("scene: BVH depth %d exceeds the traversal stack (64)", hd);
        return UVD_ERR_INVALID;
      }
    }
    int32_t* pre = (int32_t*)arrive;  // arrival counters are free again
    k_preorder<<<grid_for(ni, 256), 256, 0, st>>>(left, pint, rf, rl, ni, pre);
    note_launch();
    k_emit<<<grid_for(ni, 256), 256, 0, st>>>(s->tri, M, left, right, rf, rl, ibox, pre, s->nodes, cp);
    note_launch();
    s->root = 0;
  }
  HostTrace::mark("bvh: depth+emit");
  UVD_TRY(build_octants(s, st));
  UVD_TRY(build_hnodes(s, st));
  HostTrace::mark("bvh: octants+hnodes");
  UVD_CUDA_TRY(cudaGetLastError());
  if (order_out) {
    sc.keep(vals);  // ownership passes to the caller
    *order_out = vals;
  }
  return UVD_OK;
}

}  // namespace uvd
