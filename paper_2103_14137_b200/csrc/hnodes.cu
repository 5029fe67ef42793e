// hnodes.cu — half-precision copies of the top of the BVH (the "H nodes").
//
// ncu puts the assembly walk against the L1 data pipe (76 % of its wavefront
// peak): every node step delivers the node's 56 bytes to every active lane
// (4 + 4 + 4 + 2 wavefronts per warp), and an 8-byte wider node costs +7 %
// kernel time.  The top levels of the tree — depth <= kHDepth,
// about 60 % of a C5 segment's node visits — are therefore also stored as
// 32-byte H nodes: the twelve child-box planes as fp16 (relative to the scene
// centre), in (child 0, child 1) half2 pairs per plane and ray octant, plus the
// two child refs.  The walk tests them with six HFMA2 (both children at once),
// half the bytes of a full node.
//
// Exactness (the decisions do not change, only which boxes are visited).  For
// a plane b (relative to the centre c), the walk computes in fp16
//   t = fl16(b·inv_h − fl16(o·inv_h)),  inv_h = fl16(1/d),  o = lamp − c,
// which is the exact slab parameter of a plane shifted by at most
//   |b − o|·(2^-10 + 2^-22) + |o|·2^-11  <=  1.25·2^-10·L_axis
// (|b − o| <= L_axis, the scene extent; |o| <= L_axis / 2).  Every box is
// padded outward by that bound + 1e-4 m before rounding outward to fp16, so
// the computed interval of the padded box contains the exact interval of the
// true box, as the fp32 nodes' padding does for their rounding; t_min / t_max
// are rounded outward to fp16.  Lanes whose 1/d exceeds 2048 in some axis (fp16
// range) and scenes larger than ±16 m around their centre use the fp32 nodes
// only (the H root is then not entered).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "uvd_internal.cuh"

namespace uvd {

// depth-first collection of the nodes at depth <= max_depth (one thread: at
// most 2^(max_depth+1) nodes); hmap[h] = full node index of H node h
__global__ void k_h_collect(const Node* __restrict__ nodes, uint32_t root, int max_depth, int cap,
                            int32_t* __restrict__ hmap, int* __restrict__ n_out) {
  if (threadIdx.x | blockIdx.x) return;
  uint32_t stk[128];
  int dep[128];
  int sp = 0, n = 0;
  if (!ref_is_leaf(root)) { stk[sp] = root; dep[sp++] = 0; }
  while (sp) {
    --sp;
    const uint32_t r = stk[sp];
    const int d = dep[sp];
    if (n >= cap) break;
    hmap[n++] = (int32_t)r;
    if (d >= max_depth) continue;
    const uint2 ch = *reinterpret_cast<const uint2*>(&nodes[r].d);
    if (!ref_is_leaf(ch.y) && sp < 127) { stk[sp] = ch.y; dep[sp++] = d + 1; }
    if (!ref_is_leaf(ch.x) && sp < 127) { stk[sp] = ch.x; dep[sp++] = d + 1; }
  }
  *n_out = n;
}

// outward roundings (each step rounds toward the same side, so the composition does)
__device__ __forceinline__ __half h_down(double v) { return __float2half_rd(__double2float_rd(v)); }
__device__ __forceinline__ __half h_up(double v) { return __float2half_ru(__double2float_ru(v)); }

// one H node in one octant copy: planes padded outward and rounded outward to
// fp16, swapped to (entry, exit) for the octant; refs into the same copy
// (copies are `cap` nodes apart; the count nh comes from k_h_collect on the
// device, so the host never waits for it)
__global__ void k_h_build(const Node* __restrict__ nodes, const int32_t* __restrict__ hmap,
                          const int* __restrict__ n_h, int cap, int64_t nn, float3 ctr, float3 pad,
                          HNode* __restrict__ hn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 8 * cap) return;
  const int nh = *n_h;
  const int o = i / cap, h = i - o * cap;
  if (h >= nh) return;
  const Node nd = nodes[hmap[h]];
  // child k: lo/hi per axis (fp32 boxes of the base array)
  const float lo[2][3] = {{nd.a.x, nd.a.z, nd.c.x}, {nd.b.x, nd.b.z, nd.c.z}};
  const float hi[2][3] = {{nd.a.y, nd.a.w, nd.c.y}, {nd.b.y, nd.b.w, nd.c.w}};
  const double cc[3] = {ctr.x, ctr.y, ctr.z}, pp[3] = {pad.x, pad.y, pad.z};
  HNode out;
  for (int ax = 0; ax < 3; ++ax) {
    __half en[2], ex[2];
    for (int k = 0; k < 2; ++k) {
      const bool empty = lo[k][ax] > hi[k][ax];  // the dummy child of a one-leaf root: keep it empty
      const __half l = empty ? __float2half(1.0f) : h_down((double)lo[k][ax] - cc[ax] - pp[ax]);
      const __half u = empty ? __float2half(-1.0f) : h_up((double)hi[k][ax] - cc[ax] + pp[ax]);
      const bool neg = (o >> ax) & 1;  // 1/d < 0 on this axis: the ray enters at hi
      en[k] = neg ? u : l;
      ex[k] = neg ? l : u;
    }
    out.p[2 * ax] = __halves2half2(en[0], en[1]);
    out.p[2 * ax + 1] = __halves2half2(ex[0], ex[1]);
  }
  const uint32_t cr[2] = {nd.d.x, nd.d.y};
  for (int k = 0; k < 2; ++k) {
    uint32_t r = cr[k];
    if (!ref_is_leaf(r)) {
      int hc = -1;
      for (int q = 0; q < nh; ++q)
        if ((uint32_t)hmap[q] == r) { hc = q; break; }
      r = hc >= 0 ? kHalfRef | (uint32_t)(hc + o * cap) : r + (uint32_t)(o * nn);
    }
    out.ref[k] = r;
  }
  hn[i] = out;
}

int build_hnodes(uvd_scene* s, cudaStream_t st) {
  Alloc& al = s->alloc;
  if (s->hnodes) al.put(s->hnodes);
  s->hnodes = nullptr;
  s->n_h = 0;
  const char* e = getenv("UVD_HDEPTH");
  const int depth = e ? atoi(e) : kHDepth;
  const int64_t nn = s->n_nodes;
  // H nodes need the octant copies, fp16-safe coordinates and room for the flag bit
  const double hx = 0.5 * ((double)s->bbox[3] - s->bbox[0]), hy = 0.5 * ((double)s->bbox[4] - s->bbox[1]),
               hz = 0.5 * ((double)s->bbox[5] - s->bbox[2]);
  if (depth < 0 || !s->onodes || ref_is_leaf(s->root) || 8 * nn >= ((int64_t)1 << 30) ||
      std::max(hx, std::max(hy, hz)) > 15.0)
    return UVD_OK;
  const int cap = std::min(4096, (2 << std::min(depth, 11)) - 1);
  Scratch sc(al, st);
  int32_t* hmap = (int32_t*)sc.get(cap * sizeof(int32_t) + 16);
  if (!hmap) { set_error("scene: out of device memory (H nodes)"); return UVD_ERR_NOMEM; }
  int* dn = (int*)(hmap + cap);
  k_h_collect<<<1, 1, 0, st>>>(s->nodes, s->root, depth, cap, hmap, dn);
  note_launch();
  s->hnodes = (HNode*)al.get((size_t)8 * cap * sizeof(HNode));
  if (!s->hnodes) { set_error("scene: out of device memory (H nodes)"); return UVD_ERR_NOMEM; }
  const float3 ctr = make_float3(0.5f * (s->bbox[0] + s->bbox[3]), 0.5f * (s->bbox[1] + s->bbox[4]),
                                 0.5f * (s->bbox[2] + s->bbox[5]));
  // 1.25·2^-10·L per axis (the fp16 slab error bound above) + 1e-4 m
  const double k = 1.25 / 1024.0;
  const float3 pad = make_float3((float)(k * 2 * hx + 1e-4), (float)(k * 2 * hy + 1e-4), (float)(k * 2 * hz + 1e-4));
  k_h_build<<<(8 * cap + 127) / 128, 128, 0, st>>>(s->nodes, hmap, dn, cap, nn, ctr, pad, s->hnodes);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  s->n_h = cap;  // the stride between octant copies (the walk enters node 0 of its copy)
  s->hcenter[0] = ctr.x; s->hcenter[1] = ctr.y; s->hcenter[2] = ctr.z;
  return UVD_OK;
}

}  // namespace uvd
