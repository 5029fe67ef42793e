// uvd_internal.cuh — shared internals of libuvd (CUDA path only; the oracle
// under oracle/ shares nothing with this tree).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/uvd.h"

namespace uvd {

// ------------------------------------------------------------------ errors --
void set_error(const char* fmt, ...);
void clear_error();
void note_launch(int n = 1);  // kernel launch accounting (uvd_launch_count)

#define UVD_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::uvd::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                       cudaGetErrorString(_e));                                   \
      return UVD_ERR_CUDA;                                                        \
    }                                                                             \
  } while (0)

#define UVD_TRY(expr)            \
  do {                           \
    int _s = (expr);             \
    if (_s != UVD_OK) return _s; \
  } while (0)

// -------------------------------------------------------------- constants --
// Readings of the paper.  Written out here independently
// of the oracle (the two sides share no code or constant tables).
constexpr double kSelfEps = 1e-4;     // Q6: open segment t in (1e-4/d, 1 - 1e-4/d)
constexpr double kMinDist = 1e-9;     // domain error below 1e-9 m
constexpr double kEdgeTol = 1e-12;    // watertight acceptance of fp64 margins
constexpr double kParallel = 1e-12;   // |det| <= 1e-12 |D||E1xE2| -> no crossing
#ifndef UVD_LEAF_MAX
#define UVD_LEAF_MAX 2
#endif
constexpr int kLeafMax = UVD_LEAF_MAX;
#ifndef UVD_ROWS_DFS
#define UVD_ROWS_DFS 1  // 3D rows follow the BVH leaf (DFS) order: row r = leaf-ordered triangle r
#endif  // triangles per BVH leaf (subtree collapse), <= 8
constexpr int kCovBlocksMax = 1024;   // coverage partial sums (fixed, deterministic order)
// Q20 free-space test direction (tilted off the axes).
constexpr double kFreeDirX = 0.0123, kFreeDirY = 0.0371, kFreeDirZ = 1.0;

// BVH child reference: >= 0 internal node index; leaf = 0x80000000 | start<<3 | (count-1)
__host__ __device__ inline bool ref_is_leaf(uint32_t r) { return (r & 0x80000000u) != 0; }
__host__ __device__ inline uint32_t ref_start(uint32_t r) { return (r & 0x7fffffffu) >> 3; }
__host__ __device__ inline uint32_t ref_count(uint32_t r) { return (r & 7u) + 1u; }
__host__ __device__ inline uint32_t make_leaf(uint32_t start, uint32_t count) {
  return 0x80000000u | (start << 3) | (count - 1u);
}

// BVH2 node with both child boxes (64 B, one 128-B line holds two nodes).
struct __align__(16) Node {
  float4 a;  // child0 lo.x hi.x lo.y hi.y
  float4 b;  // child1 lo.x hi.x lo.y hi.y
  float4 c;  // child0 lo.z hi.z, child1 lo.z hi.z
  uint4 d;   // child0 ref, child1 ref, (unused), (unused)
};  // (the octant copies, bvh.cu k_octant_nodes, pair the children's planes instead)

// H node (hnodes.cu): the two child boxes of a top-level node as fp16 planes
// relative to the scene centre, (child 0, child 1) pairs per plane in (entry,
// exit) order for one ray octant — p[0..5] = entry x, exit x, entry y, exit y,
// entry z, exit z — and the child refs (an H child carries kHalfRef)
struct __align__(16) HNode {
  __half2 p[6];
  uint32_t ref[2];
};
constexpr uint32_t kHalfRef = 0x40000000u;  // internal ref into the H node copies
#ifndef UVD_HDEPTH
#define UVD_HDEPTH 6
#endif
constexpr int kHDepth = UVD_HDEPTH;          // H nodes: the nodes at depth <= kHDepth

// ------------------------------------------------------------------ memory --
struct Alloc {
  uvd_allocator user{};
  bool has_user = false;
  int device = 0;
  cudaStream_t stream = nullptr;
  void* get(size_t bytes);
  void put(void* p);
};

// Host-side trace (UVD_TRACE_HOST=1, development): wall-clock marks of the
// stages of a call and the time spent in allocator callbacks, to stderr.
struct HostTrace {
  static bool on();
  static void mark(const char* what);      // time since the previous mark
  static void alloc_time(double us);        // accumulated into the next mark
};

// Call-scoped device buffers: every buffer taken through get() is returned
// (stream-ordered on the call's stream) at every exit of the call, error
// returns included; release(p) hands one back early, keep(p) moves ownership out.
struct Scratch {
  Alloc al;
  std::vector<void*> ps;
  Scratch(const Alloc& a, cudaStream_t st) : al(a) { al.stream = st; }
  ~Scratch() { for (void* p : ps) al.put(p); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  void* get(size_t bytes) {
    void* p = al.get(bytes);
    if (p) ps.push_back(p);
    return p;
  }
  void keep(void* p) { ps.erase(std::remove(ps.begin(), ps.end(), p), ps.end()); }
  void release(void* p) {
    keep(p);
    al.put(p);
  }
};

// Every entry point runs on the device its scene (or its buffers) lives on and
// restores the caller's current device on return.
struct DeviceGuard {
  int prev = -1, dev = -1;
  explicit DeviceGuard(int d) : dev(d) {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (d >= 0 && prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};
// device of a device pointer (-1 if unknown: the current device stays)
int pointer_device(const void* p);

// NVTX range around an entry point: visible in ncu --nvtx / nsys
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// per-device cached launch geometry (SM count; occupancy-derived grids)
constexpr int kMaxDevices = 64;
int sm_count(int dev);
size_t device_total_mem(int dev);  // cached per device

// ------------------------------------------------------------------- scene --
struct Wall {  // 2.5D wall (host-prepared from the polygon description)
  float e0x, e0y, e1x, e1y;
  int32_t boundary;  // 1 = room boundary (normal into the room), 0 = obstacle
  int32_t n_seg;
  int64_t first_patch;
};

}  // namespace uvd

struct uvd_scene {
  uvd::Alloc alloc;
  int32_t kind = 0;
  int64_t N = 0;  // patches (rows of A)
  int64_t M = 0;  // triangles
  float bbox[6] = {0, 0, 0, 0, 0, 0};
  double total_area = 0.0;
  // canonical patch attributes (device)
  float* centroid = nullptr;  // N*3
  float* normal = nullptr;    // N*3
  double* area = nullptr;     // N
  int64_t* orig_id = nullptr; // N
  // BVH (device)
  float4* tri = nullptr;      // M*3: (v0, owner patch), (v1, orig tri), (v2, 0)  leaf order
  float4* ptri = nullptr;     // EXTRUDED only: 2N*3 patch-ordered wall triangles (area model)
  uvd::Node* nodes = nullptr; // max(M-1, 1) BVH2 nodes
  uvd::Node* onodes = nullptr; // 8 x max(M-1, 1): the nodes with each child box stored (near, far) per ray octant
  int64_t n_nodes = 0;
  uint32_t root = 0;          // root ref
  float* front_free = nullptr; // [N] front radius of every patch (free.cu)
  uvd::HNode* hnodes = nullptr; // 8 octant copies of the H nodes (hnodes.cu), or nullptr
  int32_t n_h = 0;              // H nodes per copy
  float hcenter[3] = {0, 0, 0}; // origin of the H nodes' fp16 coordinates
  // 2.5D description (device + host copies) for the floorplan vantage test
  uvd::Wall* walls = nullptr;  // device
  int64_t n_walls = 0;
  std::vector<uvd::Wall> h_walls;
  float* poly_xy = nullptr;    // device, obstacles' vertices
  int32_t* poly_off = nullptr; // device, n_obstacles+1 offsets
  int32_t n_poly = 0;
  int64_t n_poly_xy = 0, n_poly_off = 0;  // element counts of poly_xy / poly_off (export)
  float bounds[4] = {0, 0, 0, 0};
  float wall_height = 0.f;
  // in-kernel error flag (device int)
  int* err_flag = nullptr;
  // coverage partials, one buffer per stream the scene's coverage ran on (a
  // call on another stream never shares one); guarded by cov_mu
  struct CovScratch { cudaStream_t stream; double* p; };
  std::vector<CovScratch> cov_part;  // each 3 * kCovBlocksMax + 3 doubles
  std::mutex cov_mu;
};

namespace uvd {
// per-thread pinned staging buffer (64 B, allocated once, never freed) for the
// scalars synchronising calls return: no allocation on the critical path
void* host_stage();
// launchers implemented in the .cu files
int build_bvh(uvd_scene* s, float4* tri_in, uint32_t** order_out, cudaStream_t st);
int build_octants(uvd_scene* s, cudaStream_t st);
int build_hnodes(uvd_scene* s, cudaStream_t st);
int sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, Alloc& al, cudaStream_t st);
// free.cu: empty regions at the segment ends (front radius per patch, lamp radius per sample)
int front_radius(uvd_scene* s, cudaStream_t st);
int lamp_radius(const uvd_scene* s, const float* lamps, int64_t n, float* out, cudaStream_t st);
// assemble.cu: flag 3 on the scene when a lamp coordinate is outside the fp32 padding's range
int check_lamps(const uvd_scene* s, const float* lamps, const int64_t* dcols, int64_t n_cols, int L, cudaStream_t st);
// fluence.cu: the a7 products without allocation (uvd_lp_solve graphs them)
Alloc matrix_alloc(const uvd_matrix_out* A, int dev, cudaStream_t st);
size_t fluence_ws_bytes(int64_t n, int64_t k, bool csc, int dev);
int fluence_check(const uvd_matrix_out* A, int64_t n, int64_t k, const double* x);
int fluence_run(const uvd_matrix_out* A, int64_t n, int64_t k, int transpose, const double* x, double* out,
                cudaStream_t st, void* ws);
}  // namespace uvd
