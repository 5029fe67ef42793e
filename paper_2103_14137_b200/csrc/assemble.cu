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

#include "traverse.cuh"
#include "uvd_internal.cuh"

namespace uvd {

constexpr int kAsmWarps = 8;
constexpr int kAsmThreads = kAsmWarps * 32;

struct AsmParams {
  const float4* __restrict__ tri;
  const Node* __restrict__ nodes;
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
  unsigned long long* __restrict__ counters;  // [4] or nullptr (instrumented kernel)
  int* __restrict__ err;
};

// warp-cooperative any-hit walk; returns false for active lanes whose segment is
// blocked (inactive lanes return true: the caller ANDs with its own mask).
template <bool COUNT>
__device__ __forceinline__ bool warp_trace_clear(const AsmParams& P, uint32_t* __restrict__ stack,
                                                 bool active, const Ray32& r32, D3 O, D3 D,
                                                 double dd, double t_lo, double t_hi,
                                                 int owner, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  bool occluded = false;
  uint32_t live = __ballot_sync(0xffffffffu, active);
  if (!live) return !occluded;
  int sp = 0;
  if (lane == 0) stack[0] = P.root;
  sp = 1;
  __syncwarp();
  while (sp > 0) {
    --sp;
    uint32_t ref = stack[sp];
    if (ref_is_leaf(ref)) {
      uint32_t st = ref_start(ref), nt = ref_count(ref);
      for (uint32_t k = 0; k < nt; ++k) {
        const float4* t = P.tri + 3 * (int64_t)(st + k);
        float4 a = __ldg(t), b = __ldg(t + 1), c = __ldg(t + 2);
        bool test = active && !occluded && __float_as_int(a.w) != owner;
        if (COUNT) cnt[2] += __popc(__ballot_sync(0xffffffffu, test));
        if (test) occluded = seg_hits_tri(O, D, dd, t_lo, t_hi, a, b, c);
      }
      live = __ballot_sync(0xffffffffu, active && !occluded);
      if (!live) break;
    } else {
      const Node* nd = P.nodes + ref;
      float4 na = __ldg(&nd->a), nb = __ldg(&nd->b), nc = __ldg(&nd->c);
      uint4 ndd = __ldg(&nd->d);
      bool me = active && !occluded;
      if (COUNT) {
        cnt[1] += 2 * __popc(__ballot_sync(0xffffffffu, me));
        cnt[3] += 1;
      }
      bool h0 = me && slab(r32, na.x, na.y, na.z, na.w, nc.x, nc.y, 1.0f);
      bool h1 = me && slab(r32, nb.x, nb.y, nb.z, nb.w, nc.z, nc.w, 1.0f);
      uint32_t m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
      __syncwarp();
      if (m0 && m1) {
        // descend into the child more lanes want first (pushed last)
        bool first0 = __popc(m0) >= __popc(m1);
        if (lane == 0) {
          stack[sp] = first0 ? ndd.y : ndd.x;
          stack[sp + 1] = first0 ? ndd.x : ndd.y;
        }
        sp += 2;
      } else if (m0 | m1) {
        if (lane == 0) stack[sp] = m0 ? ndd.x : ndd.y;
        sp += 1;
      }
      if (sp > kStackDepth - 2) {  // cannot happen for depth < 126; fail loudly
        if (lane == 0) atomicExch(P.err, 2);
        break;
      }
      __syncwarp();
    }
  }
  return !occluded;
}

template <bool COUNT>
__global__ void __launch_bounds__(kAsmThreads) k_assemble(AsmParams P) {
  __shared__ uint32_t s_stack[kAsmWarps][kStackDepth];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* stack = s_stack[warp];
  unsigned long long cnt[4] = {0, 0, 0, 0};  // warp-uniform tallies (COUNT only)
  const int64_t total = P.n_cols * P.tiles;
  for (int64_t item = (int64_t)blockIdx.x * kAsmWarps + warp; item < total;
       item += (int64_t)gridDim.x * kAsmWarps) {
    const int64_t c = item / P.tiles, tile = item - c * P.tiles;
    const int64_t j = P.cols ? P.cols[c] : c;
    const int64_t r = tile * 32 + lane;
    const bool valid = r < P.N;
    float cx = 0.f, cy = 0.f, cz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
    if (valid) {
      cx = P.centroid[3 * r]; cy = P.centroid[3 * r + 1]; cz = P.centroid[3 * r + 2];
      nx = P.normal[3 * r]; ny = P.normal[3 * r + 1]; nz = P.normal[3 * r + 2];
    }
    double acc = 0.0;
    for (int l = 0; l < P.L; ++l) {
      const float* pl = P.lamps + 3 * (j * P.L + l);
      const float px = pl[0], py = pl[1], pz = pl[2];
      // a4: ray p -> c in fp64 (exact differences of fp32 inputs), front-face cull
      D3 O = d3(px, py, pz);
      D3 D = d3((double)cx - (double)px, (double)cy - (double)py, (double)cz - (double)pz);
      double dd = ddot3(D, D);
      double d = sqrt(dd);
      double cosd = -(D.x * (double)nx + D.y * (double)ny + D.z * (double)nz);  // <p - c, n>
      bool front = valid && cosd > 0.0;
      if (valid && d < kMinDist) {
        atomicExch(P.err, 1);
        front = false;
      }
      uint32_t fm = __ballot_sync(0xffffffffu, front);
      if (COUNT) cnt[0] += __popc(fm);
      bool vis = front;
      if (fm) {
        // a5: occlusion of the open segment, t in (1e-4/d, 1 - 1e-4/d)
        double t_lo = front ? kSelfEps / d : 0.0;
        Ray32 r32 = make_ray32(px, py, pz, (float)D.x, (float)D.y, (float)D.z);
        vis = warp_trace_clear<COUNT>(P, stack, front, r32, O, D, dd, t_lo, 1.0 - t_lo, (int)r, cnt) &&
              front;
      }
      uint32_t vm = __ballot_sync(0xffffffffu, vis);
      if (P.vis_bits && lane == 0 && tile < P.words)
        P.vis_bits[(c * P.L + l) * P.words + tile] = vm;
      // a6: Eq. 7 in fp64
      if (vis) acc += cosd / (dd * d);
    }
    const float a = (float)(acc * P.scale);
    if (P.values) P.values[c * P.ld + r] = a;
    if (P.col_sumsq) {
      double q = (double)a * (double)a;
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if (lane == 0 && q != 0.0) atomicAdd(P.col_sumsq + c, q);
    }
  }
  if (COUNT && lane == 0)
    for (int k = 0; k < 4; ++k)
      if (cnt[k]) atomicAdd(P.counters + k, cnt[k]);
}

template <bool COUNT>
static int grid_size_assemble() {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assemble<COUNT>, kAsmThreads, 0);
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
  if (P.col_sumsq) UVD_CUDA_TRY(cudaMemsetAsync(P.col_sumsq, 0, n_cols * sizeof(double), st));
  if (P.counters) {
    static int grid_c = 0;
    if (!grid_c) grid_c = grid_size_assemble<true>();
    k_assemble<true><<<grid_c, kAsmThreads, 0, st>>>(P);
  } else {
    static int grid = 0;
    if (!grid) grid = grid_size_assemble<false>();
    k_assemble<false><<<grid, kAsmThreads, 0, st>>>(P);
  }
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  if (dcols) al.put(dcols);
  return UVD_OK;
}
