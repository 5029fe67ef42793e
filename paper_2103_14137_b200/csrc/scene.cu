// scene.cu — uvd_scene_create / query / patches / destroy, error handling and
// the allocator (SURVEY §8(a) row a1 "scene ingest and canonical patch
// attributes"; §8(b) boundary).
//
// Canonical patch attributes are computed in fp64 with explicitly rounded
// intrinsics (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn: no FMA
// contraction) and rounded once to fp32, so they are bit-identical to any
// plain IEEE fp64 evaluation of the same formulas (include/uvd.h documents
// them).
#include <cuda_runtime.h>

#include <chrono>

#include <algorithm>
#include <atomic>
#include <string>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "uvd_internal.cuh"

namespace uvd {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }

static std::atomic<unsigned long long> g_launches{0};

void* host_stage() {
  static thread_local void* p = nullptr;
  if (!p && cudaMallocHost(&p, 64) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  return p;
}
void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

int pointer_device(const void* p) {
  if (!p) return -1;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ? a.device : -1;
}

// total device memory, queried once per device (cudaMemGetInfo took 0.1–20 ms
// per call on the bench box: it sat in every scene build)
size_t device_total_mem(int dev) {
  static size_t cache[kMaxDevices] = {0};
  if (dev < 0 || dev >= kMaxDevices) return 0;
  if (!cache[dev]) {
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, dev) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    cache[dev] = pr.totalGlobalMem;
  }
  return cache[dev];
}

int sm_count(int dev) {
  static int cache[kMaxDevices] = {0};
  if (dev < 0 || dev >= kMaxDevices) return 148;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      v = 148;
    }
    cache[dev] = v;
  }
  return cache[dev];
}

bool HostTrace::on() {
  static const bool v = [] { const char* e = getenv("UVD_TRACE_HOST"); return e && atoi(e) != 0; }();
  return v;
}
static thread_local std::chrono::steady_clock::time_point g_trace_t = std::chrono::steady_clock::now();
static thread_local double g_trace_alloc_us = 0.0;
static thread_local int g_trace_allocs = 0;
void HostTrace::alloc_time(double us) { g_trace_alloc_us += us; ++g_trace_allocs; }
void HostTrace::mark(const char* what) {
  if (!on()) return;
  const auto t = std::chrono::steady_clock::now();
  fprintf(stderr, "[uvd-host] %-28s %9.1f us  (allocator %d calls %8.1f us)\n", what,
          std::chrono::duration<double, std::micro>(t - g_trace_t).count(), g_trace_allocs, g_trace_alloc_us);
  g_trace_t = t;
  g_trace_alloc_us = 0.0;
  g_trace_allocs = 0;
}

void* Alloc::get(size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  if (has_user) {
    if (!HostTrace::on()) return user.alloc(bytes, device, (void*)stream, user.ctx);
    const auto t = std::chrono::steady_clock::now();
    void* p = user.alloc(bytes, device, (void*)stream, user.ctx);
    HostTrace::alloc_time(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count());
    return p;
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
void Alloc::put(void* p) {
  if (!p) return;
  if (has_user) {
    if (!HostTrace::on()) { user.free(p, device, (void*)stream, user.ctx); return; }
    const auto t = std::chrono::steady_clock::now();
    user.free(p, device, (void*)stream, user.ctx);
    HostTrace::alloc_time(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count());
  } else {
    cudaFreeAsync(p, stream);
  }
}

// --------------------------------------------------------- fp64 helpers --
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// 3D patch = triangle: c = fl32(((a+b)+c)/3), n = fl32(cross(b-a, c-a)/|.|),
// area = |cross|/2 (P:158, P:248 mean irradiance needs |s_i|).
__global__ void k_tri_attrs(const float* __restrict__ V, int64_t nv, const int32_t* __restrict__ F,
                            int64_t nt, float4* __restrict__ tri_in, float* __restrict__ cen,
                            float* __restrict__ nrm, double* __restrict__ area,
                            unsigned long long* __restrict__ bad) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int32_t i0 = F[3 * t], i1 = F[3 * t + 1], i2 = F[3 * t + 2];
  if (i0 < 0 || i1 < 0 || i2 < 0 || i0 >= nv || i1 >= nv || i2 >= nv) {
    atomicMin(bad, (unsigned long long)t);
    return;
  }
  const float* pa = V + 3 * (int64_t)i0;
  const float* pb = V + 3 * (int64_t)i1;
  const float* pc = V + 3 * (int64_t)i2;
  double ax = pa[0], ay = pa[1], az = pa[2];
  double bx = pb[0], by = pb[1], bz = pb[2];
  double cx = pc[0], cy = pc[1], cz = pc[2];
  cen[3 * t + 0] = (float)ddiv(dadd(dadd(ax, bx), cx), 3.0);
  cen[3 * t + 1] = (float)ddiv(dadd(dadd(ay, by), cy), 3.0);
  cen[3 * t + 2] = (float)ddiv(dadd(dadd(az, bz), cz), 3.0);
  double ux = dsub(bx, ax), uy = dsub(by, ay), uz = dsub(bz, az);
  double vx = dsub(cx, ax), vy = dsub(cy, ay), vz = dsub(cz, az);
  double nx = dsub(dmul(uy, vz), dmul(uz, vy));
  double ny = dsub(dmul(uz, vx), dmul(ux, vz));
  double nz = dsub(dmul(ux, vy), dmul(uy, vx));
  double len = __dsqrt_rn(dadd(dadd(dmul(nx, nx), dmul(ny, ny)), dmul(nz, nz)));
  if (!(len > 0.0)) {
    atomicMin(bad, (unsigned long long)t);
    len = 1.0;
  }
  nrm[3 * t + 0] = (float)ddiv(nx, len);
  nrm[3 * t + 1] = (float)ddiv(ny, len);
  nrm[3 * t + 2] = (float)ddiv(nz, len);
  area[t] = ddiv(len, 2.0);
  tri_in[3 * t] = make_float4(pa[0], pa[1], pa[2], __int_as_float(0));
  tri_in[3 * t + 1] = make_float4(pb[0], pb[1], pb[2], __int_as_float((int)t));
  tri_in[3 * t + 2] = make_float4(pc[0], pc[1], pc[2], 0.f);
}

// 2.5D: patch i of wall w (segment s of n_seg): q_s = fl32(e0 + ((e1-e0)*s)/n_seg),
// q_{n_seg} = e1; centroid ((q_s+q_{s+1})/2, h/2); normal (-dy,dx)/len (boundary,
// into the room) or (dy,-dx)/len (obstacle, outward); area len*h.
// Triangles: quad A=(q_s,0) B=(q_{s+1},0) C=(q_{s+1},h) D=(q_s,h) split on A–C,
// wound so the right-hand normal equals n (obstacle: ABC, ACD; boundary: ACB, ADC).
__global__ void k_extrude(const Wall* __restrict__ walls, int64_t n_walls, int64_t N, float h,
                          float4* __restrict__ tri_in, float* __restrict__ cen,
                          float* __restrict__ nrm, double* __restrict__ area) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int64_t lo = 0, hi = n_walls - 1;  // last wall with first_patch <= i
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (walls[mid].first_patch <= i) lo = mid; else hi = mid - 1;
  }
  Wall w = walls[lo];
  int64_t s = i - w.first_patch;
  double ex = dsub((double)w.e1x, (double)w.e0x), ey = dsub((double)w.e1y, (double)w.e0y);
  double ns = (double)w.n_seg;
  float qax = (float)dadd((double)w.e0x, ddiv(dmul(ex, (double)s), ns));
  float qay = (float)dadd((double)w.e0y, ddiv(dmul(ey, (double)s), ns));
  float qbx, qby;
  if (s + 1 == w.n_seg) { qbx = w.e1x; qby = w.e1y; }
  else {
    qbx = (float)dadd((double)w.e0x, ddiv(dmul(ex, (double)(s + 1)), ns));
    qby = (float)dadd((double)w.e0y, ddiv(dmul(ey, (double)(s + 1)), ns));
  }
  double dx = dsub((double)qbx, (double)qax), dy = dsub((double)qby, (double)qay);
  double len = __dsqrt_rn(dadd(dmul(dx, dx), dmul(dy, dy)));
  cen[3 * i + 0] = (float)ddiv(dadd((double)qax, (double)qbx), 2.0);
  cen[3 * i + 1] = (float)ddiv(dadd((double)qay, (double)qby), 2.0);
  cen[3 * i + 2] = (float)ddiv((double)h, 2.0);
  double nx = w.boundary ? ddiv(-dy, len) : ddiv(dy, len);
  double ny = w.boundary ? ddiv(dx, len) : ddiv(-dx, len);
  nrm[3 * i + 0] = (float)nx;
  nrm[3 * i + 1] = (float)ny;
  nrm[3 * i + 2] = 0.f;
  area[i] = dmul(len, (double)h);
  float4 A = make_float4(qax, qay, 0.f, 0.f), B = make_float4(qbx, qby, 0.f, 0.f);
  float4 C = make_float4(qbx, qby, h, 0.f), D = make_float4(qax, qay, h, 0.f);
  float4 t0[3], t1[3];
  if (!w.boundary) { t0[0] = A; t0[1] = B; t0[2] = C; t1[0] = A; t1[1] = C; t1[2] = D; }
  else { t0[0] = A; t0[1] = C; t0[2] = B; t1[0] = A; t1[1] = D; t1[2] = C; }
  t0[0].w = __int_as_float((int)i); t0[1].w = __int_as_float((int)(2 * i)); t0[2].w = 0.f;
  t1[0].w = __int_as_float((int)i); t1[1].w = __int_as_float((int)(2 * i + 1)); t1[2].w = 0.f;
  for (int k = 0; k < 3; ++k) {
    tri_in[3 * (2 * i) + k] = t0[k];
    tri_in[3 * (2 * i + 1) + k] = t1[k];
  }
}

// 3D canonical order = sorted (Morton) order: permute patch attributes and set
// the owner patch id of each triangle to its sorted position.
__global__ void k_permute_patches(const uint32_t* __restrict__ order, int64_t N,
                                  const float* __restrict__ cen_in, const float* __restrict__ nrm_in,
                                  const double* __restrict__ area_in, float* __restrict__ cen,
                                  float* __restrict__ nrm, double* __restrict__ area,
                                  int64_t* __restrict__ orig) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= N) return;
  int64_t t = order[r];
  for (int k = 0; k < 3; ++k) {
    cen[3 * r + k] = cen_in[3 * t + k];
    nrm[3 * r + k] = nrm_in[3 * t + k];
  }
  area[r] = area_in[t];
  orig[r] = t;
}

__global__ void k_iota64(int64_t* __restrict__ a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

// deterministic total area: fixed-shape tree reduction in one block
__global__ void __launch_bounds__(1024) k_sum_area(const double* __restrict__ a, int64_t n,
                                                   double* __restrict__ out) {
  __shared__ double part[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) s += a[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (threadIdx.x < off) part[threadIdx.x] += part[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

static inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// vertex validation + bbox on the device: per-block min/max partials and the
// first non-finite vertex index
constexpr int kBoxThreads = 256;
__global__ void __launch_bounds__(kBoxThreads) k_vert_bbox(const float* __restrict__ V, int64_t nv,
                                                           float* __restrict__ part,
                                                           unsigned long long* __restrict__ bad) {
  __shared__ float s[6][kBoxThreads];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t v = blockIdx.x * (int64_t)kBoxThreads + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * kBoxThreads) {
    float p[3] = {V[3 * v], V[3 * v + 1], V[3 * v + 2]};
    for (int k = 0; k < 3; ++k) {
      if (!isfinite(p[k])) atomicMin(bad, (unsigned long long)v);
      lo[k] = fminf(lo[k], p[k]);
      hi[k] = fmaxf(hi[k], p[k]);
    }
  }
  for (int k = 0; k < 3; ++k) { s[k][threadIdx.x] = lo[k]; s[3 + k][threadIdx.x] = hi[k]; }
  __syncthreads();
  for (int off = kBoxThreads / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
      for (int k = 0; k < 3; ++k) {
        s[k][threadIdx.x] = fminf(s[k][threadIdx.x], s[k][threadIdx.x + off]);
        s[3 + k][threadIdx.x] = fmaxf(s[3 + k][threadIdx.x], s[3 + k][threadIdx.x + off]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[6 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_bbox_final(const float* __restrict__ part, int nb, float* __restrict__ out) {
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? INFINITY : -INFINITY;
    for (int b = 0; b < nb; ++b)
      v = threadIdx.x < 3 ? fminf(v, part[6 * b + threadIdx.x]) : fmaxf(v, part[6 * b + threadIdx.x]);
    out[threadIdx.x] = v;
  }
}

static int create_trimesh(uvd_scene* s, const uvd_scene_desc* d, cudaStream_t st) {
  if (!d->vertices || !d->tris || d->n_vertices <= 0 || d->n_tris <= 0) {
    set_error("scene: TRIMESH needs vertices and triangles");
    return UVD_ERR_INVALID;
  }
  if (d->n_tris >= (int64_t)1 << 28) {
    set_error("scene: at most 2^28 triangles supported (got %lld)", (long long)d->n_tris);
    return UVD_ERR_INVALID;
  }
  Alloc& al = s->alloc;
  Scratch sc(al, st);  // this function's temporaries, released at every exit
  const int64_t M = d->n_tris, NV = d->n_vertices;
  s->M = M;
  s->N = M;
  float* dV = (float*)sc.get(NV * 3 * sizeof(float));
  int32_t* dF = (int32_t*)sc.get(M * 3 * sizeof(int32_t));
  float4* tri_in = (float4*)sc.get(3 * M * sizeof(float4));
  float* cen_in = (float*)sc.get(M * 3 * sizeof(float));
  float* nrm_in = (float*)sc.get(M * 3 * sizeof(float));
  double* area_in = (double*)sc.get(M * sizeof(double));
  unsigned long long* bad = (unsigned long long*)sc.get(sizeof(unsigned long long));
  if (!dV || !dF || !tri_in || !cen_in || !nrm_in || !area_in || !bad) {
    set_error("scene: out of device memory (M=%lld)", (long long)M);
    return UVD_ERR_NOMEM;
  }
  const cudaMemcpyKind kind = d->device_input ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  UVD_CUDA_TRY(cudaMemcpyAsync(dV, d->vertices, NV * 3 * sizeof(float), kind, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(dF, d->tris, M * 3 * sizeof(int32_t), kind, st));
  UVD_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  {
    int nb = (int)std::min<int64_t>((NV + kBoxThreads - 1) / kBoxThreads, 1184);
    float* part = (float*)sc.get((size_t)nb * 6 * sizeof(float) + 6 * sizeof(float) + 64);
    unsigned long long* vbad = (unsigned long long*)sc.get(sizeof(unsigned long long));
    if (!part || !vbad) { set_error("scene: out of device memory"); return UVD_ERR_NOMEM; }
    float* box = part + 6 * nb;
    UVD_CUDA_TRY(cudaMemsetAsync(vbad, 0xff, sizeof(unsigned long long), st));
    k_vert_bbox<<<nb, kBoxThreads, 0, st>>>(dV, NV, part, vbad);
    note_launch();
    k_bbox_final<<<1, 32, 0, st>>>(part, nb, box);
    note_launch();
    unsigned long long h_vbad = 0;
    UVD_CUDA_TRY(cudaMemcpyAsync(s->bbox, box, 6 * sizeof(float), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaMemcpyAsync(&h_vbad, vbad, sizeof(h_vbad), cudaMemcpyDeviceToHost, st));
    UVD_CUDA_TRY(cudaStreamSynchronize(st));
    sc.release(part);
    sc.release(vbad);
    if (h_vbad != ~0ull) {
      set_error("scene: vertex %llu is not finite", h_vbad);
      return UVD_ERR_INVALID;
    }
  }
  k_tri_attrs<<<grid_for(M, 256), 256, 0, st>>>(dV, NV, dF, M, tri_in, cen_in, nrm_in, area_in, bad);
  note_launch();
  unsigned long long h_bad = 0;
  UVD_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, st));
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_bad != ~0ull) {
    set_error("scene: triangle %llu has an out-of-range index or zero area (S:32)", h_bad);
    return UVD_ERR_INVALID;
  }
  uint32_t* order = nullptr;
  UVD_TRY(build_bvh(s, tri_in, &order, st));
  sc.ps.push_back(order);  // build_bvh hands the permutation over
  s->centroid = (float*)al.get(M * 3 * sizeof(float));
  s->normal = (float*)al.get(M * 3 * sizeof(float));
  s->area = (double*)al.get(M * sizeof(double));
  s->orig_id = (int64_t*)al.get(M * sizeof(int64_t));
  if (!s->centroid || !s->normal || !s->area || !s->orig_id) {
    set_error("scene: out of device memory (patches)");
    return UVD_ERR_NOMEM;
  }
  k_permute_patches<<<grid_for(M, 256), 256, 0, st>>>(order, M, cen_in, nrm_in, area_in,
                                                       s->centroid, s->normal, s->area,
                                                       s->orig_id);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  return UVD_OK;
}

static int create_extruded(uvd_scene* s, const uvd_scene_desc* d, cudaStream_t st) {
  const float* b = d->bounds;
  for (int k = 0; k < 4; ++k)
    if (!std::isfinite(b[k])) { set_error("scene: non-finite bounds"); return UVD_ERR_INVALID; }
  if (!(b[2] > b[0] && b[3] > b[1])) { set_error("scene: degenerate bounds"); return UVD_ERR_INVALID; }
  if (!(d->wall_height > 0.f) || !std::isfinite(d->wall_height)) {
    set_error("scene: wall_height must be > 0");
    return UVD_ERR_INVALID;
  }
  if (!(d->patch_res > 0.f) || !std::isfinite(d->patch_res)) {
    set_error("scene: patch_res must be > 0");
    return UVD_ERR_INVALID;
  }
  if (d->n_obstacles < 0 || (d->n_obstacles > 0 && !d->obstacles)) {
    set_error("scene: bad obstacle list");
    return UVD_ERR_INVALID;
  }
  std::vector<Wall>& W = s->h_walls;
  W.clear();
  std::vector<float> pxy;
  std::vector<int32_t> poff(1, 0);
  float cx[4] = {b[0], b[2], b[2], b[0]}, cy[4] = {b[1], b[1], b[3], b[3]};
  for (int k = 0; k < 4; ++k) {
    Wall w{cx[k], cy[k], cx[(k + 1) % 4], cy[(k + 1) % 4], 1, 0, 0};
    W.push_back(w);
  }
  for (int p = 0; p < d->n_obstacles; ++p) {
    const uvd_polygon& P = d->obstacles[p];
    if (P.n < 3 || !P.xy) { set_error("scene: obstacle %d has fewer than 3 vertices", p); return UVD_ERR_INVALID; }
    for (int k = 0; k < P.n; ++k) {
      float x = P.xy[2 * k], y = P.xy[2 * k + 1];
      if (!std::isfinite(x) || !std::isfinite(y) || !(x > b[0] && x < b[2] && y > b[1] && y < b[3])) {
        set_error("scene: obstacle %d vertex %d outside the bounds (S:24)", p, k);
        return UVD_ERR_INVALID;
      }
      pxy.push_back(x);
      pxy.push_back(y);
      const float* u = P.xy + 2 * ((k + 1) % P.n);
      Wall w{x, y, u[0], u[1], 0, 0, 0};
      W.push_back(w);
    }
    poff.push_back((int32_t)(pxy.size() / 2));
  }
  int64_t N = 0;
  for (Wall& w : W) {
    double dx = (double)w.e1x - (double)w.e0x, dy = (double)w.e1y - (double)w.e0y;
    double len = std::sqrt(dx * dx + dy * dy);
    if (!(len > 0.0)) { set_error("scene: zero-length wall"); return UVD_ERR_INVALID; }
    double ns = std::ceil(len / (double)d->patch_res);
    w.n_seg = (int32_t)ns;
    w.first_patch = N;
    N += w.n_seg;
  }
  s->N = N;
  s->M = 2 * N;
  s->n_walls = (int64_t)W.size();
  s->n_poly = d->n_obstacles;
  for (int k = 0; k < 4; ++k) s->bounds[k] = b[k];
  s->wall_height = d->wall_height;
  s->bbox[0] = b[0]; s->bbox[1] = b[1]; s->bbox[2] = 0.f;
  s->bbox[3] = b[2]; s->bbox[4] = b[3]; s->bbox[5] = d->wall_height;
  Alloc& al = s->alloc;
  s->walls = (Wall*)al.get(W.size() * sizeof(Wall));
  s->n_poly_xy = (int64_t)std::max<size_t>(pxy.size(), 2);
  s->poly_xy = (float*)al.get(s->n_poly_xy * sizeof(float));
  s->n_poly_off = (int64_t)poff.size();
  s->poly_off = (int32_t*)al.get(poff.size() * sizeof(int32_t));
  float4* tri_in = (float4*)al.get(3 * s->M * sizeof(float4));
  s->ptri = tri_in;  // patch-ordered wall triangles (2 per patch) for the area model (NEXT-2)
  s->centroid = (float*)al.get(N * 3 * sizeof(float));
  s->normal = (float*)al.get(N * 3 * sizeof(float));
  s->area = (double*)al.get(N * sizeof(double));
  s->orig_id = (int64_t*)al.get(N * sizeof(int64_t));
  if (!s->walls || !s->poly_xy || !s->poly_off || !tri_in || !s->centroid || !s->normal ||
      !s->area || !s->orig_id) {
    set_error("scene: out of device memory (N=%lld)", (long long)N);
    return UVD_ERR_NOMEM;
  }
  UVD_CUDA_TRY(cudaMemcpyAsync(s->walls, W.data(), W.size() * sizeof(Wall), cudaMemcpyHostToDevice, st));
  if (!pxy.empty())
    UVD_CUDA_TRY(cudaMemcpyAsync(s->poly_xy, pxy.data(), pxy.size() * sizeof(float), cudaMemcpyHostToDevice, st));
  UVD_CUDA_TRY(cudaMemcpyAsync(s->poly_off, poff.data(), poff.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_extrude<<<grid_for(N, 256), 256, 0, st>>>(s->walls, s->n_walls, N, d->wall_height, tri_in,
                                              s->centroid, s->normal, s->area);
  note_launch();
  k_iota64<<<grid_for(N, 256), 256, 0, st>>>(s->orig_id, N);
  note_launch();
  UVD_TRY(build_bvh(s, tri_in, nullptr, st));
  // pageable H2D copies above may still read the host vectors: finish first
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  return UVD_OK;
}

// Every stream that used the scene must be done with it before its buffers go
// back to the allocator (a caching allocator may hand them out at once): the
// device is synchronised first (uvd.h, uvd_scene_destroy).
static void free_scene(uvd_scene* s) {
  if (!s) return;
  DeviceGuard dg(s->alloc.device);
  cudaDeviceSynchronize();
  cudaGetLastError();
  Alloc& al = s->alloc;
  for (void* p : {(void*)s->centroid, (void*)s->normal, (void*)s->area, (void*)s->orig_id,
                  (void*)s->tri, (void*)s->nodes, (void*)s->walls, (void*)s->poly_xy,
                  (void*)s->poly_off, (void*)s->err_flag, (void*)s->ptri, (void*)s->onodes, (void*)s->front_free, (void*)s->hnodes})
    al.put(p);
  for (auto& c : s->cov_part) al.put(c.p);
  cudaStreamSynchronize(al.stream);
  delete s;
}

}  // namespace uvd

using namespace uvd;

extern "C" int uvd_scene_create(const uvd_scene_desc* desc, int device, void* stream,
                                const uvd_allocator* allocator, uvd_scene** out) {
  clear_error();
  if (!desc || !out) { set_error("uvd_scene_create: null argument"); return UVD_ERR_INVALID; }
  *out = nullptr;
  if (desc->kind != UVD_SCENE_TRIMESH && desc->kind != UVD_SCENE_EXTRUDED) {
    set_error("uvd_scene_create: unknown kind %d", desc->kind);
    return UVD_ERR_INVALID;
  }
  NvtxRange nv("uvd_scene_create");
  int ndev = 0;
  UVD_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("uvd_scene_create: no device %d", device); return UVD_ERR_INVALID; }
  DeviceGuard dg(device);  // the caller's current device is restored on return
  uvd_scene* s = new uvd_scene();
  s->kind = desc->kind;
  s->alloc.device = device;
  s->alloc.stream = (cudaStream_t)stream;
  if (allocator && allocator->alloc && allocator->free) {
    s->alloc.user = *allocator;
    s->alloc.has_user = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  HostTrace::mark("scene_create: enter");
  int rc = desc->kind == UVD_SCENE_TRIMESH ? create_trimesh(s, desc, st) : create_extruded(s, desc, st);
  HostTrace::mark("scene_create: trimesh+bvh");
  if (rc == UVD_OK) rc = front_radius(s, st);  // patches (row order) and BVH are final here
  if (rc == UVD_OK && !host_stage()) {
    set_error("scene: out of pinned host memory (staging)");
    rc = UVD_ERR_NOMEM;
  }
  if (rc == UVD_OK) {
    s->err_flag = (int*)s->alloc.get(sizeof(int));
    double* dsum = (double*)s->alloc.get(sizeof(double));
    if (!s->err_flag || !dsum) { set_error("scene: out of device memory"); rc = UVD_ERR_NOMEM; }
    else {
      cudaMemsetAsync(s->err_flag, 0, sizeof(int), st);
      k_sum_area<<<1, 1024, 0, st>>>(s->area, s->N, dsum);
      note_launch();
      cudaMemcpyAsync(&s->total_area, dsum, sizeof(double), cudaMemcpyDeviceToHost, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) { set_error("scene: %s", cudaGetErrorString(e)); rc = UVD_ERR_CUDA; }
      s->alloc.put(dsum);
    }
  }
  HostTrace::mark("scene_create: radii+area+sync");
  if (rc != UVD_OK) {
    std::string msg = uvd_last_error();
    free_scene(s);
    set_error("%s", msg.c_str());
    return rc;
  }
  *out = s;
  return UVD_OK;
}

extern "C" int uvd_scene_query(const uvd_scene* s, int64_t* n_patches, int64_t* n_tris,
                               float bbox[6], double* total_area) {
  clear_error();
  if (!s) { set_error("uvd_scene_query: null scene"); return UVD_ERR_INVALID; }
  if (n_patches) *n_patches = s->N;
  if (n_tris) *n_tris = s->M;
  if (bbox) for (int k = 0; k < 6; ++k) bbox[k] = s->bbox[k];
  if (total_area) *total_area = s->total_area;
  return UVD_OK;
}

extern "C" int uvd_scene_patches(const uvd_scene* s, float* centroid, float* normal, double* area,
                                 int64_t* orig_id, void* stream) {
  clear_error();
  if (!s) { set_error("uvd_scene_patches: null scene"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_scene_patches");
  cudaStream_t st = (cudaStream_t)stream;
  if (centroid) UVD_CUDA_TRY(cudaMemcpyAsync(centroid, s->centroid, s->N * 3 * sizeof(float), cudaMemcpyDeviceToDevice, st));
  if (normal) UVD_CUDA_TRY(cudaMemcpyAsync(normal, s->normal, s->N * 3 * sizeof(float), cudaMemcpyDeviceToDevice, st));
  if (area) UVD_CUDA_TRY(cudaMemcpyAsync(area, s->area, s->N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (orig_id) UVD_CUDA_TRY(cudaMemcpyAsync(orig_id, s->orig_id, s->N * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  return UVD_OK;
}

extern "C" void uvd_scene_destroy(uvd_scene* s) { free_scene(s); }

namespace uvd {
__global__ void k_take_flag(int* flag, int* out) { *out = atomicExch(flag, 0); }
}  // namespace uvd

extern "C" int uvd_sync_status(const uvd_scene* s, void* stream) {
  clear_error();
  if (!s) { set_error("uvd_sync_status: null scene"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_sync_status");
  cudaStream_t st = (cudaStream_t)stream;
  int* hflag = (int*)host_stage();  // pinned: device-visible under unified addressing
  if (!hflag) { set_error("uvd_sync_status: out of pinned host memory"); return UVD_ERR_NOMEM; }
  // read and clear in one atomic: an error raised meanwhile by a kernel on
  // another stream stays in the flag for the next call instead of being lost
  k_take_flag<<<1, 1, 0, st>>>(s->err_flag, hflag);
  note_launch();
  UVD_CUDA_TRY(cudaGetLastError());
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  const int flag = *(volatile int*)hflag;
  if (flag) {
    if (flag == 2) {  // cannot happen: scene creation refuses trees deeper than the stacks
      set_error("traversal stack overflow (BVH deeper than 64)");
      return UVD_ERR_CUDA;
    }
    if (flag == 3) {  // assemble.cu k_check_lamps
      set_error("lamp sample outside the validated range (|coordinate| > the scene's largest + 50 m, or "
                "non-finite): the box padding does not cover its rounding");
      return UVD_ERR_INVALID;
    }
    set_error("lamp–centroid distance below 1e-9 m (S:160)");
    return UVD_ERR_DOMAIN;
  }
  return UVD_OK;
}

extern "C" const char* uvd_last_error(void) { return uvd::g_err; }
extern "C" int uvd_version(void) { return 100; }
extern "C" unsigned long long uvd_launch_count(void) { return g_launches.load(); }

extern "C" int uvd_scene_bvh(const uvd_scene* s, void* nodes, float* tri, int64_t* n_nodes, uint32_t* root,
                             void* stream) {
  clear_error();
  if (!s) { set_error("uvd_scene_bvh: null scene"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_scene_bvh");
  const int64_t nn = std::max<int64_t>(s->M - 1, 1);
  if (n_nodes) *n_nodes = nn;
  if (root) *root = s->root;
  cudaStream_t st = (cudaStream_t)stream;
  if (nodes) UVD_CUDA_TRY(cudaMemcpyAsync(nodes, s->nodes, nn * sizeof(Node), cudaMemcpyDeviceToDevice, st));
  if (tri) UVD_CUDA_TRY(cudaMemcpyAsync(tri, s->tri, s->M * 3 * sizeof(float4), cudaMemcpyDeviceToDevice, st));
  return UVD_OK;
}

// ------------------------------------------------------------ export/import --
// One scene build shipped to the other ranks ("rank 0 builds and
// runs ncclBroadcast of ≈112 MB").  A flat DEVICE buffer: a 256-B header, then
// 256-B aligned sections (patch attributes, leaf-ordered triangles, BVH nodes,
// front radii, and for 2.5D scenes the wall and polygon tables and the
// patch-ordered wall triangles).  The octant node copies are rebuilt by the
// importer (k_octant_nodes, ~0.2 ms on C5) instead of shipped (8x the nodes).
namespace uvd {
struct SceneHdr {
  uint64_t magic;
  int32_t version, kind;
  int64_t N, M, n_nodes;
  uint32_t root;
  int32_t n_poly;
  float bbox[6];
  double total_area;
  float bounds[4];
  float wall_height;
  int32_t has_ptri;
  int64_t n_walls, n_poly_xy, n_poly_off;
  uint64_t off[12];  // section offsets (bytes from the buffer start)
  uint64_t total;
};
static_assert(sizeof(SceneHdr) <= 256, "scene header fits 256 B");
constexpr uint64_t kSceneMagic = 0x3130646576557655ull;  // "UvUved01"
enum { S_CEN, S_NRM, S_AREA, S_ORIG, S_TRI, S_NODES, S_FRONT, S_WALLS, S_PXY, S_POFF, S_PTRI, S_COUNT };

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static void section_sizes(const SceneHdr& h, size_t sz[S_COUNT]) {
  sz[S_CEN] = (size_t)h.N * 3 * sizeof(float);
  sz[S_NRM] = (size_t)h.N * 3 * sizeof(float);
  sz[S_AREA] = (size_t)h.N * sizeof(double);
  sz[S_ORIG] = (size_t)h.N * sizeof(int64_t);
  sz[S_TRI] = (size_t)h.M * 3 * sizeof(float4);
  sz[S_NODES] = (size_t)h.n_nodes * sizeof(Node);
  sz[S_FRONT] = (size_t)h.N * sizeof(float);
  sz[S_WALLS] = (size_t)h.n_walls * sizeof(Wall);
  sz[S_PXY] = (size_t)h.n_poly_xy * sizeof(float);
  sz[S_POFF] = (size_t)h.n_poly_off * sizeof(int32_t);
  sz[S_PTRI] = h.has_ptri ? (size_t)h.N * 2 * 3 * sizeof(float4) : 0;
}

static SceneHdr make_hdr(const uvd_scene* s) {
  SceneHdr h;
  memset(&h, 0, sizeof(h));
  h.magic = kSceneMagic;
  h.version = 1;
  h.kind = s->kind;
  h.N = s->N;
  h.M = s->M;
  h.n_nodes = s->n_nodes;
  h.root = s->root;
  h.n_poly = s->n_poly;
  memcpy(h.bbox, s->bbox, sizeof(h.bbox));
  h.total_area = s->total_area;
  memcpy(h.bounds, s->bounds, sizeof(h.bounds));
  h.wall_height = s->wall_height;
  h.has_ptri = s->ptri != nullptr;
  h.n_walls = s->walls ? s->n_walls : 0;
  h.n_poly_xy = s->kind == UVD_SCENE_EXTRUDED ? s->n_poly_xy : 0;
  h.n_poly_off = s->kind == UVD_SCENE_EXTRUDED ? s->n_poly_off : 0;
  size_t sz[S_COUNT];
  section_sizes(h, sz);
  uint64_t o = 256;
  for (int k = 0; k < S_COUNT; ++k) {
    h.off[k] = o;
    o += al256(sz[k]);
  }
  h.total = o;
  return h;
}
}  // namespace uvd

extern "C" int uvd_scene_export(const uvd_scene* s, void* buf, size_t* bytes, void* stream) {
  clear_error();
  if (!s || !bytes) { set_error("uvd_scene_export: null argument"); return UVD_ERR_INVALID; }
  DeviceGuard dg(s->alloc.device);
  NvtxRange nv("uvd_scene_export");
  const SceneHdr h = make_hdr(s);
  if (!buf) { *bytes = h.total; return UVD_OK; }
  if (*bytes < h.total) {
    set_error("uvd_scene_export: buffer of %zu bytes, need %llu", *bytes, (unsigned long long)h.total);
    *bytes = h.total;
    return UVD_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* b = (char*)buf;
  size_t sz[S_COUNT];
  section_sizes(h, sz);
  const void* src[S_COUNT] = {s->centroid, s->normal, s->area, s->orig_id, s->tri, s->nodes, s->front_free,
                              s->walls, s->poly_xy, s->poly_off, s->ptri};
  UVD_CUDA_TRY(cudaMemcpyAsync(b, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  for (int k = 0; k < S_COUNT; ++k)
    if (sz[k]) UVD_CUDA_TRY(cudaMemcpyAsync(b + h.off[k], src[k], sz[k], cudaMemcpyDeviceToDevice, st));
  UVD_CUDA_TRY(cudaStreamSynchronize(st));  // the header is a stack variable
  *bytes = h.total;
  return UVD_OK;
}

extern "C" int uvd_scene_import(const void* buf, size_t bytes, int device, void* stream,
                                const uvd_allocator* allocator, uvd_scene** out) {
  clear_error();
  if (!buf || !out) { set_error("uvd_scene_import: null argument"); return UVD_ERR_INVALID; }
  *out = nullptr;
  NvtxRange nv("uvd_scene_import");
  int ndev = 0;
  UVD_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("uvd_scene_import: no device %d", device); return UVD_ERR_INVALID; }
  DeviceGuard dg(device);
  cudaStream_t st = (cudaStream_t)stream;
  SceneHdr h;
  if (bytes < sizeof(h)) { set_error("uvd_scene_import: buffer too small"); return UVD_ERR_INVALID; }
  UVD_CUDA_TRY(cudaMemcpyAsync(&h, buf, sizeof(h), cudaMemcpyDeviceToHost, st));
  UVD_CUDA_TRY(cudaStreamSynchronize(st));
  if (h.magic != kSceneMagic || h.version != 1 || h.total > bytes || h.N < 1 || h.M < 1 ||
      (h.kind != UVD_SCENE_TRIMESH && h.kind != UVD_SCENE_EXTRUDED)) {
    set_error("uvd_scene_import: not a uvd_scene_export buffer (or truncated)");
    return UVD_ERR_INVALID;
  }
  const SceneHdr ref = [&] {  // the section layout the header must describe
    SceneHdr r = h;
    size_t sz[S_COUNT];
    section_sizes(r, sz);
    uint64_t o = 256;
    for (int k = 0; k < S_COUNT; ++k) { r.off[k] = o; o += al256(sz[k]); }
    r.total = o;
    return r;
  }();
  if (memcmp(ref.off, h.off, sizeof(h.off)) != 0 || ref.total != h.total) {
    set_error("uvd_scene_import: inconsistent section table");
    return UVD_ERR_INVALID;
  }
  uvd_scene* s = new uvd_scene();
  s->kind = h.kind;
  s->alloc.device = device;
  s->alloc.stream = st;
  if (allocator && allocator->alloc && allocator->free) {
    s->alloc.user = *allocator;
    s->alloc.has_user = true;
  }
  s->N = h.N; s->M = h.M; s->n_nodes = h.n_nodes; s->root = h.root; s->n_poly = h.n_poly;
  memcpy(s->bbox, h.bbox, sizeof(h.bbox));
  s->total_area = h.total_area;
  memcpy(s->bounds, h.bounds, sizeof(h.bounds));
  s->wall_height = h.wall_height;
  s->n_walls = h.n_walls;
  s->n_poly_xy = h.n_poly_xy;
  s->n_poly_off = h.n_poly_off;
  size_t sz[S_COUNT];
  section_sizes(h, sz);
  void** dst[S_COUNT] = {(void**)&s->centroid, (void**)&s->normal, (void**)&s->area, (void**)&s->orig_id,
                         (void**)&s->tri, (void**)&s->nodes, (void**)&s->front_free, (void**)&s->walls,
                         (void**)&s->poly_xy, (void**)&s->poly_off, (void**)&s->ptri};
  int rc = UVD_OK;
  const char* b = (const char*)buf;
  for (int k = 0; k < S_COUNT && rc == UVD_OK; ++k) {
    if (!sz[k]) continue;
    *dst[k] = s->alloc.get(sz[k]);
    if (!*dst[k]) { set_error("uvd_scene_import: out of device memory"); rc = UVD_ERR_NOMEM; break; }
    if (cudaMemcpyAsync(*dst[k], b + h.off[k], sz[k], cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      set_error("uvd_scene_import: %s", cudaGetErrorString(cudaGetLastError()));
      rc = UVD_ERR_CUDA;
    }
  }
  if (rc == UVD_OK) rc = build_octants(s, st);
  if (rc == UVD_OK) rc = build_hnodes(s, st);
  if (rc == UVD_OK) {
    s->err_flag = (int*)s->alloc.get(sizeof(int));
    if (!s->err_flag || !host_stage()) { set_error("uvd_scene_import: out of memory"); rc = UVD_ERR_NOMEM; }
    else if (cudaMemsetAsync(s->err_flag, 0, sizeof(int), st) != cudaSuccess ||
             cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("uvd_scene_import: %s", cudaGetErrorString(cudaGetLastError()));
      rc = UVD_ERR_CUDA;
    }
  }
  if (rc != UVD_OK) {
    std::string msg = uvd_last_error();
    free_scene(s);
    set_error("%s", msg.c_str());
    return rc;
  }
  *out = s;
  return UVD_OK;
}
