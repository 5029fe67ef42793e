/*
 * uvd.h — C-ABI of the B200-native irradiance-matrix engine (libuvd.so).
 *
 * The hot path of arXiv 2103.14137 "Optimized Coverage Planning for UV Surface
 * Disinfection" (SURVEY §8(a) rows a1–a8): assemble the occlusion-tested
 * irradiance matrix A[patch i, vantage configuration j] (§IV-C, PAPER.md
 * P:223–254), then the fluence products A·t and Aᵀ·y (Eq. 5; the
 * LP of Eq. 8/9) and the area coverage (P:9).
 *
 * Conventions: lengths in metres, power in W, time in s,
 * irradiance in W/m², fluence in J/m².  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, Q# = reading n in DESIGN.md §Readings.
 *
 * Ownership: the caller owns every input; the library copies what it needs
 * during the call and retains no caller pointer.  A scene owns its device
 * buffers (allocated through the uvd_allocator, default cudaMallocAsync) and
 * releases them in uvd_scene_destroy.  Outputs are caller-allocated DEVICE
 * buffers unless a parameter says "host".
 *
 * Streams: every call enqueues on `stream` (a cudaStream_t, NULL = legacy
 * default stream).  Calls that return host scalars synchronise that stream:
 * uvd_scene_create, uvd_vantage_sample, uvd_sync_status, uvd_coverage (and
 * uvd_static_columns when asked for its choice).
 * A scene's data are immutable after creation; const calls on one scene may
 * run concurrently on different streams or threads (the only per-scene
 * mutable state — coverage partial sums — is kept per stream; the in-kernel
 * error flag is shared, see uvd_sync_status).
 * Devices: every call runs on the device of its scene (uvd_fluence /
 * uvd_lp_solve: of their `out` / `t` buffer) and restores the caller's current
 * device before returning.
 *
 * Profiling: every entry point is an NVTX range named after it.
 *
 * Errors: no exception crosses the ABI.  Calls return UVD_OK (0) or a
 * negative uvd_status and set a thread-local message (uvd_last_error).  On
 * error, outputs are unspecified.  In-kernel domain errors (lamp–centroid
 * distance < 1e-9 m) set a per-scene device flag reported by
 * uvd_sync_status.
 *
 * Environment (read per call; defaults are the measured best):
 *   UVD_BVH=sah|ploc|karras   BVH builder of uvd_scene_create (default sah)
 *   UVD_SAH_HUGE=n, UVD_SAH_CHUNK=n   nodes above n triangles split over CTAs
 *                             in chunks (default 65536 / 32768; tests only)
 *   UVD_OCT=0                 no octant node copies (default: built when they
 *                             take <= 1/16 of device memory)
 *   UVD_ASM_SUPER=k           assembly work order: super-tiles of 2^k tiles,
 *                             < 0 column-major (default: 11 when the traversal
 *                             data exceeds 2x the L2, else column-major)
 *   UVD_FIXUP_CAP=n           capacity of the exact re-trace list (tests only)
 *   UVD_FREE=0                no empty end regions (free.cu) in the walk's box
 *                             tests (dev A/B); UVD_FREE_CAP=r caps the front
 *                             radius search at r m (default 0.1)
 *   UVD_HNODES=0              the walk skips the fp16 copies of the top BVH
 *                             levels (hnodes.cu; dev A/B); UVD_HDEPTH=d builds
 *                             them for depth <= d (default 6, read by
 *                             uvd_scene_create / uvd_scene_import)
 *   UVD_MULTI_PART_MAX=bytes  uvd_fluence_multi's scratch cap before it falls
 *                             back to one pass per product (default 4 GB; tests)
 *   UVD_TRACE_HOST=1          wall-clock marks of a scene build's host stages
 *                             and allocator-callback time, to stderr (development)
 *   UVD_LP_*                  PDHG tuning knobs of uvd_lp_solve (lp.cu; they
 *                             change the iterates, not the optimum)
 * The others never change a result: every setting gives bit-identical A and
 * visibility bits (tests/test_gpu_order.py, tests/test_gpu_bvh.py,
 * tests/test_gpu_hnodes.py).
 */
#ifndef UVD_H_
#define UVD_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define UVD_API __attribute__((visibility("default")))
#else
#define UVD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  UVD_OK = 0,
  UVD_ERR_INVALID = -1,   /* bad argument / non-finite input / zero-area triangle */
  UVD_ERR_DOMAIN = -2,    /* lamp–centroid distance < 1e-9 m                    */
  UVD_ERR_EMPTY = -3,     /* zero feasible vantage configurations               */
  UVD_ERR_CAPACITY = -4,  /* caller buffer too small; required size returned            */
  UVD_ERR_NOMEM = -5,     /* device allocation failed                                    */
  UVD_ERR_CUDA = -6       /* CUDA runtime failure (message = cudaGetErrorString)          */
} uvd_status;

/* Optional device allocator (e.g. bound to PyTorch's caching allocator).
 * alloc returns a device pointer (NULL on failure); free releases it.
 * Both are called on the creating thread, stream-ordered on `stream`. */
typedef struct {
  void* (*alloc)(size_t bytes, int device, void* stream, void* ctx);
  void (*free)(void* ptr, int device, void* stream, void* ctx);
  void* ctx;
} uvd_allocator;

/* ------------------------------------------------------------------ a1/a2 */
typedef struct uvd_scene uvd_scene;     /* opaque, immutable after create */

enum { UVD_SCENE_TRIMESH = 0, UVD_SCENE_EXTRUDED = 1 };

/* A simple polygon, CCW, n >= 3 vertices xy[2n] (host memory). */
typedef struct {
  const float* xy;
  int32_t n;
} uvd_polygon;

/* Scene description (pointers are HOST memory unless device_input != 0).
 *  TRIMESH  ("simplicial complex with N triangles"): vertices[n_vertices*3]
 *           fp32, tris[n_tris*3] int32 (0-based, right-hand winding gives the
 *           outward normal n(s), Q14).  Patch i = triangle.
 *  EXTRUDED (2.5D world): room bounds {x0,y0,x1,y1}, wall height
 *           h, obstacle polygons strictly inside the bounds, patch resolution
 *           res.  Walls = the bounds' 4 edges (CCW) then each polygon's edges in
 *           order; each wall of length len is split into ceil(len/res) equal
 *           patches, patch = vertical rectangle (2 triangles). */
typedef struct {
  int32_t kind;
  const float* vertices;
  int64_t n_vertices;
  const int32_t* tris;
  int64_t n_tris;
  float bounds[4];
  float wall_height;
  const uvd_polygon* obstacles;
  int32_t n_obstacles;
  float patch_res;
  int32_t device_input;   /* TRIMESH: 1 = vertices/tris are DEVICE pointers on `device` */
} uvd_scene_desc;

/* Build a scene on `device`: copy the input, compute the canonical patch
 * attributes (a1), build the BVH over all triangles (a2: Morton codes, radix
 * sort, top-down binned-SAH splits, bottom-up refit — PLOC clustering or the
 * Karras LBVH when the environment sets UVD_BVH=ploc / karras — then nodes in
 * depth-first preorder, leaves of <= 2 triangles).  Synchronises `stream`.
 * Canonical patch attributes (fp64 arithmetic, rounded once to fp32):
 *   3D : c = fl32((a+b+c)/3), n = fl32(cross(b-a,c-a)/|.|), area = |cross|/2;
 *   2.5D: q_s = fl32(e0 + ((e1-e0)*s)/n_seg) (q_nseg = e1), c = fl32((q_s+q_{s+1})/2, h/2),
 *         n = (-dy,dx)/len for boundary walls (into the room), (dy,-dx)/len for
 *         obstacle walls (out of the obstacle), area = len*h.
 * Patch (row) order: 2.5D = wall order; 3D = BVH leaf (depth-first) order, so
 * adjacent rows are adjacent leaves, with orig_id mapping back to the input
 * triangle index.
 * Errors: INVALID (non-finite vertex, index out of range, zero-area triangle,
 * polygon outside bounds / n<3, res<=0, h<=0), NOMEM, CUDA. */
UVD_API int uvd_scene_create(const uvd_scene_desc* desc, int device, void* stream,
                     const uvd_allocator* allocator, uvd_scene** out);

/* Host scalars: number of patches N (rows of A), number of triangles M,
 * bbox {xmin,ymin,zmin,xmax,ymax,zmax} of all vertices, total patch area. */
UVD_API int uvd_scene_query(const uvd_scene* scene, int64_t* n_patches, int64_t* n_tris, float bbox[6],
                    double* total_area);

/* Copy the canonical patch attributes into caller DEVICE buffers (any may be
 * NULL): centroid[N*3], normal[N*3] fp32, area[N] fp64, orig_id[N] int64. */
UVD_API int uvd_scene_patches(const uvd_scene* scene, float* centroid, float* normal, double* area,
                      int64_t* orig_id, void* stream);

/* Release the scene.  Synchronises the scene's device first (every stream
 * that used the scene must be done before its buffers go back to the
 * allocator), then frees them. */
UVD_API void uvd_scene_destroy(uvd_scene* scene);

/* Ship one scene build to other ranks (rank 0 builds, broadcasts).
 * uvd_scene_export writes the scene into a flat DEVICE buffer of *bytes bytes
 * on the scene's device (buf = NULL: *bytes receives the size; too small:
 * UVD_ERR_CAPACITY with the size): patch attributes, leaf-ordered triangles,
 * BVH nodes, front radii (and the 2.5D wall tables), not the octant node
 * copies.  Synchronises `stream`.
 * uvd_scene_import creates an independent scene on `device` from such a
 * buffer (DEVICE memory on that device, e.g. after an NCCL broadcast): the
 * same scene bit for bit (every call on it gives the results of the
 * exporter), octant copies rebuilt locally.  INVALID for a buffer that is not
 * a uvd_scene_export image.  Synchronises `stream`. */
UVD_API int uvd_scene_export(const uvd_scene* scene, void* buf, size_t* bytes, void* stream);
UVD_API int uvd_scene_import(const void* buf, size_t bytes, int device, void* stream,
                             const uvd_allocator* allocator, uvd_scene** out);

/* Introspection of the scene's BVH (a2), for structural tests and tree-quality
 * tools.  *n_nodes = max(M-1, 1), *root = the root reference (HOST).  nodes
 * (DEVICE, optional): n_nodes records of 64 B in depth-first preorder —
 * float4 a = child0 (lo.x, hi.x, lo.y, hi.y), float4 b = child1 (same),
 * float4 c = (child0 lo.z, hi.z, child1 lo.z, hi.z), uint32 refs[4] = (child0,
 * child1, 0, 0); a reference with bit 31 set is a leaf: triangles
 * [(ref & 0x7fffffff) >> 3, + (ref & 7) + 1) of `tri`; else a node index.
 * Boxes are padded outward (1e-5 m + 1e-6·|x| + 4·eps32·max|coord|).
 * tri (DEVICE, optional): M × 12 floats in leaf order, (v0, owner patch as
 * int bits), (v1, input triangle index as int bits), (v2, 0).  Asynchronous. */
UVD_API int uvd_scene_bvh(const uvd_scene* scene, void* nodes, float* tri, int64_t* n_nodes, uint32_t* root,
                  void* stream);

/* ---------------------------------------------------------------------- a3 */
enum { UVD_ROBOT_DISC2D = 0, UVD_ROBOT_TOWER = 1, UVD_ROBOT_FLOAT3D = 2, UVD_ROBOT_ARM = 3 };

/* Vantage sampling.  Cell-centred grid of spacing ρ:
 * x = lo + (a + 1/2)ρ, a = 0..floor((hi-lo)/ρ)-1 (Q9), candidates ordered x
 * fastest, then y, then z.
 *  DISC2D  (EXTRUDED scenes; planar disc robot): grid over the bounds at
 *          z = lamp_z; feasible iff inside the bounds, 2D distance to every wall
 *          >= clearance and outside every obstacle polygon.
 *  FLOAT3D (TRIMESH; Floatbot): grid over the mesh bbox; feasible iff the
 *          point is >= clearance from every triangle and in free space (Q20).
 *  TOWER   (TRIMESH; Towerbot): floor grid over the bbox xy; lamp_samples
 *          points z_l = lamp_z0 + (l+1/2)(lamp_z1-lamp_z0)/L (Q11); feasible
 *          iff every sample is >= clearance from every triangle and sample 0 is free.
 *  ARM     (TRIMESH; Armbot proxy, Q12): grid over bbox xy × [zmin,zmax]; feasible
 *          iff >= clearance, free, and within `reach` (3D) of a feasible base: floor
 *          grid point at z = base_z that is >= base_clearance and free.
 * Free space (Q20): the nearest triangle hit along p + t(0.0123, 0.0371, 1), t>0,
 * exists and is front-facing.
 * Output: lamp_xyz[cap * L * 3] fp32 DEVICE (L = lamp_samples for TOWER, else 1),
 * raw_index[cap] int64 DEVICE (optional), *out_k HOST = number of feasible
 * configurations.  If K > cap: returns UVD_ERR_CAPACITY with *out_k = K and
 * nothing written (call with cap = 0 to size).  K == 0: UVD_ERR_EMPTY.
 * Synchronises `stream`. */
typedef struct {
  int32_t robot;
  float spacing, clearance;
  float lamp_z, lamp_z0, lamp_z1;
  float reach, zmin, zmax;
  int32_t lamp_samples;
  float base_clearance, base_z;
} uvd_vantage_opts;

UVD_API int uvd_vantage_sample(const uvd_scene* scene, const uvd_vantage_opts* opts, float* lamp_xyz,
                       int64_t* raw_index, int64_t cap, int64_t* out_k, void* stream);

/* ------------------------------------------------------------------ a4–a6 */
/* Lamp model: total radiant flux P split over L = samples_per_config
 * isotropic point samples of power P/L each.
 * Irradiance model (`model`):
 *  UVD_MODEL_CENTROID (0, the hot path, BASELINE north_star): point source at
 *    the patch centroid, all-or-nothing centroid visibility (Eq. 7, Q4/Q5).
 *  UVD_MODEL_AREA (1, NEXT-2: Eq. 4 as written; Q23): mean
 *    irradiance over the patch, A = (P/L)/(4π|s_i|) Σ_l Σ_s vis(p_l → c_s) Ω_s,
 *    each patch triangle split `subdiv` times at edge midpoints (4^subdiv
 *    sub-triangles), Ω_s the exact solid angle of sub-triangle s (Van Oosterom
 *    & Strackee 1983), c_s = fl32 of its centroid the visibility target; the
 *    front-facing test is the patch's.  Exact for unoccluded patches. */
enum { UVD_MODEL_CENTROID = 0, UVD_MODEL_AREA = 1 };
typedef struct {
  double power_w;
  int32_t samples_per_config;
  int32_t model;    /* UVD_MODEL_CENTROID (default) or UVD_MODEL_AREA */
  int32_t subdiv;   /* UVD_MODEL_AREA: subdivision level m, 0..6 */
} uvd_lamp;

enum { UVD_DENSE_COLMAJOR = 0, UVD_CSC = 1 };

/* Matrix output (all DEVICE pointers).
 *  DENSE_COLMAJOR: values[n_cols * ld] fp32; local column c occupies
 *                  values[c*ld .. c*ld + N); rows N..ld-1 are written as 0.
 *                  ld >= N and ld % 32 == 0 (torch shape (n_cols, ld)).
 *  CSC:            colptr[n_cols+1] int64, rowidx[nnz_cap] int32, values[nnz_cap]
 *                  fp32, rows ascending within a column; entries are the nonzero
 *                  A[i,j] (a patch seen by at least one lamp sample).  Two-phase:
 *                  if nnz > nnz_cap the call returns UVD_ERR_CAPACITY after
 *                  writing colptr (colptr[n_cols] = nnz); call with nnz_cap = 0
 *                  to size.  The CSC path synchronises `stream` (to read nnz).
 *  vis_bits  (optional): [n_cols][L][ceil(N/32)] uint32, bit (i%32) of word i/32 =
 *            patch i front-facing and unoccluded from lamp sample l.
 *  col_sumsq (optional): [n_cols] fp64 Σ_i A[i,c]² (for ‖A‖_F).
 *  counters  (optional): 6 uint64 accumulated by the call (instrumented,
 *            slower path, for the roofline accounting): [0] front-facing rays
 *            that entered traversal, [1] per-ray child-box tests, [2] per-ray
 *            triangle tests, [3] node fetches, [4] entries the fp32 pass left
 *            undecided and re-traced with fp64 triangle tests, [5] reserved. */
typedef struct {
  int32_t format;
  int64_t ld;
  float* values;
  int64_t* colptr;
  int32_t* rowidx;
  int64_t nnz_cap;
  uint32_t* vis_bits;
  double* col_sumsq;
  unsigned long long* counters;
  /* optional (parity tools and tests): the entries the fp32 pass left
   * undecided and re-traced with exact fp64 triangle tests (DESIGN.md §6,
   * k_fixup), as (local column << 32) | row, in no particular order.  At most
   * fixup_cap are written to fixup_list; *fixup_count (DEVICE int64) receives
   * their total.  NULL fixup_list / fixup_count: not reported. */
  uint64_t* fixup_list;
  int64_t fixup_cap;
  int64_t* fixup_count;
  /* optional: allocator of the call's scratch in uvd_fluence, uvd_lp_solve and
   * uvd_static_columns (stream-ordered on the call's stream, returned before
   * the call does); NULL = cudaMallocAsync / cudaFreeAsync (the ABI default). */
  const uvd_allocator* allocator;
} uvd_matrix_out;

/* Assemble columns of A (a4 cull, a5 occlusion, a6 Eq. 7):
 *   A[i,j] = Σ_l vis_ijl · (P/L) · <p_jl - c_i, n_i> / (4π |p_jl - c_i|³)
 * (fp64, rounded once to fp32), vis_ijl = [<p_jl - c_i, n_i> > 0] and no scene
 * triangle other than patch i's own meets the open segment p_jl -> c_i at
 * t ∈ (1e-4/d, 1 - 1e-4/d) (inclusive triangle edges; Q5–Q8, Q15).
 * lamp_xyz: DEVICE [k_total * L * 3] (configuration j -> samples j*L .. j*L+L-1).
 * cols: HOST [n_cols] global configuration ids of this call's columns (local
 * column c <-> cols[c]); NULL means all, n_cols = k_total.  Asynchronous;
 * call uvd_sync_status to collect in-kernel DOMAIN errors and the lamp-range
 * check (every lamp coordinate finite and within the scene's largest
 * |coordinate| + 50 m).
 * UVD_MODEL_AREA (NEXT-2): dense output only (CSC returns INVALID); vis_bits
 * bit = some sub-triangle of the patch seen from lamp sample l. */
UVD_API int uvd_irradiance_matrix(const uvd_scene* scene, const float* lamp_xyz, int64_t k_total,
                          const int64_t* cols, int64_t n_cols, const uvd_lamp* lamp,
                          uvd_matrix_out* out, void* stream);

/* Synchronise `stream` and report the scene's in-kernel error flag, read and
 * cleared in one device atomic: UVD_OK, UVD_ERR_DOMAIN (a lamp–centroid
 * distance < 1e-9 m), UVD_ERR_INVALID (a lamp coordinate of uvd_irradiance_matrix
 * or uvd_cubemap_matrix non-finite or beyond the scene's largest |coordinate| + 50 m, the range the
 * BVH's fp32 box padding covers; the matrix is then not trusted), or
 * UVD_ERR_CUDA for a traversal-stack overflow (cannot
 * happen: scene creation refuses BVHs deeper than 62 levels with
 * UVD_ERR_INVALID).  The flag is per SCENE, not per stream: the call reports
 * errors raised by any assembly on this scene, on any stream, that completed
 * before it; an error raised later stays for the next call.  Callers that
 * assemble on several streams and need per-stream attribution synchronise
 * those streams first. */
UVD_API int uvd_sync_status(const uvd_scene* scene, void* stream);

/* ---------------------------------------------------------------------- a7 */
/* Fluence products on a local column shard (Eq. 5), fp64 accumulation:
 *  transpose = 0:  out[n] = A · x      (x = dwell times t[k], s; out = μ, J/m²)
 *  transpose = 1:  out[k] = Aᵀ · x     (x = y[n]; out = g)
 * A is a uvd_matrix_out previously filled by uvd_irradiance_matrix (dense or CSC),
 * n = number of patches, k = number of local columns.  x, out DEVICE fp64.
 * For A·t, columns with t_k == 0 are skipped.  Dense: the summation order is
 * fixed (deterministic).  CSC: A·t accumulates with fp64 atomics (order of the
 * per-row additions not fixed: results may differ by a few fp64 ulps), Aᵀ·y is
 * deterministic.  Asynchronous. */
UVD_API int uvd_fluence(const uvd_matrix_out* A, int64_t n, int64_t k, int transpose, const double* x,
                double* out, void* stream);

/* The step's fluence products in ONE pass over a dense A (a7; SURVEY §8(a):
 * μ = A·t, the ever-visible denominator A·𝟙, and g = Aᵀ·y of Eq. 5 / Eq. 9):
 *   ax[n]  = A · x   (x[k] DEVICE fp64, e.g. dwell times; NULL ax: not computed)
 *   a1[n]  = A · 𝟙   (row sums; NULL: not computed)
 *   aty[k] = Aᵀ · y  (y[n] DEVICE fp64; NULL aty: not computed)
 * At least one output; an output needs its input vector (ax needs x, aty needs
 * y).  Dense A only (CSC: INVALID; use uvd_fluence).  A is read once instead of
 * once per product.  Deterministic: ax and a1 sum over the columns in order
 * (ax equals uvd_fluence's A·x whenever that call does not split its columns:
 * zero x_k add exact zeros), aty sums fixed row blocks in order (it may differ
 * from uvd_fluence's Aᵀ·y in the last fp64 bits).  Scratch (aty: one fp64 per
 * 128 rows and column, ceil(n/128) × k doubles) through the allocator of A;
 * above 4 GB of it (env UVD_MULTI_PART_MAX, tests) the call makes one pass per
 * product instead (then equal to uvd_fluence's results).  Asynchronous. */
UVD_API int uvd_fluence_multi(const uvd_matrix_out* A, int64_t n, int64_t k, const double* x, const double* y,
                              double* ax, double* a1, double* aty, void* stream);

/* ---------------------------------------------------------------------- a8 */
/* Coverage (P:9 "fraction of the surface area"):
 *   out[0] = Σ_i |s_i| [μ_i >= μ_min]      (covered area, inclusive, Q16)
 *   out[1] = Σ_i |s_i|                     (total area)
 *   out[2] = Σ_i |s_i| [a_rowsum_i > 0]    (ever-visible area; = out[1] if NULL)
 * mu, a_rowsum: DEVICE fp64 [N] in canonical patch order.  out: HOST.
 * Deterministic reduction order.  Synchronises `stream`. */
UVD_API int uvd_coverage(const uvd_scene* scene, const double* mu, double mu_min, const double* a_rowsum,
                 double out[3], void* stream);

/* ------------------------------------------------------------------ NEXT-3 */
/* The paper's own irradiance pipeline, the "visibility cube" (P:244–250,
 * P:364), for a head-to-head comparison with uvd_irradiance_matrix: per lamp
 * sample 6 cube faces of face_res² pixels (512), face f of pixel (a,b)
 * looking along +X (1,u,v), −X (−1,u,v), +Y (u,1,v), −Y (u,−1,v), +Z (u,v,1),
 * −Z (u,v,−1) with u = −1 + (2a+1)/R, v = −1 + (2b+1)/R; each pixel carries
 * e = (P/L)·Ω_px/(4π), Ω_px its exact solid angle (the emission texture E,
 * P:250); the pixel's nearest surface (closest triangle hit, ties to the lower
 * input triangle index; the Z-buffer) receives e if front-facing;
 * A[i,j] = F_i/|s_i|.  Dense output only.  hits (optional, DEVICE
 * int32 [n_cols][L][6][R][R]): the winning input triangle per pixel, −1 none,
 * −2 back-facing (for tests).  Flux sums use fp64 atomics (order not fixed).
 * Asynchronous. */
UVD_API int uvd_cubemap_matrix(const uvd_scene* scene, const float* lamp_xyz, int64_t k_total,
                       const int64_t* cols, int64_t n_cols, const uvd_lamp* lamp, int32_t face_res,
                       uvd_matrix_out* out, int32_t* hits, void* stream);

/* ------------------------------------------------------------------ NEXT-4 */
/* Static single-point baseline (P:7, "places the disinfection light to
 * have maximum coverage over the obstacle space, allowing it to irradiate the
 * surfaces for as long as necessary"; P:53 the static Towerbot
 * for a time budget).  For each local column j of a dense A (n = scene N rows):
 *   out[3j]   = Σ_i |s_i| [A_ij > 0]            visible area (m²)
 *   out[3j+1] = min_{i: A_ij > 0} A_ij           (+inf if none): dwell to cover
 *               every visible patch = μ_min / out[3j+1] (s)
 *   out[3j+2] = Σ_i |s_i| [A_ij · t_budget ≥ μ_min]  area covered in t_budget
 * out: DEVICE fp64 [3k].
 * choice (HOST [2], optional): [0] = the static lamp's column — the largest
 * visible area, ties to the shorter dwell μ_min / out[3j+1], then the lower
 * index (reading Q24); [1] = the column covering most area within t_budget
 * (ties to the lower index); -1 when k = 0.  dwell (HOST, optional): μ_min /
 * min A of choice[0] (s; +inf if it sees nothing).  Deterministic.
 * Asynchronous unless choice or dwell is requested (then synchronises). */
UVD_API int uvd_static_columns(const uvd_scene* scene, const uvd_matrix_out* A, int64_t k, double t_budget,
                       double mu_min, double* out, int64_t choice[2], double* dwell, void* stream);

/* ------------------------------------------------------------------ NEXT-1 */
/* Relaxed dwell-time LP, Eq. 9 (§IV-D first stage):
 *   minimise Σ_k t_k + Σ_i p_i σ_i
 *   s.t.     (A·t)_i + σ_i ≥ μ_min  (every patch i),   Σ_k t_k ≤ T_max,   t, σ ≥ 0
 * and its dual  maximise μ_min Σ_i y_i − T_max y_b  s.t.  (Aᵀy)_k − y_b ≤ 1,
 * y_i ≤ p_i, y ≥ 0.  Solved by reflected restarted Halpern PDHG (Lu & Yang
 * 2024) with Chambolle–Pock diagonal preconditioning (α = 1): the coverage
 * rows are dualised, the budget is kept as a set (exact weighted projection
 * onto {t ≥ 0, Σt ≤ T_max}); every iteration is one A·t and one Aᵀ·y
 * (uvd_fluence kernels, zero-t columns skipped) plus fused fp64 vector
 * kernels.  The paper used Gurobi's interior-point method; any optimal
 * (t, σ) is acceptable (the optimum need not be unique, Q17): the solver's
 * contract is the KKT tolerance below.
 *
 * A: this process's column shard (dense or CSC, as filled by
 *    uvd_irradiance_matrix), n patches, k local columns.  A ≥ 0 is assumed
 *    (irradiance), so row/column absolute sums are plain sums.
 * t: DEVICE [k] fp64, in: initial dwell times (zeros are fine), out: solution.
 * sigma: DEVICE [n] fp64 out (slacks σ).  y: DEVICE [n+1] fp64 out (duals of
 *    the n coverage rows, then of the budget row).
 * Multi-GPU (columns sharded): set `allreduce` to a function that
 *    reduces `count` fp64 values at the DEVICE pointer `buf` in place across
 *    ranks (op 0 = sum, 1 = max), enqueued on or synchronised with `stream`;
 *    the library calls it once per iteration for the partial A·t (n values), a
 *    few times per iteration for the budget projection's sums, and at checks.
 *    No CUDA graph is used in that mode.  NULL: single process.
 * Termination (relative KKT, as in PDLP): ‖primal residual‖₂ ≤ eps(1+‖q‖₂),
 *    ‖dual residual‖₂ ≤ eps(1+‖c‖₂), |primal − dual objective| ≤
 *    eps(1+|primal|+|dual|), q = (μ_min 𝟙, −T_max), c = (𝟙, p); checked every
 *    `check_every` iterations on the operator output T(z).
 * Synchronises `stream` at every check.  Deterministic for a given launch
 * sequence (fixed reduction orders; CSC A·t uses fp64 atomics). */
typedef struct {
  double mu_min;          /* μ_min, J/m² (280) */
  double t_max;           /* T_max, s (1800) */
  const double* penalty;  /* DEVICE [n] p_i, or NULL: penalty_scalar for every patch */
  double penalty_scalar;  /* paper: p_i > ‖A‖_F */
  double eps;             /* relative KKT tolerance; 0 → 1e-6 */
  int64_t max_iter;       /* 0 → 200000 */
  int32_t check_every;    /* 0 → 64 */
  int32_t use_graph;      /* capture check_every iterations in one CUDA graph (single process, non-NULL stream) */
  double primal_weight;   /* initial ω; 0 → ‖T^½c‖/‖Σ^½q‖ (PDLP's rule in the preconditioned space) */
  int (*allreduce)(double* buf, int64_t count, int op, void* stream, void* ctx);
  void* allreduce_ctx;
} uvd_lp_opts;

typedef struct {
  int32_t status;         /* 0 converged within eps, 1 iteration limit */
  int32_t restarts;
  int64_t iterations;
  double primal_obj;      /* Σ t + Σ p σ */
  double dual_obj;        /* μ_min Σ y − T_max y_b */
  double rel_primal_res, rel_dual_res, rel_gap;
  double sum_t;           /* Σ_k t_k over all ranks */
  double primal_weight;   /* final ω */
  int32_t averaged;       /* reserved (0) */
} uvd_lp_result;

UVD_API int uvd_lp_solve(const uvd_matrix_out* A, int64_t n, int64_t k, const uvd_lp_opts* opts, double* t,
                 double* sigma, double* y, uvd_lp_result* result, void* stream);

/* Thread-local message of the last failing call on this thread ("" if none). */
UVD_API const char* uvd_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
UVD_API int uvd_version(void);

/* Number of CUDA kernels this library has launched in this process (all
 * devices, all threads) — for launch accounting in benchmarks. */
UVD_API unsigned long long uvd_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* UVD_H_ */
