"""Thin Python binding of libuvd (include/uvd.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C-ABI; this
module only converts between torch tensors / numpy arrays and the ABI's plain
pointers, and binds the ABI's allocator callback to PyTorch's caching
allocator.  There is no CPU fallback: if libuvd.so is missing or CUDA is not
available, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UVD_LIB", os.path.join(_HERE, "libuvd.so"))  # UVD_LIB: dev builds

UVD_OK, UVD_ERR_INVALID, UVD_ERR_DOMAIN, UVD_ERR_EMPTY, UVD_ERR_CAPACITY, UVD_ERR_NOMEM, UVD_ERR_CUDA = (
    0, -1, -2, -3, -4, -5, -6)
TRIMESH, EXTRUDED = 0, 1
DISC2D, TOWER, FLOAT3D, ARM = 0, 1, 2, 3
DENSE_COLMAJOR, CSC = 0, 1


class UvdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"uvd error {code}: {msg}")
        self.code = code


# ----------------------------------------------------------------- structs --
_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p)


class _Allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


class _Polygon(C.Structure):
    _fields_ = [("xy", C.POINTER(C.c_float)), ("n", C.c_int32)]


class _SceneDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("vertices", C.POINTER(C.c_float)), ("n_vertices", C.c_int64),
                ("tris", C.POINTER(C.c_int32)), ("n_tris", C.c_int64), ("bounds", C.c_float * 4),
                ("wall_height", C.c_float), ("obstacles", C.POINTER(_Polygon)),
                ("n_obstacles", C.c_int32), ("patch_res", C.c_float), ("device_input", C.c_int32)]


class _VantageOpts(C.Structure):
    _fields_ = [("robot", C.c_int32), ("spacing", C.c_float), ("clearance", C.c_float),
                ("lamp_z", C.c_float), ("lamp_z0", C.c_float), ("lamp_z1", C.c_float),
                ("reach", C.c_float), ("zmin", C.c_float), ("zmax", C.c_float),
                ("lamp_samples", C.c_int32), ("base_clearance", C.c_float), ("base_z", C.c_float)]


class _Lamp(C.Structure):
    _fields_ = [("power_w", C.c_double), ("samples_per_config", C.c_int32), ("model", C.c_int32),
                ("subdiv", C.c_int32)]


class _MatrixOut(C.Structure):
    _fields_ = [("format", C.c_int32), ("ld", C.c_int64), ("values", C.c_void_p),
                ("colptr", C.c_void_p), ("rowidx", C.c_void_p), ("nnz_cap", C.c_int64),
                ("vis_bits", C.c_void_p), ("col_sumsq", C.c_void_p), ("counters", C.c_void_p),
                ("fixup_list", C.c_void_p), ("fixup_cap", C.c_int64), ("fixup_count", C.c_void_p),
                ("allocator", C.POINTER(_Allocator))]


_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p)


class _LpOpts(C.Structure):
    _fields_ = [("mu_min", C.c_double), ("t_max", C.c_double), ("penalty", C.c_void_p),
                ("penalty_scalar", C.c_double), ("eps", C.c_double), ("max_iter", C.c_int64),
                ("check_every", C.c_int32), ("use_graph", C.c_int32), ("primal_weight", C.c_double),
                ("allreduce", _ALLREDUCE_FN), ("allreduce_ctx", C.c_void_p)]


class _LpResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("restarts", C.c_int32), ("iterations", C.c_int64),
                ("primal_obj", C.c_double), ("dual_obj", C.c_double), ("rel_primal_res", C.c_double),
                ("rel_dual_res", C.c_double), ("rel_gap", C.c_double), ("sum_t", C.c_double),
                ("primal_weight", C.c_double), ("averaged", C.c_int32)]


_lib = None


def lib():
    """Load libuvd.so (built in-tree by __graft_entry__.build()); fail loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.uvd_scene_create.argtypes = [C.POINTER(_SceneDesc), C.c_int, C.c_void_p,
                                       C.POINTER(_Allocator), C.POINTER(C.c_void_p)]
        L.uvd_scene_query.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_float), C.POINTER(C.c_double)]
        L.uvd_scene_patches.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        L.uvd_scene_bvh.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_uint32), C.c_void_p]
        L.uvd_scene_export.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t), C.c_void_p]
        L.uvd_scene_import.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.POINTER(_Allocator),
                                       C.POINTER(C.c_void_p)]
        L.uvd_scene_destroy.argtypes = [C.c_void_p]
        L.uvd_scene_destroy.restype = None
        L.uvd_vantage_sample.argtypes = [C.c_void_p, C.POINTER(_VantageOpts), C.c_void_p, C.c_void_p,
                                         C.c_int64, C.POINTER(C.c_int64), C.c_void_p]
        L.uvd_irradiance_matrix.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                            C.POINTER(_Lamp), C.POINTER(_MatrixOut), C.c_void_p]
        L.uvd_sync_status.argtypes = [C.c_void_p, C.c_void_p]
        L.uvd_fluence.argtypes = [C.POINTER(_MatrixOut), C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
        L.uvd_fluence_multi.argtypes = [C.POINTER(_MatrixOut), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.uvd_coverage.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                   C.POINTER(C.c_double), C.c_void_p]
        L.uvd_cubemap_matrix.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                         C.POINTER(_Lamp), C.c_int32, C.POINTER(_MatrixOut), C.c_void_p,
                                         C.c_void_p]
        L.uvd_static_columns.argtypes = [C.c_void_p, C.POINTER(_MatrixOut), C.c_int64, C.c_double, C.c_double,
                                         C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_void_p]
        L.uvd_lp_solve.argtypes = [C.POINTER(_MatrixOut), C.c_int64, C.c_int64, C.POINTER(_LpOpts),
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_LpResult), C.c_void_p]
        L.uvd_last_error.restype = C.c_char_p
        L.uvd_version.restype = C.c_int
        L.uvd_launch_count.restype = C.c_ulonglong
        _lib = L
    return _lib


EXPORTS = ("uvd_scene_create", "uvd_scene_query", "uvd_scene_patches", "uvd_scene_bvh", "uvd_scene_destroy",
           "uvd_scene_export", "uvd_scene_import",
           "uvd_vantage_sample", "uvd_irradiance_matrix", "uvd_sync_status", "uvd_fluence", "uvd_fluence_multi",
           "uvd_coverage", "uvd_cubemap_matrix", "uvd_static_columns", "uvd_lp_solve", "uvd_last_error", "uvd_version", "uvd_launch_count")


def _check(rc):
    if rc != UVD_OK:
        raise UvdError(rc, lib().uvd_last_error().decode(errors="replace"))
    return rc


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


# ------------------------------------------------- torch caching allocator --
@_ALLOC_FN
def _torch_alloc(nbytes, device, stream, ctx):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream)
    except Exception:  # noqa: BLE001 — the C side reports NOMEM
        return None


@_FREE_FN
def _torch_free(ptr, device, stream, ctx):
    torch.cuda.caching_allocator_delete(ptr)


_TORCH_ALLOCATOR = _Allocator(_torch_alloc, _torch_free, None)


def _new_desc(fmt) -> _MatrixOut:
    """A uvd_matrix_out whose call scratch comes from torch's caching allocator."""
    m = _MatrixOut()
    m.format = fmt
    m.allocator = C.pointer(_TORCH_ALLOCATOR)
    return m


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2103_14137_b200 needs a CUDA device (no CPU fallback)")


# ------------------------------------------------------------------- scene --
class Scene:
    """uvd_scene_create from a synth-style dict: TRIMESH {vertices, tris} or
    EXTRUDED {bounds, wall_height, obstacles, patch_res}.  TRIMESH vertices /
    tris may be numpy arrays (host; the host->device copy is part of the call)
    or CUDA tensors (float32 (nv,3) / int32 (nt,3), already resident)."""

    def __init__(self, desc: dict | None, device: int | None = None, stream=None, torch_allocator: bool = True,
                 _image: torch.Tensor | None = None):
        _require_cuda()
        self.device = torch.cuda.current_device() if device is None else device
        if _image is not None:  # uvd_scene_import of a uvd_scene_export image
            h = C.c_void_p()
            self._alloc = _TORCH_ALLOCATOR if torch_allocator else None
            with torch.cuda.device(self.device):
                _check(lib().uvd_scene_import(_ptr(_image), _image.numel(), self.device, _stream(stream),
                                              C.byref(self._alloc) if self._alloc else None, C.byref(h)))
            self._h = h
            self._query()
            return
        d = _SceneDesc()
        keep = []
        if "vertices" in desc:
            V, F = desc["vertices"], desc["tris"]
            d.kind = TRIMESH
            if isinstance(V, torch.Tensor) and V.is_cuda:
                assert V.dtype == torch.float32 and F.dtype == torch.int32 and F.is_cuda
                V, F = V.contiguous(), F.contiguous()
                d.device_input = 1
                d.vertices = C.cast(C.c_void_p(V.data_ptr()), C.POINTER(C.c_float))
                d.tris = C.cast(C.c_void_p(F.data_ptr()), C.POINTER(C.c_int32))
            else:
                V = np.ascontiguousarray(V, np.float32)
                F = np.ascontiguousarray(F, np.int32)
                d.vertices = V.ctypes.data_as(C.POINTER(C.c_float))
                d.tris = F.ctypes.data_as(C.POINTER(C.c_int32))
            keep += [V, F]
            d.n_vertices = V.shape[0]
            d.n_tris = F.shape[0]
        else:
            d.kind = EXTRUDED
            for k in range(4):
                d.bounds[k] = float(desc["bounds"][k])
            d.wall_height = float(desc["wall_height"])
            d.patch_res = float(desc["patch_res"])
            obs = [np.ascontiguousarray(p, np.float32).reshape(-1, 2) for p in desc["obstacles"]]
            keep += obs
            polys = (_Polygon * max(1, len(obs)))()
            for k, p in enumerate(obs):
                polys[k].xy = p.ctypes.data_as(C.POINTER(C.c_float))
                polys[k].n = len(p)
            keep.append(polys)
            d.obstacles = polys
            d.n_obstacles = len(obs)
        h = C.c_void_p()
        self._alloc = _TORCH_ALLOCATOR if torch_allocator else None
        with torch.cuda.device(self.device):
            _check(lib().uvd_scene_create(C.byref(d), self.device, _stream(stream),
                                          C.byref(self._alloc) if self._alloc else None, C.byref(h)))
        self._h = h
        self._query()

    def _query(self):
        n, m = C.c_int64(), C.c_int64()
        bb = (C.c_float * 6)()
        area = C.c_double()
        _check(lib().uvd_scene_query(self._h, C.byref(n), C.byref(m), bb, C.byref(area)))
        self.N, self.M = n.value, m.value
        self.bbox = np.array(bb[:], np.float32)
        self.total_area = area.value

    def export(self, stream=None) -> torch.Tensor:
        """uvd_scene_export: the scene as a flat uint8 CUDA tensor (for a broadcast)."""
        nb = C.c_size_t()
        _check(lib().uvd_scene_export(self.handle, None, C.byref(nb), _stream(stream)))
        buf = torch.empty(nb.value, dtype=torch.uint8, device=f"cuda:{self.device}")
        _check(lib().uvd_scene_export(self.handle, _ptr(buf), C.byref(nb), _stream(stream)))
        return buf

    @classmethod
    def from_image(cls, image: torch.Tensor, device: int | None = None, stream=None,
                   torch_allocator: bool = True) -> "Scene":
        """uvd_scene_import: a scene from a Scene.export() image (uint8 CUDA tensor)."""
        assert image.is_cuda and image.dtype == torch.uint8 and image.is_contiguous()
        return cls(None, device=image.device.index if device is None else device, stream=stream,
                   torch_allocator=torch_allocator, _image=image)

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("scene is closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None:
            lib().uvd_scene_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def ld(self):
        return (self.N + 31) // 32 * 32

    def patches(self, stream=None):
        dev = torch.device("cuda", self.device)
        cen = torch.empty((self.N, 3), dtype=torch.float32, device=dev)
        nrm = torch.empty((self.N, 3), dtype=torch.float32, device=dev)
        area = torch.empty(self.N, dtype=torch.float64, device=dev)
        orig = torch.empty(self.N, dtype=torch.int64, device=dev)
        _check(lib().uvd_scene_patches(self.handle, _ptr(cen), _ptr(nrm), _ptr(area), _ptr(orig),
                                       _stream(stream)))
        return dict(centroid=cen, normal=nrm, area=area, orig_id=orig)

    def bvh(self, stream=None) -> dict:
        """uvd_scene_bvh: the BVH nodes (n_nodes, 16) as raw 32-bit words (float
        boxes viewed as int32; refs in columns 12–13) and the leaf-ordered
        triangles (M, 12) float32, plus the root reference."""
        n = C.c_int64()
        root = C.c_uint32()
        _check(lib().uvd_scene_bvh(self.handle, None, None, C.byref(n), C.byref(root), _stream(stream)))
        nodes = torch.empty((n.value, 16), dtype=torch.int32, device=f"cuda:{self.device}")
        tri = torch.empty((self.M, 12), dtype=torch.float32, device=f"cuda:{self.device}")
        _check(lib().uvd_scene_bvh(self.handle, _ptr(nodes), _ptr(tri), C.byref(n), C.byref(root), _stream(stream)))
        return {"nodes": nodes, "tri": tri, "root": int(root.value)}

    def vantage(self, opts: dict, stream=None):
        """uvd_vantage_sample: returns (lamps (K, L, 3) fp32, raw_index (K,) int64)."""
        o = _VantageOpts()
        for name, _ in _VantageOpts._fields_:
            if name in opts:
                setattr(o, name, opts[name])
        L = int(opts.get("lamp_samples", 1)) if opts["robot"] == TOWER else 1
        k = C.c_int64()
        rc = lib().uvd_vantage_sample(self.handle, C.byref(o), None, None, 0, C.byref(k), _stream(stream))
        if rc not in (UVD_OK, UVD_ERR_CAPACITY):
            _check(rc)
        K = k.value
        dev = torch.device("cuda", self.device)
        lamps = torch.empty((K, L, 3), dtype=torch.float32, device=dev)
        raw = torch.empty(K, dtype=torch.int64, device=dev)
        _check(lib().uvd_vantage_sample(self.handle, C.byref(o), _ptr(lamps), _ptr(raw), K, C.byref(k),
                                        _stream(stream)))
        return lamps, raw

    def irradiance(self, lamps: torch.Tensor, cols=None, power_w: float = 80.0, vis_bits: bool = False,
                   col_sumsq: bool = False, counters: bool = False, out: torch.Tensor | None = None,
                   stream=None, area_subdiv: int | None = None, fixups: int = 0) -> dict:
        """uvd_irradiance_matrix (dense column-major).  lamps: (K_total, L, 3)
        fp32 on the device; cols: None or a host sequence of global column ids.
        Returns dict(A=(n_cols, ld) fp32, [vis_bits (n_cols, L, words) int32],
        [col_sumsq (n_cols,) fp64], [counters (6,) int64: rays, box tests,
        triangle tests, node fetches, entries re-traced in fp64, 0 — instrumented kernel],
        [fixups (m,) int64 (local column << 32 | row) of the entries the fp32 pass
        left undecided (re-traced exactly), up to `fixups` of them, and
        fixup_count (the total)])."""
        assert lamps.is_cuda and lamps.dtype == torch.float32 and lamps.is_contiguous()
        K, L = lamps.shape[0], lamps.shape[1]
        ccols = None
        if cols is not None:
            ccols = np.ascontiguousarray(cols, np.int64)
            n_cols = len(ccols)
        else:
            n_cols = K
        ld = self.ld()
        dev = lamps.device
        A = out if out is not None else torch.empty((n_cols, ld), dtype=torch.float32, device=dev)
        assert A.shape == (n_cols, ld) and A.dtype == torch.float32 and A.is_contiguous()
        res = dict(A=A)
        m = _new_desc(DENSE_COLMAJOR)
        m.ld = ld
        m.values = A.data_ptr()
        if vis_bits:
            vb = torch.empty((n_cols, L, (self.N + 31) // 32), dtype=torch.int32, device=dev)
            m.vis_bits = vb.data_ptr()
            res["vis_bits"] = vb
        if col_sumsq:
            cs = torch.empty(n_cols, dtype=torch.float64, device=dev)
            m.col_sumsq = cs.data_ptr()
            res["col_sumsq"] = cs
        if counters:
            ct = torch.zeros(6, dtype=torch.int64, device=dev)
            m.counters = ct.data_ptr()
            res["counters"] = ct
        if fixups:
            fl = torch.empty(int(fixups), dtype=torch.int64, device=dev)
            fc = torch.zeros(1, dtype=torch.int64, device=dev)
            m.fixup_list, m.fixup_cap, m.fixup_count = fl.data_ptr(), int(fixups), fc.data_ptr()
            res["_fixups"] = (fl, fc)
        lamp = _Lamp(float(power_w), int(L), 0 if area_subdiv is None else 1,
                     0 if area_subdiv is None else int(area_subdiv))
        _check(lib().uvd_irradiance_matrix(
            self.handle, _ptr(lamps), K,
            ccols.ctypes.data_as(C.c_void_p) if ccols is not None else None, n_cols,
            C.byref(lamp), C.byref(m), _stream(stream)))
        res["_desc"] = m
        if fixups:
            fl, fc = res.pop("_fixups")
            n_fix = int(fc.item())
            res["fixups"] = fl[:min(n_fix, int(fixups))]
            res["fixup_count"] = n_fix
        return res

    def irradiance_csc(self, lamps: torch.Tensor, cols=None, power_w: float = 80.0,
                       nnz_cap: int | None = None, vis_bits: bool = False, col_sumsq: bool = False,
                       stream=None) -> dict:
        """uvd_irradiance_matrix with CSC output (nonzero entries only).  With
        nnz_cap=None the call is made twice (size, then fill).  Returns
        dict(colptr (n_cols+1,) int64, rowidx (nnz,) int32, values (nnz,) fp32, nnz, ...)."""
        assert lamps.is_cuda and lamps.dtype == torch.float32 and lamps.is_contiguous()
        K, L = lamps.shape[0], lamps.shape[1]
        ccols = None if cols is None else np.ascontiguousarray(cols, np.int64)
        n_cols = K if ccols is None else len(ccols)
        dev = lamps.device
        colptr = torch.empty(n_cols + 1, dtype=torch.int64, device=dev)
        res = dict(colptr=colptr)
        m = _new_desc(CSC)
        m.colptr = colptr.data_ptr()
        if vis_bits:
            vb = torch.empty((n_cols, L, (self.N + 31) // 32), dtype=torch.int32, device=dev)
            m.vis_bits = vb.data_ptr()
            res["vis_bits"] = vb
        lamp = _Lamp(float(power_w), int(L))
        cptr = ccols.ctypes.data_as(C.c_void_p) if ccols is not None else None
        cap = 0 if nnz_cap is None else int(nnz_cap)
        for _attempt in range(2 if nnz_cap is None else 1):
            rowidx = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            values = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
            m.nnz_cap = cap
            m.rowidx = rowidx.data_ptr() if cap else 0
            m.values = values.data_ptr() if cap else 0
            cs = None
            if col_sumsq and cap:
                cs = torch.empty(n_cols, dtype=torch.float64, device=dev)
                m.col_sumsq = cs.data_ptr()
            rc = lib().uvd_irradiance_matrix(self.handle, _ptr(lamps), K, cptr, n_cols, C.byref(lamp),
                                             C.byref(m), _stream(stream))
            if rc == UVD_ERR_CAPACITY and nnz_cap is None:
                cap = int(colptr[-1].item())
                continue
            _check(rc)
            nnz = int(colptr[-1].item())
            res.update(rowidx=rowidx[:nnz], values=values[:nnz], nnz=nnz, _desc=m)
            if cs is not None:
                res["col_sumsq"] = cs
            return res
        raise UvdError(UVD_ERR_CAPACITY, "CSC capacity negotiation failed")

    def sync_status(self, stream=None):
        _check(lib().uvd_sync_status(self.handle, _stream(stream)))

    def cubemap(self, lamps: torch.Tensor, face_res: int = 512, cols=None, power_w: float = 80.0,
                hits: bool = False, out: torch.Tensor | None = None, stream=None) -> dict:
        """NEXT-3: the paper's visibility-cube irradiance (uvd_cubemap_matrix),
        dense (n_cols, ld) fp32; hits=True also returns the per-pixel winning
        input triangle (n_cols, L, 6, R, R) int32 (-1 none, -2 back-facing)."""
        assert lamps.is_cuda and lamps.dtype == torch.float32 and lamps.is_contiguous()
        K, L = lamps.shape[0], lamps.shape[1]
        ccols = None if cols is None else np.ascontiguousarray(cols, np.int64)
        n_cols = K if ccols is None else len(ccols)
        ld = self.ld()
        A = out if out is not None else torch.empty((n_cols, ld), dtype=torch.float32, device=lamps.device)
        m = _dense_desc(A)
        h = torch.full((n_cols, L, 6, face_res, face_res), -3, dtype=torch.int32, device=lamps.device) if hits else None
        lamp = _Lamp(float(power_w), int(L), 0, 0)
        _check(lib().uvd_cubemap_matrix(self.handle, _ptr(lamps), K,
                                        ccols.ctypes.data_as(C.c_void_p) if ccols is not None else None, n_cols,
                                        C.byref(lamp), int(face_res), C.byref(m), _ptr(h), _stream(stream)))
        res = {"A": A}
        if hits:
            res["hits"] = h
        return res

    def static_baseline(self, A: torch.Tensor, t_budget: float = 1800.0, mu_min: float = 280.0,
                        stream=None) -> dict:
        """NEXT-4 static single-point baseline (uvd_static_columns) on a dense
        (k, ld) A: per-column visible area, min positive entry and area covered
        in t_budget; the chosen column maximises the visible area, ties broken
        by the smaller dwell μ_min / min A, then the lower index (reading Q24)."""
        k = A.shape[0]
        out = torch.empty((k, 3), dtype=torch.float64, device=A.device)
        m = _dense_desc(A)
        choice = (C.c_int64 * 2)()
        dwell = C.c_double()
        _check(lib().uvd_static_columns(self.handle, C.byref(m), k, float(t_budget), float(mu_min),
                                        _ptr(out), choice, C.byref(dwell), _stream(stream)))
        o = out.cpu().numpy()
        return {"visible_area": o[:, 0], "min_irradiance": o[:, 1], "covered_at_budget": o[:, 2],
                "column": int(choice[0]), "dwell_s": float(dwell.value), "best_budget_column": int(choice[1])}

    def coverage(self, mu: torch.Tensor, mu_min: float = 280.0, rowsum: torch.Tensor | None = None,
                 stream=None) -> np.ndarray:
        out = (C.c_double * 3)()
        _check(lib().uvd_coverage(self.handle, _ptr(mu), float(mu_min), _ptr(rowsum), out, _stream(stream)))
        return np.array(out[:], np.float64)


def _dense_desc(A: torch.Tensor) -> _MatrixOut:
    m = _new_desc(DENSE_COLMAJOR)
    m.ld = A.shape[1]
    m.values = A.data_ptr()
    return m


def fluence(A: torch.Tensor, n: int, x: torch.Tensor, transpose: bool = False,
            out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """uvd_fluence on a dense (n_cols, ld) A: μ = A·x (x: (n_cols,) fp64) or
    g = Aᵀ·x (x: (n,) fp64)."""
    k = A.shape[0]
    assert x.dtype == torch.float64 and x.is_cuda and x.is_contiguous()
    if out is None:
        out = torch.empty(k if transpose else n, dtype=torch.float64, device=A.device)
    m = _dense_desc(A)
    _check(lib().uvd_fluence(C.byref(m), n, k, int(bool(transpose)), _ptr(x), _ptr(out), _stream(stream)))
    return out


def fluence_multi(A: torch.Tensor, n: int, x: torch.Tensor | None = None, y: torch.Tensor | None = None,
                  rowsum: bool = False, stream=None):
    """uvd_fluence_multi on a dense (n_cols, ld) A, one pass over A: returns
    (A·x or None, A·𝟙 or None, Aᵀ·y or None) for x (n_cols,) / y (n,) fp64."""
    k = A.shape[0]
    for v in (x, y):
        assert v is None or (v.dtype == torch.float64 and v.is_cuda and v.is_contiguous())
    ax = torch.empty(n, dtype=torch.float64, device=A.device) if x is not None else None
    a1 = torch.empty(n, dtype=torch.float64, device=A.device) if rowsum else None
    aty = torch.empty(k, dtype=torch.float64, device=A.device) if y is not None else None
    m = _dense_desc(A)
    _check(lib().uvd_fluence_multi(C.byref(m), n, k, _ptr(x), _ptr(y), _ptr(ax), _ptr(a1), _ptr(aty),
                                   _stream(stream)))
    return ax, a1, aty


def fluence_csc(csc: dict, n: int, x: torch.Tensor, transpose: bool = False,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """uvd_fluence on a CSC matrix from Scene.irradiance_csc."""
    k = csc["colptr"].shape[0] - 1
    assert x.dtype == torch.float64 and x.is_cuda and x.is_contiguous()
    if out is None:
        out = torch.empty(k if transpose else n, dtype=torch.float64, device=x.device)
    m = _new_desc(CSC)
    m.colptr = csc["colptr"].data_ptr()
    m.rowidx = csc["rowidx"].data_ptr() if csc["nnz"] else csc["colptr"].data_ptr()
    m.values = csc["values"].data_ptr() if csc["nnz"] else csc["colptr"].data_ptr()
    m.nnz_cap = csc["nnz"]
    _check(lib().uvd_fluence(C.byref(m), n, k, int(bool(transpose)), _ptr(x), _ptr(out), _stream(stream)))
    return out


def version() -> int:
    return int(lib().uvd_version())


def launch_count() -> int:
    """Kernels libuvd has launched in this process (uvd_launch_count)."""
    return int(lib().uvd_launch_count())


class _DevView:
    """Zero-copy view of a device fp64 buffer (for the allreduce callback)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def lp_solve(A, n: int, mu_min: float = 280.0, t_max: float = 1800.0, penalty=None, t0=None,
             eps: float = 1e-6, max_iter: int = 200000, check_every: int = 64, use_graph: bool = True,
             primal_weight: float = 0.0, distributed: bool = False, allreduce=None, stream=None) -> dict:
    """uvd_lp_solve: the relaxed dwell-time LP of Eq. 9 on this
    process's column shard of A (dense (k, ld) tensor, or a CSC dict from
    Scene.irradiance_csc).  penalty: float (every patch) or (n,) fp64 CUDA
    tensor; None = 10·‖A‖_F is the caller's job (pass it).  distributed: sum the
    per-iteration partials across torch.distributed ranks (columns sharded);
    allreduce: or any callable(tensor, op) reducing a CUDA fp64 tensor in place
    across the column shards (op "sum" or "max")."""
    if isinstance(A, dict):
        m = _new_desc(CSC)
        m.colptr = A["colptr"].data_ptr()
        m.rowidx = A["rowidx"].data_ptr() if A["nnz"] else A["colptr"].data_ptr()
        m.values = A["values"].data_ptr() if A["nnz"] else A["colptr"].data_ptr()
        m.nnz_cap = A["nnz"]
        k = A["colptr"].shape[0] - 1
        dev = A["colptr"].device
    else:
        m = _dense_desc(A)
        k = A.shape[0]
        dev = A.device
    if penalty is None:
        raise ValueError("lp_solve: pass the penalty (the paper: p_i > ||A||_F, P:274)")
    o = _LpOpts()
    o.mu_min, o.t_max, o.eps = float(mu_min), float(t_max), float(eps)
    if isinstance(penalty, torch.Tensor):
        assert penalty.dtype == torch.float64 and penalty.is_cuda and penalty.numel() == n
        o.penalty = penalty.data_ptr()
    else:
        o.penalty_scalar = float(penalty)
    o.max_iter, o.check_every, o.use_graph = int(max_iter), int(check_every), int(bool(use_graph))
    o.primal_weight = float(primal_weight)
    cb = None
    if distributed and allreduce is None:
        import torch.distributed as dist

        def allreduce(x, op):
            dist.all_reduce(x, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    if allreduce is not None:
        def _allreduce(buf, count, op, strm, ctx):
            try:
                s = torch.cuda.ExternalStream(strm) if strm else torch.cuda.current_stream()
                with torch.cuda.stream(s):
                    allreduce(torch.as_tensor(_DevView(buf, count), device=dev), "max" if op == 1 else "sum")
                return 0
            except Exception:  # noqa: BLE001 — reported to the C side as a failure code
                return 1
        cb = _ALLREDUCE_FN(_allreduce)
        o.allreduce = cb
    t = torch.zeros(k, dtype=torch.float64, device=dev) if t0 is None else t0.clone()
    sigma = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n + 1, dtype=torch.float64, device=dev)
    r = _LpResult()
    _check(lib().uvd_lp_solve(C.byref(m), int(n), int(k), C.byref(o), _ptr(t) if k else C.c_void_p(0),
                              _ptr(sigma), _ptr(y), C.byref(r), _stream(stream)))
    del cb
    return {"t": t, "sigma": sigma, "y": y[:n], "y_budget": y[n:], "status": int(r.status),
            "iterations": int(r.iterations), "restarts": int(r.restarts), "primal_obj": r.primal_obj,
            "dual_obj": r.dual_obj, "rel_primal_res": r.rel_primal_res, "rel_dual_res": r.rel_dual_res,
            "rel_gap": r.rel_gap, "sum_t": r.sum_t, "primal_weight": r.primal_weight,
            "averaged": bool(r.averaged)}
