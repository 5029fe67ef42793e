"""Sampled parity statistics of a GPU-computed irradiance matrix against the
fp64 oracle (TEST INFRASTRUCTURE ONLY: used by tests/, tools/parity_sample.py
and bench.py's cpu_baseline leg).

The caller passes plain numpy arrays read back from the GPU (values, visibility
bits) and the GPU's column -> grid-candidate map; every oracle INPUT (patches,
lamp samples) is recomputed here from the scene description — nothing the CUDA
path produced is fed to the oracle.  Bars (BASELINE.json north_star, SURVEY
§8c): visibility bit-exact on rays the oracle does not flag degenerate
(|margin| < 1e-6 or |cosθ| < 1e-6, reading Q8), entries within 1e-5 relative
on rows with no degenerate ray, degenerate fraction < 1e-4.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

REL_A = 1e-5


def oracle_lamps(desc: dict, vopts: dict, raw_ids, n_threads: int = 0) -> dict:
    """The oracle's own verdict and lamp samples for grid candidates `raw_ids`
    (the GPU's feasible columns): returns dict(samples (R, L, 3), feasible,
    ambiguous)."""
    v = O.vantage(desc, vopts, idx=np.asarray(raw_ids, np.int64), n_threads=n_threads)
    return dict(samples=v["samples"], feasible=v["feasible"], ambiguous=v["ambiguous"])


def compare_pairs(pat: dict, lamps: np.ndarray, rows, cols, gA, gvis, P: float = 80.0,
                  n_threads: int = 0) -> dict:
    """Oracle entries for pairs (input patch rows[q], column cols[q] of `lamps`
    (K, L, 3)) against the GPU's values gA[q] and visibility gvis[q, l]."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    ref = O.irradiance_pairs(pat, lamps, rows, cols, P=P, n_threads=n_threads)
    return stats_from(pat, lamps, rows, cols, gA, gvis, ref)


def stats_from(pat: dict, lamps: np.ndarray, rows, cols, gA, gvis, ref: dict) -> dict:
    """compare_pairs on oracle results `ref` already computed for these pairs."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    gA = np.asarray(gA, np.float64)
    gvis = np.asarray(gvis, bool)
    deg = ref["deg"]
    # which degeneracy (reporting only): the lamp (nearly) in the patch's plane,
    # |cos θ| < 1e-6, or a ray within 1e-6 of a triangle edge / the t range
    c = pat["centroid"][rows].astype(np.float64)
    nrm = pat["normal"][rows].astype(np.float64)
    D = np.asarray(lamps, np.float64)[cols] - c[:, None, :]
    cos = (D * nrm[:, None, :]).sum(-1) / np.sqrt((D * D).sum(-1))
    deg_cos = deg & (np.abs(cos) < 1e-6)
    ok = ~deg
    mism = (gvis != ref["vis"]) & ok
    rows_ok = ~deg.any(1)
    rA = ref["A"]
    err = np.abs(gA - rA)
    bad = rows_ok & (err > REL_A * np.abs(rA))
    pos = rows_ok & (rA > 0)
    rel = err[pos] / rA[pos]
    return dict(pairs=int(len(rows)), rays=int(deg.size), mismatches=int(mism.sum()),
                degenerate_rays=int(deg.sum()), degenerate_fraction=float(deg.mean()) if deg.size else 0.0,
                degenerate_cos=int(deg_cos.sum()), degenerate_margin=int((deg & ~deg_cos).sum()),
                entries_checked=int(rows_ok.sum()), entries_beyond_tol=int(bad.sum()),
                max_rel_err=float(rel.max()) if rel.size else 0.0,
                visible_fraction=float(ref["vis"].mean()) if deg.size else 0.0,
                mismatch_at=np.argwhere(mism)[:5].tolist(), bad_at=np.nonzero(bad)[0][:5].tolist())


def merge(a: dict, b: dict) -> dict:
    """Combine two compare_pairs results (counts add, maxima max)."""
    out = {}
    for k in ("pairs", "rays", "mismatches", "degenerate_rays", "entries_checked", "entries_beyond_tol",
              "degenerate_cos", "degenerate_margin"):
        out[k] = a.get(k, 0) + b.get(k, 0)
    out["degenerate_fraction"] = out["degenerate_rays"] / max(out["rays"], 1)
    out["max_rel_err"] = max(a["max_rel_err"], b["max_rel_err"])
    out["visible_fraction"] = (a.get("visible_fraction", 0.0) * a["rays"] + b.get("visible_fraction", 0.0) * b["rays"]) / max(out["rays"], 1)
    return out
