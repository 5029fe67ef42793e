"""BVH quality (development tool): the SAH cost of the GPU tree (uvd_scene_bvh)
against a CPU top-down binned-SAH tree over the same triangles, to size the
gain a better builder could bring to k_assemble.

SAH cost = Σ_internal SA(node)/SA(root)·C_t + Σ_leaf SA(leaf)/SA(root)·n·C_i
with C_t = 1, C_i = 1 (leaves of <= 2 triangles in both trees).

usage: python tools/bvh_quality.py [C4|C5|ward]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import configs, ward  # noqa: E402

LEAF = np.int64(0x80000000)


def sa(lo, hi):
    d = np.maximum(hi - lo, 0)
    return 2 * (d[..., 0] * d[..., 1] + d[..., 1] * d[..., 2] + d[..., 0] * d[..., 2])


def gpu_sah(sc):
    b = sc.bvh()
    words = b["nodes"].cpu().numpy()
    boxes = words.view(np.float32)
    refs = words[:, 12:14].astype(np.int64) & 0xFFFFFFFF
    c0lo = boxes[:, [0, 2, 8]]; c0hi = boxes[:, [1, 3, 9]]
    c1lo = boxes[:, [4, 6, 10]]; c1hi = boxes[:, [5, 7, 11]]
    root_sa = sa(np.minimum(c0lo[0], c1lo[0]), np.maximum(c0hi[0], c1hi[0]))
    cost = 1.0  # root
    stack = [0]
    nodes = leaves = 0
    while stack:
        n = stack.pop()
        nodes += 1
        for side, (lo, hi) in enumerate(((c0lo[n], c0hi[n]), (c1lo[n], c1hi[n]))):
            r = refs[n, side]
            s = sa(lo, hi) / root_sa
            if r & LEAF:
                cost += s * ((r & 7) + 1)
                leaves += 1
            else:
                cost += s
                stack.append(int(r))
    return cost, nodes, leaves


def cpu_sah_tree(lo, hi, leaf_max=2, bins=32):
    """top-down binned SAH (centroid bins), returns the SAH cost"""
    cen = 0.5 * (lo + hi)
    root_sa = sa(lo.min(0), hi.max(0))
    cost = 0.0
    stack = [np.arange(len(lo))]
    nodes = 0
    while stack:
        idx = stack.pop()
        blo, bhi = lo[idx].min(0), hi[idx].max(0)
        if len(idx) <= leaf_max:
            cost += sa(blo, bhi) / root_sa * len(idx)
            continue
        cost += sa(blo, bhi) / root_sa
        nodes += 1
        c = cen[idx]
        best = (np.inf, None)
        for ax in range(3):
            cmin, cmax = c[:, ax].min(), c[:, ax].max()
            if cmax <= cmin:
                continue
            b = np.minimum(((c[:, ax] - cmin) / (cmax - cmin) * bins).astype(np.int64), bins - 1)
            cnt = np.bincount(b, minlength=bins)
            blo_ = np.full((bins, 3), np.inf); bhi_ = np.full((bins, 3), -np.inf)
            np.minimum.at(blo_, b, lo[idx]); np.maximum.at(bhi_, b, hi[idx])
            llo = np.minimum.accumulate(blo_, 0); lhi = np.maximum.accumulate(bhi_, 0)
            rlo = np.minimum.accumulate(blo_[::-1], 0)[::-1]; rhi = np.maximum.accumulate(bhi_[::-1], 0)[::-1]
            lc = np.cumsum(cnt); rc = lc[-1] - lc
            for k in range(bins - 1):
                if lc[k] == 0 or rc[k] == 0:
                    continue
                v = sa(llo[k], lhi[k]) * lc[k] + sa(rlo[k + 1], rhi[k + 1]) * rc[k]
                if v < best[0]:
                    best = (v, (ax, k, b))
        if best[1] is None:  # all centroids equal: split in half
            h = len(idx) // 2
            stack += [idx[:h], idx[h:]]
            continue
        ax, k, b = best[1]
        stack += [idx[b <= k], idx[b > k]]
    return cost, nodes


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "C4"
    desc = {"C4": configs.c4_scene, "C5": configs.c5_scene, "ward": lambda: ward.ward(4, 1, 0.1)}[which]()
    from paper_2103_14137_b200 import uvd
    sc = uvd.Scene(desc)
    t0 = time.time()
    g = gpu_sah(sc)
    V = desc["vertices"][desc["tris"]].astype(np.float64)
    lo, hi = V.min(1), V.max(1)
    c = cpu_sah_tree(lo, hi)
    print({"scene": which, "M": len(lo), "gpu_ploc_sah": g[0], "gpu_nodes_reached": g[1],
           "cpu_binned_sah": c[0], "ratio_gpu_over_cpu": g[0] / c[0], "s": round(time.time() - t0, 1)})


if __name__ == "__main__":
    main()
