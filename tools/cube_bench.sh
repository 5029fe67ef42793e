timeout 800 python -m pytest tests/test_gpu_cube.py -q 2>&1 | tail -3
python - <<'PY'
import sys, os, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2103_14137_b200 import uvd as U
from synth import configs
sc = U.Scene(configs.c4_scene())
lam, _ = sc.vantage(configs.FLOAT_OPTS)
K = lam.shape[0]
cols = list(range(K // 3, K // 3 + 64))
out = {}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def best(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
for R in (128, 512):
    ms = best(lambda: sc.cubemap(lam, face_res=R, cols=cols))
    rays = len(cols) * 6 * R * R
    out[f"cube_R{R}"] = {"ms": ms, "cols": len(cols), "rays_per_s": rays / (ms / 1e3), "entries_per_s": len(cols) * sc.N / (ms / 1e3)}
    print(R, out[f"cube_R{R}"], flush=True)
ms = best(lambda: sc.irradiance(lam, cols=cols))
a = sc.irradiance(lam, cols=cols)
out["shadow_ray_centroid"] = {"ms": ms, "entries_per_s": len(cols) * sc.N / (ms / 1e3)}
ms1 = best(lambda: sc.irradiance(lam, cols=cols, area_subdiv=1))
a1 = sc.irradiance(lam, cols=cols, area_subdiv=1)
out["shadow_ray_area_m1"] = {"ms": ms1, "entries_per_s": len(cols) * sc.N / (ms1 / 1e3)}
# agreement cube(512) vs area model m=1 and centroid model, over lit patches
c512 = sc.cubemap(lam, face_res=512, cols=cols)["A"][:, :sc.N].double()
am = a1["A"][:, :sc.N].double(); cm = a["A"][:, :sc.N].double()
lit = am > 0
out["agreement"] = {"median_rel_cube_vs_area_m1": float(((c512 - am).abs() / am)[lit].median()),
                    "median_rel_centroid_vs_area_m1": float(((cm - am).abs() / am)[lit].median()),
                    "total_flux_ratio_cube_over_area": float((c512.sum() / am.sum()))}
print(out, flush=True)
json.dump(out, open("gpurun_out/cube_r01.json", "w"), indent=1)
PY
