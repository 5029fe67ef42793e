"""Compare vantage sets from the two BVH builders and check differing
candidates against the oracle (debug tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2103_14137_b200 import uvd
    from synth import configs
    sc = uvd.Scene(configs.c5_scene())
    _, raw = sc.vantage(configs.ARM_OPTS)
    np.save(sys.argv[2], raw.cpu().numpy())
    sys.exit(0)

for b in ("karras", "ploc"):
    subprocess.check_call([sys.executable, __file__, "child", f"/tmp/raw_{b}.npy"], env=dict(os.environ, UVD_BVH=b))
ka, pl = np.load("/tmp/raw_karras.npy"), np.load("/tmp/raw_ploc.npy")
diff = np.setxor1d(ka, pl)
print("karras", len(ka), "ploc", len(pl), "differ", len(diff))
from oracle import oracle as O  # noqa: E402
from synth import configs  # noqa: E402
sel = np.sort(diff[:40])
v = O.vantage(configs.c5_scene(), configs.ARM_OPTS, idx=sel)
for q, f, a in zip(v["idx"], v["feasible"], v["ambiguous"]):
    print(q, "in_karras", q in ka, "in_ploc", q in pl, "oracle feasible", f, "ambiguous", a)
