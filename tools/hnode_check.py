"""Full-size check that the fp16 H nodes change no decision: C4 (both robots)
and C5 assembled with UVD_HNODES (or the variable named on the command
line, e.g. UVD_QNODES) =0 and =1, A compared bit for bit on the device,
fix-up lists compared as sets.  usage: python tools/hnode_check.py [VAR]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from synth import configs  # noqa: E402

__graft_entry__.build()
from paper_2103_14137_b200 import uvd  # noqa: E402

VAR = sys.argv[1] if len(sys.argv) > 1 else "UVD_HNODES"
for c in (configs.c4("float"), configs.c4("tower"), configs.c5()):
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    out = {}
    for h in ("0", "1"):
        os.environ[VAR] = h
        torch.cuda.synchronize()
        t0 = time.time()
        r = sc.irradiance(lamps, fixups=1 << 24)
        sc.sync_status()
        torch.cuda.synchronize()
        out[h] = (r["A"], np.sort(r["fixups"].cpu().numpy().astype(np.uint64)), time.time() - t0)
        del r
    eqA = torch.equal(out["0"][0].view(torch.int32), out["1"][0].view(torch.int32))
    eqF = np.array_equal(out["0"][1], out["1"][1])
    print(json.dumps({"var": VAR, "workload": c["name"], "N": sc.N, "K": lamps.shape[0], "A_equal": bool(eqA),
                      "fixups_equal": bool(eqF), "n_fixups": int(len(out["1"][1])),
                      "s_off": out["0"][2], "s_on": out["1"][2]}), flush=True)
    del out
    sc.close()
    torch.cuda.empty_cache()
os.environ.pop(VAR)
