"""Summarise an `ncu --nvtx --csv` launch list per NVTX range (uvd_* entry
point) and per kernel: launches, time, share, DRAM bytes per launch.
usage: python tools/nvtx_summary.py launches.csv [steps]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(ln for ln in open(sys.argv[1]) if ln.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
rng_col = [h for h in hdr if "Push/Pop_Range" in h][0]
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[1:]:
    rng = r[ix[rng_col]].split(":")[1] if ":" in r[ix[rng_col]] else "(none)"
    k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    m = r[ix["Metric Name"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    key = (rng, k)
    if m == "gpu__time_duration.sum":
        per[key]["n"] += 1
        per[key]["ns"] += v
    elif m.startswith("dram__bytes"):
        per[key]["dram"] += v
tot = sum(d["ns"] for d in per.values())
by_rng = collections.defaultdict(float)
for (rng, k), d in per.items():
    by_rng[rng] += d["ns"]
print("| NVTX range (entry point) | GPU time share |")
print("|---|---|")
for rng, ns in sorted(by_rng.items(), key=lambda x: -x[1]):
    print(f"| {rng} | {ns / tot * 100:.2f} % |")
print()
print("| range | kernel | launches | ms per launch | share | DRAM GB per launch |")
print("|---|---|---|---|---|---|")
for (rng, k), d in sorted(per.items(), key=lambda x: -x[1]["ns"]):
    if d["ns"] / tot < 1e-4:
        continue
    print(f"| {rng} | {k} | {int(d['n'])} | {d['ns'] / d['n'] / 1e6:.3f} | {d['ns'] / tot * 100:.2f} % | "
          f"{d['dram'] / d['n'] / 1e9:.3f} |")
