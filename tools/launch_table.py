"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_*)
per kernel: launches, total time, share, DRAM bytes per launch, GB/s.

usage: python tools/launch_table.py launches.csv [top]
"""
import collections
import csv
import sys

T = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
B = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    seen = set()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        if (r[idi], name) not in seen:
            seen.add((r[idi], name))
            cnt[name] += 1
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= T[r[ui]]
        elif "bytes" in r[mi]:
            v *= B[r[ui]]
        agg[name][r[mi]] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    print(f"total {tot / 1e3:.3f} ms over {sum(cnt.values())} launches")
    print("| kernel | launches | ms | share | DRAM GB/launch | GB/s |")
    print("|---|---|---|---|---|---|")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])[:top]:
        t = a["gpu__time_duration.sum"]
        b = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        print(f"| {n} | {cnt[n]} | {t / 1e3:.3f} | {100 * t / tot:.1f} % | {b / 1e9 / cnt[n]:.3f} | "
              f"{b / (t * 1e-6) / 1e9 if t else 0:.0f} |")


if __name__ == "__main__":
    main()
