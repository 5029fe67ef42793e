"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[iu], 1e-6)
    name = r[ik].split("(")[0]
    tot[name] += float(r[iv].replace(",", "")) * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':50s} {'launches':>8s} {'ms (cold, serialised)':>22s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:50]:50s} {cnt[k]:8d} {v:22.2f} {v / T * 100:5.1f}%")
print(f"total {T:.1f} ms over {sum(cnt.values())} launches")
