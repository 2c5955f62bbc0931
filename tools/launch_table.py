"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
for r in rows[hi + 1:]:
    if len(r) > iv:
        agg[r[ik].split("(")[0][-40:]].append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-9))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:42s} n={len(v):5d} total={sum(v) * 1e3:9.3f} ms mean={sum(v) / len(v) * 1e6:9.2f} us "
          f"share={100 * sum(v) / tot:5.1f}%")
