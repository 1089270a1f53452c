"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python scripts/launch_summary.py gpurun_out/launches_X.csv [iterations]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    n = r[ki].split("(")[0].replace("void ", "")
    tot[n] += float(r[vi].replace(",", ""))
    cnt[n] += 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for n in sorted(tot, key=lambda n: -tot[n])[:20]:
    per = f"  {tot[n] / iters / 1e3:8.2f} us/iteration" if iters else ""
    print(f"{n:40s} {cnt[n]:6d} launches {tot[n] / cnt[n] / 1e3:9.2f} us avg {tot[n] / 1e6:9.3f} ms{per}")
