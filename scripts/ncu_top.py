"""Top utilisation metrics (pct of peak) of one kernel in an ncu report:
which unit is closest to its ceiling.
    python scripts/ncu_top.py report.ncu-rep kernel_regex [launch_index] [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kern], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, d = rows[0], rows[2 + idx]
vals = []
for h, v in zip(hdr, d):
    if ("pct_of_peak_sustained_elapsed" in h and ".avg." in h) or h.endswith("pct_of_peak_sustained_elapsed") and ".sum" not in h and ".max" not in h and ".min" not in h:
        try:
            vals.append((float(v), h))
        except ValueError:
            pass
print(d[hdr.index("Kernel Name")][:60], "time_us", d[hdr.index("gpu__time_duration.sum")])
for f, h in sorted(vals, reverse=True)[:n]:
    print(f"{f:6.1f}  {h}")
