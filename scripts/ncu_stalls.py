"""Top stall-sampled SASS instructions of one kernel in an ncu report, with
the CUDA source line each belongs to (needs -lineinfo + --import-source on).
    python scripts/ncu_stalls.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "-c", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
src_line, src_txt = None, ""
seen, items, total = set(), [], 0
for r in rows[3:]:
    if len(r) <= i_s:
        continue
    if r[0]:
        src_line, src_txt = r[0], r[1].strip()
        continue
    addr = r[2]
    if addr in seen or not r[i_s].isdigit():
        continue
    seen.add(addr)
    v = int(r[i_s])
    total += v
    items.append((v, addr[-5:], r[3].strip(), src_line, src_txt))
print("total stall samples", total)
for v, a, ins, ln, txt in sorted(items, reverse=True)[:n]:
    print(f"{v:6d} {100.0 * v / max(total, 1):5.1f}%  {a}  {ins[:42]:42s}  L{ln}: {txt[:60]}")
