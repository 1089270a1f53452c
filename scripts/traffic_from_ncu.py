"""Per-iteration DRAM traffic and L1->L2 request utilisation of the two pass
kernels from one `ncu --set full` capture of scripts/profile_run.py (one
iteration = NB stream passes + NB link passes), for bench.py's
roofline.traffic and profiles/.
    python scripts/traffic_from_ncu.py report.ncu-rep CONFIG > profiles/traffic_r1.json"""
import csv
import io
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(d, m):
    return float(d[ix[m]]) * scale.get(units[ix[m]], 1.0)


# The capture window holds one iteration's worth of launches (NB stream
# passes, NB link passes, one epilogue), possibly straddling two iterations.
per = {}
for d in data:
    name = d[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].replace("numpmp_dev::", "")
    # stream side: the stream passes (+ the v refresh they wait for); link side:
    # the link passes and the link epilogue
    key = "k_stream_pass" if ("stream_pass" in name or "refresh_v" in name) else "k_link_pass"
    e = per.setdefault(key, {"dram_bytes": 0.0, "ncu_us": 0.0, "launches": 0, "xbar_req_pct": [], "l2_hit_pct": []})
    e["dram_bytes"] += val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    e["ncu_us"] += float(d[ix["gpu__time_duration.sum"]]) / (1e3 if units[ix["gpu__time_duration.sum"]] == "nsecond" else 1.0)
    e["launches"] += 1
    t_us = float(d[ix["gpu__time_duration.sum"]]) / (1e3 if units[ix["gpu__time_duration.sum"]] == "nsecond" else 1.0)
    e["xbar_req_pct"].append((t_us, float(d[ix["l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"]])))
    e["l2_hit_pct"].append((t_us, float(d[ix["lts__t_sector_hit_rate.pct"]])))
for e in per.values():  # time-weighted over the launches of the iteration
    for k in ("xbar_req_pct", "l2_hit_pct"):
        tot = sum(t for t, _ in e[k])
        e[k] = round(sum(t * v for t, v in e[k]) / tot, 1) if tot > 0 else None
    e["ncu_us"] = round(e["ncu_us"], 1)
print(json.dumps({"source": f"{rep} (ncu --set full --clock-control none, scripts/profile_run.py {cfg}; one iteration)",
                  "config": cfg, "per_iteration": per}, indent=1))
