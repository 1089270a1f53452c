"""Summarise an ncu report (raw page) for the PMP kernels: time, DRAM
bytes, L2 hit rate, L1 data-pipe split, occupancy."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("l1_data_pipe_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("l1_smem_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("l1_gld_tout_pct", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum.pct_of_peak_sustained_elapsed"),
    ("lsu_wb_pct", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed"),
    ("lts_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("smem_bank_conf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
]
w = csv.writer(sys.stdout)
w.writerow(["kernel"] + [k for k, _ in want])
for d in data:
    name = d[idx["Kernel Name"]].split("(")[0].replace("void ", "")
    vals = []
    for k, m in want:
        if m not in idx:
            vals.append("NA")
            continue
        v = d[idx[m]]
        u = units[idx[m]]
        try:
            f = float(v)
            if k.endswith("_MB"):
                f = f * {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(u, 1.0)
            vals.append(f"{f:.1f}")
        except ValueError:
            vals.append(v)
    w.writerow([name] + vals)
