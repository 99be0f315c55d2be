"""Summarise an .ncu-rep: key throughput metrics + top stall reasons per kernel.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "inst",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
}
idx = {name: i for i, name in enumerate(h)}
ki = idx.get("Kernel Name")
for r in rows[2:]:
    if not re.search(kre, r[ki]):
        continue
    print(r[ki][:90])
    for m, lab in want.items():
        if m in idx:
            print(f"   {lab:15s} {r[idx[m]]} {rows[1][idx[m]]}")
    stalls = []
    for name, i in idx.items():
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if v > 0:
                stalls.append((v, name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot = sum(v for v, _ in stalls) or 1
    print("   stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:6]))
