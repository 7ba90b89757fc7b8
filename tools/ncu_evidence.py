"""Curated ncu evidence for one captured launch (the north_star's asks: HBM/L2
bytes moved for the gather, FP32 pipe utilisation of the scoring, and what
bounds the kernel).  Usage: python tools/ncu_evidence.py REPORT [label]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
col = {n: i for i, n in enumerate(h)}

WANT = [
    ("kernel", "Kernel Name"),
    ("duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM read rate", "dram__bytes_read.sum.per_second"),
    ("DRAM peak fraction", "dram__bytes_read.sum.pct_of_peak_sustained_elapsed"),
    ("L2 sectors (tex) pct of peak", "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed"),
    ("L2 throughput pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
    ("L2 read sectors from the SMs", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("L2 -> L1/smem bytes", "l1tex__m_xbar2l1tex_read_bytes.sum"),
    ("L1/shared wavefronts pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("shared-memory wavefronts pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("FP32 (FMA pipe) active pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("ALU pipe active pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("LSU pipe pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("issue active pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    ("warps active per scheduler", "smsp__warps_active.avg.per_cycle_active"),
    ("instructions", "smsp__inst_executed.sum"),
    ("registers", "launch__registers_per_thread"),
    ("smem per block", "launch__shared_mem_per_block_dynamic"),
]
print(f"== {label}")
for name, key in WANT:
    if key in col:
        i = col[key]
        print(f"  {name:32s} {v[i]:>22s} {u[i]}")
stalls = sorted(((float(v[i].replace(",", "")), n) for n, i in col.items()
                 if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")),
                reverse=True)
print("  stall cycles per issued instruction (top):")
for val, n in stalls[:8]:
    print(f"    {n[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {val:6.3f}")
