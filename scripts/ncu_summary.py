"""Summarise an ncu report: key metrics, stall reasons, opcode mix, top stall lines.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [--lines N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units, rows = raw[0], raw[1], raw[2:]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum",
        "smsp__inst_executed_pipe_lsu.sum", "lts__t_bytes.sum",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
for r in rows:
    print(r[h.index("Kernel Name")][:60])
    for k in keys:
        if k in h:
            print(f"   {k:60s} {r[h.index(k)]} {units[h.index(k)]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
ie, smp = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
data = [r for r in src[2:] if len(r) == len(hh) and r[ie].isdigit()]
seen, uniq = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)
stall = [i for i, n in enumerate(hh) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(int(r[ie]) for r in uniq)
st = Counter()
for r in uniq:
    for i in stall:
        st[hh[i]] += int(r[i])
print("instructions", tot, "stalls:", st.most_common(8))
op, ops = Counter(), Counter()
for r in uniq:
    t = r[1].split()
    if not t:
        continue
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += int(r[ie])
    ops[o] += int(r[smp])
for k, v in op.most_common(22):
    print(f"  {k:10s} {v:9d} {100 * v / tot:5.1f}%  samples {ops[k]}")
print("top stall lines:")
for r in sorted(uniq, key=lambda r: -int(r[smp]))[:nlines]:
    print(" ", r[0][-5:], r[smp], r[ie], r[1][:58], [(hh[i][6:], r[i]) for i in stall if int(r[i]) > max(2, int(r[smp]) // 4)])
