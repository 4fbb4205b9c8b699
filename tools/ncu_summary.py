"""Summarise an ncu report (raw page): duration, DRAM bytes, issue/pipe utilisation, stall reasons per issue, and the
per-opcode instruction / stall-sample mix of the source page.  Usage: python tools/ncu_summary.py <report.ncu-rep>"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__average_warp_latency_per_inst_issued.ratio"]
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h} = {vals[i]} {units[i]}")
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(vals[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v >= 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r2 = list(csv.reader(io.StringIO(src)))
h2, data = r2[1], r2[2:]
iS, iA, iE = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)"), h2.index("Instructions Executed")
samp, ex = collections.Counter(), collections.Counter()
for r in data:
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    samp[op] += int(float(r[iA] or 0))
    ex[op] += int(float(r[iE] or 0))
tot_s, tot_e = sum(samp.values()), sum(ex.values())
print(f"instructions executed {tot_e}, stall samples {tot_s}")
for op, v in ex.most_common(16):
    print(f"  {op:8s} executed {v:9d} ({100 * v / tot_e:5.1f}%)  samples {samp[op]:5d} ({100 * samp[op] / max(tot_s, 1):5.1f}%)")
