"""Turn the ncu metrics CSV of one bench step's GEMV launches into profiles/r02_ncu_traffic.json.
usage: python tools/traffic_from_ncu.py gpurun_out/traffic.csv"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_18172_b200 as sb  # noqa: E402

FUSED = [("qkv_proj", 6144, 4096), ("o_proj", 4096, 4096), ("gate_up_proj", 28672, 4096), ("down_proj", 4096, 14336)]
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iid, iname, imet, ival, iunit = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = {}
for r in rows[1:]:
    if "gemv_mma" not in r[iname]:
        continue
    v = float(r[ival].replace(",", ""))
    unit = r[iunit]
    if unit in ("Kbyte", "KB"):
        v *= 1e3
    elif unit in ("Mbyte", "MB"):
        v *= 1e6
    elif unit in ("Gbyte", "GB"):
        v *= 1e9
    elif unit in ("usecond",):
        v *= 1e3
    elif unit in ("msecond",):
        v *= 1e6
    per.setdefault(int(r[iid]), {})[r[imet]] = v
ids = sorted(per)[:4]
out = {"kernel": "gemv_mma_kernel<4,4,1,false>", "launches": []}
tot_t, tot_a = 0.0, 0
for i, (name, M, N) in zip(ids, FUSED):
    m = per[i]
    t = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a = sb.algorithmic_bytes(M, N, 4, act="sbvr", l=8)
    out["launches"].append({"gemv": name, "dram_read_bytes": m.get("dram__bytes_read.sum"),
                            "dram_write_bytes": m.get("dram__bytes_write.sum"), "traffic_bytes": t,
                            "algorithmic_bytes": a, "traffic_over_algorithmic": round(t / a, 4),
                            "ncu_duration_ns": m.get("gpu__time_duration.sum")})
    tot_t += t
    tot_a += a
out["traffic_bytes_per_launch_mean"] = tot_t / len(ids)
out["algorithmic_bytes_per_launch_mean"] = tot_a / len(ids)
out["traffic_over_algorithmic"] = round(tot_t / tot_a, 4)
out["source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control "
                 "none -k regex:gemv_mma on bench.py (first 4 GEMV launches = one step: qkv, o, gate_up, down)")
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                  "r02_ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
