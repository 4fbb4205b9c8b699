"""Summarise tools/ab.sh output: min us per (variant, shape)."""
import json
import sys
tag, res = None, {}
for l in open(sys.argv[1]):
    l = l.strip()
    if l.startswith("== "):
        tag = l[3:]
        continue
    try:
        d = json.loads(l)
    except Exception:
        continue
    key = (tag, d["shape"] + (f"/T{d['T']}" if d.get("T", 1) != 1 else ""))
    res[key] = min(res.get(key, 1e9), d["us"])
tags = sorted({t for t, _ in res}, key=lambda t: (t != "cur", t))
shapes = sorted({s for _, s in res}, key=lambda s: list(k[1] for k in res).index(s))
print("variant".ljust(12) + "".join(s.rjust(14) for s in shapes))
for t in tags:
    print(t.ljust(12) + "".join(f"{res.get((t, s), float('nan')):14.3f}" for s in shapes))
