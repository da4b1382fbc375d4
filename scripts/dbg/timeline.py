"""Summarise the warm contraction's role timeline (CVB_TC_DEBUG=16 dump,
CVB_TC_TS_FILE): per tile, when each role passed its waits (CTAs 0-3, first
64 tiles of each launch).  usage: python scripts/dbg/timeline.py FILE [launch]"""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
per_launch = 4 * 64 * 32
n = raw.size // per_launch
launch = int(sys.argv[2]) if len(sys.argv) > 2 else n // 2
ts = raw[launch * per_launch:(launch + 1) * per_launch].reshape(4, 64, 32).astype(np.int64)
names = {0: "plan copy issued", 1: "MMA has plan", 6: "MMA acc free", 2: "MMA tile done",
         3: "A tile done", 20: "epi acc full", 21: "epi chunk0 done", 4: "epi tile done",
         5: "B tile done"}
for k in range(4):
    names[24 + k] = f"B piece{k} issued"
    names[12 + k] = f"MMA B{k} full"
    names[16 + k] = f"A stage{k} free/issue"
    names[8 + k] = f"MMA A{k} full"
rows = []
for cta in range(4):
    t = ts[cta]
    valid = [i for i in range(1, 63) if t[i, 2] > 0 and t[i + 1, 2] > 0 and t[i, 1] > 0]
    for i in valid:
        base = t[i, 1]
        rows.append({e: (t[i, e] - base) if t[i, e] > 0 else np.nan for e in names})
        rows[-1]["period"] = t[i + 1, 2] - t[i, 2]
print(f"launch {launch} of {n}, {len(rows)} tiles; ns relative to 'MMA has plan' (median, p90)")
for e in sorted(names, key=lambda e: np.nanmedian([r[e] for r in rows])):
    v = np.array([r[e] for r in rows], dtype=float)
    print(f"  {names[e]:24s} {np.nanmedian(v):8.0f} {np.nanpercentile(v, 90):8.0f}")
p = np.array([r["period"] for r in rows], dtype=float)
print(f"  tile period (MMA done to MMA done): median {np.median(p):.0f} ns, mean {p.mean():.0f}")
