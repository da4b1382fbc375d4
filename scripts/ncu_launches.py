"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
`bench.py --profile-only --steps 1 --warmup 0`: the second half of the list
is one graph-replayed step.  usage: python scripts/ncu_launches.py CSV OUTDIR"""
import csv, sys
from collections import defaultdict

src, outdir = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
unit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
data = [(r[ki], float(r[vi].replace(",", "")) * unit[r[ui]]) for r in rows[1:]]
step = data[len(data) // 2:]
with open(f"{outdir}/ncu_launches_C4_step.csv", "w") as f:
    f.write("idx,kernel,us\n")
    for i, (k, t) in enumerate(step):
        f.write(f'{i},"{k[:90]}",{t:.2f}\n')
tot = sum(t for _, t in step)
agg = defaultdict(lambda: [0, 0.0])
for k, t in step:
    key = k.split("(")[0]
    agg[key][0] += 1
    agg[key][1] += t
lines = ["one C4 step (the second, graph-replayed half of `bench.py --profile-only --steps 1 "
         "--warmup 0` under ncu --metrics gpu__time_duration.sum --clock-control none; per-launch "
         "times are cold-cache and serialised)",
         f"launches {len(step)}, sum of kernel time {tot / 1e3:.3f} ms", ""]
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k[:60]:60s} {c:3d} launches {t / 1e3:8.3f} ms  {100 * t / tot:5.1f}%")
con = [t for k, t in step if "partial_contract_tcp" in k]
gat = [t for k, t in step if "gather_fast" in k]
lines += ["", "per-iteration contraction / gather (us):",
          "contract " + " ".join(f"{t:.0f}" for t in con),
          "gather   " + " ".join(f"{t:.0f}" for t in gat)]
open(f"{outdir}/ncu_launches_C4_summary.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
