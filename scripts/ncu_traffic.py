"""profiles/ncu_traffic_<CFG>.json from a warm `ncu --set full` capture:
dram__bytes_read.sum + dram__bytes_write.sum per kernel (one launch each).
usage: python scripts/ncu_traffic.py REPORT CFG SOURCE_NOTE"""
import csv, io, json, subprocess, sys

rep, cfg, note = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv",
                      "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    key = ("partial_contract_tcp_kernel" if "partial_contract_tcp" in name else
           "gather_fast_kernel" if "gather_fast" in name else name.split("(")[0])
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(r[i].replace(",", "")) * scale[units[i]]
    res.setdefault(key, int(tot))
res["source"] = note
json.dump(res, open(f"profiles/ncu_traffic_{cfg}.json", "w"), indent=1)
print(cfg, res)
