"""Summarise an ncu report: headline metrics, stall reasons, top stall SASS lines."""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
NCU = "/usr/local/cuda/bin/ncu"


def run(*a):
    return subprocess.run([NCU, "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate"]
seen = set()
for r in rows[1:]:
    if r[mi] in want and (r[ki], r[mi]) not in seen:
        seen.add((r[ki], r[mi]))
        print(f"{r[ki][:50]:50s} {r[mi]:28s} {r[vi]} {r[ui]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
for r in raw[2:]:
    print("==", r[h.index("Kernel Name")][:60])
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
                # tcgen05: tensor-pipe busy time, its shared-memory operand reads, TMEM traffic
                "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
        if key in h:
            print(f"   {key} = {r[h.index(key)]} {raw[1][h.index(key)]}")
    items = []
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                items.append((float(r[i].replace(",", "")), name[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1
    print("   stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(items, reverse=True)[:6]))
for view in ("sass", "cuda"):
    text = run("--page", "source", "--csv", "--print-source", view)
    blocks, cur = [], None
    for row in csv.reader(io.StringIO(text)):
        if row and row[0] == "Kernel Name":
            cur = [row[1], None, []]
            blocks.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = row
        elif cur is not None:
            cur[2].append(row)
    for name, sh, data in blocks:
        if sh is None or not data:
            continue
        ci = {x: i for i, x in enumerate(sh)}
        col = "Warp Stall Sampling (All Samples)"
        if col not in ci:
            continue
        f = lambda x, c: float((x[ci[c]] or "0").replace(",", "")) if x[ci[c]] not in ("-", "") else 0.0
        tot = sum(f(x, col) for x in data) or 1
        print(f"== [{view}] {name[:70]}: top stall lines")
        for x in sorted(data, key=lambda x: -f(x, col))[:ntop]:
            loc = x[ci["Source"]].strip()[:90]
            print(f"   {100*f(x, col)/tot:5.1f}% {x[ci['Instructions Executed']]:>9} {loc}")
