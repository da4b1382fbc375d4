"""Instrument partial_tc.cu in place with per-role wait-cycle accumulators
(for a variant build only; restore with git checkout afterwards).  The dump
goes to row 63 of the CVB_TC_TS_FILE timeline (CVB_TC_DEBUG & 16); the
per-event stamps are disabled so they do not perturb the measurement."""
import re
import sys

p = sys.argv[1]
s = open(p).read()
waits = [  # (substring identifying the wait, counter, recording thread)
    ("wait_full(U(C.plan_full[s]), (uint32_t)(it / NPL));", None, None),
]
lines = s.split("\n")
role = None
out = []
counters = {"B": (12, 13), "MMA": (0, 1, 2, 3), "L": (15,), "A": (5, 6), "E": (8, 9)}
for ln in lines:
    if "B producer: F1 pieces" in ln: role = "B"
    elif "MMA issuer ---" in ln: role = "MMA"
    elif "plan loader: one bulk" in ln: role = "L"
    elif "A producers:" in ln: role = "A"
    elif "epilogue (128 threads" in ln: role = "E"
    m = re.match(r"^(\s*)(wait_(full|empty)\(U\(C\.(\w+)\[.*)$", ln)
    if m and role:
        bar = m.group(4)
        idx = {("B", "plan_full"): 12, ("B", "b_empty"): 13, ("MMA", "plan_full"): 0,
               ("MMA", "acc_empty"): 1, ("MMA", "b_full"): 2, ("MMA", "a_full"): 3,
               ("L", "plan_empty"): 15, ("A", "plan_full"): 5, ("A", "a_empty"): 6,
               ("E", "plan_full"): 8, ("E", "acc_full"): 9}[(role, bar)]
        who = {"A": "tid == 128", "E": "tid == 256"}.get(role, "(lane == 0)")
        ln = f"{m.group(1)}{{ const long long _t0 = clock64(); {m.group(2)} if ({who}) wacc[{idx}] += clock64() - _t0; }}"
    out.append(ln)
s = "\n".join(out)
s = s.replace("""        const int64_t t = atomicAdd(tile_counter(P), 1);  // dynamic tile scheduler""",
              """        const long long _ta = clock64();
        const int64_t t = atomicAdd(tile_counter(P), 1);  // dynamic tile scheduler
        wacc[16] += clock64() - _ta;""")
s = s.replace("""  const uint32_t tmem = C.tmem;
  pdl_trigger();""", """  const uint32_t tmem = C.tmem;
  long long wacc[18] = {0};
  const long long t_start = clock64();
  pdl_trigger();""")
s = s.replace("""  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc""", """  if (T.ts != nullptr && blockIdx.x < 4 && (tid == 0 || tid == 32 || tid == 64 || tid == 128 || tid == 256)) {
    unsigned long long* w = T.ts + ((int64_t)blockIdx.x * 64 + 63) * 32;
    for (int i = 0; i < 18; ++i)
      if (wacc[i] != 0) w[i] = (unsigned long long)wacc[i];
    const int tot = tid == 0 ? 14 : tid == 32 ? 4 : tid == 64 ? 17 : tid == 128 ? 7 : 10;
    w[tot] = (unsigned long long)(clock64() - t_start);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc""")
s = s.replace("""  if (T.ts != nullptr && blockIdx.x < 4 && it < 64) {
    unsigned long long t;""", """  if (false) {
    unsigned long long t;""")
assert s.count("wacc[") >= 14, s.count("wacc[")
open(p, "w").write(s)
