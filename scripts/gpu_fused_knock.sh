# usage (GPU box): bash scripts/gpu_fused_knock.sh TAG — fused kernel knock-outs (C4 step times)
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1
mkdir -p gpurun_out
for dbg in 128 160 143 0; do
CVB_TC_DEBUG=$dbg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare --no-e2e > gpurun_out/bk_${TAG}_$dbg.json 2> gpurun_out/bk_${TAG}_$dbg.err; echo bench rc $?
python - $dbg <<PY
import json,sys
d=json.loads(open("gpurun_out/bk_${TAG}_$dbg.json").read().strip().splitlines()[-1])
print("dbg", sys.argv[1], "value",d["value"],"ms_per_step",d["ms_per_step"])
PY
tail -2 gpurun_out/bk_${TAG}_$dbg.err
done
