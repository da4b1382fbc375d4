# usage (GPU box): bash scripts/gpu_quick_r2.sh TAG [tests...] — selected gpu tests + a quick C4 bench line
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
mkdir -p gpurun_out
if [ $# -gt 0 ]; then
timeout 1500 python -m pytest "$@" -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?
tail -4 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare --no-e2e > gpurun_out/bq_$TAG.json 2> gpurun_out/bq_$TAG.err; echo bench rc $?
python - <<PY
import json
d=json.loads(open("gpurun_out/bq_$TAG.json").read().strip().splitlines()[-1])
print("value",d["value"],"ms_per_step",d["ms_per_step"])
k=d["kernel_ms"]; print("contract",[round(x,3) for x in k["contract_ms"]]); print("gather",[round(x,3) for x in k["gather_ms"]])
PY
