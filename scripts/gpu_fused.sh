# usage (GPU box): bash scripts/gpu_fused.sh TAG [tests...] — fused-vs-unfused tests and C4 step times
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
mkdir -p gpurun_out
if [ $# -gt 0 ]; then
timeout 900 python -m pytest "$@" -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc $?
tail -15 gpurun_out/pytest_$TAG.log
fi
for f in 1 0 1 0; do
CVB_FUSED=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare --no-e2e > gpurun_out/bf_${TAG}_$f.json 2> gpurun_out/bf_${TAG}_$f.err; echo bench rc $?
python - $f <<PY
import json,sys
d=json.loads(open("gpurun_out/bf_${TAG}_$f.json").read().strip().splitlines()[-1])
print("fused", sys.argv[1], "value",d["value"],"ms_per_step",d["ms_per_step"])
PY
done
