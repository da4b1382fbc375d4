# usage (GPU box): bash scripts/gpu_splits.sh TAG — C4 step time per range-split setting
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1
mkdir -p gpurun_out
for cfg in "1 serial" "2 serial" "4 serial" "8 serial" "16 serial" "4 side" "8 side"; do
  set -- $cfg
  CVB_PIPELINE_SPLITS=$1 CVB_SPLIT_MODE=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare --no-e2e > gpurun_out/sp_${TAG}_$1_$2.json 2> gpurun_out/sp_${TAG}_$1_$2.err
  python - $1 $2 <<PY
import json,sys
d=json.loads(open("gpurun_out/sp_${TAG}_$1_$2.json").read().strip().splitlines()[-1])
print(sys.argv[1:], "value",d["value"],"ms_per_step",d["ms_per_step"])
PY
done
