# usage (on the GPU box, from the repo root): bash scripts/gpu_check.sh TAG [bench args...]
set -x
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-run}; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?
tail -15 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
tail -5 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
