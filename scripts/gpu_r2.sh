# usage (GPU box, repo root): bash scripts/gpu_r2.sh TAG [pytest selector]
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-run}; SEL=${2:-tests}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest $SEL -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?
tail -30 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
tail -3 gpurun_out/bench_$TAG.err
cut -c1-600 gpurun_out/bench_$TAG.json
