# usage (GPU box): bash scripts/gpu_r2t.sh TAG test-files...
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
mkdir -p gpurun_out
nproc; free -g | head -2; lscpu | grep -E "Model name|Socket|Core"
timeout 2400 python -m pytest "$@" -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?
tail -25 gpurun_out/pytest_gpu_$TAG.log
