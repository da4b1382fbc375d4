set -x
cd ${GRAFT_REPO_ROOT:-.}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo smoke rc $?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu1.log 2>&1; echo pytest rc $?
tail -30 gpurun_out/pytest_gpu1.log
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc $?
tail -5 gpurun_out/bench1.err
cat gpurun_out/bench1.json
