# probe + gpu tests + bench (no compare/e2e/cpu) — fast iteration loop
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-q}
timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe_$TAG.log 2>&1; echo probe rc $?; tail -4 gpurun_out/tc_probe_$TAG.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
tail -3 gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('ms/iter', d['value'], 'clocks', d['clocks'])
print('contract', d['kernel_ms']['contract_ms']); print('gather', d['kernel_ms']['gather_ms'])
print('roofline', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
