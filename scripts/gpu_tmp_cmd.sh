timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_dn.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_dn.log
for c in C2 C3 C4 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['compare'])" || tail -3 gpurun_out/ab.err
done
