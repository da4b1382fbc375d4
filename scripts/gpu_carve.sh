cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for C in -1 70 60 100; do
  CVB_GF_CARVEOUT=$C timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-compare --no-e2e > gpurun_out/carve_$C.json 2>/dev/null
  python -c "
import json,statistics
d=json.loads(open('gpurun_out/carve_$C.json').read().strip().splitlines()[-1])
print('carve $C value',d['value'],'gather warm',round(statistics.mean(d['kernel_ms']['gather_ms'][1:]),4))"
done
