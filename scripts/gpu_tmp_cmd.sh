for rep in 1 2 3; do for v in 65 60 70; do
  CVB_GF_CARVEOUT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json,statistics; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']
print('carve=$v', d['value'], 'warm %.4f gather %.4f' % (statistics.mean(k['contract_ms'][1:]), statistics.mean(k['gather_ms'][1:])))" || tail -3 gpurun_out/ab.err
done; done
