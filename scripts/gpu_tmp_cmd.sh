nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json,statistics; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']
print(d['value'], 'contract it0 %.3f warm %.4f gather %.4f' % (k['contract_ms'][0], statistics.mean(k['contract_ms'][1:]), statistics.mean(k['gather_ms'][1:])), d['clocks'])" || tail -3 gpurun_out/ab.err
done
