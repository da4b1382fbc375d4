# A/B of prebuilt library variants in variants_tmp/*/ (swapped in place), alternating, per carveout
cd ${GRAFT_REPO_ROOT:-.}
cp paper_2505_16942_b200/libcorrvol_b200.so /tmp/lib_orig.so
for rep in 1 2; do
for C in ${CARVES:--1 65}; do
for d in variants_tmp/*/; do
  cp $d/libcorrvol_b200.so paper_2505_16942_b200/libcorrvol_b200.so
  CVB_GF_CARVEOUT=$C timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json,statistics; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']
print('$d carve $C', d['value'], 'contract it0 %.3f warm %.4f gather %.4f' % (k['contract_ms'][0], statistics.mean(k['contract_ms'][1:]), statistics.mean(k['gather_ms'][1:])))" || tail -3 gpurun_out/ab.err
done; done; done
cp /tmp/lib_orig.so paper_2505_16942_b200/libcorrvol_b200.so
