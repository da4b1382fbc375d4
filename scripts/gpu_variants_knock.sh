# knockout masks (args) for each prebuilt library variant in ${VARDIR:-variants_tmp}/*/
cd ${GRAFT_REPO_ROOT:-.}
cp paper_2505_16942_b200/libcorrvol_b200.so /tmp/lib_orig.so
for d in ${VARDIR:-variants_tmp}/*/; do
  cp $d/libcorrvol_b200.so paper_2505_16942_b200/libcorrvol_b200.so
  for M in "$@"; do
    CVB_TC_DEBUG=$M timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/var.json 2>gpurun_out/var.err
    python -c "
import json; d=json.load(open('gpurun_out/var.json')); k=d['kernel_ms']
print('$d mask $M', d['value'], 'contract it0 %.3f warm %.3f gather %.3f' % (k['contract_ms'][0], sum(k['contract_ms'][1:])/11, sum(k['gather_ms'])/12))" || tail -3 gpurun_out/var.err
  done
done
cp /tmp/lib_orig.so paper_2505_16942_b200/libcorrvol_b200.so
