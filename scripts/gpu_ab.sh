# A/B of prebuilt library variants in abvar/*/ (swapped in place), alternating.
# usage (GPU box): bash scripts/gpu_ab.sh [reps] ; with TESTS="tests/..." also runs those gpu tests per variant
cd ${GRAFT_REPO_ROOT:-.}
cp paper_2505_16942_b200/libcorrvol_b200.so /tmp/lib_orig.so
if [ -n "$TESTS" ]; then
for d in abvar/*/; do
  cp $d/libcorrvol_b200.so paper_2505_16942_b200/libcorrvol_b200.so
  timeout 900 python -m pytest $TESTS -m gpu -x -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "$d pytest rc $?"; tail -3 gpurun_out/ab_tests.log
done
fi
for rep in $(seq ${1:-2}); do
for d in abvar/*/; do
  cp $d/libcorrvol_b200.so paper_2505_16942_b200/libcorrvol_b200.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json,statistics; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernel_ms']
print('$d', d['value'], 'contract it0 %.3f warm %.4f gather %.4f' % (k['contract_ms'][0], statistics.mean(k['contract_ms'][1:]), statistics.mean(k['gather_ms'][1:])))" || tail -3 gpurun_out/ab.err
done; done
cp /tmp/lib_orig.so paper_2505_16942_b200/libcorrvol_b200.so
