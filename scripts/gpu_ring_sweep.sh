cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in partial256 dense64; do
  timeout 900 $CS --tool racecheck python scripts/sanitize_ring.py $c > gpurun_out/race_$c.log 2>&1; echo race $c rc $?
  grep -E "RACECHECK SUMMARY" gpurun_out/race_$c.log
done
VARDIR=variants_tmp bash scripts/gpu_variants.sh
VARDIR=variants_tmp bash scripts/gpu_variants.sh
