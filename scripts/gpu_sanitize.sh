# compute-sanitizer memcheck / racecheck / synccheck over small cases of every kernel family
cd ${GRAFT_REPO_ROOT:-.}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc $?"; grep -E "ERROR SUMMARY|Error|error" gpurun_out/sanitize_$tool.log | head -5
done
