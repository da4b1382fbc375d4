cd ${GRAFT_REPO_ROOT:-.}
timeout 120 python scripts/tc_probe.py > gpurun_out/tc_probe.log 2>&1; echo probe rc $?
cat gpurun_out/tc_probe.log | tail -20
