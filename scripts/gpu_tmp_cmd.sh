timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_plan.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_plan.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plan_kernel --csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/plan_ncu.csv 2>&1
grep gpu__time gpurun_out/plan_ncu.csv | awk -F'","' '{print $NF}' | tr -d '"' | tail -12 | tr '\n' ' '; echo
bash scripts/gpu_ab.sh 3
