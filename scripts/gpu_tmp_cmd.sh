TESTS="tests/test_gpu_configs.py tests/test_gpu_parity.py" bash scripts/gpu_ab.sh 3
