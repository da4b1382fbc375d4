TESTS="tests/test_gpu_configs.py" bash scripts/gpu_ab.sh 3
