TESTS="tests/test_gpu_configs.py tests/test_gpu_fullsize.py" bash scripts/gpu_ab.sh 4
