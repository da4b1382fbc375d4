bash scripts/gpu_ab.sh 3
