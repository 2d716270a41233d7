bash scripts/gpu_quick.sh
bash scripts/gpu_ab2.sh
