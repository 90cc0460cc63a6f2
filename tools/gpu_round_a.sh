bash tools/gpu_k1c_tune.sh
bash tools/ab_k2.sh
