bash tools/gpu_round2.sh r02am
