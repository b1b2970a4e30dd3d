tag=r02av
bash tools/gpu_round2.sh $tag
ZF_RANDOM_MR_SEEDS=30 timeout 2400 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_mr30.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_mr30.log
