tag=r02ar
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_RANDOM_MR_SEEDS=40 timeout 2400 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_mr40.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_mr40.log
