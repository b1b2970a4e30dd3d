tag=r02ay
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_RANDOM_SEEDS=2000 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_random2000.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_random2000.log
ZF_RANDOM_MR_SEEDS=100 timeout 2400 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_mr100.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_mr100.log
