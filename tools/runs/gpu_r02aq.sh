tag=r02aq
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_RANDOM_SEEDS=1500 timeout 3000 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_random1500.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_random1500.log
