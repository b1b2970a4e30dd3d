tag=r02as
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_RANDOM_MR_SEEDS=60 timeout 2400 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_mr60.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_mr60.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
