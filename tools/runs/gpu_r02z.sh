tag=r02z
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random > gpurun_out/${tag}_pytest_random.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_random.log
