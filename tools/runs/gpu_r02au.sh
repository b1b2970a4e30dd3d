tag=r02au
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
ZF_RANDOM_SEEDS=1000 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_configurations > gpurun_out/${tag}_pytest_random1000.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_random1000.log
CFGS="rs1:;rs0:-DZF_REFRESH_SUBSET=0;rs1b:-DZF_REFRESH_SUBSET=1;rs0b:-DZF_REFRESH_SUBSET=0 -DZF_X=1" bash tools/k3_exp.sh $tag nopytest > gpurun_out/${tag}_k3exp_summary.txt 2>&1
