tag=r02ag
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${tag}_pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_parity.log
CFGS="perm1:;perm0:-DZF_K3_PERM=0;perm1b:-DZF_K3_PERM=1 -DZF_K3_PERM_B=1;perm0b:-DZF_K3_PERM=0 -DZF_K3_PERM_B=1" bash tools/k3_exp.sh $tag nopytest > gpurun_out/${tag}_k3exp_summary.txt 2>&1
