tag=r02i
mkdir -p gpurun_out
export ZF_NVCC_EXTRA="-DZF_K3_PROF"
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" > gpurun_out/${tag}_build.log 2>&1
for run in "100000 1e-5" "10000 1e-5"; do
ZF_K3_PROF_PRINT=1 ZF_OPTS='{"param_subset": true}' timeout 300 python tools/k3_steps.py $run 8 >> gpurun_out/${tag}_k3prof.log 2>&1
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>&1
