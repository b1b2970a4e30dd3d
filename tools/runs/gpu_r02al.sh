tag=r02al
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "nonfinite_on or waits_for" > gpurun_out/${tag}_pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_new.log
timeout 900 python tools/mutate_gpu.py -k "lagged refresh" --out gpurun_out/${tag}_m1.json > gpurun_out/${tag}_gpu_mutation.log 2>&1
timeout 900 python tools/mutate_gpu.py -k "K3 AdamW non-finite" --out gpurun_out/${tag}_m2.json >> gpurun_out/${tag}_gpu_mutation.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
bash tools/runs/gpu_r02ak.sh
