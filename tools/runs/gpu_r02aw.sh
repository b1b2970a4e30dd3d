tag=r02aw
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 3000 python tools/mutate_gpu.py -k "subset" --out gpurun_out/${tag}_gpu_mutation.json > gpurun_out/${tag}_gpu_mutation.log 2>&1
