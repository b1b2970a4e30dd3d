tag=r02aj
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
for k in "peer reduce" "peer gather" "lagged refresh" "non-finite" "dense AdamW" "K6 smax" "K7 Zen-auto" "f1 refresh gather"; do
  timeout 1200 python tools/mutate_gpu.py -k "$k" --out gpurun_out/${tag}_m_$(echo $k | tr ' ' '_').json >> gpurun_out/${tag}_gpu_mutation.log 2>&1
done
