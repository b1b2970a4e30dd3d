tag=r02an
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
for k in "k_patch" "remap step delta" "H1 one-step" "warm-up one step" "K6 sums squared" "X1 copy gated"; do
  timeout 1200 python tools/mutate_gpu.py -k "$k" --out gpurun_out/${tag}_m_$(echo $k | tr ' ' '_').json >> gpurun_out/${tag}_gpu_mutation.log 2>&1
done
