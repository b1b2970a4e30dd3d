tag=r02p
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
for mb in 32 64 128 256; do
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --refresh-group-mb $mb > gpurun_out/${tag}_bench_rg$mb.jsonl 2> gpurun_out/${tag}_bench_rg$mb.err
done
