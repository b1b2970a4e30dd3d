tag=r02c
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/${tag}_pytest_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_multirank.log
timeout 900 python bench.py --no-k1pct --no-lr1e3 --no-lagged --no-cpu-baseline > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
timeout 900 python bench.py --gpus 2 --colocate --no-k1pct --no-lr1e3 --no-lagged --no-cpu-baseline > gpurun_out/${tag}_bench_7b_colocate2.jsonl 2> gpurun_out/${tag}_bench_7b_colocate2.err
timeout 600 python tools/retention_sweep.py --out gpurun_out/${tag}_retention.json > gpurun_out/${tag}_retention.log 2>&1
