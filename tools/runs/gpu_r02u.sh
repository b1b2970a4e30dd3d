tag=r02u
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python bench.py --shard-of 8 --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --also-cpu-update --refresh-group-mb 0 > gpurun_out/${tag}_bench_7b_shard8_cpu_update.jsonl 2> gpurun_out/${tag}_bench_7b_shard8_cpu_update.err
timeout 900 python bench.py --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --no-e2e --also-state-offload --also-auto 0.15 --refresh-group-mb 0 > gpurun_out/${tag}_bench_7b_f2auto_f3swap.jsonl 2> gpurun_out/${tag}_bench_7b_f2auto_f3swap.err
