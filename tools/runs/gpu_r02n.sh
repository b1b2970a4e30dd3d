tag=r02n
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
SECONDS=0; timeout 1200 python bench.py --no-k1pct --no-lr1e3 --no-lagged --no-cpu-baseline > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err; echo "wall_s=$SECONDS" >> gpurun_out/${tag}_bench_7b.err
SECONDS=0; timeout 1200 python bench.py > gpurun_out/${tag}_bench_7b_full.jsonl 2> gpurun_out/${tag}_bench_7b_full.err; echo "wall_s=$SECONDS" >> gpurun_out/${tag}_bench_7b_full.err
