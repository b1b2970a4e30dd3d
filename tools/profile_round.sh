# On the GPU box: launch list (ncu) + full default bench lines.  usage: bash tools/profile_round.sh <tag>
tag=${1:-r01}
python -m paper_2505_12242_b200._build >/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"k_(update|column_norms|topk|scatter)" --log-file gpurun_out/${tag}_launches_7b.csv python bench.py --steps 4 --warmup 2 --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS:---also-k1pct} > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
timeout 300 python bench.py --model gpt2-small --no-e2e > gpurun_out/${tag}_bench_gpt2.jsonl 2> gpurun_out/${tag}_bench_gpt2.err
tail -c 400 gpurun_out/${tag}_bench_7b.jsonl
