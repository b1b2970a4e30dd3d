# On the GPU box: the round's evidence.  usage: bash tools/profile_round.sh <tag>
#  1. launch list of the default bench command (ncu: per-launch time + DRAM bytes)
#  2. one full ncu capture of K3 (the dominant kernel)
#  3. bench lines: default (7B k=10%, + k=1%, + f3 state swap, + Zen-auto), GPT-2, 13B,
#     and rank 0's shard of the 8-GPU 13B config with offload (per-rank e2e)
tag=${1:-r01}
python -m paper_2505_12242_b200._build >/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_(update|column_norms|topk|scatter|accumulate|zen_auto)" \
    --log-file gpurun_out/${tag}_launches_7b.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 1300 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 \
    -o gpurun_out/${tag}_k3_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_k3_full.log 2>&1
ncu -i gpurun_out/${tag}_k3_full.ncu-rep --page details > gpurun_out/${tag}_k3_full.txt 2>&1
ncu -i gpurun_out/${tag}_k3_full.ncu-rep --page raw --csv > gpurun_out/${tag}_k3_full_raw.csv 2>&1
timeout 900 python bench.py --also-k1pct --also-state-offload --also-auto 0.15 > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
timeout 300 python bench.py --model gpt2-small --no-e2e > gpurun_out/${tag}_bench_gpt2.jsonl 2> gpurun_out/${tag}_bench_gpt2.err
timeout 600 python bench.py --model llama2-13b --no-cpu-baseline > gpurun_out/${tag}_bench_13b.jsonl 2> gpurun_out/${tag}_bench_13b.err
timeout 600 python bench.py --model llama2-13b --shard-of 8 --no-cpu-baseline > gpurun_out/${tag}_bench_13b_shard8.jsonl 2> gpurun_out/${tag}_bench_13b_shard8.err
timeout 600 python bench.py --shard-of 8 --no-cpu-baseline > gpurun_out/${tag}_bench_7b_shard8.jsonl 2> gpurun_out/${tag}_bench_7b_shard8.err
tail -c 300 gpurun_out/${tag}_bench_7b.jsonl
