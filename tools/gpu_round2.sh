# On the GPU box: tests + bench + ncu evidence for one tag.  usage: bash tools/gpu_round2.sh <tag> [quick]
#  1. pytest -m gpu, smoke()
#  2. default bench line (7B k=10% + k=1% + lr 1e-3 + lagged), 2 co-located ranks
#  3. ncu launch list of the default bench command; full K3 captures (7B k=10%, 7B k=1%, GPT-2)
#  4. GPT-2 / 13B / dp8-shard bench lines
tag=${1:-r02a}
mode=${2:-full}
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
timeout 600 python bench.py --gpus 2 --colocate --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_7b_colocate2.jsonl 2> gpurun_out/${tag}_bench_7b_colocate2.err
timeout 600 python bench.py --gpus 2 --colocate --exchange peer --no-cpu-baseline --no-e2e --no-k1pct --no-lr1e3 --no-lagged > gpurun_out/${tag}_bench_7b_colocate2_peer.jsonl 2> gpurun_out/${tag}_bench_7b_colocate2_peer.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.jsonl 2> gpurun_out/${tag}_bench_reference.err
[ "$mode" = quick ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_(update|column_norms|topk|scatter|accumulate|zen_auto|adam)" \
    --log-file gpurun_out/${tag}_launches_7b.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --refresh-group-mb 0 \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
for spec in "7b_k10:--ratio-ppm 100000" "7b_k1:--ratio-ppm 10000" "gpt2_k10:--model gpt2-small"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout 1300 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 \
      -o gpurun_out/${tag}_k3_${name} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --refresh-group-mb 0 $args \
      > gpurun_out/${tag}_k3_${name}.log 2>&1
  ncu -i gpurun_out/${tag}_k3_${name}.ncu-rep --page details > gpurun_out/${tag}_k3_${name}.txt 2>&1
  ncu -i gpurun_out/${tag}_k3_${name}.ncu-rep --page raw --csv > gpurun_out/${tag}_k3_${name}_raw.csv 2>&1
done
timeout 300 python bench.py --model gpt2-small --no-e2e --no-lagged --steps 4000 > gpurun_out/${tag}_bench_gpt2.jsonl 2> gpurun_out/${tag}_bench_gpt2.err
timeout 600 python bench.py --model llama2-13b --no-cpu-baseline > gpurun_out/${tag}_bench_13b.jsonl 2> gpurun_out/${tag}_bench_13b.err
timeout 600 python bench.py --model llama2-13b --shard-of 8 --no-cpu-baseline --no-lagged --steps 300 > gpurun_out/${tag}_bench_13b_shard8.jsonl 2> gpurun_out/${tag}_bench_13b_shard8.err
timeout 600 python bench.py --shard-of 8 --no-cpu-baseline --no-lagged --steps 600 > gpurun_out/${tag}_bench_7b_shard8.jsonl 2> gpurun_out/${tag}_bench_7b_shard8.err
rm -f gpurun_out/*.ncu-rep.tmp
du -sh gpurun_out
