tag=r02l
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
NCCL_DEBUG=INFO timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k nccl_one_rank -s > gpurun_out/${tag}_nccl_one_rank.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.jsonl 2> gpurun_out/${tag}_bench_reference.err
timeout 300 python bench.py --model gpt2-small --no-e2e --no-lagged --steps 4000 > gpurun_out/${tag}_bench_gpt2.jsonl 2> gpurun_out/${tag}_bench_gpt2.err
timeout 600 python bench.py --model llama2-13b --shard-of 8 --no-cpu-baseline --no-lagged --steps 300 > gpurun_out/${tag}_bench_13b_shard8.jsonl 2> gpurun_out/${tag}_bench_13b_shard8.err
timeout 600 python bench.py --shard-of 8 --no-cpu-baseline --no-lagged --steps 600 > gpurun_out/${tag}_bench_7b_shard8.jsonl 2> gpurun_out/${tag}_bench_7b_shard8.err
