tag=r02aa
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 600 python bench.py --gpus 2 --colocate --no-cpu-baseline --no-e2e --no-k1pct --no-lr1e3 --no-lagged > gpurun_out/${tag}_bench_colocate2.jsonl 2> gpurun_out/${tag}_bench_colocate2.err
timeout 600 python bench.py --gpus 3 --colocate --exchange peer --no-cpu-baseline --no-e2e --no-k1pct --no-lr1e3 --no-lagged --model gpt2-small > gpurun_out/${tag}_bench_colocate3_peer_gpt2.jsonl 2> gpurun_out/${tag}_bench_colocate3_peer_gpt2.err
