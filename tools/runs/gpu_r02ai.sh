tag=r02ai
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "past_the" > gpurun_out/${tag}_pytest_tables.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_tables.log
timeout 900 python tools/mutate_gpu.py -k "bias correction past the table" --out gpurun_out/${tag}_gpu_mutation_tables.json > gpurun_out/${tag}_gpu_mutation_tables.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
