tag=r02b
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
gcc -O3 -march=native -fopenmp tools/host_membw.c -o /tmp/hm && /tmp/hm 4 16 > gpurun_out/${tag}_host_membw.json; /tmp/hm 4 8 >> gpurun_out/${tag}_host_membw.json
timeout 900 python bench.py --no-k1pct --no-lr1e3 --no-lagged --no-cpu-baseline > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
CFGS='base:;cpair:-DZF_K3_CPAIR=1' bash tools/k3_exp.sh ${tag}e
