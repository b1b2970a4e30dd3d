tag=r02h
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1.json 2>gpurun_out/${tag}_timeline_h1.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 1200 python bench.py --no-k1pct --no-lr1e3 --no-lagged --no-cpu-baseline > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
