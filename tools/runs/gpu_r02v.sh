tag=r02v
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 1 0 12 > gpurun_out/${tag}_timeline_k7.json 2>gpurun_out/${tag}_timeline_k7.err
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1.json 2>gpurun_out/${tag}_timeline_h1.err
timeout 900 python bench.py --no-cpu-baseline --no-k1pct --no-lr1e3 --no-lagged --no-e2e --also-auto 0.15 --refresh-group-mb 0 > gpurun_out/${tag}_bench_7b_auto.jsonl 2> gpurun_out/${tag}_bench_7b_auto.err
