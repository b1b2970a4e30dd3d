tag=r02f
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1.json 2>gpurun_out/${tag}_timeline_h1.err
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 4 12 > gpurun_out/${tag}_timeline_h1s4.json 2>gpurun_out/${tag}_timeline_h1s4.err
timeout 1200 python bench.py > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err
