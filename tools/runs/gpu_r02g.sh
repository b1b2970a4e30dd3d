tag=r02g
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1.json 2>gpurun_out/${tag}_timeline_h1.err
ZF_X1_NO_WAITVALUE=1 ZF_TRACE_STEP=1 timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1_nowv.json 2>gpurun_out/${tag}_timeline_h1_nowv.err
