tag=r02d
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 300 python tools/e2e_timeline.py 0 8 12 > gpurun_out/${tag}_timeline_h1.json 2>gpurun_out/${tag}_timeline.err
timeout 300 python tools/e2e_timeline.py 1 0 12 > gpurun_out/${tag}_timeline_k7.json 2>>gpurun_out/${tag}_timeline.err
CFGS='base:;sleep32:-DZF_MBAR_SLEEP_NS=32;sleep128:-DZF_MBAR_SLEEP_NS=128;sleep512:-DZF_MBAR_SLEEP_NS=512' bash tools/k3_exp.sh ${tag}e nopytest
