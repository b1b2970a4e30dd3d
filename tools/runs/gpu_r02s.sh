tag=r02s
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
for run in "100000 1e-5" "100000 1e-3" "10000 1e-5"; do
ZF_OPTS='{"param_subset": true};{"param_subset": false}' timeout 600 python tools/k3_steps.py $run 12 2>/dev/null | grep '^{' >> gpurun_out/${tag}_psub.jsonl
done
