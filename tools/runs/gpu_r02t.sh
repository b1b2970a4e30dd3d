tag=r02t
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
ZF_REFRESH_PTILE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "step and not fullsize and not shard" > gpurun_out/${tag}_pytest.log 2>&1; tail -1 gpurun_out/${tag}_pytest.log >> gpurun_out/${tag}_pytest.log
for env in 1 0; do
for run in "100000 1e-5" "100000 1e-3" "10000 1e-5"; do
ZF_REFRESH_PTILE=$env ZF_OPTS='{"param_subset": true}' timeout 600 python tools/k3_steps.py $run 12 2>/dev/null | grep '^{' | sed "s/^{/{\"ptile\": $env, /" >> gpurun_out/${tag}_k3.jsonl
done
done
