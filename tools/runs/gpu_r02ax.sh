tag=r02ax
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "params_changed" > gpurun_out/${tag}_pytest_poke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_poke.log
timeout 1200 python tools/mutate_gpu.py -k "ignores psub_valid" --out gpurun_out/${tag}_m.json > gpurun_out/${tag}_gpu_mutation.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
