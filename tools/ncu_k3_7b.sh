# Full ncu capture of one K3 launch on the Llama-2-7B bench workload (one GPU).
# usage: bash tools/ncu_k3_7b.sh <tag>
tag=${1:-k3}
python -m paper_2505_12242_b200._build >/dev/null
timeout 1300 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 \
  -o gpurun_out/${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page details > gpurun_out/${tag}.txt 2>&1
tail -2 gpurun_out/${tag}.log
