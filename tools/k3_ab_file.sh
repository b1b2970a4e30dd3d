# A/B of two K3 sources on the same box: copy the baseline to tools/_k_update_base.cu.txt first (the box has no .git), then run.
run() {
  for args in "" "--ratio-ppm 10000" "--model llama2-13b"; do
    timeout 300 python bench.py $args --steps 12 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_launch']; print('$1', '$args', round(d['ms_per_step'],4), 'k3', round(p['k3_update'],4))"
  done
}
cp paper_2505_12242_b200/csrc/k_update.cu /tmp/k_update_new.cu
cp tools/_k_update_base.cu.txt paper_2505_12242_b200/csrc/k_update.cu
python -m paper_2505_12242_b200._build >/dev/null; run base
cp /tmp/k_update_new.cu paper_2505_12242_b200/csrc/k_update.cu
python -m paper_2505_12242_b200._build >/dev/null; run new
