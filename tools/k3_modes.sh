python -m paper_2505_12242_b200._build >/dev/null
for m in ${MODES:-0 1 2 3}; do
ZF_K3_DEBUG_MODE=$m python bench.py --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', d['ms_per_step'], d['phases_ms_per_launch']['k3_update'])"
done
