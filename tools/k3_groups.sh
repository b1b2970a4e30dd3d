for g in ${GROUPS_LIST:-1 2}; do
  ZF_NVCC_EXTRA="-DZF_K3_GROUPS=$g" python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
  python bench.py --steps 10 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('groups $g', d['ms_per_step'], d['phases_ms_per_launch']['k3_update'])"
done
