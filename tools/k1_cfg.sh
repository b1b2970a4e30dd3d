# K1 variants (rows per block, rows in flight, threads), live timing of the K1 phase (refresh every step).
IFS=';' read -ra ALL <<< "${CFGS:-base:}"
for c in "${ALL[@]}"; do
  name=${c%%:*}; flags=${c#*:}
  export ZF_NVCC_EXTRA="$flags"
  python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>/tmp/build.err || { echo "build $name failed"; continue; }
  timeout 150 python bench.py --refresh 1 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('cfg $name', round(d['phases_ms_per_launch']['k1_norms'],4), round(d['k1_roofline']['frac'],3))" || tail -3 /tmp/b.err
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
