# Time K3 variants built with extra nvcc flags.  The bench process gets the same
# ZF_NVCC_EXTRA (bench.py calls _build.build(), which rebuilds when the flags differ).
# usage: CFGS="name1:-DFOO=1 -DBAR=2;name2:" bash tools/k3_cfg.sh
IFS=';' read -ra ALL <<< "${CFGS:-base:}"
for c in "${ALL[@]}"; do
  name=${c%%:*}; flags=${c#*:}
  export ZF_NVCC_EXTRA="$flags"
  python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>/tmp/build.err || { echo "build $name failed"; tail -3 /tmp/build.err; continue; }
  timeout 150 python bench.py --steps ${STEPS:-10} --warmup 4 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('cfg $name', round(d['ms_per_step'],3), round(d['phases_ms_per_launch']['k3_update'],3))" || tail -3 /tmp/b.err
  grep "k3 prof" /tmp/b.err | tail -1
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
