# A/B of the K3 unit shape rule: ZF_K3_GEOM=rows (full rows, else single-row segments) vs the
# default search (R rows x c columns with the fewest units).
python -m paper_2505_12242_b200._build >/dev/null
for geo in rows auto; do
  for args in "--model llama2-13b" "--ratio-ppm 10000" ""; do
    ZF_K3_GEOM=$geo timeout 300 python bench.py $args --steps 12 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$geo', '$args', round(d['ms_per_step'],3), 'k3', round(d['phases_ms_per_launch']['k3_update'],3), 'sec', round(d['roofline']['frac_sector'],3))"
  done
done
