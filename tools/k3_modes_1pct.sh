# K3 phase ceilings at k = 1% (debug modes: 0 full, 1 stream stages only, 2 no AdamW, 3 no compaction)
python -m paper_2505_12242_b200._build >/dev/null
for m in 0 1 2 3; do
ZF_K3_DEBUG_MODE=$m timeout 300 python bench.py --ratio-ppm 10000 --steps 12 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mode $m', round(d['ms_per_step'],3), 'k3', round(d['phases_ms_per_launch']['k3_update'],3), 'k1', round(d['phases_ms_per_launch']['k1_norms'],3), 'sectorGBs', round(r['achieved_sector_GBs']))"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_update -s 3 -c 1 python bench.py --ratio-ppm 10000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '"k_update\|k_update' | tr ',' ' ' | awk '{print $(NF-2), $NF}'
