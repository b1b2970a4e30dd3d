# Experiment: does writing back partial p sectors without having read them cost DRAM reads?
# mode 0 = normal, mode 4 = p tile never read (garbage results).  ncu DRAM bytes + live timing.
python -m paper_2505_12242_b200._build >/dev/null
for m in ${MODES:-0 4}; do
  ZF_K3_DEBUG_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_update -s 3 -c 2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ptraffic_ncu_$m.csv 2>&1
  ZF_K3_DEBUG_MODE=$m timeout 300 python bench.py --steps 8 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', d['ms_per_step'], d['phases_ms_per_launch']['k3_update'])"
done
grep -h "k_update" gpurun_out/ptraffic_ncu_*.csv | cut -c1-400
