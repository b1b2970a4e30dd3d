# Per-launch K3 time + DRAM bytes (+ L2 sectors, instructions) on the Llama-2-7B bench
# workload (ncu, application-only: the bench's nvidia-smi sampler is not profiled).
# usage: bash tools/ncu_k3_traffic.sh <tag> [extra bench args]
tag=${1:-k3traffic}; shift
python -m paper_2505_12242_b200._build >/dev/null
timeout 900 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__inst_executed.sum \
  --clock-control none --csv -k regex:"k_update|k_adam" -s 3 -c 8 --log-file gpurun_out/${tag}.csv \
  python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-k1pct --no-lr1e3 "$@" > gpurun_out/${tag}.log 2>&1
