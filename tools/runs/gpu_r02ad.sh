tag=r02ad
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
SECONDS=0; timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_bench_reference.jsonl 2> gpurun_out/${tag}_bench_reference.err; echo "wall_s=$SECONDS" >> gpurun_out/${tag}_bench_reference.err
SECONDS=0; timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${tag}_bench_7b.jsonl 2> gpurun_out/${tag}_bench_7b.err; echo "wall_s=$SECONDS" >> gpurun_out/${tag}_bench_7b.err
