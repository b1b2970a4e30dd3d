tag=r02ak
mkdir -p gpurun_out
python -m paper_2505_12242_b200._build > gpurun_out/${tag}_build.log 2>&1
timeout 300 python tools/sanitize.py > gpurun_out/${tag}_sanitize_plain.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_sanitize_plain.log
for tool in memcheck synccheck; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/${tag}_sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_sanitize_$tool.log
done
timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/${tag}_sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_sanitize_racecheck.log
