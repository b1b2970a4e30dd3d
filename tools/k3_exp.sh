# K3 compile-flag experiments on the GPU box: for each config, build, a quick parity subset
# (multi-step zf_step tests, bit-exact vs the oracle), then per-step K3 timings (k3_steps.py)
# at k=10% lr 1e-5 / 1e-3 and k=1% lr 1e-5.
# usage: CFGS="name1:-DFOO=1;name2:-DBAR=2" bash tools/k3_exp.sh <tag> [nopytest]
tag=${1:-exp}
IFS=';' read -ra ALL <<< "${CFGS:-base:}"
mkdir -p gpurun_out
out=gpurun_out/${tag}_k3exp.jsonl
: > $out
for c in "${ALL[@]}"; do
  name=${c%%:*}; flags=${c#*:}
  export ZF_NVCC_EXTRA="$flags"
  python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>gpurun_out/${tag}_${name}_build.err || { echo "{\"cfg\": \"$name\", \"build\": \"failed\"}" >> $out; continue; }
  if [ "$2" != nopytest ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "step and not fullsize and not shard" > gpurun_out/${tag}_${name}_pytest.log 2>&1
    echo "{\"cfg\": \"$name\", \"pytest\": \"$(tail -1 gpurun_out/${tag}_${name}_pytest.log)\"}" >> $out
  fi
  for run in "100000 1e-5" "100000 1e-3" "10000 1e-5"; do
    ZF_OPTS='{"param_subset": true}' timeout 300 python tools/k3_steps.py $run 12 2>/dev/null | grep '^{' | sed "s/^{/{\"cfg\": \"$name\", /" >> $out
  done
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
cat $out | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'steady' in d: print(d['cfg'], d['ppm'], d['lr'], 'refresh %.3f steady %.3f avg %.3f' % (d['refresh'], d['steady'], d['avg']))
    else: print(d)
"
