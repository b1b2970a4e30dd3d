# A/B of K3b compile-time knobs: per-step K3a / K3b times (tools/k3_steps.py).
# usage: CFGS="name1:-DFOO;name2:" bash tools/k3b_flags.sh [ppm] [lr]
IFS=';' read -ra ALL <<< "${CFGS:-base:}"
for c in "${ALL[@]}"; do
  name=${c%%:*}; flags=${c#*:}
  export ZF_NVCC_EXTRA="$flags"
  python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>/tmp/build.err || { echo "build $name failed"; tail -3 /tmp/build.err; continue; }
  ZF_OPTS='{"param_subset": true}' timeout 300 python tools/k3_steps.py ${1:-100000} ${2:-1e-5} 6 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('cfg $name', d['ppm'], d['lr'], 'K3a', d['k3a_ms'][1:4], 'K3b', d['k3b_ms'][1:4], 'avg %.3f' % d['avg'])"
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
