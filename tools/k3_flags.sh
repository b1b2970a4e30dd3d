# A/B of K3 compile-time knobs on the per-step K3 timing harness (tools/k3_steps.py).
# usage: CFGS="name1:-DFOO=1;name2:-DBAR=2" bash tools/k3_flags.sh [ppm] [lr]
IFS=';' read -ra ALL <<< "${CFGS:-base:}"
for c in "${ALL[@]}"; do
  name=${c%%:*}; flags=${c#*:}
  export ZF_NVCC_EXTRA="$flags"
  python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null 2>/tmp/build.err || { echo "build $name failed"; tail -3 /tmp/build.err; continue; }
  ZF_OPTS='{"param_subset": true}' timeout 300 python tools/k3_steps.py ${1:-100000} ${2:-1e-5} 8 2>&1 | sed "s/^/cfg $name /" | grep -v Warn
done
unset ZF_NVCC_EXTRA
python -c "from paper_2505_12242_b200 import _build; _build.build(force=True)" >/dev/null
