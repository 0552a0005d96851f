#!/bin/bash
# Kernel-time sweep over env knobs: tools/sweep_knobs.sh "<cfg[:atx]> ..." "<VAR=a,b ...>" tag
# e.g. tools/sweep_knobs.sh "C2 C3" "MPSP_PD=1,2 MPSP_MINB=1,4" s1
CFGS="$1"; KNOBS="$2"; TAG="${3:-k}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
combos=("")
for kv in $KNOBS; do
  var=${kv%%=*}; vals=${kv#*=}; new=()
  for c in "${combos[@]}"; do for v in ${vals//,/ }; do new+=("$c $var=$v"); done; done
  combos=("${new[@]}")
done
for c in $CFGS; do
  cfg=${c%%:*}; op=ax; [[ "$c" == *:atx ]] && op=atx
  for combo in "${combos[@]}"; do
    log=gpurun_out/sweep_${TAG}.log
    env $combo timeout 300 python bench.py --config $cfg --op $op --steps 10 --warmup 3 --no-cpu --no-e2e --no-per-config > $log 2>&1
    echo "$c [$combo ] $(python -c "import json; d=json.loads(open('$log').read().strip().splitlines()[-1]); r=d['roofline']; print('kern_ms=%.4f frac=%.3f' % (r['kernel_ms'], r['frac_of_t_roof']))" 2>&1 | tail -1)"
  done
done
