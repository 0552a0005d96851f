#!/bin/bash
# Kernel-time sweep of environment knobs under gpurun:
#   tools/knobs.sh "<ENV=V[,ENV2=V2] ...|base>" "<cfg[:atx] ...>"
COMBOS="$1"; CFGS="$2"
python -c "import __graft_entry__ as g; g.build()" || exit 1
for combo in $COMBOS; do
  envs=""; [ "$combo" != "base" ] && envs=$(echo $combo | tr ',' ' ')
  for c in $CFGS; do
    cfg=${c%%:*}; op=ax; [[ "$c" == *:atx ]] && op=atx
    env $envs timeout 300 python bench.py --config $cfg --op $op --steps 10 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/k.log 2>&1
    echo "$combo $c $(python -c "import json; d=json.loads(open('gpurun_out/k.log').read().strip().splitlines()[-1]); print('%.4f' % d['roofline']['kernel_ms'])" 2>&1 | tail -1)"
  done
done
