#!/bin/bash
# Bench prebuilt tuning variants (paper_1411_2377_b200/<name>.so, built here by
#   python -m paper_1411_2377_b200._build --name=<name>.so -D...)
# on the given configs.  Run under gpurun from the repo root.
#   tools/variants.sh "<name1 name2 ...>" "<cfg[:atx] ...>" <tag>
VARS="$1"; CFGS="$2"; TAG="${3:-v}"
mkdir -p gpurun_out
for v in $VARS; do
  for c in $CFGS; do
    cfg=${c%%:*}; op=ax; [[ "$c" == *:atx ]] && op=atx
    log=gpurun_out/var_${TAG}_${v}_${cfg}_${op}.log
    MPSP_LIB=$v.so timeout 600 python bench.py --config $cfg --op $op --steps 10 --warmup 3 --no-cpu --no-e2e --no-per-config > $log 2>&1
    echo "$v $c rc=$? $(python -c "import json; d=json.loads(open('$log').read().strip().splitlines()[-1]); r=d['roofline']; print('kern_ms=%.4f frac=%.3f MACs=%.2fT' % (r['kernel_ms'], r['frac_of_t_roof'], r['macs_achieved_T']))" 2>&1 | tail -1)"
  done
done
