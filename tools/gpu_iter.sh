#!/bin/bash
# One GPU iteration: parity tests, benches for the given configs, optional ncu
# capture of the spmv kernel on one config.  Run under gpurun from the repo root.
#   tools/gpu_iter.sh "<pytest -k expr or ALL|NONE>" "<configs>" "<ncu config or NONE>" <tag>
K="$1"; CFGS="$2"; NCU="$3"; TAG="${4:-x}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ "$K" != "NONE" ]; then
  if [ "$K" == "ALL" ]; then timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1
  else timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; fi
  echo "pytest=$? $(tail -1 gpurun_out/pytest_$TAG.log)"
fi
for c in $CFGS; do
  cfg=${c%%:*}; op=ax; [[ "$c" == *:atx ]] && op=atx
  timeout 600 python bench.py --config $cfg --op $op --steps 10 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/bench_${TAG}_${cfg}_${op}.log 2>&1
  echo "bench $c rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${TAG}_${cfg}_${op}.log').read().strip().splitlines()[-1]); r=d['roofline']; print('kern_ms=%.4f t_roof_ms=%.4f frac=%.3f bound=%s MACs=%.2fT GB/s=%.0f sm=%s' % (r['kernel_ms'], r['t_roof_ms'], r['frac_of_t_roof'], r['bound'], r['macs_achieved_T'], r['hbm_achieved_gbs'], d['clocks']['sm_mhz']))" 2>&1 | tail -1)"
done
if [ "$NCU" != "NONE" ]; then
  cfg=${NCU%%:*}; op=ax; [[ "$NCU" == *:atx ]] && op=atx
  CMD="python bench.py --config $cfg --op $op --steps 2 --warmup 1 --no-cpu --no-e2e --no-per-config"
  timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu=$?"
fi
