#!/bin/bash
# Profiling pass under gpurun: full ncu capture of one kernel per (config, op,
# kernel regex) triple and the launch list of the default bench.
#   tools/prof.sh <tag> "C2:ax:spmv_sell C4:ax:spmv_long ..." [launchlist]
TAG="$1"; SPECS="$2"; LL="${3:-}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for s in $SPECS; do
  IFS=: read cfg op rx <<< "$s"
  CMD="python bench.py --config $cfg --op $op --steps 2 --warmup 1 --no-cpu --no-e2e --no-per-config"
  timeout 600 $CMD > gpurun_out/plain_${TAG}_${cfg}_${op}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${cfg}_${op}_${rx} $CMD > gpurun_out/ncu_${TAG}_${cfg}_${op}_${rx}.log 2>&1
  echo "ncu $s rc=$?"
done
if [ -n "$LL" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config"
  timeout 600 $CMD > gpurun_out/plain_${TAG}_ll.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_ll_${TAG}.log 2>&1
  echo "launchlist rc=$?"
fi
