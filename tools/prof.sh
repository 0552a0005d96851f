#!/bin/bash
# Profiling pass under gpurun: full ncu capture of one kernel per (config, op,
# kernel regex) triple, text summaries written into gpurun_out/ (reports kept
# in /tmp/prof on the box; copied back only while gpurun_out stays small),
# and the launch list of the default bench.
#   tools/prof.sh <tag> "C2:ax:spmv_sell C4:ax:spmv_wrow ..." [LL]
TAG="$1"; SPECS="$2"; LL="${3:-}"
mkdir -p gpurun_out /tmp/prof
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
for s in $SPECS; do
  IFS=: read cfg op rx <<< "$s"
  CMD="python bench.py --config $cfg --op $op --steps 2 --warmup 1 --no-cpu --no-e2e --no-per-config"
  rep=/tmp/prof/prof_${TAG}_${cfg}_${op}_${rx}
  timeout 600 $CMD > gpurun_out/plain_${TAG}_${cfg}_${op}.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 \
      -o $rep $CMD > gpurun_out/ncu_${TAG}_${cfg}_${op}_${rx}.log 2>&1
  echo "ncu $s rc=$?"
  if [ -f $rep.ncu-rep ]; then
    python tools/ncu_summary.py $rep.ncu-rep "$cfg $op $rx" > gpurun_out/sum_${TAG}_${cfg}_${op}_${rx}.txt 2>&1
    python tools/ncu_lines.py $rep.ncu-rep 60 > gpurun_out/lines_${TAG}_${cfg}_${op}_${rx}.txt 2>&1
    python tools/ncu_opmix.py $rep.ncu-rep > gpurun_out/opmix_${TAG}_${cfg}_${op}_${rx}.txt 2>&1
    sz=$(du -sm gpurun_out | cut -f1)
    rsz=$(du -sm $rep.ncu-rep | cut -f1)
    if [ $((sz + rsz)) -lt 55 ]; then cp $rep.ncu-rep gpurun_out/; fi
  fi
done
if [ -n "$LL" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config"
  timeout 600 $CMD > gpurun_out/plain_${TAG}_ll.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_ll_${TAG}.log 2>&1
  echo "launchlist rc=$?"
fi
