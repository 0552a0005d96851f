#!/bin/bash
# Full bench lines (cpu_baseline, e2e, roofline) for every config and op, one
# JSON line each, into gpurun_out/bench_all_$TAG.jsonl.  Run under gpurun.
TAG="${1:-x}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/bench_all_$TAG.jsonl
: > $out
for c in C1:ax C1:atx C2:ax C2:atx C3:ax C4:ax C4:atx C5:ax; do
  cfg=${c%%:*}; op=${c#*:}
  timeout 900 python bench.py --config $cfg --op $op --steps 10 --warmup 3 --cpu-seconds 8 \
    > gpurun_out/bench_all_${TAG}_${cfg}_${op}.log 2>&1
  tail -1 gpurun_out/bench_all_${TAG}_${cfg}_${op}.log >> $out
  echo "$c rc=$?"
done
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
echo "default rc=$?"
