mkdir -p gpurun_out /tmp/prof
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
CMD="python bench.py --config C2 --p 2048 --op ax --steps 2 --warmup 1 --no-cpu --no-e2e --no-per-config"
rep=/tmp/prof/prof_w2048
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:spmv_wide -s 1 -c 1 -o $rep $CMD > gpurun_out/ncu_w2048.log 2>&1
echo ncu=$?
python tools/ncu_summary.py $rep.ncu-rep "C2@p2048 ax spmv_wide" > gpurun_out/sum_w2048.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 50 > gpurun_out/lines_w2048.txt 2>&1
python tools/ncu_opmix.py $rep.ncu-rep > gpurun_out/opmix_w2048.txt 2>&1
