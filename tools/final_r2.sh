#!/bin/bash
# Round-2 final measurement pass (run under gpurun from the repo root):
# smoke, GPU tests, default bench line, launch list, ncu summaries of the C5
# and C2 SpMV kernels, and a bounded fuzz sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/m2_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/m2_pytest.log 2>&1; echo "pytest=$? $(tail -1 gpurun_out/m2_pytest.log)"
timeout 600 python bench.py > gpurun_out/m2_bench.json 2> gpurun_out/m2_bench.err; echo bench=$?
bash tools/prof.sh r2m "C5:ax:spmv_sell" LL > gpurun_out/m2_prof.log 2>&1; echo prof=$?; cat gpurun_out/m2_prof.log
timeout 420 python tools/fuzz.py 360 $RANDOM > gpurun_out/m2_fuzz.log 2>&1; echo "fuzz=$? $(tail -2 gpurun_out/m2_fuzz.log)"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m2_bench_ref.json 2> gpurun_out/m2_bench_ref.err; echo ref=$?
