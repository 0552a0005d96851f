python -c "import __graft_entry__ as g; g.build()"
for T in 32 64 128 256 1000; do
  MPSP_LONG_T=$T timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_T$T.log 2>&1
  echo "T=$T $(python -c "import json; d=json.loads(open('gpurun_out/sw_T$T.log').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'])")"
done
for M in 1 6; do for c in C2 C4:atx; do cfg=${c%%:*}; op=ax; [[ "$c" == *:atx ]] && op=atx
  MPSP_MINB=$M timeout 300 python bench.py --config $cfg --op $op --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_M${M}_$cfg$op.log 2>&1
  echo "MINB=$M $c $(python -c "import json; d=json.loads(open('gpurun_out/sw_M${M}_$cfg$op.log').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'])")"
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k tie_prone 2>&1 | tail -2
