#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full captures of the GEMMs
# and the memory-bound kernels.  Usage (under gpurun): bash tools/gpu_session.sh [tests|bench|ncu|all]
set -u
OUT=gpurun_out
mkdir -p $OUT
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $OUT/pytest_gpu.log 2>&1
  tail -3 $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
fi
if [[ $what == bench || $what == all || $what == ncu ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
  tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
fi
if [[ $what == ncu || $what == all ]]; then
  T=$(python -c "import json;print(json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])['config']['threshold_M'])")
  echo "threshold $T"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-accuracy --no-configs --threshold $T > $OUT/ncu_launch_run.log 2>&1
  python tools/launches.py $OUT/launches.csv
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8_tc2 -s 3 -c 3 \
      -o $OUT/prof_gemm -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accuracy --no-configs --threshold $T > $OUT/ncu_gemm.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_quant|k_select|k_stats|k_absmax|k_cols|k_fallback" -s 6 -c 6 \
      -o $OUT/prof_mem -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accuracy --no-configs --threshold $T > $OUT/ncu_mem.log 2>&1
  ls -la $OUT
fi
