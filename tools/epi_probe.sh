#!/bin/bash
# GEMM epilogue probes at one shape (under gpurun): bash tools/epi_probe.sh M N K
# XG_GEMM_DEBUG bits (gemm_tc.cuh): 2 no epilogue, 4 TMEM drain only, 8 no TMA store,
# 64 no dequant math (D_F GEMM), 1 no TMA operand loads, 32 no MMA (33: epilogue alone).  Results are wrong under probes: timing only.
OUT=gpurun_out
for d in ${DBGS:-0 2 8 64}; do
  line=$(XG_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-accuracy --m $1 --n $2 --k $3 2>/dev/null | tail -1)
  echo "dbg=$d $* $(echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('df', round(r['gemm_df_ms'],4), 'comp', round(r['gemm_comp_ms'],4), d['clocks']['sm_mhz'])" 2>&1 | tail -1)" | tee -a $OUT/epi_probe.txt
done
