#!/bin/bash
# Pipeline timing across BASELINE.json's single-GPU shapes (under gpurun):
#   bash tools/shapes.sh [launches]   -> gpurun_out/shapes.txt (+ launch lists per shape)
OUT=gpurun_out
mode=${1:-}
mkdir -p $OUT
for shp in "4096 4096 4096" "8192 8192 8192" "16384 11008 4096" "8192 8192 16384"; do
  set -- $shp
  line=$(timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-accuracy --m $1 --n $2 --k $3 2>/dev/null | tail -1)
  echo "${XG_TAG:-} $shp $(echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],4), 'df', round(r['gemm_df_ms'],4), 'comp', round(r['gemm_comp_ms'],4), d['clocks']['sm_mhz'])")" | tee -a $OUT/shapes.txt
done
if [[ $mode == launches ]]; then
  for shp in "16384 11008 4096" "4096 4096 4096"; do
    set -- $shp
    tag=$1x$2x$3
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$tag.csv \
        python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-accuracy --m $1 --n $2 --k $3 > /dev/null 2>&1
    python tools/launches.py $OUT/launches_$tag.csv > $OUT/launches_$tag.txt
  done
fi
