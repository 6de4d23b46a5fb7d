# A/B of environment variants at several shapes (student-t C3 data via bench.py):
#   SHAPES="4096 4096 4096;8192 8192 8192" bash tools/ab_env.sh "A=0" "XG_X=1" ...
SHAPES=${SHAPES:-"4096 4096 4096;8192 8192 8192"}
IFS=';' read -ra SH <<< "$SHAPES"
VARS=("$@")
for rep in 1 2; do
for v in "${VARS[@]}"; do
  for shp in "${SH[@]}"; do
    set -- $shp
    echo "$rep | $v | $shp | $(env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-e2e --no-accuracy --m $1 --n $2 --k $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), {k: v//1000 for k, v in d['stage_ns'].items() if k in ('quant','reduce','gemm_df','gemm_comp')})")"
  done
done
done
