for v in "A=0" "XG_COLS_FUSED_MAXC=8" "A=0" "XG_COLS_FUSED_MAXC=8"; do
  for shp in "8192 8192 16384" "65536 16384 16384"; do set -- $shp
  echo "$v $shp $(env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-accuracy --m $1 --n $2 --k $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['stage_ns']['quant']//1000)")"
  done
done
