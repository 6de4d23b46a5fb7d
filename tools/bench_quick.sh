# quick pipeline timing under env variants: bash tools/bench_quick.sh "ENV=.. ENV2=.." ...
for v in "$@"; do
  echo "== $v"
  env $v python bench.py --steps 10 --no-cpu-baseline --threshold 0.01539926526059492 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],4), {k: v//1000 for k, v in d['stage_ns'].items()}, 'df', round(r['gemm_df_ms'],4), 'comp', round(r['gemm_comp_ms'],4), d['clocks']['sm_mhz'])"
done
