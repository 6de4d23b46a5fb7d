for i in 1 2 3; do python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-accuracy --m 16384 --n 11008 --k 4096 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],4), 'df', round(r['gemm_df_ms'],4), 'comp', round(r['gemm_comp_ms'],4))"; done
SHAPE=16384,11008,4096 ITERS=30 CFGS=0,2 python tools/gemm_ceiling.py
