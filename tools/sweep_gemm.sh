for gm in 8 16 32; do for pf in 0 8 16; do
  echo "== group $gm pf $pf"
  XG_GEMM_GROUP=$gm XG_GEMM_PF=$pf ITERS=30 GAP=0.3 CFGS=0,2 python tools/gemm_ceiling.py
done; done
