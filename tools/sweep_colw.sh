# Column-kernel shape sweep: per XG_COLW variant, the ncu launch time of k_cols_w4.
for v in 16x2x1 24x2x1 20x2x1 24x1x1; do
  XG_COLW=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cols_w4 --csv \
     --log-file gpurun_out/colw_$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
     --threshold 0.01539926526059492 > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/colw_$v.csv | head -2
done
