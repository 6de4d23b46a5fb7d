# Row-kernel shape sweep (ncu launch times of the r4 kernels).
for v in "XG_R4SEL=4x8" "XG_R4SEL=2x8" "XG_R4SEL=8x6" "XG_R4SEL=4x12" "XG_R4SEL=4x6" "XG_R4Q=3" "XG_R4Q=5" "XG_R4Q=2"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_r4" --csv \
     --log-file gpurun_out/rows.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
     --threshold 0.01539926526059492 > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/rows.csv | head -2
done
