# Same-box A/B of two library builds: the in-tree one and a copy of the baseline build placed in
# paper_2403_06924_b200/lib/ab/ beforehand (loaded through XG_LIB_PATH; delete it afterwards):
# kernel durations from an ncu launch list of tools/c3_once.py, then the bench at SHAPES.
B=paper_2403_06924_b200/lib/ab/libxigemm_b200.so
for rep in 1 2; do
  for lib in new base; do
    if [ $lib = base ]; then export XG_LIB_PATH=$B; else unset XG_LIB_PATH; fi
    CALLS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-k_}" -c ${KCOUNT:-20} \
      --csv python tools/c3_once.py 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[h.index('Kernel Name')].split('(')[0][-40:]].append(float(r[h.index('Metric Value')]))
print('$rep $lib', {k: round(sum(v)/len(v),1) for k,v in d.items()})"
  done
done
unset XG_LIB_PATH
