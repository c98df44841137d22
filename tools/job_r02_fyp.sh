cd $GRAFT_REPO_ROOT
for v in fyp5; do
  if [ $v = base ]; then unset EMIE_CU_LIBRARY; else export EMIE_CU_LIBRARY=$PWD/exp/$v/libemie_cu.so; fi
  for G in 1 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stream_tma" --csv --log-file gpurun_out/fyp_${v}_$G.csv python tools/fypeer_time.py $G > gpurun_out/fyp_${v}_$G.log 2>&1
  python - <<P
import csv
lines=open('gpurun_out/fyp_${v}_$G.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.DictReader(lines[i:]))
x=[float(r['Metric Value'].replace(',','')) for r in rows if 'FyPeer' in r['Kernel Name']]
print('$v G=$G', len(x), sum(x)/max(1,len(x)))
P
  done
done
