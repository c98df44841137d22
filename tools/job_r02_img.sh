cd $GRAFT_REPO_ROOT
export EMIE_CU_GREENS_IMG=1
for lib in base imgx1; do
  if [ $lib = base ]; then unset EMIE_CU_LIBRARY; else export EMIE_CU_LIBRARY=$PWD/exp/$lib/libemie_cu.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"chunk_image|assemble_kernel" --csv --log-file gpurun_out/imgx_$lib.csv python tools/time_greens.py --config 3 --reps 1 > gpurun_out/imgx_$lib.log 2>&1
  python - <<P
import csv
lines=open('gpurun_out/imgx_$lib.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
agg={}
for r in csv.DictReader(lines[i:]):
    n=r['Kernel Name'][:40]; agg.setdefault(n,[]).append(float(r['Metric Value'].replace(',','')))
for n,v in agg.items(): print('$lib', n, len(v), round(sum(v)/1e6,2), 'ms')
P
done
