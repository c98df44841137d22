cd $GRAFT_REPO_ROOT
echo "== cfg3 split"; EMIE_CU_GREENS_IMG=1 timeout 300 python tools/time_greens.py --config 3 --reps 2 2>&1 | tail -1
echo "== cfg3 fused"; timeout 300 python tools/time_greens.py --config 3 --reps 2 2>&1 | tail -1
echo "== cfg4 split"; timeout 300 python tools/time_greens.py --config 4 --reps 2 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"chunk_image|assemble_kernel" --csv --log-file gpurun_out/imgx.csv env EMIE_CU_GREENS_IMG=1 python tools/time_greens.py --config 3 --reps 1 > /dev/null 2>&1
python - <<P
import csv
lines=open('gpurun_out/imgx.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
agg={}
for r in csv.DictReader(lines[i:]):
    n=r['Kernel Name'][:40]; agg.setdefault(n,[]).append(float(r['Metric Value'].replace(',','')))
for n,v in agg.items(): print(n, len(v), round(sum(v)/1e6,2), 'ms')
P
