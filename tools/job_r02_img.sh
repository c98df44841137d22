cd $GRAFT_REPO_ROOT
for mb in 1024 2048 4096; do echo "== $mb"; EMIE_CU_GREENS_IMG_MB=$mb timeout 300 python tools/time_greens.py --config 3 --reps 3 2>&1 | tail -1; done
