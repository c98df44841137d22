cd $GRAFT_REPO_ROOT
for r in 0 3 0 3 0 3; do echo "== reserve $r GB"; timeout 300 python tools/cold_build.py warm $r 2>&1 | tail -4 | head -2; done
