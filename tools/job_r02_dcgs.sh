cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -q tests/test_gpu_solve.py 2>&1 | tail -5
