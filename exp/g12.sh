cd $GRAFT_REPO_ROOT
PNPULA_TIME_CREATE=1 timeout 600 python exp/e2e_probe.py 2>&1 | tail -16
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
