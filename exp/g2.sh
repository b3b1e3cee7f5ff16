cd $GRAFT_REPO_ROOT
PYTHONPATH=. timeout 600 python exp/graph_probe.py c1 c2 c4 c3 t5 c5 2>&1 | tail -20
