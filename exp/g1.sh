cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_graphs.py -x -q 2>&1 | tail -15
PYTHONPATH=. timeout 600 python exp/graph_probe.py c1 c2 c4 t5 2>&1 | tail -20
