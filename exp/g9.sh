cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py tests/test_gpu_tv.py tests/test_gpu_poisson.py tests/test_gpu_rgb.py tests/test_gpu_ddfb.py -x -q 2>&1 | tail -15
