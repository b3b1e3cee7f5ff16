import sys, numpy as np
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
from test_gpu_poisson import poisson_problem, gpu_poisson
for kern in ("gauss5", "gauss9"):
    kw, pb = poisson_problem(58, 61, kernel=kern)
    try:
        g = gpu_poisson(kw, 3, 1, seed=1)
        print(kern, "ok", float(g["x"].mean()))
    except Exception as e:
        print(kern, "FAIL", e)
