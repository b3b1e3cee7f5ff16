"""Diagnostics (not a test): rel-L2 errors of x / mean / var of the fp32 GPU chains against the fp64
oracle for the configurations the parity tests use, plus kappa = rms(x) / rms(std), the
conditioning factor of reading R44.  Run on a GPU box from the repo root."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import oracle  # noqa: E402
from gpu_common import gpu_run, make_problem, rel_l2  # noqa: E402


def report(name, g, o, n):
    kappa = np.sqrt(np.mean(o["mean"] ** 2 + o["var"] * (n - 1) / n)) / np.sqrt(np.mean(o["var"]))
    ex, em, ev = rel_l2(g["x"], o["x"]), rel_l2(g["mean"], o["mean"]), rel_l2(g["var"], o["var"])
    print(f"{name:28s} x {ex:.2e} mean {em:.2e} var {ev:.2e} kappa {kappa:6.2f} "
          f"var/(2 kappa max(x,mean)) {ev / (2 * kappa * max(ex, em)):.3f}", flush=True)


for kernel, z in [("gauss9", False), ("random5", True), ("gauss5", True)]:
    kw, pb = make_problem(64, 72, kernel=kernel, z=z)
    report(f"chain50 {kernel} z={z}", gpu_run(kw, 50, 10, 870), oracle.run(pb, 50, 10, 870), 40)
kw, pb = make_problem(66, 70, op="mask", z=True)
report("chain50 mask", gpu_run(kw, 50, 5, 871), oracle.run(pb, 50, 5, 871), 45)

from test_gpu_poisson import gpu_poisson, poisson_problem  # noqa: E402
for kernel, shape in [("gauss9", (70, 83)), ("random5", (61, 57))]:
    kw, pb = poisson_problem(*shape, kernel=kernel)
    report(f"poisson {kernel}", gpu_poisson(kw, 50, 10, seed=870), oracle.run(pb, 50, 10, seed=870), 40)

from test_gpu_tv import gpu_tv, tv_problem  # noqa: E402
for op, kernel, shape in [("conv", "gauss9", (70, 83)), ("conv", "random5", (61, 57)), ("mask", None, (64, 66))]:
    kw, pb = tv_problem(*shape, op=op, kernel=kernel or "gauss9")
    report(f"tv {op} {kernel}", gpu_tv(kw, 50, 10, seed=872), oracle.run(pb, 50, 10, seed=872), 40)

from test_gpu_rgb import rgb_problem, run as rgb_run  # noqa: E402
for op, kernel in [("conv", "random5"), ("conv", "gauss9"), ("mask", None), ("poisson", "gauss9")]:
    kw, pb = rgb_problem(53, 61, op=op, kernel=kernel or "")
    report(f"rgb {op} {kernel}", rgb_run(kw, 30, 5, 870), oracle.run(pb, 30, 5, 870), 25)
