"""Diagnostics: where the first pnpula_create of a process spends its time (c5 inputs);
run with PNPULA_TIME_CREATE=1 in a fresh process."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2511_00870_b200 import Sampler  # noqa: E402

torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
wl = bench.workload("c5", 1)
kw = bench.build_inputs(wl, (0, 0, wl["ny"], wl["nx"]), pinned=True)
kw.pop("_pin")
for rep in range(2):
    t0 = time.perf_counter()
    s = Sampler(**kw, tiles=wl["tiles"])
    t1 = time.perf_counter()
    s.reset(0, 1)
    s.advance(2)
    s.synchronize()
    t2 = time.perf_counter()
    s.close()
    print(f"rep {rep}: create {1e3 * (t1 - t0):.1f} ms, reset + 2 iterations {1e3 * (t2 - t1):.1f} ms", flush=True)
