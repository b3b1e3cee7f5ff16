"""Diagnostics: where the end-to-end time goes (create / reset / advance / moments)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_00870_b200 import Sampler
wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c5", 1)
kw = bench.build_inputs(wl, (0, 0, wl["ny"], wl["nx"]), pinned=True)
kw.pop("_pin")
shp = ((wl["nc"],) if wl.get("nc", 1) > 1 else ()) + (wl["ny"], wl["nx"])
pm = torch.empty(shp, dtype=torch.float32, pin_memory=True).numpy()
pv = torch.empty(shp, dtype=torch.float32, pin_memory=True).numpy()
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    s = Sampler(**kw, tiles=wl["tiles"]); t.append(time.perf_counter())
    s.reset(0, 1); s.synchronize(); t.append(time.perf_counter())
    s.advance(1); s.synchronize(); t.append(time.perf_counter())
    s.advance(19); s.synchronize(); t.append(time.perf_counter())
    s.moments(out=(pm, pv)); t.append(time.perf_counter())
    s.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: create {d[0]:.1f} reset {d[1]:.1f} first iter {d[2]:.1f} next 19 {d[3]:.1f} moments {d[4]:.1f} close {d[5]:.1f} ms")
