"""Per-iteration device time, graph replay vs direct launches, on the bench workloads."""
import sys, time
import torch
import bench
from paper_2511_00870_b200 import FLAG_NO_GRAPH, Sampler

for name in sys.argv[1:]:
    wl = bench.workload(name, 1)
    kw = bench.build_inputs(wl, (0, 0, wl["ny"], wl["nx"]))
    kw.pop("_pin", None)
    for flags in (FLAG_NO_GRAPH, 0):
        s = Sampler(**kw, tiles=wl["tiles"], flags=flags)
        s.reset(0, 1)
        s.advance(5)
        s.synchronize()
        K = 200 if wl["ny"] * wl["nx"] <= 4 << 20 else 30
        t0 = time.perf_counter()
        s.advance(K)
        t1 = time.perf_counter()
        s.synchronize()
        t2 = time.perf_counter()
        print(f"{name} {'graph ' if flags == 0 else 'direct'} host-enqueue {1e3 * (t1 - t0) / K:.4f} ms/it, "
              f"wall {1e3 * (t2 - t0) / K:.4f} ms/it", flush=True)
        s.close()
