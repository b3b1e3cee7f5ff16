"""Summarise ncu output for profiles/ (diagnostics only; runs here, on the .ncu-rep / CSV files
that gpurun brings back).

    python tools_ncu_summary.py launches <launches.csv>           # per-kernel share of the launch list
    python tools_ncu_summary.py report <file.ncu-rep> [...]        # key metrics per captured launch
    python tools_ncu_summary.py traffic <cnn.ncu-rep> <update.ncu-rep> <pixels> <workload>
                                                                   # -> profiles/ncu_traffic.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block", "shared mem/block"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts (tensor) %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts (LSU)"),
    ("smsp__pcsamp_warps_issue_stalled_long_scoreboard", "stall samples: long scoreboard"),
    ("smsp__pcsamp_warps_issue_stalled_no_instructions", "stall samples: no instruction"),
    ("smsp__pcsamp_warps_issue_stalled_barrier", "stall samples: barrier"),
    ("smsp__pcsamp_warps_issue_stalled_wait", "stall samples: wait"),
    ("smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "stall samples: math pipe throttle"),
    ("smsp__pcsamp_warps_issue_stalled_mio_throttle", "stall samples: MIO throttle"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        res.append(d)
    return res


def find(d, key):
    for h, (v, u) in d.items():
        if h == key or h.endswith("." + key) or h.endswith(key) and key.count(".") >= 2 and h.split(".", 2)[-1] == key:
            return v, u
    return None, None


def report(reps):
    for rep in reps:
        print(f"### {os.path.basename(rep)}")
        for i, d in enumerate(raw(rep)):
            name = d.get("Kernel Name", ("?", ""))[0]
            print(f"\nlaunch {i}: `{name}`\n")
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                v, u = find(d, k)
                if v is not None:
                    print(f"| {label} (`{k}`) | {v} {u} |")
        print()


def launches(fn):
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    all_ns = sum(tot.values())
    print("| kernel | launches | total ms | mean us/launch | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / cnt[k] / 1e3:.1f} | {v / all_ns * 100:.1f}% |")


def traffic(cnn_rep, upd_rep, px, workload):
    def total_bytes(rep):
        t = 0.0
        n = 0
        for d in raw(rep):
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = find(d, k)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                t += float(v.replace(",", "")) * scale
            n += 1
        return t, n
    cb, cn = total_bytes(cnn_rep)
    ub, un = total_bytes(upd_rep)
    out = {"workload": workload, "pixels_per_gpu": px,
           "cnn_bytes_per_px": cb / px, "cnn_launches_captured": cn,
           "update_bytes_per_px": ub / un / px, "update_launches_captured": un,
           "source": [os.path.basename(cnn_rep), os.path.basename(upd_rep)],
           "note": "dram__bytes_read.sum + dram__bytes_write.sum from ncu --set full; CNN summed over the "
                   "launches of one evaluation, update per launch"}
    os.makedirs("profiles", exist_ok=True)
    json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(sys.argv[2:])
    elif cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5])
