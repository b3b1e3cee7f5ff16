"""Analyse a PNPULA_CNN_TRACE dump (diagnostics only).
codes: 1/2 producer empty-wait done / fill arrived; 3/4/5 MMA: start / inputs ready / issued+committed;
6 epi tfull done, 7 TMEM loaded, 9 exchange barrier passed, 10 before ring-slot wait, 11 slot free, 8 full arrived."""
import sys
import numpy as np


def load(fn):
    a = np.fromfile(fn, dtype=np.uint64)
    n = int(a[0]); r = a[1:1 + n]
    t = (r >> np.uint64(20)).astype(np.int64)
    code = ((r >> np.uint64(16)) & np.uint64(0xf)).astype(int)
    s = ((r >> np.uint64(4)) & np.uint64(0xfff)).astype(int)
    l = (r & np.uint64(0xf)).astype(int)
    t = t - t.min()
    return {(c, si, li): ti for ti, c, si, li in zip(t, code, s, l)}


def d(ev, a, b, si, li):
    if (a, si, li) in ev and (b, si, li) in ev:
        return ev[(b, si, li)] - ev[(a, si, li)]
    return None


def report(fn, steps=range(24, 30)):
    ev = load(fn)
    L = max(li for c, si, li in ev) + 1
    print(fn)
    for si in steps:
        t0 = min((ev[(3, si, j)] for j in range(L) if (3, si, j) in ev), default=0)
        parts = []
        for j in range(L):
            if (3, si, j) not in ev:
                continue
            seg = [('wfull', 3, 10), ('wtmem', 10, 4), ('issue', 4, 5), ('->tfull', 5, 6), ('ld', 6, 7),
                   ('wempty', 7, 9), ('st', 9, 8), ('epi', 6, 8)]
            parts.append(f"L{j} " + ' '.join(f"{nm}={d(ev, a, b, si, j)}" for nm, a, b in seg if d(ev, a, b, si, j) is not None))
        print(f"s={si} t={t0}: " + ' | '.join(parts))




def summary(fn, lo=20, hi=None):
    """Mean per-step segment durations (cycles) over steps [lo, hi) for every layer."""
    ev = load(fn)
    L = max(li for c, si, li in ev) + 1
    S = max(si for c, si, li in ev) + 1
    hi = hi or S - 20
    segs = [('wfull', 3, 14), ('wtmem', 14, 4), ('issue', 4, 5), ('ld', 6, 7), ('wempty', 7, 9), ('st', 9, 8)]
    print(fn, f"steps {lo}..{hi}, step time {np.mean([ev[(3, s + 1, 1)] - ev[(3, s, 1)] for s in range(lo, hi) if (3, s, 1) in ev and (3, s + 1, 1) in ev]):.0f}")
    for l in range(L):
        out = []
        for nm, a, b in segs:
            v = [d(ev, a, b, s, l) for s in range(lo, hi)]
            v = [x for x in v if x is not None]
            if v:
                out.append(f"{nm}={np.mean(v):.0f}")
        print(f"  L{l}: " + ' '.join(out))


if __name__ == "__main__":
    for fn in sys.argv[1:]:
        summary(fn)
