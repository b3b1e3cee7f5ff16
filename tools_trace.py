"""Analyse a PNPULA_CNN_TRACE dump (diagnostics only)."""
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
    return t, code, s, l

for fn in sys.argv[1:]:
    t, code, s, l = load(fn)
    print(fn, 'events', len(t), 'span', t.max())
    ev = {}
    for ti, c, si, li in zip(t, code, s, l):
        ev[(c, si, li)] = ti
    # per step: MMA issue start/end, epilogue done
    steps = sorted(set(si for c, si, li in ev if c == 3))
    L = max(li for c, si, li in ev) + 1
    print('step  ' + '  '.join(f'L{j}:wait(3->4)/issue(4->5)/tfull(6)/done(8)' for j in range(min(L,3))))
    prev = None
    for si in steps[:40]:
        row = []
        for j in range(L):
            if (3, si, j) in ev:
                w = ev[(4, si, j)] - ev[(3, si, j)]
                iss = ev[(5, si, j)] - ev[(4, si, j)]
                tf = ev.get((6, si, j), -1) - ev[(5, si, j)]
                dn = ev.get((8, si, j), -1) - ev.get((6, si, j), 0) if (8, si, j) in ev else -1
                row.append(f'{w:5d}/{iss:4d}/{tf:5d}/{dn:5d}')
            else:
                row.append(' ' * 23)
        t0 = min(ev[(3, si, j)] for j in range(L) if (3, si, j) in ev)
        print(f'{si:4d} {t0 - (prev or t0):6d} ' + ' | '.join(row))
        prev = t0
