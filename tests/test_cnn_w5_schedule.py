"""CPU check of the wide TMEM accumulator schedule of the tcgen05 CNN kernel (cnn_kernels.cu,
wide_slots / mma_step / epi_step, R46) -- host-side logic, no GPU -- for both
widths W = T + 2 (T = 3: 5 slots, T = 4: 6 slots):

* every fill's MMA window is one contiguous run of slots inside the W slots (never split);
* every output row's three contributions (dy = -1, 0, +1) land in the slots its global row
  mod T prescribes (so a row's accumulation order never depends on the tiling), in at most two
  slots;
* with the kernel's wait rule (fill f of a unit waits until the epilogue drained
  O0 + max(0, f - (T - 1)) rows, rows drained in order), no slot is ever written while it still
  holds an undrained row of another output row, for random unit sequences per CTA; and the
  epilogue can never be two rows past the awaited one (the row-parity barriers stay unambiguous).
"""
import numpy as np
import pytest


def wide_slots(o, T):
    m = o % T
    q2, q0 = m + 2, (m + 2) % T
    return q2, (None if q0 == q2 else q0)


def contribution_slot(o, q, T):
    """slot of output row o's contribution from the fill in which it is row f-2+q (q = 2: dy = -1,
    its first fill; q = 1: dy = 0; q = 0: dy = +1, its last) -- from the window rule b = o_f mod T."""
    fresh = o + (2 - q)            # global row of the fresh row of that fill
    return fresh % T + q


@pytest.mark.parametrize("T", [3, 4])
def test_slot_map(T):
    for o in range(-7, 50):
        main, second = wide_slots(o, T)
        used = {contribution_slot(o, q, T) for q in range(3)}
        assert used == ({main} if second is None else {main, second})
        assert contribution_slot(o, 2, T) == main and max(used) <= T + 1


@pytest.mark.parametrize("T", [3, 4])
@pytest.mark.parametrize("seed", range(10))
def test_wide_windows_no_overwrite(T, seed):
    rng = np.random.default_rng(seed)
    owner = {}          # slot -> sequence index of the row whose partial sum it holds
    drained = 0
    seq = 0
    completed = []      # rows completed by the MMA, not yet drained (in order)
    for _unit in range(12):
        o_first = int(rng.integers(-8, 5000))
        nout = int(rng.integers(1, 40))
        O0 = seq
        for f in range(nout + 2):
            need = O0 + max(0, f - (T - 1))
            while drained < need:
                assert completed and completed[0] == drained, "wait rule asks for a row not yet completed"
                r = completed.pop(0)
                for s in [k for k, v in owner.items() if v == r]:
                    del owner[s]
                drained += 1
            while completed and rng.random() < 0.5:   # the epilogue may run ahead of the wait ...
                r = completed.pop(0)
                for s in [k for k, v in owner.items() if v == r]:
                    del owner[s]
                drained += 1
            assert drained <= need + 1                 # ... but never two phases past it
            ilo, ihi = max(f - 2, 0), min(f, nout - 1)
            b = (o_first + f) % T
            q0 = ilo - (f - 2)
            slots = [b + q0 + i for i in range(ihi - ilo + 1)]
            assert 0 <= slots[0] and slots[-1] <= T + 1
            for i, ic in enumerate(range(ilo, ihi + 1)):
                s = slots[i]
                assert s == contribution_slot(o_first + ic, q0 + i, T)
                r = O0 + ic
                assert owner.get(s, r) == r, f"slot {s} overwritten while holding row {owner.get(s)}"
                owner[s] = r
            if 0 <= f - 2 < nout:
                completed.append(O0 + f - 2)
        seq += nout
