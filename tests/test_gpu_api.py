"""C-ABI behaviour on the GPU beyond the numerics (include/pnpula.h): global-scope outputs equal
the local ones on one rank, z is zeros without a z block, calls before reset fail with E_STATE,
invalid arguments are rejected, contexts are independent, the memory pool can be trimmed, and
the launch counter counts every kernel."""
import numpy as np
import pytest

from gpu_common import make_problem
from paper_2511_00870_b200 import SCOPE_GLOBAL_ON_ROOT, SCOPE_LOCAL, Sampler
from paper_2511_00870_b200 import _lib as L

pytestmark = pytest.mark.gpu


def test_global_scope_equals_local_on_one_rank():
    kw, _ = make_problem(70, 90, kernel="gauss9", z=True)
    s = Sampler(**kw, tiles=(2, 3))
    try:
        s.run(12, 4, 5)
        xl, zl, _ = s.state(SCOPE_LOCAL)
        xg, zg, _ = s.state(SCOPE_GLOBAL_ON_ROOT)
        ml, vl, _ = s.moments(SCOPE_LOCAL)
        mg, vg, _ = s.moments(SCOPE_GLOBAL_ON_ROOT)
    finally:
        s.close()
    for a, b in ((xl, xg), (zl, zg), (ml, mg), (vl, vg)):
        np.testing.assert_array_equal(a, b)


def test_z_is_zero_without_z_block_and_state_before_reset():
    kw, _ = make_problem(40, 40, kernel="gauss5", z=False)
    s = Sampler(**kw)
    try:
        with pytest.raises(Exception):
            s.advance(1)                       # reset must come first (E_STATE)
        with pytest.raises(Exception):
            s.moments()                        # no chain yet
        s.run(3, 0, 1)
        x, z, t = s.state()
        assert t == 3 and not z.any() and np.isfinite(x).all()
        with pytest.raises(Exception):
            s.advance(-1)                      # invalid n_iter
    finally:
        s.close()


def test_invalid_configurations_are_rejected():
    kw, _ = make_problem(32, 32, kernel="gauss5")
    for bad in (dict(gamma=0.0), dict(sigma2=-1.0), dict(rho=1.0, kappa=2.0)):
        with pytest.raises(Exception):
            Sampler(**{**kw, **bad})
    with pytest.raises(Exception):
        Sampler(**kw, tiles=(16, 1))             # 2-row tiles < halo width 4 (5x5 kernel)


def test_independent_contexts_and_pool_trim():
    kw1, _ = make_problem(48, 40, kernel="gauss5", z=True)
    kw2, _ = make_problem(30, 50, op="mask", z=True)
    a = Sampler(**kw1)
    b = Sampler(**kw2)
    try:
        a.run(6, 2, 1)
        b.run(6, 2, 1)
        xa, _, _ = a.state()
        xb, _, _ = b.state()
    finally:
        a.close()
        b.close()
    ref = Sampler(**kw1)
    try:
        ref.run(6, 2, 1)
        xr, _, _ = ref.state()
    finally:
        ref.close()
    np.testing.assert_array_equal(xa, xr)        # a second live context does not disturb the first
    assert xb.shape == (30, 50)
    lib = L.load()
    assert lib.pnpula_release_memory(0) == 0    # unused pool memory back to the driver
    assert lib.pnpula_release_memory(99) != 0   # no such device


def test_launch_counter_counts_kernels():
    kw, _ = make_problem(64, 64, kernel="gauss9", cnn=(8, 32))
    s = Sampler(**kw)
    try:
        s.reset(0, 1)
        s.kernel_time("all", reset=True)
        s.advance(5)
        _, n = s.kernel_time("all")
    finally:
        s.close()
    assert n == 5 * 3                            # two CNN chunks + one update per iteration
