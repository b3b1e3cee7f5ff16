"""The x / z / moment update fused into the last CNN chunk (cnn_kernels.cu, FU):
the folded layer's epilogue hands every completed G row to the chunk's producer warps, which
evaluate g = H^T(eta H x - y) in a streaming separable stencil (or the mask term) and the K7 tail
 for every tile pixel, in the per-pixel order of update_sep_kernel / update_mask_kernel.  The fused chain must therefore equal the unfused one
(PNPULA_FUSE=0 at create: G stored, then the update kernel) BIT FOR BIT -- over 3x3 / 5x5 / 9x9
stencils, the mask operator, Poisson's x step, the AXDA z block, box prox, several column strips
and row units per CTA, tiled grids, graph replays and the layer-wise chain -- and the fused run
must launch no x-update kernel.  The unfused path itself is pinned to the oracle elsewhere
(test_gpu_parity, test_gpu_c3_chain, test_gpu_poisson).  The fused path is opt-in (PNPULA_FUSE=1;
measured slower)."""
import numpy as np
import pytest

from gpu_common import make_problem
from paper_2511_00870_b200 import FLAG_CNN_LAYERWISE, FLAG_NO_GRAPH, Sampler
from test_gpu_poisson import poisson_problem

pytestmark = pytest.mark.gpu


def _run(kw, n_iter, burn_in, seed, monkeypatch, fuse, tiles=(1, 1), flags=0, max_ctas=None):
    monkeypatch.setenv("PNPULA_FUSE", "1" if fuse else "0")
    if max_ctas:
        monkeypatch.setenv("PNPULA_MAX_CTAS", str(max_ctas))
    else:
        monkeypatch.delenv("PNPULA_MAX_CTAS", raising=False)
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        s.set_timing(True)
        s.run(n_iter, burn_in, seed)
        _, n_upd = s.kernel_time("update")
        x, z, _ = s.state()
        mean, var, _ = s.moments()
        z1 = s.z1() if kw.get("op") == "poisson" else None
        return dict(x=x, z=z, mean=mean, var=var, z1=z1, n_upd=n_upd)
    finally:
        s.close()
        monkeypatch.delenv("PNPULA_FUSE", raising=False)
        monkeypatch.delenv("PNPULA_MAX_CTAS", raising=False)


def _same(a, b):
    for k in ("x", "z", "mean", "var", "z1"):
        if a[k] is None:
            assert b[k] is None, k
            continue
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


CASES = {
    "conv9_box": dict(ny=150, nx=300, op="conv", kernel="gauss9", z=False),
    "conv5_z": dict(ny=97, nx=260, op="conv", kernel="gauss5", z=True),
    "mask_z": dict(ny=130, nx=250, op="mask", z=True),
    "conv9_z_ragged": dict(ny=61, nx=395, op="conv", kernel="gauss9", z=True),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fused_equals_unfused_bitwise(name, monkeypatch):
    c = dict(CASES[name])
    ny, nx = c.pop("ny"), c.pop("nx")
    kw, _ = make_problem(ny, nx, cnn=(8, 32), **c)
    a = _run(kw, 12, 4, 31, monkeypatch, fuse=False)
    b = _run(kw, 12, 4, 31, monkeypatch, fuse=True)
    assert a["n_upd"] > 0 and b["n_upd"] == 0, (a["n_upd"], b["n_upd"])
    _same(a, b)


@pytest.mark.parametrize("tiles,flags,max_ctas", [((2, 2), 0, None), ((3, 1), FLAG_NO_GRAPH, None),
                                                  ((1, 1), 0, 2), ((1, 2), FLAG_CNN_LAYERWISE, None)])
def test_fused_tilings_units_graphs_layerwise(tiles, flags, max_ctas, monkeypatch):
    kw, _ = make_problem(140, 280, kernel="gauss9", cnn=(8, 32), z=True)
    ref = _run(kw, 10, 3, 77, monkeypatch, fuse=False)
    got = _run(kw, 10, 3, 77, monkeypatch, fuse=True, tiles=tiles, flags=flags, max_ctas=max_ctas)
    assert got["n_upd"] == 0
    _same(ref, got)


def test_fused_poisson_x_step(monkeypatch):
    kw, _ = poisson_problem(96, 270, kernel="gauss9", cnn=(8, 32))
    a = _run(kw, 10, 3, 5, monkeypatch, fuse=False, tiles=(2, 1))
    b = _run(kw, 10, 3, 5, monkeypatch, fuse=True, tiles=(2, 1))
    # the z1 block kernel (timed with the update class) still runs; the x-update launches do not
    assert b["n_upd"] < a["n_upd"], (a["n_upd"], b["n_upd"])
    _same(a, b)


def test_unfusable_configs_fall_back(monkeypatch):
    # non-separable kernel / 16-channel net: the update kernel runs (no fused path compiled)
    kw, _ = make_problem(80, 90, kernel="random5", cnn=(8, 32))
    assert _run(kw, 3, 0, 1, monkeypatch, fuse=True)["n_upd"] > 0
    kw, _ = make_problem(80, 90, kernel="gauss5", cnn=(4, 16))
    assert _run(kw, 3, 0, 1, monkeypatch, fuse=True)["n_upd"] > 0
