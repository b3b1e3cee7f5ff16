"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(bench.workload + bench.build_inputs: whole 4096 x 8192 image on one GPU, 1x1 tile grid, the
bench's inputs and step sizes, x0 = 0): after four iterations (three non-trivial denoiser
evaluations: x0 = 0 makes the first one constant) the library's state is compared, at sampled
pixels, with the oracle evaluated on a crop around each sample that contains the sample's whole
four-iteration dependency cone (radius 4h, h = 8), with the noise indexed by
global pixel (oracle origin).  Samples cover the image corners and edges, CNN strip seams
(122-column strips) and interior points.  The denoiser runs in bf16: compared with the
bf16-emulating oracle; TV / fp32 paths with the plain fp64 oracle."""
import numpy as np
import pytest

import bench
import oracle
from paper_2511_00870_b200 import Sampler

pytestmark = pytest.mark.gpu

N_ITER, SEED, H = 4, 2511, 8
MARGIN = N_ITER * H + 2


def _samples(ny, nx):
    pts = [(0, 0), (0, nx - 1), (ny - 1, 0), (ny - 1, nx - 1), (ny // 2, 0), (0, nx // 2), (ny - 1, nx // 3),
           (ny // 3, nx - 1)]
    pts += [(1000, 122 * k - 1) for k in (1, 7, 30)] + [(2047, 122 * k) for k in (2, 45)]
    rng = np.random.default_rng(7)
    pts += [(int(rng.integers(0, ny)), int(rng.integers(0, nx))) for _ in range(6)]
    return [(i, j) for i, j in pts if i < ny and j < nx]


def _crop_oracle(wl, si, sj, bf16):
    ny, nx = wl["ny"], wl["nx"]
    i0, j0 = max(si - MARGIN, 0), max(sj - MARGIN, 0)
    i1, j1 = min(si + MARGIN + 1, ny), min(sj + MARGIN + 1, nx)
    kw = bench.build_inputs(wl, (i0, j0, i1 - i0, j1 - j0))
    okw = {k: v for k, v in kw.items() if k in ("sigma2", "gamma", "mask", "weights", "biases", "n_layers",
                                                "channels", "alpha", "eps", "lam", "c_lo", "c_hi", "rho", "kappa",
                                                "z_lo", "z_hi", "eta", "rho1", "kappa1", "tv_beta", "den_kind",
                                                "ddfb_gammas", "ht_eps")}
    if wl["op"] == "mask":
        okw.update(op="mask")
    else:
        okw.update(op="poisson" if wl["op"] == "poisson" else "conv", ksep=kw["kernel_sep"])
    pb = oracle.Problem(y=kw["y"], **okw)
    out = oracle.run(pb, N_ITER, 0, SEED, bf16_emulate=bf16, origin=(i0, j0))
    return {k: out[k][..., si - i0, sj - j0] for k in ("x", "z", "z1", "zh", "mean")}


def _close(a, b, atol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= atol * np.maximum(1.0, np.abs(b))))


@pytest.mark.parametrize("name,bf16,atol", [("c5", True, 2e-3), ("p5", True, 2e-3), ("t5", False, 1e-5),
                                            ("r5", True, 2e-3), ("c3", True, 2e-3), ("d5", True, 2e-3)])
def test_full_size_sampled_parity(name, bf16, atol):
    wl = bench.workload(name, 1)
    ny, nx = wl["ny"], wl["nx"]
    kw = bench.build_inputs(wl, (0, 0, ny, nx))
    kw.pop("_pin", None)
    s = Sampler(**kw, tiles=wl["tiles"])
    try:
        s.run(N_ITER, 0, SEED)
        x, z, _ = s.state()
        mean, _, _ = s.moments(want_var=False)
        z1 = s.z1() if wl["op"] == "poisson" else None
        zh = s.tv_zh() if wl.get("tv") else None
    finally:
        s.close()
    assert np.isfinite(x).all()
    for si, sj in _samples(ny, nx):
        o = _crop_oracle(wl, si, sj, bf16)
        assert _close(x[..., si, sj], o["x"], atol), (si, sj, x[..., si, sj], o["x"])
        assert _close(mean[..., si, sj], o["mean"], atol), (si, sj)
        if wl["z"]:
            assert _close(z[..., si, sj], o["z"], atol), (si, sj, z[..., si, sj], o["z"])
        if z1 is not None:
            assert _close(z1[..., si, sj], o["z1"], atol), (si, sj, z1[..., si, sj], o["z1"])
        if zh is not None:
            assert _close(zh[si, sj], o["zh"], atol), (si, sj, zh[si, sj], o["zh"])
