"""Halo-exchange overlap (pnpula_host.cpp enqueue_step): with NCCL halo messages on
a row-strip grid, each iteration updates the h boundary rows of every tile first, runs the
exchange on a second stream while the interior rows update, and the next kernels wait for
both.  The chain must be bitwise equal to the serial order (PNPULA_OVERLAP=0) and to the
untiled chain; the launch count shows the split (3 update launches per tile and channel).
Exercised on one GPU through NCCL self send/recv (PNPULA_FLAG_HALO_VIA_NCCL)."""
import os

import numpy as np
import pytest

import synth
from gpu_common import make_problem
from paper_2511_00870_b200 import FLAG_HALO_VIA_NCCL, Sampler, params

pytestmark = pytest.mark.gpu


def _run(kw, tiles, flags, overlap, n=9, burn=3, seed=21):
    old = os.environ.get("PNPULA_OVERLAP")
    os.environ["PNPULA_OVERLAP"] = "1" if overlap else "0"
    try:
        s = Sampler(**kw, tiles=tiles, flags=flags)
    finally:
        if old is None:
            del os.environ["PNPULA_OVERLAP"]
        else:
            os.environ["PNPULA_OVERLAP"] = old
    try:
        s.run(n, burn, seed)
        x, z, t = s.state()
        mean, var, _ = s.moments()
        out = dict(x=x, z=z, mean=mean, var=var)
        if kw.get("op") == "poisson":
            out["z1"] = s.z1()
        if kw.get("tv_beta", 0) > 0:
            out["zh"] = s.tv_zh()
        _, launches = s.kernel_time("all")
        return out, launches
    finally:
        s.close()


def _cases():
    kw_cnn, _ = make_problem(96, 70, kernel="gauss9", cnn=(8, 32), z=True)
    kw_mask, _ = make_problem(80, 66, op="mask", z=True, cnn=(4, 16))
    ky, kx = synth.gaussian_factors(5, 1.0)
    y = synth.observe_poisson(90, 64, synth.outer(ky, kx), 250.0)
    hp = params.poisson_pnp(250.0)
    kw_ptv = dict(ny=90, nx=64, y=y, sigma2=1.0, op="poisson", kernel_sep=(ky, kx),
                  gamma=0.99 / (250.0 ** 2 / hp["rho1"] + 8.0 / 1e-3), eta=250.0, rho1=hp["rho1"],
                  kappa1=hp["kappa1"], rho=1e-3, kappa=0.99e-3 / 8, tv_beta=13.0,
                  x0=(synth.ground_truth(90, 64) * 0.8 + 0.1).astype(np.float32))
    k2 = synth.outer(*synth.gaussian_factors(9, 2.0))
    s2 = synth.noise_sigma2_blur(96, 72, k2, 25.0)
    w, b = synth.dncnn_weights(4, 32, image_channels=3)
    hpg = params.gaussian_pnp(s2, 1.0, 1.0)
    kw_rgb = dict(ny=96, nx=72, y=synth.observe_blur_rgb(96, 72, k2, s2), kernel_sep=synth.gaussian_factors(9, 2.0),
                  sigma2=s2, gamma=hpg["gamma"], lam=hpg["lam"], c_lo=0.0, c_hi=1.0, weights=w, biases=b,
                  n_layers=4, channels=32, alpha=1.0, eps=hpg["eps"])
    return {"cnn_z": kw_cnn, "mask_z": kw_mask, "poisson_tv": kw_ptv, "rgb_cnn": kw_rgb}


@pytest.mark.parametrize("case", ["cnn_z", "mask_z", "poisson_tv", "rgb_cnn"])
@pytest.mark.parametrize("tiles", [(2, 1), (3, 1)])
def test_overlapped_exchange_bitwise(case, tiles):
    kw = _cases()[case]
    on, n_on = _run(kw, tiles, FLAG_HALO_VIA_NCCL, True)
    off, n_off = _run(kw, tiles, FLAG_HALO_VIA_NCCL, False)
    ref, _ = _run(kw, (1, 1), 0, True)
    for k in on:
        np.testing.assert_array_equal(on[k], off[k], err_msg=k)
        np.testing.assert_array_equal(on[k], ref[k], err_msg=k)
    nc = kw["y"].shape[0] if kw["y"].ndim == 3 else 1
    # overlap: top band + bottom band + interior launches instead of one per tile and channel
    assert n_on - n_off == 9 * 2 * tiles[0] * nc
