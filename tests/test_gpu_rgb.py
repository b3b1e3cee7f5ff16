"""Colour (C = 3) images through the C ABI vs the oracle (reading R43):
planar channels, H / mask / box / z blocks per channel with Philox streams 4c + s, the colour
DnCNN (layer 1: 27 im2col taps in K = 32; last layer: P -> 3 folded into N = 48)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import rel_l2
from paper_2511_00870_b200 import FLAG_CNN_LAYERWISE, FLAG_HALO_VIA_NCCL, FLAG_NO_GRAPH, Sampler, params

pytestmark = pytest.mark.gpu


def rgb_problem(ny, nx, op="conv", kernel="random5", cnn=None, z=True, box=True):
    C = 3
    kw = {}
    if op == "mask":
        s2 = synth.noise_sigma2_mask(ny, nx, 15.0)
        y, m = synth.observe_mask_rgb(ny, nx, s2)
        kw.update(op="mask", mask=m)
        okw = dict(op="mask", mask=m)
    else:
        if kernel.startswith("gauss"):
            ky, kx = synth.gaussian_factors(9, 2.0)
            k2 = synth.outer(ky, kx)
            kw["kernel_sep"], okw = (ky, kx), dict(op=op, ksep=(ky, kx))
        else:
            k = synth.random_kernel(5, 5, seed=5)
            k2 = k.astype(np.float64)
            kw["kernel"], okw = k, dict(op=op, kernel=k)
        kw["op"] = op
        if op == "poisson":
            y = np.stack([synth.observe_poisson(ny, nx, k2, 250.0) * (1.0 + 0.2 * c) for c in range(C)])
            y = np.floor(y).astype(np.float32)
            s2 = 1.0
        else:
            s2 = synth.noise_sigma2_blur(ny, nx, k2, 25.0)
            y = synth.observe_blur_rgb(ny, nx, k2, s2)
    hp = params.gaussian_pnp(s2, 1.0, 1.0, rho=1e-2 if z else 0.0)
    common = dict(sigma2=s2, gamma=hp["gamma"],
                  x0=(synth.ground_truth_rgb(ny, nx) * 0.8 + 0.1).astype(np.float32))
    if box:
        common.update(lam=hp["lam"], c_lo=0.0, c_hi=1.0)
    if z:
        common.update(rho=hp["rho"], kappa=hp["kappa"], z_lo=0.0, z_hi=1.0)
    if op == "poisson":
        pp = params.poisson_pnp(250.0)
        common.update(eta=250.0, rho1=pp["rho1"], kappa1=pp["kappa1"], z_hi=np.inf,
                      gamma=0.99 / (250.0 ** 2 / pp["rho1"] + 1.0 / hp["rho"] + 1.0 / hp["lam"]))
    if cnn is not None:
        w, b = synth.dncnn_weights(cnn[0], cnn[1], seed=2514, image_channels=C)
        common.update(weights=w, biases=b, n_layers=cnn[0], channels=cnn[1], alpha=1.0, eps=hp["eps"])
    kw.update(common, ny=ny, nx=nx, y=y)
    pb = oracle.Problem(y=y, **okw, **common)
    return kw, pb


def run(kw, n_iter, burn_in, seed, tiles=(1, 1), flags=0):
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        s.run(n_iter, burn_in, seed)
        x, z, t = s.state()
        mean, var, _ = s.moments()
        out = dict(x=x, z=z, mean=mean, var=var)
        if kw.get("op") == "poisson":
            out["z1"] = s.z1()
        return out
    finally:
        s.close()


@pytest.mark.parametrize("K,P,shape,flags", [
    (4, 32, (40, 130), 0),
    (8, 32, (70, 150), 0),
    (8, 32, (70, 150), FLAG_CNN_LAYERWISE),
    (3, 64, (33, 140), 0),
])
def test_colour_denoiser_residual(K, P, shape, flags):
    ny, nx = shape
    kw, _ = rgb_problem(ny, nx, cnn=(K, P))
    s = Sampler(**kw, flags=flags)
    try:
        s.reset(0, 1)
        G = s.denoiser_residual()
    finally:
        s.close()
    assert G.shape == (3, ny, nx)
    ref = oracle.dncnn_residual(kw["x0"], kw["weights"], kw["biases"], K, P)
    ref16 = oracle.dncnn_residual(kw["x0"], kw["weights"], kw["biases"], K, P, bf16_emulate=True)
    assert rel_l2(G, ref) <= 2e-2
    assert rel_l2(G, ref16) <= 2e-3
    for c in range(3):   # every channel, not just the aggregate
        assert rel_l2(G[c], ref16[c]) <= 2e-3


@pytest.mark.parametrize("op,kernel", [("conv", "random5"), ("conv", "gauss9"), ("mask", None), ("poisson", "gauss9")])
def test_colour_chain_fp32_path(op, kernel):
    kw, pb = rgb_problem(53, 61, op=op, kernel=kernel or "")
    g = run(kw, 30, 5, 870)
    o = oracle.run(pb, 30, 5, 870)
    keys = ("x", "z", "mean") + (("z1",) if op == "poisson" else ())
    for k in keys:
        assert g[k].shape == (3, 53, 61)
        assert rel_l2(g[k], o[k]) <= 1e-5, k
    assert rel_l2(g["var"], o["var"]) <= 1e-5   # SURVEY A16; conditioning: DESIGN.md R44


def test_colour_chain_with_cnn():
    kw, pb = rgb_problem(45, 140, kernel="gauss9", cnn=(8, 32))
    g = run(kw, 20, 4, 871)
    o16 = oracle.run(pb, 20, 4, 871, bf16_emulate=True)
    o = oracle.run(pb, 20, 4, 871)
    assert rel_l2(g["x"], o16["x"]) <= 2e-3 and rel_l2(g["mean"], o16["mean"]) <= 2e-3
    assert rel_l2(g["x"], o["x"]) <= 2e-2


@pytest.mark.parametrize("tiles,flags", [((2, 2), 0), ((3, 1), FLAG_HALO_VIA_NCCL), ((1, 2), FLAG_NO_GRAPH)])
def test_colour_tiled_equals_untiled(tiles, flags):
    kw, _ = rgb_problem(64, 70, kernel="gauss9", cnn=(4, 32))
    a = run(kw, 12, 3, 5)
    t = run(kw, 12, 3, 5, tiles=tiles, flags=flags)
    for k in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(a[k], t[k], err_msg=k)


def test_channel_zero_equals_grayscale():
    kw, _ = rgb_problem(40, 44)
    g = {**kw, "y": kw["y"][0], "x0": kw["x0"][0]}
    a = run(kw, 10, 2, 9)
    b = run(g, 10, 2, 9)
    for k in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(a[k][0], b[k], err_msg=k)


def test_colour_checkpoint_resume():
    kw, _ = rgb_problem(48, 50, kernel="gauss9", cnn=(4, 32))
    ref = run(kw, 9, 2, 31)
    s = Sampler(**kw, tiles=(2, 1))
    try:
        s.run(4, 2, 31)
        blob = s.save_checkpoint()
    finally:
        s.close()
    s = Sampler(**kw, tiles=(2, 1))
    try:
        s.load_checkpoint(blob)
        s.advance(5)
        x, z, t = s.state()
        mean, var, _ = s.moments()
    finally:
        s.close()
    assert t == 9
    for k, v in (("x", x), ("z", z), ("mean", mean), ("var", var)):
        np.testing.assert_array_equal(ref[k], v, err_msg=k)


def test_colour_rejections():
    kw, _ = rgb_problem(32, 32, cnn=(4, 16))
    with pytest.raises(Exception):
        Sampler(**kw)          # the colour DnCNN needs P >= 32
    kw, _ = rgb_problem(32, 32, z=False)
    w, g, ht = synth.ddfb_weights(2, 16, seed=3, image_channels=3)
    with pytest.raises(Exception):   # the colour DDFB adjoint (N = 48 folded columns) needs P >= 32
        Sampler(**kw, weights=w, n_layers=2, channels=16, alpha=1.0, eps=0.1, den_kind="ddfb", ddfb_gammas=g,
                ht_eps=ht)


# ---------------------------------------------------------------- colour DDFB and colour TV
def ddfb_rgb_problem(ny, nx, K=4, P=32):
    kw, pb = rgb_problem(ny, nx, kernel="gauss9", z=False)
    w, g, ht = synth.ddfb_weights(K, P, seed=7, image_channels=3)
    extra = dict(weights=w, n_layers=K, channels=P, alpha=1.0, eps=0.1, den_kind="ddfb", ddfb_gammas=g, ht_eps=ht)
    kw.update(extra)
    pb = oracle.Problem(**{**pb.__dict__, **extra})
    return kw, pb


def tv_rgb_problem(ny, nx, op="conv"):
    kw, pb = rgb_problem(ny, nx, op=op, kernel="gauss9", z=False, box=False)
    hp = params.tv_gaussian(kw["sigma2"], rho=1e-3)
    extra = dict(gamma=hp["gamma"], rho=hp["rho"], kappa=hp["kappa"], tv_beta=hp["tv_beta"])
    kw.update(extra)
    pb = oracle.Problem(**{**pb.__dict__, **extra})
    return kw, pb


@pytest.mark.parametrize("K,P,shape", [(1, 32, (40, 70)), (2, 64, (33, 140)), (4, 32, (45, 130)), (4, 64, (37, 61))])
def test_colour_ddfb_residual(K, P, shape):
    kw, _ = ddfb_rgb_problem(*shape, K=K, P=P)
    s = Sampler(**kw)
    try:
        s.reset(0, 1)
        G = s.denoiser_residual()
    finally:
        s.close()
    assert G.shape == (3,) + shape
    args = (kw["x0"], kw["weights"], kw["ddfb_gammas"], K, P, kw["ht_eps"])
    ref, ref16 = oracle.ddfb_residual(*args), oracle.ddfb_residual(*args, bf16_emulate=True)
    assert rel_l2(G, ref) <= 2e-2
    for c in range(3):
        assert rel_l2(G[c], ref16[c]) <= 2e-3, c


def test_colour_ddfb_chain_vs_oracle():
    kw, pb = ddfb_rgb_problem(45, 70)
    g = run(kw, 20, 4, 873)
    o16 = oracle.run(pb, 20, 4, 873, bf16_emulate=True)
    o = oracle.run(pb, 20, 4, 873)
    for k in ("x", "mean"):
        assert rel_l2(g[k], o16[k]) <= 2e-3, k
        assert rel_l2(g[k], o[k]) <= 2e-2, k


@pytest.mark.parametrize("op", ["conv", "mask"])
def test_colour_tv_chain_fp32_path(op):
    kw, pb = tv_rgb_problem(53, 61, op=op)
    s = Sampler(**kw)
    try:
        s.run(30, 5, 874)
        x, zv, _ = s.state()
        zh = s.tv_zh()
        mean, var, _ = s.moments()
    finally:
        s.close()
    o = oracle.run(pb, 30, 5, 874)
    for k, v in (("x", x), ("z", zv), ("zh", zh), ("mean", mean)):
        assert v.shape == (3, 53, 61)
        assert rel_l2(v, o[k]) <= 1e-5, k
    assert rel_l2(var, o["var"]) <= 1e-5   # R44
    assert np.all(x >= 0)


@pytest.mark.parametrize("case,tiles,flags", [("tv", (2, 2), 0), ("tv", (3, 1), FLAG_HALO_VIA_NCCL),
                                              ("ddfb", (2, 2), 0), ("ddfb", (3, 1), FLAG_HALO_VIA_NCCL)])
def test_colour_ddfb_tv_tiled_bitwise(case, tiles, flags):
    kw, _ = tv_rgb_problem(60, 66) if case == "tv" else ddfb_rgb_problem(60, 66)

    def go(t, f):
        s = Sampler(**kw, tiles=t, flags=f)
        try:
            s.run(10, 3, 55)
            x, z, _ = s.state()
            mean, var, _ = s.moments()
            out = dict(x=x, z=z, mean=mean, var=var)
            if case == "tv":
                out["zh"] = s.tv_zh()
            return out
        finally:
            s.close()
    a, b = go((1, 1), 0), go(tiles, flags)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
