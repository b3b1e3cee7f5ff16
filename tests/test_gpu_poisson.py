"""GPU parity for the Poisson-deconvolution iteration (sec:poisson_deconvolution P:727-744,
P:777-782; readings R31-R34): the C-ABI library (OP_POISSON: two AXDA blocks, KL
prox, z1 on tile (+) r_H) against the pinned oracle on the same seeded inputs, and the
bitwise tiling invariance of x, z2, z1 and the moments."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import rel_l2
from paper_2511_00870_b200 import Sampler, params
from paper_2511_00870_b200._lib import FLAG_HALO_VIA_NCCL

pytestmark = pytest.mark.gpu


def poisson_problem(ny, nx, *, kernel="gauss9", cnn=None, eta=250.0, box=True):
    if kernel.startswith("gauss"):
        L = int(kernel[5:])
        ky, kx = synth.gaussian_factors(L, 1.0 if L == 5 else 2.0)
        k2 = synth.outer(ky, kx)
        ks, ko = dict(kernel_sep=(ky, kx)), dict(ksep=(ky, kx))
    else:
        L = int(kernel[6:])
        k = synth.random_kernel(L, L, seed=L)
        k2 = k.astype(np.float64)
        ks, ko = dict(kernel=k), dict(kernel=k)
    y = synth.observe_poisson(ny, nx, k2, eta)
    hp = params.poisson_pnp(eta)
    common = dict(gamma=hp["gamma"], rho=hp["rho"], kappa=hp["kappa"], z_lo=0.0, z_hi=np.inf,
                  eta=hp["eta"], rho1=hp["rho1"], kappa1=hp["kappa1"],
                  x0=(synth.ground_truth(ny, nx) * 0.8 + 0.1).astype(np.float32))
    if box:
        common.update(lam=hp["lam"], c_lo=0.0, c_hi=1.0)
    if cnn is not None:
        K, P = cnn
        w, b = synth.dncnn_weights(K, P, seed=2513)
        common.update(weights=w, biases=b, n_layers=K, channels=P, alpha=1.0, eps=hp["eps"])
    kw = dict(ny=ny, nx=nx, y=y, sigma2=1.0, op="poisson", **ks, **common)
    pb = oracle.Problem(y=y, sigma2=1.0, op="poisson", **ko, **common)
    return kw, pb


def gpu_poisson(kw, n_iter, burn_in, seed, tiles=(1, 1), flags=0):
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        s.run(n_iter, burn_in, seed)
        x, z, t = s.state()
        z1 = s.z1()
        mean, var, _ = s.moments()
        return dict(x=x, z=z, z1=z1, mean=mean, var=var)
    finally:
        s.close()


@pytest.mark.parametrize("kernel,shape", [("gauss9", (70, 83)), ("random5", (61, 57))])
def test_poisson_chain_fp32_path_vs_oracle(kernel, shape):
    ny, nx = shape
    kw, pb = poisson_problem(ny, nx, kernel=kernel)
    g = gpu_poisson(kw, 50, 10, seed=870)
    o = oracle.run(pb, 50, 10, seed=870)
    assert rel_l2(g["x"], o["x"]) <= 1e-5
    assert rel_l2(g["z"], o["z"]) <= 1e-5
    assert rel_l2(g["z1"], o["z1"]) <= 1e-5
    assert rel_l2(g["mean"], o["mean"]) <= 1e-5
    assert rel_l2(g["var"], o["var"]) <= 1e-5   # SURVEY A16; conditioning: DESIGN.md R44
    assert np.all(g["z1"] >= 0) and np.all(g["z"] >= 0)


def test_poisson_chain_with_cnn_vs_oracle():
    ny, nx = 64, 72
    kw, pb = poisson_problem(ny, nx, cnn=(4, 16))
    g = gpu_poisson(kw, 30, 5, seed=871)
    o = oracle.run(pb, 30, 5, seed=871)
    ob = oracle.run(pb, 30, 5, seed=871, bf16_emulate=True)
    assert rel_l2(g["x"], o["x"]) <= 2e-2
    assert rel_l2(g["z1"], o["z1"]) <= 2e-2
    assert rel_l2(g["x"], ob["x"]) <= 2e-3
    assert rel_l2(g["z1"], ob["z1"]) <= 2e-3


@pytest.mark.parametrize("tiles,flags", [((2, 2), 0), ((3, 1), 0), ((1, 3), FLAG_HALO_VIA_NCCL)])
def test_poisson_tiled_bitwise(tiles, flags):
    ny, nx = 66, 75
    kw, _ = poisson_problem(ny, nx, kernel="random5", cnn=(4, 16))
    a = gpu_poisson(kw, 12, 4, seed=5)
    b = gpu_poisson(kw, 12, 4, seed=5, tiles=tiles, flags=flags)
    for k in ("x", "z", "z1", "mean", "var"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_poisson_rejects_bad_kappa1():
    kw, _ = poisson_problem(40, 40, kernel="gauss5")
    kw = dict(kw, kappa1=kw["rho1"] * 1.5)
    with pytest.raises(Exception):
        Sampler(**kw)
