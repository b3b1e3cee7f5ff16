"""GPU parity for the DDFB prior (Example sec:denoiser:cnn:ddfb P:378-395; DESIGN.md readings
R39-R42): the library's 2K single-operator tcgen05 launches (W_K v; proj(v - W_k^* u); HT(u +
gamma_k W_k p); v - proj(v - gamma_K W_K^* u)) against the pinned oracle, alone and inside the
chain, plus bitwise tiling invariance."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import rel_l2
from paper_2511_00870_b200 import Sampler, params
from paper_2511_00870_b200._lib import FLAG_HALO_VIA_NCCL

pytestmark = pytest.mark.gpu


def ddfb_problem(ny, nx, K=4, P=32, kernel="gauss5"):
    L = int(kernel[5:])
    ky, kx = synth.gaussian_factors(L, 1.0 if L == 5 else 2.0)
    k2 = synth.outer(ky, kx)
    s2 = synth.noise_sigma2_blur(ny, nx, k2, 25.0)
    y = synth.observe_blur(ny, nx, k2, s2)
    hp = params.gaussian_pnp(s2, 1.0, 1.0)
    w, g, ht = synth.ddfb_weights(K, P, seed=11 * K + P)
    common = dict(sigma2=s2, gamma=hp["gamma"], lam=hp["lam"], c_lo=0.0, c_hi=1.0, weights=w, n_layers=K,
                  channels=P, alpha=1.0, eps=hp["eps"], ddfb_gammas=g, ht_eps=ht,
                  x0=(synth.ground_truth(ny, nx) * 1.1 - 0.05).astype(np.float32))
    kw = dict(ny=ny, nx=nx, y=y, kernel_sep=(ky, kx), den_kind="ddfb", **common)
    pb = oracle.Problem(y=y, op="conv", ksep=(ky, kx), den_kind="ddfb", **common)
    return kw, pb


@pytest.mark.parametrize("K,P,shape", [(4, 32, (70, 83)), (4, 64, (66, 131)), (2, 16, (40, 300)), (1, 32, (33, 47))])
def test_ddfb_residual_vs_oracle(K, P, shape):
    ny, nx = shape
    kw, pb = ddfb_problem(ny, nx, K, P)
    s = Sampler(**kw)
    try:
        s.reset(0, 1)
        G = s.denoiser_residual()
    finally:
        s.close()
    x0 = np.asarray(kw["x0"], np.float64)
    ref = oracle.ddfb_residual(x0, kw["weights"], kw["ddfb_gammas"], K, P, kw["ht_eps"])
    refb = oracle.ddfb_residual(x0, kw["weights"], kw["ddfb_gammas"], K, P, kw["ht_eps"], bf16_emulate=True)
    assert rel_l2(G, ref) <= 2e-2
    assert rel_l2(G, refb) <= 2e-3


def test_chain_with_ddfb_vs_oracle():
    kw, pb = ddfb_problem(64, 72, 4, 32)
    s = Sampler(**kw)
    try:
        s.run(30, 5, 873)
        x, _, _ = s.state()
        mean, var, _ = s.moments()
    finally:
        s.close()
    o = oracle.run(pb, 30, 5, 873)
    ob = oracle.run(pb, 30, 5, 873, bf16_emulate=True)
    assert rel_l2(x, o["x"]) <= 2e-2 and rel_l2(mean, o["mean"]) <= 2e-2
    assert rel_l2(x, ob["x"]) <= 2e-3 and rel_l2(mean, ob["mean"]) <= 2e-3


@pytest.mark.parametrize("tiles,flags", [((2, 2), 0), ((3, 1), FLAG_HALO_VIA_NCCL)])
def test_ddfb_tiled_bitwise(tiles, flags):
    kw, _ = ddfb_problem(66, 75, 4, 16)
    out = []
    for t, f in [((1, 1), 0), (tiles, flags)]:
        s = Sampler(**kw, tiles=t, flags=f)
        try:
            s.run(10, 3, 9)
            x, _, _ = s.state()
            m, v, _ = s.moments()
            out.append((x, m, v))
        finally:
            s.close()
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)
