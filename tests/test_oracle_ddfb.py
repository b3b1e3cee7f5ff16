"""Pins of the oracle's DDFB denoiser (Example sec:denoiser:cnn:ddfb, eq:ddfb_operator P:382-385,
eq:dfb_operator:T P:390-393; readings R39-R42) against things other than itself:

* W_k = 0 -> D(v) = proj_[0,1](v);
* a torch fp64 implementation with F.conv2d for W_k and F.conv_transpose2d for W_k^* (library
  routines, not the oracle's loops), for K = 1..4 and non-trivial HT clipping;
* the bf16-emulation mode against the same torch chain with explicit bfloat16 casts at the
  GPU's rounding points;
* the output box: D(v) in [0, 1];
* tiled chain with the DDFB prior bitwise equal to the untiled chain.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth


def _torch_ddfb(v, w, gammas, K, P, ht, emul=False):
    t = torch.from_numpy(np.asarray(v, np.float64))[None, None]
    W = torch.from_numpy(np.asarray(w, np.float64)).reshape(K, P, 1, 3, 3)
    bf = (lambda a: a.to(torch.bfloat16).to(torch.float64)) if emul else (lambda a: a)
    Wk = lambda k, s=1.0: bf(s * W[k - 1])
    u = bf(F.conv2d(bf(t), Wk(K), padding=1))                       # u0 = W_K v
    for k in range(1, K):
        a = F.conv_transpose2d(u, Wk(k), padding=1)                  # W_k^* u
        p = torch.clamp(t - a, 0.0, 1.0)
        u = bf(torch.clamp(u + F.conv2d(bf(p), Wk(k, float(gammas[k - 1])), padding=1), -ht, ht))
    a = F.conv_transpose2d(u, Wk(K, float(gammas[K - 1])), padding=1)
    d = torch.clamp(t - a, 0.0, 1.0)
    return (t - d)[0, 0].numpy()


def test_ddfb_zero_operator_is_box_projection():
    v = synth.ground_truth(9, 11) * 3 - 1
    w = np.zeros(4 * 8 * 9, np.float32)
    G = oracle.ddfb_residual(v, w, np.ones(4, np.float32), 4, 8, 0.05)
    np.testing.assert_allclose(G, v - np.clip(v, 0, 1), atol=0)


@pytest.mark.parametrize("K,P", [(1, 4), (2, 8), (4, 16)])
def test_ddfb_matches_torch(K, P):
    w, g, ht = synth.ddfb_weights(K, P, seed=K * 31 + P)
    v = synth.ground_truth(13, 17) * 1.4 - 0.2
    G = oracle.ddfb_residual(v, w, g, K, P, ht)
    ref = _torch_ddfb(v, w, g, K, P, ht)
    np.testing.assert_allclose(G, ref, atol=1e-12)
    d = v - G
    assert d.min() >= 0.0 and d.max() <= 1.0
    # the hard-tanh must actually clip somewhere for this pin to cover it
    if K > 1:
        t = torch.from_numpy(np.asarray(v, np.float64))[None, None]
        u0 = F.conv2d(t, torch.from_numpy(w.astype(np.float64)).reshape(K, P, 1, 3, 3)[K - 1], padding=1)
        assert float(u0.abs().max()) > ht


def test_ddfb_bf16_emulation_matches_torch_casts():
    K, P = 4, 16
    w, g, ht = synth.ddfb_weights(K, P, seed=5)
    v = synth.ground_truth(12, 15) * 1.2 - 0.1
    G = oracle.ddfb_residual(v, w, g, K, P, ht, bf16_emulate=True)
    np.testing.assert_allclose(G, _torch_ddfb(v, w, g, K, P, ht, emul=True), atol=1e-12)


@pytest.mark.parametrize("tiles", [(2, 2), (3, 1)])
def test_chain_with_ddfb_tiled_equals_untiled(tiles):
    ny, nx = 40, 37
    ky, kx = synth.gaussian_factors(5, 1.0)
    k2 = synth.outer(ky, kx)
    s2 = synth.noise_sigma2_blur(ny, nx, k2, 25.0)
    y = synth.observe_blur(ny, nx, k2, s2)
    w, g, ht = synth.ddfb_weights(4, 8, seed=2)
    pb = oracle.Problem(y=y, sigma2=s2, gamma=1e-4, op="conv", ksep=(ky, kx), weights=w, n_layers=4, channels=8,
                        alpha=1.0, eps=0.05, den_kind="ddfb", ddfb_gammas=g, ht_eps=ht, lam=0.05, c_lo=0, c_hi=1)
    a = oracle.run(pb, 5, 1, 870)
    t = oracle.run(pb, 5, 1, 870, tiles=tiles)
    for k in ("x", "mean", "var"):
        np.testing.assert_array_equal(a[k], t[k])


# ---------------------------------------------------------------- colour DDFB (W_k : C -> P)
def _torch_ddfb_c(v, w, gammas, K, P, C, ht, emul=False):
    t = torch.from_numpy(np.asarray(v, np.float64))[None]
    W = torch.from_numpy(np.asarray(w, np.float64)).reshape(K, P, C, 3, 3)
    bf = (lambda a: a.to(torch.bfloat16).to(torch.float64)) if emul else (lambda a: a)
    Wk = lambda k, s=1.0: bf(s * W[k - 1])
    u = bf(F.conv2d(bf(t), Wk(K), padding=1))                       # u0 = W_K v   (C -> P)
    for k in range(1, K):
        a = F.conv_transpose2d(u, Wk(k), padding=1)                  # W_k^* u      (P -> C)
        p = torch.clamp(t - a, 0.0, 1.0)
        u = bf(torch.clamp(u + F.conv2d(bf(p), Wk(k, float(gammas[k - 1])), padding=1), -ht, ht))
    a = F.conv_transpose2d(u, Wk(K, float(gammas[K - 1])), padding=1)
    d = torch.clamp(t - a, 0.0, 1.0)
    return (t - d)[0].numpy()


@pytest.mark.parametrize("K,P,C", [(1, 4, 3), (2, 8, 3), (4, 16, 3), (3, 6, 2)])
def test_colour_ddfb_matches_torch(K, P, C):
    w, g, ht = synth.ddfb_weights(K, P, seed=K * 7 + P, image_channels=C)
    v = synth.ground_truth_rgb(11, 14, C=C) * 1.4 - 0.2
    G = oracle.ddfb_residual(v, w, g, K, P, ht)
    np.testing.assert_allclose(G, _torch_ddfb_c(v, w, g, K, P, C, ht), atol=1e-12)
    np.testing.assert_allclose(oracle.ddfb_residual(v, w, g, K, P, ht, bf16_emulate=True),
                               _torch_ddfb_c(v, w, g, K, P, C, ht, emul=True), atol=1e-12)
    d = v - G
    assert d.min() >= 0.0 and d.max() <= 1.0
    assert oracle.ddfb_param_count(K, P, C) == w.size
    if K > 1:   # the channels are coupled through W_k: G of channel 0 depends on the others
        v2 = v.copy()
        v2[1:] = 0.5
        assert not np.allclose(oracle.ddfb_residual(v2, w, g, K, P, ht)[0], G[0])


def test_colour_ddfb_zero_operator_and_table_count():
    v = synth.ground_truth_rgb(7, 9) * 3 - 1
    G = oracle.ddfb_residual(v, np.zeros(4 * 8 * 3 * 9, np.float32), np.ones(4, np.float32), 4, 8, 0.05)
    np.testing.assert_allclose(G, v - np.clip(v, 0, 1), atol=0)
    assert oracle.ddfb_param_count(4, 64, 3) == 6912   # Table I, DDFB (K = 4)


def test_colour_ddfb_chain_iterations_against_rederivation():
    """one and two iterations of a C = 3 chain with the DDFB prior vs a scipy / torch re-derivation
    (H per channel, the DDFB residual from the torch chain above, streams 4c + s)."""
    from scipy.signal import convolve2d
    ny, nx, C, K, P, seed = 10, 12, 3, 3, 8, 17
    k = synth.random_kernel(5, 5, seed=4).astype(np.float64)
    s2 = 2e-3
    y = synth.observe_blur_rgb(ny, nx, k, s2, C=C)
    w, g, ht = synth.ddfb_weights(K, P, seed=9, image_channels=C)
    x0 = (synth.ground_truth_rgb(ny, nx, C=C) * 0.8 + 0.1).astype(np.float32)
    pb = oracle.Problem(y=y, sigma2=s2, gamma=4e-4, op="conv", kernel=k.astype(np.float32), weights=w, n_layers=K,
                        channels=P, alpha=1.0, eps=0.05, den_kind="ddfb", ddfb_gammas=g, ht_eps=ht, lam=0.05,
                        c_lo=0.0, c_hi=1.0, x0=x0)
    x = x0.astype(np.float64)
    for t in range(2):
        G = _torch_ddfb_c(x, w, g, K, P, C, ht)
        xn = np.empty_like(x)
        for c in range(C):
            grad = convolve2d(convolve2d(x[c], k, mode="same") - y[c], k[::-1, ::-1], mode="same") / s2
            xn[c] = (x[c] - pb.gamma * grad - (pb.alpha * pb.gamma / pb.eps ** 2) * G[c]
                     + (pb.gamma / pb.lam) * (np.clip(x[c], 0, 1) - x[c])
                     + np.sqrt(2 * pb.gamma) * oracle.normal_field(seed, t + 1, ny, nx, 4 * c))
        x = xn
        out = oracle.run(pb, t + 1, t + 1, seed)
        np.testing.assert_allclose(out["x"], x, rtol=0, atol=1e-10)
