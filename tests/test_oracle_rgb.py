"""Pins of the oracle's C-channel (RGB; reading R43) chain against things other than itself:

* the colour DnCNN residual (layer 1 C -> P, layer K P -> C) against torch.nn.functional.conv2d
  in fp64 (PyTorch cross-correlation, zero padding: an independent library routine);
* channel 0 of a C = 3 chain without a prior equals the grayscale chain on channel 0's data
  (same Philox streams 0 / 1), bit for bit;
* one and two iterations of every channel against a dense re-derivation (scipy convolve2d for H,
  the mask shared by the channels, noise streams 4c + s from oracle.normal_field), with the
  z block and the box term, and with the colour CNN residual taken from torch;
* the Poisson z1 block per channel (stream 4c + 2).
"""
import numpy as np
import pytest
import torch
from scipy.signal import convolve2d

import oracle
import synth


def _torch_dncnn(x, w, b, K, P, C):
    a = torch.from_numpy(np.asarray(x, np.float64))[None]
    off = boff = 0
    cin = C
    for k in range(1, K + 1):
        cout = C if k == K else P
        wk = torch.from_numpy(np.asarray(w[off:off + cout * cin * 9], np.float64).reshape(cout, cin, 3, 3))
        bk = torch.from_numpy(np.asarray(b[boff:boff + cout], np.float64))
        a = torch.nn.functional.conv2d(a, wk, bk, padding=1)
        if k < K:
            a = torch.relu(a)
        off += cout * cin * 9
        boff += cout
        cin = cout
    return a[0].numpy()


@pytest.mark.parametrize("K,P,C", [(4, 16, 3), (3, 8, 2), (2, 5, 3)])
def test_colour_dncnn_residual_vs_torch(K, P, C):
    rng = np.random.default_rng(K * 10 + C)
    x = rng.uniform(-0.2, 1.2, size=(C, 13, 17))
    w, b = synth.dncnn_weights(K, P, seed=3 + K, image_channels=C)
    b = (b + rng.uniform(-0.3, 0.3, size=b.shape)).astype(np.float32)   # biases large enough to matter
    G = oracle.dncnn_residual(x, w, b, K, P)
    np.testing.assert_allclose(G, _torch_dncnn(x, w, b, K, P, C), rtol=0, atol=1e-12)
    assert oracle.dncnn_param_count(K, P, C) == w.size + b.size


def _rgb_problem(ny, nx, op="conv", z=True, cnn=None, C=3):
    k = synth.random_kernel(5, 5, seed=11)
    s2 = 2e-3
    if op == "mask":
        y, m = synth.observe_mask_rgb(ny, nx, s2, C=C)
        kw = dict(op="mask", mask=m)
    else:
        y = synth.observe_blur_rgb(ny, nx, k.astype(np.float64), s2, C=C)
        kw = dict(op="conv", kernel=k)
    common = dict(sigma2=s2, gamma=4e-4, lam=0.05, c_lo=0.0, c_hi=1.0,
                  x0=(synth.ground_truth_rgb(ny, nx, C=C) * 0.8 + 0.1).astype(np.float32))
    if z:
        common.update(rho=5e-3, kappa=0.99 * 5e-3, z_lo=0.0, z_hi=1.0)
    if cnn:
        w, b = synth.dncnn_weights(cnn[0], cnn[1], seed=5, image_channels=C)
        common.update(weights=w, biases=b, n_layers=cnn[0], channels=cnn[1], alpha=1.0, eps=0.05)
    return oracle.Problem(y=y, **kw, **common), k


def test_channel_zero_equals_grayscale_chain():
    pb, k = _rgb_problem(23, 29)
    out = oracle.run(pb, 12, 4, seed=870)
    g = oracle.Problem(**{**pb.__dict__, "y": pb.y[0], "x0": pb.x0[0]})
    out1 = oracle.run(g, 12, 4, seed=870)
    for key in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(out[key][0], out1[key], err_msg=key)
        assert not np.array_equal(out[key][1], out1[key])   # the other channels draw other streams


@pytest.mark.parametrize("op,cnn", [("conv", None), ("mask", None), ("conv", (3, 8))])
def test_rgb_iterations_against_dense_rederivation(op, cnn):
    ny, nx, C, seed = 9, 11, 3, 41
    pb, k = _rgb_problem(ny, nx, op=op, cnn=cnn)
    kd = np.asarray(k, np.float64)
    y = np.asarray(pb.y, np.float64)
    x = np.asarray(pb.x0, np.float64)
    z = np.zeros_like(x)
    g, r, kp, lam = pb.gamma, pb.rho, pb.kappa, pb.lam
    for t in range(2):
        G = _torch_dncnn(x, pb.weights, pb.biases, cnn[0], cnn[1], C) if cnn else np.zeros_like(x)
        xn = np.empty_like(x)
        for c in range(C):
            if op == "mask":
                m = pb.mask.astype(np.float64)
                grad = m * (m * x[c] - y[c]) / pb.sigma2
            else:
                grad = convolve2d(convolve2d(x[c], kd, mode="same") - y[c], kd[::-1, ::-1], mode="same") / pb.sigma2
            xi = oracle.normal_field(seed, t + 1, ny, nx, 4 * c)
            xn[c] = (x[c] - g * grad - (g / r) * (x[c] - z[c]) - (pb.alpha * g / pb.eps ** 2) * G[c]
                     + (g / lam) * (np.clip(x[c], 0, 1) - x[c]) + np.sqrt(2 * g) * xi)
            ze = oracle.normal_field(seed, t + 1, ny, nx, 4 * c + 1)
            z[c] = np.clip(z[c] - (kp / r) * (z[c] - xn[c]) + np.sqrt(2 * kp) * ze, 0, 1)
        x = xn
        out = oracle.run(pb, t + 1, t + 1, seed)
        np.testing.assert_allclose(out["x"], x, rtol=0, atol=1e-11)
        np.testing.assert_allclose(out["z"], z, rtol=0, atol=1e-11)


def test_rgb_poisson_z1_block_per_channel():
    ny, nx, C, seed = 8, 10, 3, 5
    rng = np.random.default_rng(3)
    k = synth.random_kernel(3, 3, seed=2).astype(np.float64)
    eta = 40.0
    y = rng.poisson(eta * rng.uniform(0.1, 1, (C, ny, nx))).astype(np.float32)
    pb = oracle.Problem(y=y, sigma2=1.0, gamma=1e-3, op="poisson", kernel=k.astype(np.float32), eta=eta,
                        rho1=10.0, kappa1=9.9, rho=0.05, kappa=0.0495, z_lo=0.0, z_hi=np.inf,
                        x0=rng.uniform(0, 1, (C, ny, nx)).astype(np.float32))
    out = oracle.run(pb, 1, 1, seed)
    x0 = np.asarray(pb.x0, np.float64)
    for c in range(C):
        Hx0 = convolve2d(x0[c], k, mode="same")
        grad = eta * convolve2d(eta * Hx0, k[::-1, ::-1], mode="same") / pb.rho1   # z1^0 = 0
        xn = x0[c] - pb.gamma * grad - (pb.gamma / pb.rho) * x0[c] + np.sqrt(2 * pb.gamma) * oracle.normal_field(
            seed, 1, ny, nx, 4 * c)
        np.testing.assert_allclose(out["x"][c], xn, rtol=0, atol=1e-11)
        w1 = (pb.kappa1 / pb.rho1) * eta * convolve2d(xn, k, mode="same") + np.sqrt(2 * pb.kappa1) * \
            oracle.normal_field(seed, 1, ny, nx, 4 * c + 2)
        z1 = 0.5 * ((w1 - pb.kappa1) + np.sqrt((w1 - pb.kappa1) ** 2 + 4 * pb.kappa1 * y[c].astype(np.float64)))
        np.testing.assert_allclose(out["z1"][c], z1, rtol=0, atol=1e-11)


def test_rgb_rejects_tiles():
    pb, _ = _rgb_problem(12, 12)
    with pytest.raises(ValueError):
        oracle.run(pb, 1, 0, 1, tiles=(2, 1))
