"""Pins of the oracle's TV-prior iteration (item:prior_choice:tv P:786-809; DESIGN.md readings
R35-R38) against things other than itself:

* D / D^T: SPEC examples, constant image, adjoint dot test, ||D||^2 <= 8 and close
  to 8 (power iteration), a dense D built from numpy.diff;
* the l2,1 prox: SPEC closed-form example, shrink-to-zero, tau = 0, and a numerical
  minimiser of tau ||u|| + ||u - g||^2 / 2 (scipy);
* one and two full iterations (x by PSGLA with p = 1_{R+}, z ~ D x) against a dense-matrix
  re-derivation (scipy convolve2d for H, numpy.diff for D);
* the tiled chain bitwise equal to the untiled one.
"""
import numpy as np
import pytest
from scipy.optimize import minimize
from scipy.signal import convolve2d

import oracle
import synth


def test_grad2d_examples():
    gv, gh = oracle.grad2d(np.array([[1.0], [3.0], [6.0]]))
    np.testing.assert_array_equal(gv.ravel(), [2.0, 3.0, 0.0])
    np.testing.assert_array_equal(gh.ravel(), [0.0, 0.0, 0.0])
    gv, gh = oracle.grad2d(np.full((4, 5), 2.5))
    assert not gv.any() and not gh.any()


def _dense_D(ny, nx):
    """Rows: vertical then horizontal differences, built from numpy.diff of unit images."""
    Dv = np.zeros((ny * nx, ny * nx))
    Dh = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros((ny, nx))
        e.ravel()[n] = 1.0
        dv = np.zeros((ny, nx))
        dv[:-1, :] = np.diff(e, axis=0)
        dh = np.zeros((ny, nx))
        dh[:, :-1] = np.diff(e, axis=1)
        Dv[:, n] = dv.ravel()
        Dh[:, n] = dh.ravel()
    return Dv, Dh


def test_grad2d_matches_dense_and_adjoint():
    rng = np.random.default_rng(35)
    for ny, nx in [(6, 6), (5, 9), (1, 7), (8, 1)]:
        x = rng.normal(size=(ny, nx))
        gv, gh = oracle.grad2d(x)
        Dv, Dh = _dense_D(ny, nx)
        np.testing.assert_allclose(gv.ravel(), Dv @ x.ravel(), atol=1e-14)
        np.testing.assert_allclose(gh.ravel(), Dh @ x.ravel(), atol=1e-14)
        uv, uh = rng.normal(size=(ny, nx)), rng.normal(size=(ny, nx))
        lhs = np.sum(gv * uv) + np.sum(gh * uh)
        rhs = np.sum(x * oracle.grad2d_adj(uv, uh))
        assert lhs == pytest.approx(rhs, rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(oracle.grad2d_adj(uv, uh).ravel(), Dv.T @ uv.ravel() + Dh.T @ uh.ravel(),
                                   atol=1e-13)


def test_grad2d_norm_bound():
    ny, nx = 32, 32
    v = np.random.default_rng(1).normal(size=(ny, nx))
    for _ in range(300):
        v = oracle.grad2d_adj(*oracle.grad2d(v))
        v /= np.linalg.norm(v)
    gv, gh = oracle.grad2d(v)
    nrm2 = np.sum(gv ** 2) + np.sum(gh ** 2)
    assert 7.8 < nrm2 <= 8.0


def test_prox_l21_examples_and_minimiser():
    assert oracle.prox_l21(3.0, 4.0, 1.0) == pytest.approx((2.4, 3.2), abs=1e-15)
    assert oracle.prox_l21(0.3, -0.4, 0.5) == (0.0, 0.0)
    assert oracle.prox_l21(0.3, -0.4, 0.0) == (0.3, -0.4)
    assert oracle.prox_l21(0.0, 0.0, 0.7) == (0.0, 0.0)
    rng = np.random.default_rng(36)
    for _ in range(40):
        g = rng.normal(0, 3, size=2)
        tau = float(rng.uniform(0, 4))
        obj = lambda u: tau * np.hypot(u[0], u[1]) + 0.5 * np.sum((u - g) ** 2)
        ref = minimize(obj, g * 0.5 + 1e-3, method="Nelder-Mead", options={"xatol": 1e-10, "fatol": 1e-14,
                                                                          "maxiter": 4000}).x
        out = np.array(oracle.prox_l21(g[0], g[1], tau))
        assert obj(out) <= obj(ref) + 1e-10
        np.testing.assert_allclose(out, ref, atol=1e-5)


def _dense_conv(ny, nx, k):
    H = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros(ny * nx)
        e[n] = 1.0
        H[:, n] = convolve2d(e.reshape(ny, nx), k, mode="same").ravel()
    return H


def _tv_problem(ny, nx, seed=4):
    rng = np.random.default_rng(seed)
    k = rng.uniform(0, 1, size=(3, 3))
    k /= k.sum()
    y = (convolve2d(rng.uniform(0, 1, (ny, nx)), k, mode="same") + 0.05 * rng.normal(size=(ny, nx)))
    return oracle.Problem(y=y.astype(np.float32), sigma2=0.05 ** 2, gamma=2e-3, op="conv",
                          kernel=k.astype(np.float32), rho=0.05, kappa=0.05 * 0.99 / 8, tv_beta=4.0,
                          x0=rng.uniform(0, 1, (ny, nx)).astype(np.float32))


@pytest.mark.parametrize("n_iter", [1, 2])
def test_tv_iterations_against_dense_matrices(n_iter):
    ny, nx = 6, 7
    pb = _tv_problem(ny, nx)
    seed = 41
    H = _dense_conv(ny, nx, np.asarray(pb.kernel, np.float64))
    Dv, Dh = _dense_D(ny, nx)
    y = np.asarray(pb.y, np.float64).ravel()
    x = np.asarray(pb.x0, np.float64).ravel()
    zv = np.zeros(ny * nx)
    zh = np.zeros(ny * nx)
    g, r, k, tau = pb.gamma, pb.rho, pb.kappa, pb.kappa * pb.tv_beta
    for t in range(n_iter):
        xi, zev, zeh = (oracle.normal_field(seed, t + 1, ny, nx, s).ravel() for s in (0, 1, 3))
        # PSGLA x-step with p = 1_{R+}: projection after the Langevin step
        v = (x - g * H.T @ (H @ x - y) / pb.sigma2 - (g / r) * (Dv.T @ (Dv @ x - zv) + Dh.T @ (Dh @ x - zh))
             + np.sqrt(2 * g) * xi)
        x = np.maximum(v, 0.0)
        # z-step: prox of kappa beta ||.||_{2,1} (block soft threshold per pixel)
        wv = zv - (k / r) * (zv - Dv @ x) + np.sqrt(2 * k) * zev
        wh = zh - (k / r) * (zh - Dh @ x) + np.sqrt(2 * k) * zeh
        nrm = np.hypot(wv, wh)
        sc = np.where(nrm > tau, 1 - tau / np.where(nrm > 0, nrm, 1), 0.0)
        zv, zh = wv * sc, wh * sc
    out = oracle.run(pb, n_iter=n_iter, burn_in=n_iter, seed=seed)
    np.testing.assert_allclose(out["x"].ravel(), x, rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["z"].ravel(), zv, rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["zh"].ravel(), zh, rtol=0, atol=1e-12)


@pytest.mark.parametrize("tiles", [(2, 2), (3, 1), (1, 3)])
def test_tv_tiled_equals_untiled(tiles):
    ny, nx = 27, 25
    ky, kx = synth.gaussian_factors(5, 1.0)
    k2 = synth.outer(ky, kx)
    s2 = synth.noise_sigma2_blur(ny, nx, k2, 25.0)
    y = synth.observe_blur(ny, nx, k2, s2)
    pb = oracle.Problem(y=y, sigma2=s2, gamma=1e-4, op="conv", ksep=(ky, kx), rho=1e-3, kappa=0.99e-3 / 8,
                        tv_beta=40.0)
    a = oracle.run(pb, n_iter=6, burn_in=2, seed=870)
    t = oracle.run(pb, n_iter=6, burn_in=2, seed=870, tiles=tiles)
    for key in ("x", "z", "zh", "mean", "var"):
        np.testing.assert_array_equal(a[key], t[key])
    assert np.all(a["x"] >= 0)


def test_poisson_tv_iteration_against_dense_matrices():
    """Poisson noise with the TV prior: f1 = 0, z1 ~ eta H x (KL prox, stream 2),
    z = (z_v, z_h) ~ D x (l2,1 prox, streams 1 / 3), x by PSGLA on R+."""
    ny, nx = 6, 7
    rng = np.random.default_rng(12)
    k = rng.uniform(0, 1, size=(3, 3))
    k /= k.sum()
    eta = 30.0
    y = rng.poisson(eta * convolve2d(rng.uniform(0.1, 1, (ny, nx)), k, mode="same")).astype(np.float32)
    pb = oracle.Problem(y=y, sigma2=1.0, gamma=1e-3, op="poisson", kernel=k.astype(np.float32), eta=eta,
                        rho1=10.0, kappa1=9.9, rho=0.05, kappa=0.05 * 0.99 / 8, tv_beta=3.0,
                        x0=rng.uniform(0, 1, (ny, nx)).astype(np.float32))
    seed = 17
    H = _dense_conv(ny, nx, np.asarray(pb.kernel, np.float64))
    Dv, Dh = _dense_D(ny, nx)
    x = np.asarray(pb.x0, np.float64).ravel()
    yy = np.asarray(y, np.float64).ravel()
    z1, zv, zh = np.zeros(ny * nx), np.zeros(ny * nx), np.zeros(ny * nx)
    g, r, kp, tau, e, r1, k1 = pb.gamma, pb.rho, pb.kappa, pb.kappa * pb.tv_beta, eta, pb.rho1, pb.kappa1
    for t in range(2):
        xi, zev, zeh, ze1 = (oracle.normal_field(seed, t + 1, ny, nx, s).ravel() for s in (0, 1, 3, 2))
        v = (x - (g / r1) * e * H.T @ (e * H @ x - z1) - (g / r) * (Dv.T @ (Dv @ x - zv) + Dh.T @ (Dh @ x - zh))
             + np.sqrt(2 * g) * xi)
        x = np.maximum(v, 0.0)
        wv = zv - (kp / r) * (zv - Dv @ x) + np.sqrt(2 * kp) * zev
        wh = zh - (kp / r) * (zh - Dh @ x) + np.sqrt(2 * kp) * zeh
        nrm = np.hypot(wv, wh)
        sc = np.where(nrm > tau, 1 - tau / np.where(nrm > 0, nrm, 1), 0.0)
        zv, zh = wv * sc, wh * sc
        w1 = z1 - (k1 / r1) * (z1 - e * H @ x) + np.sqrt(2 * k1) * ze1
        z1 = 0.5 * ((w1 - k1) + np.sqrt((w1 - k1) ** 2 + 4 * k1 * yy))
    out = oracle.run(pb, n_iter=2, burn_in=2, seed=seed)
    for key, ref in (("x", x), ("z", zv), ("zh", zh), ("z1", z1)):
        np.testing.assert_allclose(out[key].ravel(), ref, rtol=0, atol=1e-11, err_msg=key)
    t2 = oracle.run(pb, n_iter=2, burn_in=2, seed=seed, tiles=(2, 1))
    for key in ("x", "z", "zh", "z1"):
        np.testing.assert_array_equal(out[key], t2[key])


# ---------------------------------------------------------------- colour TV (C = 3)
def test_colour_tv_iterations_against_dense_matrices():
    """Colour TV (P:795-798 with N = C x Ny x Nx): D acts on each channel plane and
    ||z||_{2,1} sums the 2-norms of the per-channel-pixel gradient pairs -- channel-wise isotropic
    TV with per-channel streams; one and two
    iterations of every channel vs the dense re-derivation, noise streams 4c + 0 / 1 / 3 (R43)."""
    ny, nx, C, seed = 6, 7, 3, 43
    rng = np.random.default_rng(8)
    k = rng.uniform(0, 1, size=(3, 3))
    k /= k.sum()
    y = np.stack([convolve2d(rng.uniform(0, 1, (ny, nx)), k, mode="same") + 0.05 * rng.normal(size=(ny, nx))
                  for _ in range(C)]).astype(np.float32)
    pb = oracle.Problem(y=y, sigma2=0.05 ** 2, gamma=2e-3, op="conv", kernel=k.astype(np.float32), rho=0.05,
                        kappa=0.05 * 0.99 / 8, tv_beta=4.0, x0=rng.uniform(0, 1, (C, ny, nx)).astype(np.float32))
    H = _dense_conv(ny, nx, np.asarray(pb.kernel, np.float64))
    Dv, Dh = _dense_D(ny, nx)
    g, r, kp, tau = pb.gamma, pb.rho, pb.kappa, pb.kappa * pb.tv_beta
    x = np.asarray(pb.x0, np.float64).reshape(C, -1).copy()
    zv, zh = np.zeros_like(x), np.zeros_like(x)
    for t in range(2):
        for c in range(C):
            xi, zev, zeh = (oracle.normal_field(seed, t + 1, ny, nx, 4 * c + s).ravel() for s in (0, 1, 3))
            yc = np.asarray(y[c], np.float64).ravel()
            v = (x[c] - g * H.T @ (H @ x[c] - yc) / pb.sigma2
                 - (g / r) * (Dv.T @ (Dv @ x[c] - zv[c]) + Dh.T @ (Dh @ x[c] - zh[c])) + np.sqrt(2 * g) * xi)
            x[c] = np.maximum(v, 0.0)
            wv = zv[c] - (kp / r) * (zv[c] - Dv @ x[c]) + np.sqrt(2 * kp) * zev
            wh = zh[c] - (kp / r) * (zh[c] - Dh @ x[c]) + np.sqrt(2 * kp) * zeh
            nrm = np.hypot(wv, wh)
            sc = np.where(nrm > tau, 1 - tau / np.where(nrm > 0, nrm, 1), 0.0)
            zv[c], zh[c] = wv * sc, wh * sc
        out = oracle.run(pb, n_iter=t + 1, burn_in=t + 1, seed=seed)
        np.testing.assert_allclose(out["x"].reshape(C, -1), x, rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["z"].reshape(C, -1), zv, rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["zh"].reshape(C, -1), zh, rtol=0, atol=1e-12)


def test_colour_tv_channel_zero_equals_grayscale():
    ny, nx = 15, 13
    ky, kx = synth.gaussian_factors(5, 1.0)
    k2 = synth.outer(ky, kx)
    y = synth.observe_blur_rgb(ny, nx, k2, 1e-3)
    common = dict(sigma2=1e-3, gamma=1e-4, op="conv", ksep=(ky, kx), rho=1e-3, kappa=0.99e-3 / 8, tv_beta=40.0)
    a = oracle.run(oracle.Problem(y=y, **common), 5, 2, 870)
    b = oracle.run(oracle.Problem(y=y[0], **common), 5, 2, 870)
    for key in ("x", "z", "zh", "mean", "var"):
        np.testing.assert_array_equal(a[key][0], b[key])
