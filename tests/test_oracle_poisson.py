"""Pins of the oracle's Poisson-deconvolution iteration (sec:poisson_deconvolution P:727-744,
P:777-782; readings R31-R34) against things other than itself:

* the KL prox against its closed-form special case (y = 0: soft threshold) and against a
  numerical minimiser of its variational definition (scipy), plus the stationarity condition;
* one full iteration (x, z1, z2) against a dense-matrix re-derivation with H built by
  scipy.signal.convolve2d (not the oracle's stencil) and the oracle's pinned normals;
* the tiled chain (line 11 exchange, z1 on worker blocks) bitwise equal to the untiled one.
"""
import numpy as np
import pytest
from scipy.optimize import minimize_scalar
from scipy.signal import convolve2d

import oracle
import synth


def test_prox_kl_zero_counts_is_soft_threshold():
    # y = 0: argmin kappa u + (u - v)^2 / 2 over u >= 0  ->  max(v - kappa, 0)
    for v in (-2.0, -0.1, 0.0, 0.2, 0.5, 3.0):
        for kappa in (0.01, 0.3, 2.0):
            assert oracle.prox_kl(v, 0.0, kappa) == pytest.approx(max(v - kappa, 0.0), abs=1e-15)


def test_prox_kl_matches_numerical_minimiser():
    rng = np.random.default_rng(31)
    for _ in range(60):
        v = float(rng.normal(0.0, 5.0))
        y = float(rng.integers(0, 40))
        kappa = float(10 ** rng.uniform(-2, 1))
        u = oracle.prox_kl(v, y, kappa)
        if y > 0:
            obj = lambda w: kappa * (w - y * np.log(w)) + 0.5 * (w - v) ** 2
            ref = minimize_scalar(obj, bounds=(1e-12, max(abs(v), y) + 10 * kappa + 10), method="bounded",
                                  options={"xatol": 1e-12}).x
            assert u == pytest.approx(ref, rel=1e-6, abs=1e-8)
            assert kappa * (1.0 - y / u) + u - v == pytest.approx(0.0, abs=1e-9 * (1 + abs(v) + y))
            assert u > 0
        else:
            assert u == pytest.approx(max(v - kappa, 0.0), abs=1e-15)


def _dense_conv(ny, nx, k):
    """Columns = H e_n with H the same-size true convolution, zero boundary (scipy)."""
    H = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros(ny * nx)
        e[n] = 1.0
        H[:, n] = convolve2d(e.reshape(ny, nx), k, mode="same", boundary="fill", fillvalue=0.0).ravel()
    return H


def _poisson_problem(ny, nx, seed=5, with_box=True):
    rng = np.random.default_rng(seed)
    k = rng.uniform(0.0, 1.0, size=(3, 5))
    k /= k.sum()
    xbar = rng.uniform(0.1, 1.0, size=(ny, nx))
    eta = 20.0
    y = rng.poisson(eta * convolve2d(xbar, k, mode="same")).astype(np.float32)
    pb = oracle.Problem(y=y, sigma2=1.0, gamma=2e-3, op="poisson", kernel=k.astype(np.float32),
                        eta=eta, rho1=10.0, kappa1=9.9, rho=0.05, kappa=0.0495, z_lo=0.0, z_hi=np.inf,
                        x0=rng.uniform(0.0, 1.0, size=(ny, nx)).astype(np.float32))
    if with_box:
        pb.lam, pb.c_lo, pb.c_hi = 0.02, 0.0, 1.0
    return pb


def test_one_poisson_iteration_against_dense_matrices():
    ny, nx = 6, 7
    pb = _poisson_problem(ny, nx)
    seed = 870
    k = np.asarray(pb.kernel, dtype=np.float64)
    H = _dense_conv(ny, nx, k)
    x0 = np.asarray(pb.x0, dtype=np.float64).ravel()
    y = np.asarray(pb.y, dtype=np.float64).ravel()
    z1_0 = np.zeros(ny * nx)
    z2_0 = np.zeros(ny * nx)
    xi = oracle.normal_field(seed, 1, ny, nx, 0).ravel()
    zeta2 = oracle.normal_field(seed, 1, ny, nx, 1).ravel()
    zeta1 = oracle.normal_field(seed, 1, ny, nx, 2).ravel()
    g, e, r1, k1, r2, k2 = pb.gamma, pb.eta, pb.rho1, pb.kappa1, pb.rho, pb.kappa
    # eq:sgs_pnp_ula_psgla:pnp_ula with f1 = 0, H2 = [eta H; I]
    x1 = (x0 - (g / r1) * (e * H.T @ (e * H @ x0 - z1_0)) - (g / r2) * (x0 - z2_0)
          + (g / pb.lam) * (np.clip(x0, pb.c_lo, pb.c_hi) - x0) + np.sqrt(2 * g) * xi)
    # eq:sgs_pnp_ula_psgla:psgla per block: z2 -> projection on R+, z1 -> KL prox
    z2_1 = np.maximum(z2_0 - (k2 / r2) * (z2_0 - x1) + np.sqrt(2 * k2) * zeta2, 0.0)
    v1 = z1_0 - (k1 / r1) * (z1_0 - e * H @ x1) + np.sqrt(2 * k1) * zeta1
    z1_1 = 0.5 * ((v1 - k1) + np.sqrt((v1 - k1) ** 2 + 4 * k1 * y))
    out = oracle.run(pb, n_iter=1, burn_in=1, seed=seed)
    np.testing.assert_allclose(out["x"].ravel(), x1, rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["z"].ravel(), z2_1, rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["z1"].ravel(), z1_1, rtol=0, atol=1e-12)


def test_two_poisson_iterations_against_dense_matrices():
    # the second iteration uses z1^1, z2^1 (coupling terms non-zero): pins the z1 residual sign
    ny, nx = 5, 6
    pb = _poisson_problem(ny, nx, seed=9, with_box=False)
    seed = 11
    k = np.asarray(pb.kernel, dtype=np.float64)
    H = _dense_conv(ny, nx, k)
    x = np.asarray(pb.x0, dtype=np.float64).ravel()
    y = np.asarray(pb.y, dtype=np.float64).ravel()
    z1 = np.zeros(ny * nx)
    z2 = np.zeros(ny * nx)
    g, e, r1, k1, r2, k2 = pb.gamma, pb.eta, pb.rho1, pb.kappa1, pb.rho, pb.kappa
    for t in range(2):
        xi, zeta2, zeta1 = (oracle.normal_field(seed, t + 1, ny, nx, s).ravel() for s in (0, 1, 2))
        xn = x - (g / r1) * (e * H.T @ (e * H @ x - z1)) - (g / r2) * (x - z2) + np.sqrt(2 * g) * xi
        z2 = np.maximum(z2 - (k2 / r2) * (z2 - xn) + np.sqrt(2 * k2) * zeta2, 0.0)
        v1 = z1 - (k1 / r1) * (z1 - e * H @ xn) + np.sqrt(2 * k1) * zeta1
        z1 = 0.5 * ((v1 - k1) + np.sqrt((v1 - k1) ** 2 + 4 * k1 * y))
        x = xn
    out = oracle.run(pb, n_iter=2, burn_in=2, seed=seed)
    np.testing.assert_allclose(out["x"].ravel(), x, rtol=0, atol=1e-11)
    np.testing.assert_allclose(out["z"].ravel(), z2, rtol=0, atol=1e-11)
    np.testing.assert_allclose(out["z1"].ravel(), z1, rtol=0, atol=1e-11)


@pytest.mark.parametrize("tiles", [(2, 2), (3, 1), (1, 3)])
def test_poisson_tiled_equals_untiled(tiles):
    ny, nx = 24, 21
    k = synth.outer(*synth.gaussian_factors(5, 1.0))
    rng = np.random.default_rng(3)
    xbar = synth.ground_truth(ny, nx, seed=2511)
    eta = 50.0
    y = rng.poisson(eta * np.clip(convolve2d(xbar, k, mode="same"), 0, None)).astype(np.float32)
    w, b = synth.dncnn_weights(4, 8, seed=7)
    pb = oracle.Problem(y=y, sigma2=1.0, gamma=1e-3, op="poisson", kernel=k.astype(np.float32), eta=eta,
                        rho1=10.0, kappa1=9.9, rho=1e-2, kappa=0.99e-2, z_lo=0.0, z_hi=np.inf,
                        lam=0.05, c_lo=0.0, c_hi=1.0, weights=w, biases=b, n_layers=4, channels=8,
                        alpha=1.0, eps=0.05)
    a = oracle.run(pb, n_iter=6, burn_in=2, seed=870)
    t = oracle.run(pb, n_iter=6, burn_in=2, seed=870, tiles=tiles)
    for key in ("x", "z", "z1", "mean", "var"):
        np.testing.assert_array_equal(a[key], t[key])
    assert np.all(a["z"] >= 0) and np.all(a["z1"] >= 0)
