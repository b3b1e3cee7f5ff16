"""The GPU chain against closed forms (BASELINE config C4: "linear-Gaussian posterior, closed-form
mean/variance check"), independent of the oracle: with no denoiser and a Gaussian Moreau term
(box [c, c]), the ULA recursion of eq:sgs_pnp_ula_psgla:pnp_ula is a Gaussian AR(1) chain whose
stationary law is N(P^-1 b, (P - gamma P^2 / 2)^-1), P = H^T H / sigma^2 + I / lambda,
b = H^T y / sigma^2 + c / lambda (SURVEY 8(c) closed forms).

* mask (diagonal P, exact per pixel, 512 x 512 in 2 x 2 tiles): pooled z-scores of the MMSE mean
  and of the variance estimate;
* blur (48 x 48, random asymmetric 5 x 5 kernel): dense P from scipy convolve2d columns, mean by a
  linear solve, variance from the dense covariance."""
import numpy as np
import pytest
from scipy.signal import convolve2d

import synth
from paper_2511_00870_b200 import Sampler

pytestmark = pytest.mark.gpu


def test_mask_chain_matches_the_closed_form():
    ny, nx = 512, 512
    s2, lam, c = 0.05, 0.1, 0.5
    y, m = synth.observe_mask(ny, nx, s2)
    p = m / s2 + 1 / lam
    gamma = 0.9 / p.max()
    mu = (m * y.astype(np.float64) / s2 + c / lam) / p
    v = 1 / (p * (1 - gamma * p / 2))
    T, burn = 20000, 200
    s = Sampler(ny=ny, nx=nx, y=y, op="mask", mask=m, sigma2=s2, gamma=gamma, lam=lam, c_lo=c, c_hi=c,
                tiles=(2, 2))
    try:
        s.run(T + burn, burn, 2024)
        mean, var, n = s.moments()
    finally:
        s.close()
    assert n == T
    phi = 1 - gamma * p
    z_mean = (mean - mu) / np.sqrt(2 / (gamma * p ** 2 * T))
    z_var = (var - v) / np.sqrt(2 * v ** 2 * (1 + phi ** 2) / ((1 - phi ** 2) * T))
    N = z_mean.size
    assert abs(z_mean.mean()) < 4 / np.sqrt(N)
    assert 0.9 < np.mean(z_mean ** 2) < 1.1
    assert abs(z_var.mean()) < 0.05
    assert 0.85 < np.mean(z_var ** 2) < 1.15


def test_blur_chain_matches_the_closed_form():
    ny, nx = 48, 48
    k = synth.random_kernel(5, 5, seed=3).astype(np.float64)
    s2, lam, c = 1e-2, 0.05, 0.5
    y = synth.observe_blur(ny, nx, k, s2)
    H = np.zeros((ny * nx, ny * nx))
    for j in range(ny * nx):
        e = np.zeros(ny * nx)
        e[j] = 1.0
        H[:, j] = convolve2d(e.reshape(ny, nx), k, mode="same").ravel()
    P = H.T @ H / s2 + np.eye(ny * nx) / lam
    b = H.T @ y.astype(np.float64).ravel() / s2 + c / lam
    mu = np.linalg.solve(P, b)
    gamma = 0.99 / np.linalg.eigvalsh(P).max()
    Sigma_diag = np.diag(np.linalg.inv(P - gamma * P @ P / 2))
    T, burn = 40000, 400
    s = Sampler(ny=ny, nx=nx, y=y, kernel=k.astype(np.float32), sigma2=s2, gamma=gamma, lam=lam, c_lo=c, c_hi=c)
    try:
        s.run(T + burn, burn, 2025)
        mean, var, _ = s.moments()
    finally:
        s.close()
    Pinv = np.linalg.inv(P)
    se = np.sqrt(2 / (gamma * T) * np.sum(Pinv ** 2, axis=0))
    z = (mean.ravel() - mu) / se
    assert abs(z.mean()) < 0.3
    assert 0.5 < np.mean(z ** 2) < 1.6
    ratio = var.ravel() / Sigma_diag
    assert abs(ratio.mean() - 1) < 0.03
