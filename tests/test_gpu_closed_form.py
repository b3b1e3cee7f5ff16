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


# ---------------------------------------------------------------- BASELINE configs[3] at its own size
def _probes_c4(n):
    """~64 probe pixels of the 2048^2 C4 image: the 4 corners, 4 edge midpoints, both sides of the
    7 seams of an 8 x 1 row-strip tiling (at 4 columns: 56), the centre -- in groups whose members
    are >= 128 px apart (Chebyshev), so one linear solve per group gives every member's diagonal
    entry (the inverse operators decay like 0.3^(d/4) here: < 1e-9 at 128 px)."""
    pts = [(0, 0), (0, n - 1), (n - 1, 0), (n - 1, n - 1), (0, n // 2), (n - 1, n // 2), (n // 2, 0),
           (n // 2, n - 1), (n // 2 + 64, n // 2 + 64)]
    for k in range(1, 8):
        r = k * n // 8
        for col in (3, n // 3, 2 * n // 3, n - 4):
            pts += [(r - 1, col), (r, col)]
    groups = []
    for p in pts:
        for g in groups:
            if all(max(abs(p[0] - q[0]), abs(p[1] - q[1])) >= 128 for q in g):
                g.append(p)
                break
        else:
            groups.append([p])
    return pts, groups


def test_c4_2048_blur_chain_matches_the_closed_form():
    """BASELINE.json configs[3] / SURVEY 8(c) C4 row: 2048^2, 9 x 9 Gaussian blur (sigma_b = 2),
    sigma^2 = 1e-2, lambda = 0.05, c = 0.5, gamma = 0.99/120, x0 = 0, burn-in 200, T = 5000, 4 seeds,
    on one GPU in 8 x 1 row strips (the tiling of the 8-GPU run).  Closed forms by conjugate gradients
    on the zero-boundary convolution (scipy.ndimage, no oracle): mu = P^-1 b over the whole image,
    and at 65 probe pixels (corners, edges, both sides of every strip seam, centre)
    var_i = e_i^T (P - gamma P^2 / 2)^-1 e_i and Var(mean_i) = (2 / (gamma T)) ||P^-1 e_i||^2."""
    from scipy.ndimage import convolve1d, correlate1d
    from scipy.sparse.linalg import LinearOperator, cg

    n = 2048
    ky, kx = synth.gaussian_factors(9, 2.0)
    k2 = synth.outer(ky, kx)
    s2, lam, c, gamma = 1e-2, 0.05, 0.5, 0.99 / 120
    y = synth.observe_blur(n, n, k2, s2)
    kyd, kxd = ky.astype(np.float64), kx.astype(np.float64)

    def H(v):
        return convolve1d(convolve1d(v, kyd, axis=0, mode="constant"), kxd, axis=1, mode="constant")

    def Ht(v):
        return correlate1d(correlate1d(v, kyd, axis=0, mode="constant"), kxd, axis=1, mode="constant")

    def Pm(v):
        v = v.reshape(n, n)
        return (Ht(H(v)) / s2 + v / lam).ravel()

    def Am(v):
        pv = Pm(v)
        return pv - gamma / 2 * Pm(pv)

    P_op = LinearOperator((n * n, n * n), matvec=Pm, dtype=np.float64)
    A_op = LinearOperator((n * n, n * n), matvec=Am, dtype=np.float64)
    b = (Ht(y.astype(np.float64)) / s2 + c / lam).ravel()
    mu, info = cg(P_op, b, rtol=1e-11, maxiter=500)
    assert info == 0
    mu = mu.reshape(n, n)
    pts, groups = _probes_c4(n)
    var_true, se_mean = {}, {}
    for g in groups:
        e = np.zeros(n * n)
        for (i, j) in g:
            e[i * n + j] = 1.0
        w, info = cg(A_op, e, rtol=1e-11, maxiter=500)
        assert info == 0
        u, info = cg(P_op, e, rtol=1e-11, maxiter=500)
        assert info == 0
        w, u = w.reshape(n, n), u.reshape(n, n)
        for (i, j) in g:
            var_true[(i, j)] = w[i, j]
            win = u[max(i - 64, 0):i + 65, max(j - 64, 0):j + 65]   # P^-1 e_i, separated from the others
            se_mean[(i, j)] = np.sqrt(2 / (gamma * 5000) * np.sum(win ** 2))

    T, burn = 5000, 200
    zm, zv, ratio = [], [], []
    for seed in (870, 871, 872, 873):
        s = Sampler(ny=n, nx=n, y=y, kernel_sep=(ky, kx), sigma2=s2, gamma=gamma, lam=lam, c_lo=c, c_hi=c,
                    tiles=(8, 1))
        try:
            s.run(T + burn, burn, seed)
            mean, var, cnt = s.moments()
        finally:
            s.close()
        assert cnt == T
        # MMSE mean at every pixel: the chain mean is exactly mu in law (linear Gaussian ULA)
        assert np.sqrt(np.mean((mean - mu) ** 2)) < 4 * np.mean(list(se_mean.values()))
        for p in pts:
            zm.append((mean[p] - mu[p]) / se_mean[p])
            ratio.append(var[p] / var_true[p])
    zm, ratio = np.array(zm), np.array(ratio)
    # pooled z-test of the probe means (4 x 65 draws) and of the probe variances: the sample
    # variance of a chain with integrated autocorrelation ~ 1/(gamma p_min) ~ 6 has relative
    # standard error ~ sqrt(2 * 6 / T) = 5 %; the pooled mean of 260 ratios is within 1 +- 1 %
    assert abs(zm.mean()) < 4 / np.sqrt(zm.size)
    assert 0.7 < np.mean(zm ** 2) < 1.4
    assert abs(ratio.mean() - 1) < 0.015, ratio.mean()
    assert np.all(np.abs(ratio - 1) < 0.3)
