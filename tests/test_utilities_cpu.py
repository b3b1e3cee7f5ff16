"""SURVEY 8(f) rank 4 utilities that need no GPU: the ||H||^2 bound for the step sizes
(against numpy's FFT and the exact value 1 for normalised non-negative kernels) and the
quality metrics of P:826-838 (closed-form cases, and SSIM against a per-window loop)."""
import numpy as np
import pytest

import synth
from paper_2511_00870_b200 import metrics, pnpula_conv_norm2_bound


def test_norm_bound_normalised_nonnegative_kernel_is_one():
    ky, kx = synth.gaussian_factors(9, 2.0)
    assert pnpula_conv_norm2_bound(synth.outer(ky, kx), 64) == pytest.approx(1.0, rel=1e-6)


def test_norm_bound_matches_numpy_fft():
    k = synth.random_kernel(5, 7, seed=3) - 0.05
    grid = 64
    ref = np.max(np.abs(np.fft.fft2(k.astype(np.float64), s=(grid, grid))) ** 2)
    assert pnpula_conv_norm2_bound(k, grid) == pytest.approx(ref, rel=1e-5)


def test_norm_bound_bounds_the_zero_boundary_operator():
    # power iteration on the same-size zero-boundary operator (scipy) stays below the bound
    from scipy.signal import convolve2d, correlate2d
    k = synth.random_kernel(5, 5, seed=9) - 0.03
    v = np.random.default_rng(0).normal(size=(40, 40))
    for _ in range(200):
        v = correlate2d(convolve2d(v, k, mode="same"), k, mode="same")
        v /= np.linalg.norm(v)
    est = np.sum(convolve2d(v, k, mode="same") ** 2)
    assert est <= pnpula_conv_norm2_bound(k, 256) * (1 + 1e-6)


def test_metrics_closed_forms():
    x = synth.ground_truth(64, 64)
    assert metrics.snr(x, 0.9 * x) == pytest.approx(20.0, abs=1e-5)        # ||x|| / ||0.1 x|| (fp32 x)
    assert metrics.psnr(np.zeros((8, 8)), np.full((8, 8), 0.1)) == pytest.approx(20.0, abs=1e-9)
    assert metrics.ssim(x, x) == pytest.approx(1.0, abs=1e-12)
    assert metrics.ssim(x, x + 0.1 * np.random.default_rng(1).normal(size=x.shape)) < 0.99


def test_ssim_matches_windowed_loop():
    rng = np.random.default_rng(5)
    a = rng.uniform(0, 1, (20, 23))
    b = np.clip(a + 0.2 * rng.normal(size=a.shape), 0, 1)
    r = np.arange(11) - 5.0
    g = np.exp(-r ** 2 / (2 * 1.5 ** 2))
    g /= g.sum()
    w = np.outer(g, g)
    vals = []
    for i in range(a.shape[0] - 10):
        for j in range(a.shape[1] - 10):
            pa, pb = a[i:i + 11, j:j + 11], b[i:i + 11, j:j + 11]
            ma, mb = np.sum(w * pa), np.sum(w * pb)
            va, vb = np.sum(w * (pa - ma) ** 2), np.sum(w * (pb - mb) ** 2)
            cab = np.sum(w * (pa - ma) * (pb - mb))
            vals.append(((2 * ma * mb + 1e-4) * (2 * cab + 9e-4)) / ((ma ** 2 + mb ** 2 + 1e-4) * (va + vb + 9e-4)))
    assert metrics.ssim(a, b) == pytest.approx(float(np.mean(vals)), rel=1e-9)
