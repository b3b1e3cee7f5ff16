"""Restoration-quality metrics of the paper's evaluation (sec:exp_settings P:826-838), evaluated
on host arrays after pnpula_get_moments (post-processing, not part of the sampling path).

snr:  eq:rsnr P:833-836, 10 log10(||xbar||^2 / ||xbar - xhat||^2)
psnr: 10 log10(peak^2 / MSE), peak = 1 for images in C = [0, 1]
ssim: Wang et al. 2004 (cited at P:831): Gaussian window sigma = 1.5 truncated to 11 x 11,
      K1 = 0.01, K2 = 0.03, dynamic range L = peak, mean of the SSIM map over the "valid"
      window positions.
"""
from __future__ import annotations

import numpy as np


def snr(xbar, xhat) -> float:
    xbar = np.asarray(xbar, np.float64)
    err = np.sum((xbar - np.asarray(xhat, np.float64)) ** 2)
    return float(10.0 * np.log10(np.sum(xbar ** 2) / err)) if err > 0 else float("inf")


def psnr(xbar, xhat, peak: float = 1.0) -> float:
    mse = np.mean((np.asarray(xbar, np.float64) - np.asarray(xhat, np.float64)) ** 2)
    return float(10.0 * np.log10(peak * peak / mse)) if mse > 0 else float("inf")


def _gauss_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    r = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-(r ** 2) / (2 * sigma * sigma))
    g /= g.sum()
    return np.outer(g, g)


def ssim(xbar, xhat, peak: float = 1.0, size: int = 11, sigma: float = 1.5) -> float:
    from scipy.signal import correlate2d
    a = np.asarray(xbar, np.float64)
    b = np.asarray(xhat, np.float64)
    w = _gauss_window(size, sigma)
    f = lambda im: correlate2d(im, w, mode="valid")
    mu_a, mu_b = f(a), f(b)
    saa = f(a * a) - mu_a ** 2
    sbb = f(b * b) - mu_b ** 2
    sab = f(a * b) - mu_a * mu_b
    c1, c2 = (0.01 * peak) ** 2, (0.03 * peak) ** 2
    m = ((2 * mu_a * mu_b + c1) * (2 * sab + c2)) / ((mu_a ** 2 + mu_b ** 2 + c1) * (saa + sbb + c2))
    return float(m.mean())
