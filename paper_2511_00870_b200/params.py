"""Hyper-parameter helpers of the paper's experimental setting (host-side, no GPU).

gaussian_pnp: P:771-774 (Gaussian noise, PnP prior, no AXDA): alpha = 1, eps = sigma,
  lambda = 0.99 / (4 ||H||^2/sigma^2 + 2 alpha L_D / eps^2),
  gamma  = 0.99 / (3 (alpha L_D/eps^2 + ||H||^2/sigma^2 + 1/lambda [+ 1/rho]))
  -- the printed gamma contains ||eta H||^2/rho, a copy of the Poisson formula;
  DESIGN.md reading R11 replaces it by ||H||^2/sigma^2 (and adds 1/rho when the AXDA
  z-block of P:538-545 is switched on).
"""
from __future__ import annotations

import math


def gaussian_pnp(sigma2: float, normH2: float = 1.0, L_D: float = 1.0, alpha: float = 1.0,
                 rho: float = 0.0) -> dict:
    eps = math.sqrt(sigma2)
    lam = 0.99 / (4 * normH2 / sigma2 + 2 * alpha * L_D / eps ** 2)
    inv = alpha * L_D / eps ** 2 + normH2 / sigma2 + 1 / lam + (1 / rho if rho > 0 else 0.0)
    gamma = 0.99 / (3 * inv)
    out = dict(alpha=alpha, eps=eps, lam=lam, gamma=gamma)
    if rho > 0:
        out.update(rho=rho, kappa=0.99 * rho)
    return out


def kernel_norm_bound(k) -> float:
    """||H||^2 <= ||k||_1^2 for a convolution (Young's inequality); = 1 for normalised non-negative kernels."""
    import numpy as np
    return float(np.abs(np.asarray(k, dtype=np.float64)).sum() ** 2)
