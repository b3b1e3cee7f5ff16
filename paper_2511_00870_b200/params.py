"""Hyper-parameter helpers of the paper's experimental setting (host-side, no GPU).

gaussian_pnp: P:771-774 (Gaussian noise, PnP prior, no AXDA): alpha = 1, eps = sigma,
  lambda = 0.99 / (4 ||H||^2/sigma^2 + 2 alpha L_D / eps^2),
  gamma  = 0.99 / (3 (alpha L_D/eps^2 + ||H||^2/sigma^2 + 1/lambda [+ 1/rho]))
  -- the printed gamma contains ||eta H||^2/rho, a copy of the Poisson formula;
  DESIGN.md reading R11 replaces it by ||H||^2/sigma^2 (and adds 1/rho when the AXDA
  z-block of P:538-545 is switched on).
poisson_pnp: P:777-782 (Poisson noise, PnP prior, AXDA blocks z1 ~ eta H x, z2 ~ x):
  alpha = 1, eps = 0.05, rho1 = 10, rho2 = 1e-3,
  lambda = 0.99 / (4 ||eta H||^2/rho1 + 4/rho2 + 2 alpha L_D/eps^2),
  gamma  = 0.99 / (3 (alpha L_D/eps^2 + ||eta H||^2/rho1 + 1/rho2 + 1/lambda)),
  kappa1 = 0.99 rho1, kappa2 = 0.99 rho2.
tv_gaussian: P:802-809 (Gaussian noise, TV prior, z ~ D x): rho = 1e-5, beta = 40,
  gamma = 0.99 (||H||^2/sigma^2 + ||D||^2/rho)^-1, kappa = 0.99 rho ||D||^-2, ||D||^2 <= 8.
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


def poisson_pnp(eta: float, normH2: float = 1.0, L_D: float = 1.0, alpha: float = 1.0, eps: float = 0.05,
                rho1: float = 10.0, rho2: float = 1e-3) -> dict:
    h2 = eta * eta * normH2 / rho1
    lam = 0.99 / (4 * h2 + 4 / rho2 + 2 * alpha * L_D / eps ** 2)
    gamma = 0.99 / (3 * (alpha * L_D / eps ** 2 + h2 + 1 / rho2 + 1 / lam))
    return dict(alpha=alpha, eps=eps, lam=lam, gamma=gamma, eta=eta, rho1=rho1, kappa1=0.99 * rho1,
                rho=rho2, kappa=0.99 * rho2)


def tv_gaussian(sigma2: float, normH2: float = 1.0, rho: float = 1e-5, beta: float = 40.0,
                normD2: float = 8.0) -> dict:
    gamma = 0.99 / (normH2 / sigma2 + normD2 / rho)
    return dict(gamma=gamma, rho=rho, kappa=0.99 * rho / normD2, tv_beta=beta)
