"""Shared builders for the GPU parity tests: one seeded problem, fed identically to the
oracle (oracle.Problem) and to the CUDA path (paper_2511_00870_b200.Sampler)."""
from __future__ import annotations

import numpy as np

import oracle
import synth
from paper_2511_00870_b200 import Sampler, params


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make_problem(ny, nx, *, op="conv", kernel="random5", cnn=None, z=False, box=True, x0="truth",
                 snr=None, seed_w=2513):
    """Returns (kwargs for Sampler, oracle.Problem).  kernel: 'random5', 'random9', 'gauss5', 'gauss9'."""
    kw = {}
    if op == "conv":
        if kernel.startswith("gauss"):
            L = int(kernel[5:])
            ky, kx = synth.gaussian_factors(L, 1.0 if L == 5 else 2.0)
            k2 = synth.outer(ky, kx)
            kw_s = dict(kernel_sep=(ky, kx))
            kw_o = dict(ksep=(ky, kx))
        else:
            L = int(kernel[6:])
            k = synth.random_kernel(L, L, seed=L)
            k2 = k.astype(np.float64)
            kw_s = dict(kernel=k)
            kw_o = dict(kernel=k)
        s2 = synth.noise_sigma2_blur(ny, nx, k2, 25.0 if snr is None else snr)
        y = synth.observe_blur(ny, nx, k2, s2)
        kw.update(kw_s)
        okw = dict(op="conv", **kw_o)
    else:
        s2 = synth.noise_sigma2_mask(ny, nx, 15.0 if snr is None else snr)
        y, m = synth.observe_mask(ny, nx, s2)
        kw.update(op="mask", mask=m)
        okw = dict(op="mask", mask=m)
    rho = 1e-2 if z else 0.0
    hp = params.gaussian_pnp(s2, 1.0, 1.0, rho=rho)
    common = dict(sigma2=s2, gamma=hp["gamma"])
    if box:
        common.update(lam=hp["lam"], c_lo=0.0, c_hi=1.0)
    if z:
        common.update(rho=hp["rho"], kappa=hp["kappa"], z_lo=0.0, z_hi=1.0)
    if cnn is not None:
        K, P = cnn
        w, b = synth.dncnn_weights(K, P, seed=seed_w)
        common.update(weights=w, biases=b, n_layers=K, channels=P, alpha=1.0, eps=hp["eps"])
    if x0 == "truth":
        common["x0"] = synth.ground_truth(ny, nx) * 0.8 + 0.1
    kw.update(common)
    pb = oracle.Problem(y=y, **okw, **common)
    kw.update(ny=ny, nx=nx, y=y)
    return kw, pb


def gpu_run(kw, n_iter, burn_in, seed, tiles=(1, 1), flags=0):
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        s.run(n_iter, burn_in, seed)
        x, z, t = s.state()
        mean, var = None, None
        if n_iter - burn_in >= 2:
            mean, var, _ = s.moments()
        return dict(x=x, z=z, t=t, mean=mean, var=var)
    finally:
        s.close()
