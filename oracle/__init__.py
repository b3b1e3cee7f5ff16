"""CPU oracle for the distributed PnP-ULA hot path (arXiv 2511.00870).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
module.  The product package ``paper_2511_00870_b200`` never imports it, and it
never imports the product package (they share no code).

The arithmetic lives in ``pnpula_oracle.c`` (plain C, fp64, plain loops, each
function citing the PAPER.md passage it follows).  This file only builds that C
file with gcc and marshals numpy arrays through ctypes.

Parity status per function:
  partition, philox, normal, conv fwd/adj, mask, dncnn residual, step-size
  check, run (untiled + tiled), KL prox, Poisson run, TV, DDFB, C-channel (RGB) run and
  residual: pinned (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pnpula_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, strict IEEE: no -ffast-math, no FMA contraction; OpenMP
    over output rows -- OMP_NUM_THREADS=1 for the single-thread timing; results do not depend on
    the thread count)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
               "-D_DEFAULT_SOURCE", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Config(C.Structure):
    _fields_ = [
        ("ny", C.c_int32), ("nx", C.c_int32), ("op", C.c_int32),
        ("kernel", C.c_void_p), ("ksep_y", C.c_void_p), ("ksep_x", C.c_void_p),
        ("kh", C.c_int32), ("kw", C.c_int32),
        ("mask", C.c_void_p), ("y", C.c_void_p), ("sigma2", C.c_double),
        ("n_layers", C.c_int32), ("channels", C.c_int32),
        ("weights", C.c_void_p), ("biases", C.c_void_p),
        ("alpha", C.c_double), ("eps", C.c_double), ("bf16_emulate", C.c_int32),
        ("lam", C.c_double), ("c_lo", C.c_double), ("c_hi", C.c_double),
        ("rho", C.c_double), ("kappa", C.c_double), ("z_lo", C.c_double), ("z_hi", C.c_double),
        ("gamma", C.c_double), ("x0", C.c_void_p),
        ("n_iter", C.c_int64), ("burn_in", C.c_int64), ("seed", C.c_uint64),
        ("tiles_y", C.c_int32), ("tiles_x", C.c_int32),
        ("i_off", C.c_int64), ("j_off", C.c_int64),
        ("eta", C.c_double), ("rho1", C.c_double), ("kappa1", C.c_double),
        ("den_kind", C.c_int32), ("ddfb_gammas", C.c_void_p), ("ht_eps", C.c_double),
        ("tv_beta", C.c_double),
        ("n_chan", C.c_int32),
    ]


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i32, i64, u32, u64, vp = C.c_double, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_void_p
        _lib.or_partition.argtypes = [i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]
        _lib.or_philox4x32_10.argtypes = [vp, vp, vp]
        _lib.or_normal.argtypes = [u64, u32, i64, i64, u32]
        _lib.or_normal.restype = d
        _lib.or_normal_field.argtypes = [u64, u32, i32, i32, u32, vp]
        _lib.or_conv_fwd.argtypes = [vp, i32, i32, vp, i32, i32, vp]
        _lib.or_conv_adj.argtypes = [vp, i32, i32, vp, i32, i32, vp]
        _lib.or_dncnn_residual.argtypes = [vp, i32, i32, i32, i32, vp, vp, i32, vp]
        _lib.or_dncnn_residual.restype = C.c_int
        _lib.or_dncnn_residual_c.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, i32, vp]
        _lib.or_dncnn_residual_c.restype = C.c_int
        _lib.or_dncnn_param_count.argtypes = [i32, i32, i32]
        _lib.or_dncnn_param_count.restype = i64
        _lib.or_check_stepsizes.argtypes = [d, d, d, d, d, d, d]
        _lib.or_check_stepsizes.restype = C.c_int
        _lib.or_run.argtypes = [C.POINTER(_Config), vp, vp, vp, vp, C.POINTER(i64)]
        _lib.or_run.restype = C.c_int
        _lib.or_run_ex.argtypes = [C.POINTER(_Config), vp, vp, vp, vp, vp, vp, C.POINTER(i64)]
        _lib.or_run_ex.restype = C.c_int
        _lib.or_prox_kl.argtypes = [d, d, d]
        _lib.or_prox_kl.restype = d
        _lib.or_grad2d.argtypes = [vp, i32, i32, vp, vp]
        _lib.or_grad2d_adj.argtypes = [vp, vp, i32, i32, vp]
        _lib.or_prox_l21.argtypes = [d, d, d, C.POINTER(d), C.POINTER(d)]
        _lib.or_ddfb_residual.argtypes = [vp, i32, i32, i32, i32, vp, vp, d, i32, vp]
        _lib.or_ddfb_residual.restype = C.c_int
        _lib.or_ddfb_residual_c.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, d, i32, vp]
        _lib.or_ddfb_residual_c.restype = C.c_int
        _lib.or_ddfb_param_count.argtypes = [i32, i32, i32]
        _lib.or_ddfb_param_count.restype = i64
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a) -> Optional[np.ndarray]:
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- primitives
def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's row loops (n <= 0: all host cores); returns the count set.
    Results do not depend on it (see OR_PARALLEL_ROWS in pnpula_oracle.c)."""
    _load()
    n = n if n > 0 else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    C.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    return int(n)


def partition(n: int, parts: int, p: int) -> tuple[int, int]:
    lo, hi = C.c_int64(), C.c_int64()
    _load().or_partition(n, parts, p, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().or_philox4x32_10(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return out


def normal(seed: int, t1: int, i: int, j: int, stream: int) -> float:
    return _load().or_normal(seed, t1, i, j, stream)


def normal_field(seed: int, t1: int, ny: int, nx: int, stream: int) -> np.ndarray:
    out = np.zeros((ny, nx), dtype=np.float64)
    _load().or_normal_field(seed, t1, ny, nx, stream, out.ctypes.data)
    return out


def conv_fwd(x, k) -> np.ndarray:
    x, k = _f64(x), _f64(k)
    out = np.zeros_like(x)
    _load().or_conv_fwd(x.ctypes.data, x.shape[0], x.shape[1], k.ctypes.data, k.shape[0], k.shape[1],
                        out.ctypes.data)
    return out


def conv_adj(r, k) -> np.ndarray:
    r, k = _f64(r), _f64(k)
    out = np.zeros_like(r)
    _load().or_conv_adj(r.ctypes.data, r.shape[0], r.shape[1], k.ctypes.data, k.shape[0], k.shape[1],
                        out.ctypes.data)
    return out


def dncnn_residual(x, weights, biases, n_layers: int, channels: int, bf16_emulate: bool = False):
    """x: (ny, nx) grayscale or (C, ny, nx) planes (layer 1 C -> P, layer K P -> C; R43)."""
    x = _f64(x)
    w, b = _f32(weights), _f32(biases)
    G = np.zeros_like(x)
    nc = x.shape[0] if x.ndim == 3 else 1
    e = _load().or_dncnn_residual_c(x.ctypes.data, x.shape[-2], x.shape[-1], nc, n_layers, channels,
                                    w.ctypes.data, b.ctypes.data, int(bf16_emulate), G.ctypes.data)
    if e:
        raise ValueError("or_dncnn_residual failed")
    return G


def ddfb_residual(x, weights, gammas, n_layers: int, channels: int, ht_eps: float, bf16_emulate: bool = False):
    """G = v - D(v) for the DDFB denoiser (eq:ddfb_operator, eq:dfb_operator:T; readings R39-R42);
    x: [ny][nx], or [C][ny][nx] with weights [K][P][C][3][3] (colour)."""
    x = _f64(x)
    w, g = _f32(weights), _f32(gammas)
    G = np.zeros_like(x)
    nc = x.shape[0] if x.ndim == 3 else 1
    e = _load().or_ddfb_residual_c(x.ctypes.data, x.shape[-2], x.shape[-1], nc, n_layers, channels,
                                   w.ctypes.data, g.ctypes.data, ht_eps, int(bf16_emulate), G.ctypes.data)
    if e:
        raise ValueError("or_ddfb_residual failed")
    return G


def ddfb_param_count(n_layers: int, channels: int, image_channels: int) -> int:
    return int(_load().or_ddfb_param_count(n_layers, channels, image_channels))


def dncnn_param_count(n_layers: int, channels: int, image_channels: int) -> int:
    return int(_load().or_dncnn_param_count(n_layers, channels, image_channels))


def check_stepsizes(L, h2_over_rho, alpha, eps, L_D, lam, gamma) -> int:
    return int(_load().or_check_stepsizes(L, h2_over_rho, alpha, eps, L_D, lam, gamma))


def grad2d(x):
    """D x = (vertical, horizontal) forward differences, zero at the last row / column (R35)."""
    x = _f64(x)
    gv, gh = np.zeros_like(x), np.zeros_like(x)
    _load().or_grad2d(x.ctypes.data, x.shape[0], x.shape[1], gv.ctypes.data, gh.ctypes.data)
    return gv, gh


def grad2d_adj(gv, gh):
    gv, gh = _f64(gv), _f64(gh)
    out = np.zeros_like(gv)
    _load().or_grad2d_adj(gv.ctypes.data, gh.ctypes.data, gv.shape[0], gv.shape[1], out.ctypes.data)
    return out


def prox_l21(gv: float, gh: float, tau: float):
    a, b = C.c_double(), C.c_double()
    _load().or_prox_l21(gv, gh, tau, C.byref(a), C.byref(b))
    return a.value, b.value


def prox_kl(v: float, y: float, kappa: float) -> float:
    """prox of kappa KL(y || .) (Poisson likelihood, closed form; reading R31)."""
    return float(_load().or_prox_kl(v, y, kappa))


# ---------------------------------------------------------------- chain
@dataclass
class Problem:
    """All inputs of one chain (host arrays; fp32 like the library's inputs)."""
    y: np.ndarray
    sigma2: float
    gamma: float
    op: str = "conv"                      # "conv" | "mask" | "poisson"
    kernel: Optional[np.ndarray] = None   # 2-D true-convolution kernel
    ksep: Optional[tuple] = None          # (ky, kx) separable factors
    mask: Optional[np.ndarray] = None
    weights: Optional[np.ndarray] = None
    biases: Optional[np.ndarray] = None
    n_layers: int = 0
    channels: int = 0
    alpha: float = 0.0
    eps: float = 1.0
    lam: float = 0.0
    c_lo: float = 0.0
    c_hi: float = 1.0
    rho: float = 0.0
    kappa: float = 0.0
    z_lo: float = -np.inf
    z_hi: float = np.inf
    x0: Optional[np.ndarray] = None
    eta: float = 0.0                      # op "poisson": y ~ Poisson(eta H x), z1 ~ eta H x
    rho1: float = 0.0
    kappa1: float = 0.0
    tv_beta: float = 0.0                  # > 0: TV prior, z ~ D x (z = vertical, zh = horizontal)
    den_kind: str = "dncnn"               # "dncnn" | "ddfb"
    ddfb_gammas: Optional[np.ndarray] = None
    ht_eps: float = 0.0
    extra: dict = field(default_factory=dict)


def run(pb: Problem, n_iter: int, burn_in: int, seed: int, tiles=(1, 1), bf16_emulate=False,
        want_var: bool = True, origin=(0, 0)) -> dict:
    """Run the chain.  origin = global coordinates of pixel (0, 0) when pb is a crop of a
    larger image (only the noise indexing uses it).  pb.y of shape (C, ny, nx) runs a C-channel
    image (R43); the returned fields then have that shape too."""
    lib = _load()
    y = _f32(pb.y)
    nc = y.shape[0] if y.ndim == 3 else 1
    ny, nx = y.shape[-2:]
    keep = [y]
    cfg = _Config()
    cfg.ny, cfg.nx = ny, nx
    cfg.op = {"conv": 0, "mask": 1, "poisson": 2}[pb.op]
    if pb.op in ("conv", "poisson"):
        if pb.ksep is not None:
            ky, kx = _f32(pb.ksep[0]), _f32(pb.ksep[1])
            keep += [ky, kx]
            cfg.ksep_y, cfg.ksep_x = ky.ctypes.data, kx.ctypes.data
            cfg.kh, cfg.kw = ky.size, kx.size
        else:
            k = _f32(pb.kernel)
            keep.append(k)
            cfg.kernel = k.ctypes.data
            cfg.kh, cfg.kw = k.shape
    else:
        m = np.ascontiguousarray(pb.mask, dtype=np.uint8)
        keep.append(m)
        cfg.mask = m.ctypes.data
    cfg.y = y.ctypes.data
    cfg.sigma2 = pb.sigma2
    if pb.n_layers and pb.alpha != 0.0:
        w = _f32(pb.weights)
        keep.append(w)
        cfg.weights = w.ctypes.data
        if pb.den_kind == "ddfb":
            gm = _f32(pb.ddfb_gammas)
            keep.append(gm)
            cfg.den_kind, cfg.ddfb_gammas, cfg.ht_eps = 1, gm.ctypes.data, pb.ht_eps
        else:
            b = _f32(pb.biases)
            keep.append(b)
            cfg.biases = b.ctypes.data
        cfg.n_layers, cfg.channels = pb.n_layers, pb.channels
    cfg.alpha, cfg.eps, cfg.bf16_emulate = pb.alpha, pb.eps, int(bf16_emulate)
    cfg.lam, cfg.c_lo, cfg.c_hi = pb.lam, pb.c_lo, pb.c_hi
    cfg.rho, cfg.kappa, cfg.z_lo, cfg.z_hi = pb.rho, pb.kappa, pb.z_lo, pb.z_hi
    cfg.gamma = pb.gamma
    if pb.x0 is not None:
        x0 = _f32(pb.x0)
        keep.append(x0)
        cfg.x0 = x0.ctypes.data
    cfg.n_iter, cfg.burn_in, cfg.seed = n_iter, burn_in, seed
    cfg.tiles_y, cfg.tiles_x = tiles
    cfg.i_off, cfg.j_off = origin
    cfg.eta, cfg.rho1, cfg.kappa1 = pb.eta, pb.rho1, pb.kappa1
    cfg.tv_beta = pb.tv_beta
    cfg.n_chan = nc
    shp = y.shape
    x = np.zeros(shp); z = np.zeros(shp); z1 = np.zeros(shp); zh = np.zeros(shp)
    mean = np.zeros(shp); var = np.zeros(shp)
    n = C.c_int64()
    have_mean = n_iter > burn_in
    have_var = want_var and n_iter - burn_in >= 2
    e = lib.or_run_ex(C.byref(cfg), x.ctypes.data, z.ctypes.data, z1.ctypes.data, zh.ctypes.data,
                      mean.ctypes.data if have_mean else None, var.ctypes.data if have_var else None, C.byref(n))
    if e:
        raise ValueError(f"or_run failed with status {e}")
    return {"x": x, "z": z, "z1": z1, "zh": zh, "mean": mean if have_mean else None, "var": var if have_var else None,
            "n": n.value}
