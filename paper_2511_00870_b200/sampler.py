"""Thin Python front-end of the C ABI (include/pnpula.h): builds a pnpula_config from
numpy arrays and wraps the context handle.  No arithmetic of the method happens here."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib as L


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


class Sampler:
    """One rank's view of a distributed PnP-ULA chain (Algorithm 1)."""

    def __init__(self, *, ny: int, nx: int, y: np.ndarray, sigma2: float, gamma: float,
                 op: str = "conv", kernel: Optional[np.ndarray] = None, kernel_sep=None,
                 mask: Optional[np.ndarray] = None,
                 weights: Optional[np.ndarray] = None, biases: Optional[np.ndarray] = None,
                 n_layers: int = 0, channels: int = 0, alpha: float = 0.0, eps: float = 1.0,
                 lam: float = 0.0, c_lo: float = 0.0, c_hi: float = 1.0,
                 rho: float = 0.0, kappa: float = 0.0, z_lo: float = -np.inf, z_hi: float = np.inf,
                 x0: Optional[np.ndarray] = None, in_rect=None, tiles=(1, 1),
                 rank: int = 0, world_size: int = 1, device: int = 0, nccl_uid: Optional[bytes] = None,
                 stream: int = 0, flags: int = 0, lipschitz_L: float = 0.0, lipschitz_LD: float = 0.0,
                 eta: float = 0.0, rho1: float = 0.0, kappa1: float = 0.0, tv_beta: float = 0.0,
                 den_kind: str = "dncnn", ddfb_gammas: Optional[np.ndarray] = None, ht_eps: float = 0.0):
        lib = L.load()
        keep = []
        cfg = L.Config()
        cfg.ny, cfg.nx = ny, nx
        cfg.tiles_y, cfg.tiles_x = tiles
        cfg.rank, cfg.world_size, cfg.device = rank, world_size, device
        if nccl_uid is not None:
            ub = (C.c_uint8 * 128).from_buffer_copy(nccl_uid)
            keep.append(ub)
            cfg.nccl_uid = C.addressof(ub)
        cfg.stream = stream
        cfg.op = {"conv": L.OP_CONV, "mask": L.OP_MASK, "poisson": L.OP_POISSON}[op]
        if op in ("conv", "poisson"):
            if kernel_sep is not None:
                ky, kx = _f32(kernel_sep[0]), _f32(kernel_sep[1])
                keep += [ky, kx]
                cfg.kernel_y, cfg.kernel_x = ky.ctypes.data, kx.ctypes.data
                cfg.kh, cfg.kw = ky.size, kx.size
            else:
                k = _f32(kernel)
                keep.append(k)
                cfg.kernel = k.ctypes.data
                cfg.kh, cfg.kw = k.shape
        else:
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            keep.append(m)
            cfg.mask = m.ctypes.data
        yy = _f32(y)
        keep.append(yy)
        cfg.y = yy.ctypes.data
        if x0 is not None:
            xx = _f32(x0)
            keep.append(xx)
            cfg.x0 = xx.ctypes.data
        r = in_rect if in_rect is not None else (0, 0, ny, nx)
        cfg.in_rect = L.Rect(*r)
        # colour images (R43): y / x0 as planes (C, h, w)
        self.nc = yy.shape[0] if yy.ndim == 3 else 1
        cfg.img_channels = self.nc
        if yy.shape[-2:] != (r[2], r[3]) or yy.ndim not in (2, 3):
            raise ValueError(f"y has shape {yy.shape}, in_rect is {r}")
        cfg.sigma2 = sigma2
        if n_layers and alpha != 0.0:
            w = _f32(weights)
            keep.append(w)
            if den_kind == "ddfb":
                gm = _f32(ddfb_gammas)
                keep.append(gm)
                den = L.Denoiser(n_layers, channels, w.ctypes.data, None, L.DEN_DDFB, gm.ctypes.data, ht_eps)
            else:
                b = _f32(biases)
                keep.append(b)
                den = L.Denoiser(n_layers, channels, w.ctypes.data, b.ctypes.data, L.DEN_DNCNN, None, 0.0)
            keep.append(den)
            cfg.den = C.pointer(den)
        cfg.alpha, cfg.eps = alpha, eps
        cfg.lam, cfg.c_lo, cfg.c_hi = lam, c_lo, c_hi
        cfg.rho, cfg.kappa, cfg.z_lo, cfg.z_hi = rho, kappa, z_lo, z_hi
        cfg.gamma = gamma
        cfg.lipschitz_L, cfg.lipschitz_LD = lipschitz_L, lipschitz_LD
        cfg.flags = flags
        cfg.eta, cfg.rho1, cfg.kappa1 = eta, rho1, kappa1
        cfg.tv_beta = tv_beta
        h = C.c_void_p()
        L.check(lib.pnpula_create(C.byref(cfg), C.byref(h)))
        self.warning = L.last_error()
        self._h = h
        self._lib = lib
        self.ny, self.nx = ny, nx
        self.has_z = rho > 0
        self.op = op
        bb = L.Rect()
        L.check(lib.pnpula_local_bbox(h, C.byref(bb)))
        self.bbox = bb.tup()
        nloc, halo = C.c_int32(), C.c_int32()
        L.check(lib.pnpula_tile_info(h, 0, None, C.byref(nloc), C.byref(halo)))
        self.n_local_tiles, self.halo = nloc.value, halo.value
        self.rank, self.world_size = rank, world_size

    # ---------------------------------------------------------------- chain
    def reset(self, burn_in: int, seed: int):
        L.check(self._lib.pnpula_reset(self._h, burn_in, seed))

    def advance(self, n_iter: int):
        L.check(self._lib.pnpula_advance(self._h, n_iter))

    def run(self, n_iter: int, burn_in: int, seed: int):
        L.check(self._lib.pnpula_run(self._h, n_iter, burn_in, seed))

    def synchronize(self):
        L.check(self._lib.pnpula_synchronize(self._h))

    def _out_shape(self, scope, planes=None):
        c = (self.nc if planes is None else planes,) if (self.nc > 1 and planes != 1) else ()
        if scope == L.SCOPE_GLOBAL_ON_ROOT:
            return c + (self.ny, self.nx) if self.rank == 0 else None
        return c + (self.bbox[2], self.bbox[3])

    def moments(self, scope: int = L.SCOPE_LOCAL, want_var: bool = True, out=None):
        """out: optional (mean, var) host arrays (e.g. pinned) to write into."""
        shp = self._out_shape(scope)
        if out is not None:
            mean, var = out
        else:
            mean = np.zeros(shp, np.float32) if shp else None
            var = np.zeros(shp, np.float32) if (shp and want_var) else None
        n = C.c_int64()
        L.check(self._lib.pnpula_get_moments(self._h, L._ptr(mean), L._ptr(var), C.byref(n), scope))
        return mean, var, n.value

    def state(self, scope: int = L.SCOPE_LOCAL):
        shp = self._out_shape(scope)
        x = np.zeros(shp, np.float32) if shp else None
        z = np.zeros(shp, np.float32) if shp else None
        t = C.c_int64()
        L.check(self._lib.pnpula_get_state(self._h, L._ptr(x), L._ptr(z), C.byref(t), scope))
        return x, z, t.value

    def z1(self, scope: int = L.SCOPE_LOCAL):
        """OP_POISSON: the AXDA block z1 (~ eta H x)."""
        shp = self._out_shape(scope)
        out = np.zeros(shp, np.float32) if shp else None
        L.check(self._lib.pnpula_get_z1(self._h, L._ptr(out), scope))
        return out

    def tv_zh(self, scope: int = L.SCOPE_LOCAL):
        """TV prior: the horizontal component z_h of z ~ D x (C planes for colour images)."""
        shp = self._out_shape(scope)
        out = np.zeros(shp, np.float32) if shp else None
        L.check(self._lib.pnpula_get_tv_zh(self._h, L._ptr(out), scope))
        return out

    def opnorm2(self, iters: int = 100) -> float:
        """||H||^2 by power iteration on the GPU (collective)."""
        out = C.c_double()
        L.check(self._lib.pnpula_opnorm2(self._h, iters, C.byref(out)))
        return out.value

    def save_checkpoint(self) -> bytes:
        """This rank's complete chain state (resume with load_checkpoint on an identical context)."""
        n = C.c_uint64()
        L.check(self._lib.pnpula_checkpoint_bytes(self._h, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        L.check(self._lib.pnpula_save_checkpoint(self._h, buf, n.value))
        return bytes(buf)

    def load_checkpoint(self, blob: bytes):
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        L.check(self._lib.pnpula_load_checkpoint(self._h, buf, len(blob)))

    def tile_info(self, i: int):
        r = L.Rect()
        L.check(self._lib.pnpula_tile_info(self._h, i, C.byref(r), None, None))
        return r.tup()

    def padded_x(self, i: int):
        r = self.tile_info(i)
        out = np.zeros((r[2] + 2 * self.halo, r[3] + 2 * self.halo), np.float32)
        L.check(self._lib.pnpula_get_padded_x(self._h, i, out.ctypes.data))
        return out

    def denoiser_residual(self):
        out = np.zeros(self._out_shape(L.SCOPE_LOCAL), np.float32)
        L.check(self._lib.pnpula_get_denoiser_residual(self._h, out.ctypes.data))
        return out

    def set_timing(self, enable: bool):
        L.check(self._lib.pnpula_set_timing(self._h, int(enable)))

    def kernel_time(self, name: str, reset: bool = False):
        ms, n = C.c_double(), C.c_int64()
        L.check(self._lib.pnpula_kernel_time(self._h, name.encode(), C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pnpula_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
