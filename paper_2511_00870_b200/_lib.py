"""ctypes binding of libpnpula.so (include/pnpula.h).  Argument marshalling only:
every step of the sampler runs inside the library's CUDA kernels.  There is no
fallback: if the shared library is missing or cannot be loaded this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# PNPULA_LIB: load an alternative build of the same library (kernel experiments only)
LIB_PATH = os.environ.get("PNPULA_LIB") or os.path.join(_PKG, "libpnpula.so")

PNPULA_OK = 0
STATUS = {0: "OK", 1: "E_INVALID_ARG", 2: "E_SHAPE", 3: "E_PARTITION_TOO_FINE", 4: "E_STEPSIZE",
          5: "E_STATS_EMPTY", 6: "E_STATE", 7: "E_CUDA", 8: "E_NCCL", 9: "E_OOM", 10: "E_UNSUPPORTED"}
OP_CONV, OP_MASK, OP_POISSON = 0, 1, 2
SCOPE_LOCAL, SCOPE_GLOBAL_ON_ROOT = 0, 1
FLAG_HALO_VIA_NCCL, FLAG_CNN_LAYERWISE, FLAG_NO_GRAPH = 0x1, 0x2, 0x4


class PnpulaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Rect(C.Structure):
    _fields_ = [("i0", C.c_int32), ("j0", C.c_int32), ("h", C.c_int32), ("w", C.c_int32)]

    def tup(self):
        return (self.i0, self.j0, self.h, self.w)


DEN_DNCNN, DEN_DDFB = 0, 1


class Denoiser(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("channels", C.c_int32),
                ("weights", C.c_void_p), ("biases", C.c_void_p),
                ("kind", C.c_int32), ("ddfb_gammas", C.c_void_p), ("ht_eps", C.c_double)]


class Config(C.Structure):
    _fields_ = [
        ("ny", C.c_int32), ("nx", C.c_int32), ("tiles_y", C.c_int32), ("tiles_x", C.c_int32),
        ("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
        ("nccl_uid", C.c_void_p), ("stream", C.c_uint64),
        ("op", C.c_int32), ("kernel", C.c_void_p), ("kernel_y", C.c_void_p), ("kernel_x", C.c_void_p),
        ("kh", C.c_int32), ("kw", C.c_int32),
        ("mask", C.c_void_p), ("y", C.c_void_p), ("x0", C.c_void_p), ("in_rect", Rect),
        ("sigma2", C.c_double),
        ("den", C.POINTER(Denoiser)), ("alpha", C.c_double), ("eps", C.c_double),
        ("lam", C.c_double), ("c_lo", C.c_double), ("c_hi", C.c_double),
        ("rho", C.c_double), ("kappa", C.c_double), ("z_lo", C.c_double), ("z_hi", C.c_double),
        ("gamma", C.c_double),
        ("lipschitz_L", C.c_double), ("lipschitz_LD", C.c_double),
        ("flags", C.c_int32),
        ("eta", C.c_double), ("rho1", C.c_double), ("kappa1", C.c_double),
        ("tv_beta", C.c_double),
        ("img_channels", C.c_int32),
    ]


class HaloMsg(C.Structure):
    _fields_ = [("src_tile", C.c_int32), ("dst_tile", C.c_int32), ("rect", Rect)]


_lib = None


def load():
    """Load libpnpula.so (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run paper_2511_00870_b200/build.py (or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i32, i64, u64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sigs = {
        "pnpula_version": ([], C.c_char_p),
        "pnpula_last_error": ([], C.c_char_p),
        "pnpula_get_unique_id": ([vp], C.c_int),
        "pnpula_create": ([C.POINTER(Config), C.POINTER(vp)], C.c_int),
        "pnpula_reset": ([vp, i64, u64], C.c_int),
        "pnpula_advance": ([vp, i64], C.c_int),
        "pnpula_run": ([vp, i64, i64, u64], C.c_int),
        "pnpula_synchronize": ([vp], C.c_int),
        "pnpula_local_bbox": ([vp, C.POINTER(Rect)], C.c_int),
        "pnpula_get_moments": ([vp, vp, vp, C.POINTER(i64), i32], C.c_int),
        "pnpula_get_state": ([vp, vp, vp, C.POINTER(i64), i32], C.c_int),
        "pnpula_get_z1": ([vp, vp, i32], C.c_int),
        "pnpula_get_tv_zh": ([vp, vp, i32], C.c_int),
        "pnpula_checkpoint_bytes": ([vp, C.POINTER(u64)], C.c_int),
        "pnpula_save_checkpoint": ([vp, vp, u64], C.c_int),
        "pnpula_load_checkpoint": ([vp, vp, u64], C.c_int),
        "pnpula_conv_norm2_bound": ([vp, i32, i32, i32, C.POINTER(d)], C.c_int),
        "pnpula_opnorm2": ([vp, i32, C.POINTER(d)], C.c_int),
        "pnpula_tile_info": ([vp, i32, C.POINTER(Rect), C.POINTER(i32), C.POINTER(i32)], C.c_int),
        "pnpula_get_padded_x": ([vp, i32, vp], C.c_int),
        "pnpula_get_denoiser_residual": ([vp, vp], C.c_int),
        "pnpula_set_timing": ([vp, i32], C.c_int),
        "pnpula_kernel_time": ([vp, C.c_char_p, C.POINTER(d), C.POINTER(i64), i32], C.c_int),
        "pnpula_destroy": ([vp], C.c_int),
        "pnpula_release_memory": ([i32], C.c_int),
        "pnpula_debug_philox": ([i32, u64, vp, i64, vp, vp], C.c_int),
        "pnpula_partition": ([i64, i64, i64, C.POINTER(i64), C.POINTER(i64)], None),
        "pnpula_halo_width": ([i32, i32, i32, i32], i32),
        "pnpula_plan_halo": ([i32, i32, i32, i32, i32, C.POINTER(HaloMsg), i32], i32),
        "pnpula_check_stepsizes": ([d, d, d, d, d, d, d], i32),
    }
    for name, (args, res) in sigs.items():
        if name == "pnpula_debug_philox" and not hasattr(lib, name) and os.environ.get("PNPULA_LIB"):
            continue   # an older experimental build (PNPULA_LIB) without the test hook
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


# names exported by include/pnpula.h (tests check the .so exports every one)
EXPORTED = ["pnpula_version", "pnpula_last_error", "pnpula_get_unique_id", "pnpula_create", "pnpula_reset",
            "pnpula_advance", "pnpula_run", "pnpula_synchronize", "pnpula_local_bbox", "pnpula_get_moments",
            "pnpula_get_state", "pnpula_get_z1", "pnpula_get_tv_zh", "pnpula_tile_info", "pnpula_get_padded_x", "pnpula_get_denoiser_residual",
            "pnpula_set_timing", "pnpula_kernel_time", "pnpula_destroy", "pnpula_partition",
            "pnpula_halo_width", "pnpula_plan_halo", "pnpula_check_stepsizes", "pnpula_checkpoint_bytes",
            "pnpula_save_checkpoint", "pnpula_load_checkpoint", "pnpula_conv_norm2_bound", "pnpula_opnorm2",
            "pnpula_release_memory", "pnpula_debug_philox"]


def last_error() -> str:
    return load().pnpula_last_error().decode()


def check(status: int):
    if status != PNPULA_OK:
        raise PnpulaError(status, last_error())


def _ptr(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------- host-only helpers
def pnpula_version() -> str:
    return load().pnpula_version().decode()


def pnpula_partition(n: int, parts: int, p: int) -> tuple[int, int]:
    lo, hi = C.c_int64(), C.c_int64()
    load().pnpula_partition(n, parts, p, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def pnpula_halo_width(op: int, kh: int, kw: int, n_layers: int) -> int:
    return int(load().pnpula_halo_width(op, kh, kw, n_layers))


def pnpula_plan_halo(ny, nx, tiles_y, tiles_x, h):
    lib = load()
    n = lib.pnpula_plan_halo(ny, nx, tiles_y, tiles_x, h, None, 0)
    if n < 0:
        raise PnpulaError(3, "tile extent smaller than halo width")
    arr = (HaloMsg * max(n, 1))()
    lib.pnpula_plan_halo(ny, nx, tiles_y, tiles_x, h, arr, n)
    return [(m.src_tile, m.dst_tile, m.rect.tup()) for m in arr[:n]]


def pnpula_check_stepsizes(L, h2_over_rho, alpha, eps, L_D, lam, gamma) -> int:
    return int(load().pnpula_check_stepsizes(L, h2_over_rho, alpha, eps, L_D, lam, gamma))


def pnpula_conv_norm2_bound(k, grid: int = 256) -> float:
    """Upper bound of ||H||^2 for the zero-boundary convolution with kernel k (max |DFT|^2)."""
    import numpy as np
    kk = np.ascontiguousarray(k, dtype=np.float32)
    out = C.c_double()
    check(load().pnpula_conv_norm2_bound(kk.ctypes.data, kk.shape[0], kk.shape[1], grid, C.byref(out)))
    return out.value


def pnpula_debug_philox(seed: int, counters, device: int = 0):
    """Test hook: raw Philox4x32-10 words and the four Box-Muller normals of each counter row
    (column quad, row, t+1, stream), computed on the GPU by the update kernels' own functions."""
    c = np.ascontiguousarray(counters, dtype=np.uint32).reshape(-1, 4)
    words = np.zeros_like(c)
    normals = np.zeros(c.shape, dtype=np.float32)
    check(load().pnpula_debug_philox(device, seed, c.ctypes.data, c.shape[0], words.ctypes.data,
                                     normals.ctypes.data))
    return words, normals


def pnpula_get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(load().pnpula_get_unique_id(buf))
    return bytes(buf)
