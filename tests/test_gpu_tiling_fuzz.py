"""Randomised bitwise tiling invariance (north_star: results bitwise independent of the tile grid;
DESIGN.md R6): seeded random image sizes (ragged against the 122-column CNN strips and the 32 x 64
update blocks), tile grids (row strips, column strips, 2-D; tiles as narrow as the halo allows),
forward operators (random / Gaussian kernels, mask), priors (none, DnCNN 4x16 / 8x32), AXDA
z-block on / off, halo exchange by device copies or NCCL self send/recv, graph replay on / off.
Every field after 7 iterations must equal the 1 x 1 chain bit for bit."""
import numpy as np
import pytest

from gpu_common import gpu_run, make_problem
from paper_2511_00870_b200 import FLAG_HALO_VIA_NCCL, FLAG_NO_GRAPH

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    op = "mask" if rng.random() < 0.3 else "conv"
    kernel = str(rng.choice(["random5", "random9", "gauss5", "gauss9"]))
    cnn = [None, (4, 16), (8, 32)][int(rng.integers(0, 3))]
    z = bool(rng.random() < 0.5)
    h = max(8 if "9" in kernel and op == "conv" else 4 if op == "conv" else 0, cnn[0] if cnn else 0)
    ny, nx = int(rng.integers(max(40, 3 * h), 200)), int(rng.integers(max(40, 3 * h), 260))
    while True:
        ty, tx = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        if (ty, tx) != (1, 1) and ny // ty >= max(h, 1) and nx // tx >= max(h, 1):
            break
    flags = (FLAG_HALO_VIA_NCCL if rng.random() < 0.4 else 0) | (FLAG_NO_GRAPH if rng.random() < 0.3 else 0)
    return dict(ny=ny, nx=nx, op=op, kernel=kernel, cnn=cnn, z=z, tiles=(ty, tx), flags=flags)


@pytest.mark.parametrize("seed", range(10))
def test_random_tilings_bitwise(seed):
    c = _case(seed)
    kw, _ = make_problem(c["ny"], c["nx"], op=c["op"], kernel=c["kernel"], cnn=c["cnn"], z=c["z"])
    a = gpu_run(kw, 7, 2, 90 + seed)
    b = gpu_run(kw, 7, 2, 90 + seed, tiles=c["tiles"], flags=c["flags"])
    for k in ("x", "z", "mean", "var"):
        if a[k] is None:
            continue
        assert np.array_equal(a[k], b[k]), (k, c)
