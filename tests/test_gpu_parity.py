"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs, element by element.  Tolerances (north_star): rel-L2 <= 1e-5 after 50
iterations on the fp32 operator path, <= 2e-2 with the bf16 denoiser; bitwise for
halo indexing and for every tile grid."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import gpu_run, make_problem, rel_l2
from paper_2511_00870_b200 import FLAG_CNN_LAYERWISE, FLAG_HALO_VIA_NCCL, Sampler

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- noise (Philox counters + Box-Muller)
def test_noise_matches_oracle():
    ny, nx = 37, 70                         # ragged: nx % 4 != 0 exercises partial quads
    y = np.zeros((ny, nx), np.float32)
    s = Sampler(ny=ny, nx=nx, y=y, sigma2=1.0, gamma=0.5, op="mask", mask=np.zeros((ny, nx), np.uint8))
    try:
        for seed, t in [(870, 1), (2 ** 40 + 3, 3)]:
            s.run(t, 0, seed)
            x, _, _ = s.state()
            # x^1 = sqrt(2*0.5) xi^1 exactly; x^t = sum of t normals.  Bound: reading R45 per normal
            # (1.2e-6 rho + 1e-7, rho = the Box-Muller radius of the lane pair) + fp32 summation
            fields = [oracle.normal_field(seed, k, ny, nx + 2, 0) for k in range(1, t + 1)]
            want = sum(f[:, :nx] for f in fields)
            rho = [np.sqrt(f[:, (np.arange(nx) & ~1)] ** 2 + f[:, (np.arange(nx) | 1)] ** 2) for f in fields]
            bound = sum(1.2e-6 * r + 1e-7 for r in rho) + t * 6e-8 * sum(np.abs(f[:, :nx]) for f in fields)
            err = np.abs(x - want)
            assert np.all(err <= bound), (err / bound).max()
    finally:
        s.close()


# ---------------------------------------------------------------- fp32 operator path
@pytest.mark.parametrize("kernel", ["random5", "random9", "gauss9", "gauss5"])
def test_one_iteration_conv(kernel):
    kw, pb = make_problem(53, 61, kernel=kernel)
    g = gpu_run(kw, 1, 0, 11)
    o = oracle.run(pb, 1, 0, 11, want_var=False)
    assert rel_l2(g["x"], o["x"]) <= 1e-6


@pytest.mark.parametrize("kernel,z", [("gauss9", False), ("random5", True), ("gauss5", True)])
def test_chain_50_fp32(kernel, z):
    kw, pb = make_problem(64, 72, kernel=kernel, z=z)
    g = gpu_run(kw, 50, 10, 870)
    o = oracle.run(pb, 50, 10, 870)
    assert rel_l2(g["x"], o["x"]) <= 1e-5
    assert rel_l2(g["mean"], o["mean"]) <= 1e-5
    assert rel_l2(g["var"], o["var"]) <= 1e-5   # SURVEY A16; conditioning: DESIGN.md R44
    if z:
        assert rel_l2(g["z"], o["z"]) <= 1e-5


def test_chain_50_mask():
    kw, pb = make_problem(66, 70, op="mask", z=True)
    g = gpu_run(kw, 50, 5, 871)
    o = oracle.run(pb, 50, 5, 871)
    assert rel_l2(g["x"], o["x"]) <= 1e-5
    assert rel_l2(g["mean"], o["mean"]) <= 1e-5
    assert rel_l2(g["z"], o["z"]) <= 1e-5


def test_stats_empty_and_bounds():
    kw, _ = make_problem(32, 32, op="mask")
    s = Sampler(**kw)
    try:
        s.run(5, 5, 1)
        with pytest.raises(Exception):
            s.moments()
        s.run(6, 5, 1)
        mean, var, n = s.moments(want_var=False)
        assert n == 1 and var is None
    finally:
        s.close()


# ---------------------------------------------------------------- halo index map (bit-exact)
@pytest.mark.parametrize("tiles,flags", [((2, 2), 0), ((3, 2), 0), ((2, 3), FLAG_HALO_VIA_NCCL)])
def test_halo_index_map(tiles, flags):
    ny, nx = 45, 53
    idx = np.arange(ny * nx, dtype=np.float32).reshape(ny, nx) + 1.0   # exact in fp32
    kw, _ = make_problem(ny, nx, kernel="random9", x0=None)
    kw["x0"] = idx
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        s.reset(0, 1)
        s.synchronize()
        h = s.halo
        pad = np.zeros((ny + 2 * h, nx + 2 * h), np.float32)
        pad[h:h + ny, h:h + nx] = idx
        for i in range(s.n_local_tiles):
            i0, j0, th, tw = s.tile_info(i)
            got = s.padded_x(i)
            want = pad[i0:i0 + th + 2 * h, j0:j0 + tw + 2 * h]
            assert np.array_equal(got, want), (i, tiles)
    finally:
        s.close()


# ---------------------------------------------------------------- B-invariance (bitwise)
@pytest.mark.parametrize("tiles,flags", [((2, 2), 0), ((3, 2), 0), ((1, 3), FLAG_HALO_VIA_NCCL),
                                         ((2, 1), FLAG_CNN_LAYERWISE)])
def test_tiled_equals_untiled_bitwise(tiles, flags):
    kw, _ = make_problem(61, 67, kernel="random5", cnn=(4, 16), z=True)
    a = gpu_run(kw, 12, 4, 5)
    b = gpu_run(kw, 12, 4, 5, tiles=tiles, flags=flags)
    for k in ("x", "z", "mean", "var"):
        assert np.array_equal(a[k], b[k]), k


# ---------------------------------------------------------------- CNN residual (tcgen05 kernel)
@pytest.mark.parametrize("K,P,shape,flags", [
    (4, 16, (40, 52), 0),
    (8, 32, (70, 150), 0),          # two fused chunks, two column strips, ragged tail
    (8, 32, (70, 150), FLAG_CNN_LAYERWISE),
    (3, 64, (33, 140), 0),
    (5, 32, (19, 300), 0),
])
def test_denoiser_residual_matches_oracle(K, P, shape, flags):
    ny, nx = shape
    kw, pb = make_problem(ny, nx, kernel="gauss5", cnn=(K, P))
    s = Sampler(**kw, flags=flags)
    try:
        s.reset(0, 1)
        G = s.denoiser_residual()
    finally:
        s.close()
    x0 = kw["x0"]
    ref = oracle.dncnn_residual(x0, kw["weights"], kw["biases"], K, P)
    ref16 = oracle.dncnn_residual(x0, kw["weights"], kw["biases"], K, P, bf16_emulate=True)
    assert rel_l2(G, ref) <= 2e-2
    assert rel_l2(G, ref16) <= 2e-3


def test_chain_50_with_cnn():
    kw, pb = make_problem(48, 56, kernel="gauss9", cnn=(8, 32))
    g = gpu_run(kw, 50, 10, 9)
    o = oracle.run(pb, 50, 10, 9)
    o16 = oracle.run(pb, 50, 10, 9, bf16_emulate=True)
    assert rel_l2(g["x"], o["x"]) <= 2e-2
    assert rel_l2(g["mean"], o["mean"]) <= 2e-2
    assert rel_l2(g["x"], o16["x"]) <= 2e-3


@pytest.mark.parametrize("case", ["cnn", "poisson", "tv"])
def test_checkpoint_resume_is_bitwise(case):
    """save after 9 iterations, load into a fresh context, advance 11: identical to 20 straight
    (x, z blocks, moments) -- SURVEY 8(f) rank 4 resume."""
    if case == "cnn":
        kw, _ = make_problem(45, 52, kernel="gauss5", cnn=(4, 16), z=True)
    elif case == "poisson":
        from test_gpu_poisson import poisson_problem
        kw, _ = poisson_problem(47, 50, kernel="random5", cnn=(4, 16))
    else:
        from test_gpu_tv import tv_problem
        kw, _ = tv_problem(47, 50, kernel="random5")
    ref = Sampler(**kw, tiles=(2, 1))
    ref.run(20, 4, 77)
    want_x, want_z, _ = ref.state()
    want_m, want_v, _ = ref.moments()
    aux = (lambda smp: smp.z1()) if case == "poisson" else (lambda smp: smp.tv_zh()) if case == "tv" else None
    want_z1 = aux(ref) if aux else None
    ref.close()
    a = Sampler(**kw, tiles=(2, 1))
    a.reset(4, 77)
    a.advance(9)
    blob = a.save_checkpoint()
    a.close()
    b = Sampler(**kw, tiles=(2, 1))
    b.load_checkpoint(blob)
    b.advance(11)
    x, z, t = b.state()
    m, v, _ = b.moments()
    assert t == 20
    np.testing.assert_array_equal(x, want_x)
    np.testing.assert_array_equal(z, want_z)
    np.testing.assert_array_equal(m, want_m)
    np.testing.assert_array_equal(v, want_v)
    if want_z1 is not None:
        np.testing.assert_array_equal(aux(b), want_z1)
    b.close()
