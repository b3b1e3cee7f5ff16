"""GPU edge and degenerate cases against the oracle: a 1x1 kernel (H = k I: no stencil halo),
a 3x1 (non-square) kernel, tiles exactly as small as the halo, images smaller than one CNN strip
and than one update block, a mask with no observed pixel and one with every pixel observed,
a chain whose burn-in leaves exactly one sample, and a seed above 2^32 (both key words used)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import gpu_run, make_problem, rel_l2
from paper_2511_00870_b200 import Sampler, params

pytestmark = pytest.mark.gpu


def _conv_problem(ny, nx, k, cnn=None, x0=True):
    s2 = 1e-2
    y = (synth.blurred_truth(ny, nx, k) + 0.1 * synth.white_noise(ny, nx)).astype(np.float32)
    hp = params.gaussian_pnp(s2, 1.0, 1.0)
    common = dict(sigma2=s2, gamma=hp["gamma"], lam=hp["lam"], c_lo=0.0, c_hi=1.0)
    if cnn:
        w, b = synth.dncnn_weights(cnn[0], cnn[1], seed=3)
        common.update(weights=w, biases=b, n_layers=cnn[0], channels=cnn[1], alpha=1.0, eps=hp["eps"])
    if x0:
        common["x0"] = (synth.ground_truth(ny, nx) * 0.8 + 0.1).astype(np.float32)
    kw = dict(ny=ny, nx=nx, y=y, kernel=k.astype(np.float32), **common)
    pb = oracle.Problem(y=y, op="conv", kernel=k.astype(np.float32), **common)
    return kw, pb


@pytest.mark.parametrize("k", [np.array([[0.7]]), np.array([[0.2], [0.5], [0.3]]), np.array([[0.25, 0.5, 0.25]])])
def test_degenerate_kernels(k):
    kw, pb = _conv_problem(29, 34, k)
    g = gpu_run(kw, 20, 5, 3)
    o = oracle.run(pb, 20, 5, 3)
    assert rel_l2(g["x"], o["x"]) <= 1e-5 and rel_l2(g["mean"], o["mean"]) <= 1e-5


def test_tiles_as_small_as_the_halo():
    # 5x5 kernel, 4x16 CNN: h = max(2*2, 4) = 4; a 16 x 12 image in 4 x 3 tiles of 4 x 4
    k = synth.random_kernel(5, 5, seed=1)
    kw, pb = _conv_problem(16, 12, k, cnn=(4, 16))
    a = gpu_run(kw, 8, 2, 5)
    t = gpu_run(kw, 8, 2, 5, tiles=(4, 3))
    for key in ("x", "mean", "var"):
        np.testing.assert_array_equal(a[key], t[key])
    ob = oracle.run(pb, 8, 2, 5, bf16_emulate=True)
    assert rel_l2(a["x"], ob["x"]) <= 2e-3


@pytest.mark.parametrize("shape", [(3, 5), (9, 130), (150, 7)])
def test_images_smaller_than_a_strip_or_block(shape):
    ny, nx = shape
    k = synth.random_kernel(3, 3, seed=2)
    kw, pb = _conv_problem(ny, nx, k, cnn=(4, 16))
    g = gpu_run(kw, 10, 2, 7)
    ob = oracle.run(pb, 10, 2, 7, bf16_emulate=True)
    assert rel_l2(g["x"], ob["x"]) <= 2e-3


@pytest.mark.parametrize("fill", [0, 1])
def test_mask_all_unobserved_or_all_observed(fill):
    ny, nx = 33, 41
    kw, pb = make_problem(ny, nx, op="mask", z=True)
    m = np.full((ny, nx), fill, np.uint8)
    kw["mask"] = m
    pb.mask = m
    g = gpu_run(kw, 30, 3, 9)
    o = oracle.run(pb, 30, 3, 9)
    assert rel_l2(g["x"], o["x"]) <= 1e-5 and rel_l2(g["z"], o["z"]) <= 1e-5


def test_single_post_burn_in_sample_and_large_seed():
    kw, pb = make_problem(40, 44, kernel="gauss5")
    s = Sampler(**kw)
    try:
        seed = (1 << 40) + 12345
        s.run(7, 6, seed)
        x, _, _ = s.state()
        mean, _, n = s.moments(want_var=False)
        assert n == 1
        np.testing.assert_array_equal(mean, x)   # Welford with n = 1: mean = the sample
        with pytest.raises(Exception):
            s.moments(want_var=True)            # variance needs n >= 2
    finally:
        s.close()
    o = oracle.run(pb, 7, 6, seed, want_var=False)
    assert rel_l2(x, o["x"]) <= 1e-5


@pytest.mark.parametrize("tiles", [(1, 1), (2, 2)])
def test_opnorm2_power_iteration(tiles):
    """||H||^2 on the GPU (power iteration over the tiled operator) vs the largest eigenvalue of
    H^T H from a dense matrix built with scipy (zero-boundary same-size convolution)."""
    from scipy.signal import convolve2d
    ny, nx = 30, 27
    k = synth.random_kernel(5, 5, seed=4) - 0.02
    H = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros(ny * nx)
        e[n] = 1.0
        H[:, n] = convolve2d(e.reshape(ny, nx), k, mode="same").ravel()
    lam = np.linalg.eigvalsh(H.T @ H)[-1]
    kw, _ = _conv_problem(ny, nx, k)
    s = Sampler(**kw, tiles=tiles)
    try:
        est = s.opnorm2(400)
    finally:
        s.close()
    # Rayleigh quotients never exceed lambda_max; the top of this spectrum is clustered
    # (0.24656, 0.24630, 0.24486, ...), so 400 iterations land within ~1 % of it
    assert lam * 0.99 <= est <= lam * (1 + 1e-5)
    # a kernel with a well-separated top eigenvalue: 2 taps, converges fast
    k2 = np.zeros((3, 3))
    k2[1, 1], k2[1, 2] = 1.0, 0.9
    H2 = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros(ny * nx)
        e[n] = 1.0
        H2[:, n] = convolve2d(e.reshape(ny, nx), k2, mode="same").ravel()
    lam2 = np.linalg.eigvalsh(H2.T @ H2)[-1]
    kw2, _ = _conv_problem(ny, nx, k2)
    s = Sampler(**kw2, tiles=tiles)
    try:
        est2 = s.opnorm2(3000)
    finally:
        s.close()
    assert lam2 * 0.999 <= est2 <= lam2 * (1 + 1e-5)
