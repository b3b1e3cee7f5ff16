"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds NO arithmetic of the method (no sampler step, no operator of
the library).  It only draws inputs shaped like the paper's workloads
(recipe in DESIGN.md "Input recipe"):

* ground truth: procedural, tile-local, piecewise-smooth texture in [0, 1]
  ("cropped ... normalized into C = [0,1]^N");
* blur kernels: normalised Gaussian (separable factors) and random asymmetric
  normalised kernels (parity cases; asymmetry exposes flip bugs);
* observations: y = conv(xbar, K) + sigma w, y = m (xbar + sigma w)
  with m ~ Bernoulli(0.3), or counts y ~ Poisson(eta conv(xbar, K))
  (P:731-735).  The data-generation convolution uses
  scipy.signal.fftconvolve (a library routine independent of both the oracle
  and the CUDA path);
* random-init DnCNN-style weights, each layer rescaled to
  spectral norm 0.9 (reading R13).

Every array is reproducible from (seed, global pixel coordinates): a rank can
generate just its own rectangle and obtain exactly the global image's values.
"""
from __future__ import annotations

import numpy as np

BLOCK = 256          # noise / mask blocks are drawn per aligned 256x256 block
GT_SEED = 2511       # ground-truth texture parameters
NOISE_SEED = 2512    # observation noise and masks
WEIGHT_SEED = 2513   # denoiser weights


# ---------------------------------------------------------------- ground truth
def _gt_params(seed: int = GT_SEED):
    rng = np.random.default_rng(seed)
    K = 16
    amps = rng.uniform(0.03, 0.12, K)
    freqs = rng.integers(-12, 13, size=(K, 2)).astype(np.float64)
    freqs[np.all(freqs == 0, axis=1)] = 1.0
    phases = rng.uniform(0, 2 * np.pi, K)
    D = 24
    centers = rng.uniform(0.0, 1.0, size=(D, 2))
    radii = rng.uniform(0.02, 0.12, D)
    vals = rng.choice([-0.3, 0.3], D)
    return amps, freqs, phases, centers, radii, vals


def ground_truth(ny: int, nx: int, rect=None, seed: int = GT_SEED) -> np.ndarray:
    """x̄ on rect = (i0, j0, h, w) (global coordinates; default whole image), fp32.
    Pixels outside [0,ny)x[0,nx) are returned as 0 (zero boundary)."""
    i0, j0, h, w = rect if rect is not None else (0, 0, ny, nx)
    amps, freqs, phases, centers, radii, vals = _gt_params(seed)
    ii = np.arange(i0, i0 + h, dtype=np.float64) / ny
    jj = np.arange(j0, j0 + w, dtype=np.float64) / nx
    out = np.full((h, w), 0.5, dtype=np.float64)
    for a, f, ph in zip(amps, freqs, phases):
        # cos(A_i + B_j) = cos A_i cos B_j - sin A_i sin B_j  (outer products)
        A = 2 * np.pi * f[0] * ii + ph
        B = 2 * np.pi * f[1] * jj
        out += a * (np.outer(np.cos(A), np.cos(B)) - np.outer(np.sin(A), np.sin(B)))
    for c, r, v in zip(centers, radii, vals):
        a0 = max(int(np.floor((c[0] - r) * ny)) - i0 - 1, 0)
        a1 = min(int(np.ceil((c[0] + r) * ny)) - i0 + 2, h)
        b0 = max(int(np.floor((c[1] - r) * nx)) - j0 - 1, 0)
        b1 = min(int(np.ceil((c[1] + r) * nx)) - j0 + 2, w)
        if a0 >= a1 or b0 >= b1:
            continue
        d2 = (ii[a0:a1, None] - c[0]) ** 2 + (jj[None, b0:b1] - c[1]) ** 2
        out[a0:a1, b0:b1] += v * (d2 < r * r)
    np.clip(out, 0.0, 1.0, out=out)
    ri = np.arange(i0, i0 + h)
    rj = np.arange(j0, j0 + w)
    out[(ri < 0) | (ri >= ny), :] = 0.0
    out[:, (rj < 0) | (rj >= nx)] = 0.0
    return out.astype(np.float32)


# ---------------------------------------------------------------- kernels
def gaussian_factors(L: int, sigma_b: float) -> tuple[np.ndarray, np.ndarray]:
    """1-D normalised Gaussian taps (fp32); the 2-D kernel is their outer product."""
    r = L // 2
    t = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-0.5 * (t / sigma_b) ** 2)
    g /= g.sum()
    g = g.astype(np.float32)
    return g.copy(), g.copy()


def outer(ky: np.ndarray, kx: np.ndarray) -> np.ndarray:
    return (ky.astype(np.float64)[:, None] * kx.astype(np.float64)[None, :])


def random_kernel(kh: int, kw: int, seed: int = 7) -> np.ndarray:
    """Random, asymmetric, non-negative kernel normalised to sum 1 (fp32)."""
    rng = np.random.default_rng(seed)
    k = rng.uniform(0.0, 1.0, size=(kh, kw))
    k[0, :] *= 3.0          # break every symmetry
    k[:, -1] *= 0.2
    k /= k.sum()
    return k.astype(np.float32)


# ---------------------------------------------------------------- noise/mask blocks
def _block_field(ny, nx, rect, seed, tag, draw):
    i0, j0, h, w = rect
    out = np.zeros((h, w), dtype=np.float64)
    bi0, bi1 = max(i0, 0) // BLOCK, (min(i0 + h, ny) - 1) // BLOCK
    bj0, bj1 = max(j0, 0) // BLOCK, (min(j0 + w, nx) - 1) // BLOCK
    for bi in range(bi0, bi1 + 1):
        for bj in range(bj0, bj1 + 1):
            rng = np.random.default_rng(np.random.SeedSequence([seed, tag, bi, bj]))
            blk = draw(rng, (BLOCK, BLOCK))
            gi0, gj0 = bi * BLOCK, bj * BLOCK
            a0, a1 = max(gi0, i0), min(gi0 + BLOCK, i0 + h, ny)
            b0, b1 = max(gj0, j0), min(gj0 + BLOCK, j0 + w, nx)
            if a0 < a1 and b0 < b1:
                out[a0 - i0:a1 - i0, b0 - j0:b1 - j0] = blk[a0 - gi0:a1 - gi0, b0 - gj0:b1 - gj0]
    return out


def white_noise(ny, nx, rect=None, seed=NOISE_SEED) -> np.ndarray:
    rect = rect if rect is not None else (0, 0, ny, nx)
    return _block_field(ny, nx, rect, seed, 1, lambda g, s: g.standard_normal(s))


def bernoulli_mask(ny, nx, p=0.3, rect=None, seed=NOISE_SEED) -> np.ndarray:
    rect = rect if rect is not None else (0, 0, ny, nx)
    return (_block_field(ny, nx, rect, seed, 2, lambda g, s: g.uniform(0, 1, s)) < p).astype(np.uint8)


# ---------------------------------------------------------------- observations
def _blur_valid(xext: np.ndarray, k2d: np.ndarray) -> np.ndarray:
    from scipy.signal import fftconvolve
    return fftconvolve(xext.astype(np.float64), k2d, mode="valid")


def blurred_truth(ny, nx, k2d, rect=None, gt_seed=GT_SEED) -> np.ndarray:
    """conv(x̄, K) (same size, zero boundary) on rect, via scipy FFT convolution."""
    i0, j0, h, w = rect if rect is not None else (0, 0, ny, nx)
    ry, rx = k2d.shape[0] // 2, k2d.shape[1] // 2
    xe = ground_truth(ny, nx, (i0 - ry, j0 - rx, h + 2 * ry, w + 2 * rx), seed=gt_seed)
    return _blur_valid(xe, k2d)


def probe_rect(ny, nx, size=256):
    s = min(size, ny, nx)
    return ((ny - s) // 2, (nx - s) // 2, s, s)


def noise_sigma2_blur(ny, nx, k2d, snr_db=25.0) -> float:
    """sigma^2 giving the input SNR measured on a fixed central probe crop."""
    hx = blurred_truth(ny, nx, k2d, probe_rect(ny, nx))
    return float(np.mean(hx ** 2) / 10 ** (snr_db / 10))


def noise_sigma2_mask(ny, nx, snr_db=15.0) -> float:
    xb = ground_truth(ny, nx, probe_rect(ny, nx)).astype(np.float64)
    return float(np.mean(xb ** 2) / 10 ** (snr_db / 10))


def observe_blur(ny, nx, k2d, sigma2, rect=None, gt_seed=GT_SEED, noise_seed=NOISE_SEED) -> np.ndarray:
    rect = rect if rect is not None else (0, 0, ny, nx)
    y = blurred_truth(ny, nx, k2d, rect, gt_seed) + np.sqrt(sigma2) * white_noise(ny, nx, rect, noise_seed)
    i0, j0, h, w = rect
    y[:max(0, -i0), :] = 0
    y[:, :max(0, -j0)] = 0
    if i0 + h > ny:
        y[ny - i0:, :] = 0
    if j0 + w > nx:
        y[:, nx - j0:] = 0
    return y.astype(np.float32)


def observe_poisson(ny, nx, k2d, eta=250.0, rect=None) -> np.ndarray:
    """Counts y ~ Poisson(eta conv(xbar, K)) (eq:likelihood:poisson_deconvolution, P:731-735;
    eta = 250 in the paper).  Drawn per aligned 256x256 block with a generator seeded by
    (seed, block) from that whole block's intensities (computed on the block alone), so any
    rectangle reproduces the global image's values exactly; zero outside the image."""
    i0, j0, h, w = rect if rect is not None else (0, 0, ny, nx)
    out = np.zeros((h, w), dtype=np.float64)
    bi0, bi1 = max(i0, 0) // BLOCK, (min(i0 + h, ny) - 1) // BLOCK
    bj0, bj1 = max(j0, 0) // BLOCK, (min(j0 + w, nx) - 1) // BLOCK
    for bi in range(bi0, bi1 + 1):
        for bj in range(bj0, bj1 + 1):
            gi0, gj0 = bi * BLOCK, bj * BLOCK
            bh, bw = min(BLOCK, ny - gi0), min(BLOCK, nx - gj0)
            lam = eta * np.clip(blurred_truth(ny, nx, k2d, (gi0, gj0, bh, bw)), 0.0, None)
            rng = np.random.default_rng(np.random.SeedSequence([NOISE_SEED, 3, bi, bj]))
            blk = rng.poisson(lam).astype(np.float64)
            a0, a1 = max(gi0, i0), min(gi0 + bh, i0 + h)
            b0, b1 = max(gj0, j0), min(gj0 + bw, j0 + w)
            if a0 < a1 and b0 < b1:
                out[a0 - i0:a1 - i0, b0 - j0:b1 - j0] = blk[a0 - gi0:a1 - gi0, b0 - gj0:b1 - gj0]
    return out.astype(np.float32)


def observe_mask(ny, nx, sigma2, p=0.3, rect=None):
    rect = rect if rect is not None else (0, 0, ny, nx)
    m = bernoulli_mask(ny, nx, p, rect)
    y = m * (ground_truth(ny, nx, rect).astype(np.float64) + np.sqrt(sigma2) * white_noise(ny, nx, rect))
    return y.astype(np.float32), m


# ---------------------------------------------------------------- colour (C = 3; reading R43)
def rgb_seeds(c: int):
    """(ground-truth seed, noise seed) of colour channel c: one texture and one noise field per plane."""
    return GT_SEED + 17 * c, NOISE_SEED + 17 * c


def ground_truth_rgb(ny, nx, rect=None, C=3) -> np.ndarray:
    """Planes [C][h][w]: channel c is the procedural texture with seed rgb_seeds(c)[0]."""
    return np.stack([ground_truth(ny, nx, rect, seed=rgb_seeds(c)[0]) for c in range(C)])


def observe_blur_rgb(ny, nx, k2d, sigma2, rect=None, C=3) -> np.ndarray:
    """y_c = conv(x̄_c, K) + sigma w_c per plane (the same blur on every channel)."""
    return np.stack([observe_blur(ny, nx, k2d, sigma2, rect, *rgb_seeds(c)) for c in range(C)])


def observe_mask_rgb(ny, nx, sigma2, p=0.3, rect=None, C=3):
    """A per-pixel mask shared by the channels, y_c = m (x̄_c + sigma w_c)."""
    rect = rect if rect is not None else (0, 0, ny, nx)
    m = bernoulli_mask(ny, nx, p, rect)
    y = np.stack([m * (ground_truth(ny, nx, rect, seed=rgb_seeds(c)[0]).astype(np.float64)
                       + np.sqrt(sigma2) * white_noise(ny, nx, rect, rgb_seeds(c)[1])) for c in range(C)])
    return y.astype(np.float32), m


# ---------------------------------------------------------------- denoiser weights
def _conv_spectral_norm(w: np.ndarray, grid: int = 64) -> float:
    """Largest singular value of the multichannel 3x3 circular convolution on a grid^2 torus
    (upper-bounds the zero-padded operator norm)."""
    cout, cin = w.shape[:2]
    W = np.zeros((cout, cin, grid, grid))
    W[:, :, :3, :3] = w
    F = np.fft.fft2(W, axes=(2, 3))              # cout x cin x g x g
    F = np.transpose(F, (2, 3, 0, 1)).reshape(-1, cout, cin)
    return float(np.max(np.linalg.svd(F, compute_uv=False)))


def dncnn_weights(n_layers: int, channels: int, seed: int = WEIGHT_SEED, target_norm: float = 0.9,
                  image_channels: int = 1):
    """Random-init DnCNN-style (C -> P, (K-2) x P -> P, P -> C; 3x3) weights, fp32 OIHW
    concatenated, and biases concatenated.  PyTorch-default-like U(-1/sqrt(fan_in), +)."""
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    cin = image_channels
    for k in range(1, n_layers + 1):
        cout = image_channels if k == n_layers else channels
        bound = 1.0 / np.sqrt(cin * 9)
        w = rng.uniform(-bound, bound, size=(cout, cin, 3, 3))
        w *= target_norm / _conv_spectral_norm(w)
        b = rng.uniform(-0.01, 0.01, size=cout)
        ws.append(w.astype(np.float32).ravel())
        bs.append(b.astype(np.float32))
        cin = cout
    return np.concatenate(ws), np.concatenate(bs)


def linear_cnn_weights(n_layers: int, channels: int, theta: float, shift: float = 10.0):
    """A DnCNN whose residual is exactly G(x) = theta * x on inputs > -shift:
    layer 1 puts x + shift in channel 0 (ReLU inactive), middle layers copy channel 0,
    the last layer outputs theta*(ch0) - theta*shift.  Used for a closed-form pin."""
    ws, bs = [], []
    cin = 1
    for k in range(1, n_layers + 1):
        cout = 1 if k == n_layers else channels
        w = np.zeros((cout, cin, 3, 3))
        b = np.zeros(cout)
        if k == 1:
            w[0, 0, 1, 1] = 1.0
            b[0] = shift
        elif k < n_layers:
            w[0, 0, 1, 1] = 1.0
        else:
            w[0, 0, 1, 1] = theta
            b[0] = -theta * shift
        ws.append(w.astype(np.float32).ravel())
        bs.append(b.astype(np.float32))
        cin = cout
    return np.concatenate(ws), np.concatenate(bs)


def ddfb_weights(n_layers: int, channels: int, seed: int = WEIGHT_SEED + 1, ht_eps: float = 0.05,
                 image_channels: int = 1):
    """Random-init DDFB weights (Example sec:denoiser:cnn:ddfb): K operators W_k : C -> P
    (3x3, fp32 [P][C][3][3] concatenated; C = image_channels), steps gamma_k = 1.8 / ||W_k||^2
    inside (0, 2/||W_k||^2), and the hard-tanh level."""
    rng = np.random.default_rng(seed)
    ws, gs = [], []
    bound = 1.0 / np.sqrt(9.0 * image_channels)
    for _ in range(n_layers):
        w = rng.uniform(-bound, bound, size=(channels, image_channels, 3, 3))
        nrm = _conv_spectral_norm(w)
        ws.append(w.astype(np.float32).ravel())
        gs.append(np.float32(1.8 / nrm ** 2))
    return np.concatenate(ws), np.asarray(gs, np.float32), float(ht_eps)
