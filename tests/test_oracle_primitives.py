"""Pins of the CPU oracle's primitives against values fixed by the paper, published
known-answer tests, and independent library routines (scipy / torch), never
against the oracle itself.  CPU only."""
import numpy as np
import pytest
import scipy.signal
import scipy.stats
import torch

import oracle
import synth
from conftest import golden


def _rows(name):
    with open(golden(name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ---------------------------------------------------------------- partition (Fig. 1)
def test_partition_matches_paper_fig1():
    for row in _rows("partition_fig1.txt"):
        n, parts = int(row[0]), int(row[1])
        want = [tuple(int(v) for v in s.split(":")) for s in row[2:]]
        got = [oracle.partition(n, parts, p) for p in range(parts)]
        assert got == want


def test_partition_covers_and_balances():
    for n in [1, 7, 20, 64, 1000, 4097]:
        for parts in range(1, min(n, 9) + 1):
            blocks = [oracle.partition(n, parts, p) for p in range(parts)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(parts - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


# ---------------------------------------------------------------- Philox KAT
def test_philox_known_answers():
    for row in _rows("philox4x32_10_kat.txt"):
        vals = [int(v, 16) for v in row]
        got = oracle.philox4x32_10(vals[0:4], vals[4:6])
        assert list(got) == vals[6:10]


# ---------------------------------------------------------------- normals
def test_normals_statistics():
    f = oracle.normal_field(870, 1, 250, 400, 0).ravel()        # 1e5 draws
    assert abs(f.mean()) < 0.01
    assert abs(f.var() - 1.0) < 0.02
    assert scipy.stats.kstest(f, "norm").pvalue > 0.01
    ac = np.corrcoef(f[:-1], f[1:])[0, 1]
    assert abs(ac) < 0.01
    g = oracle.normal_field(870, 1, 250, 400, 1).ravel()        # other stream
    assert abs(np.corrcoef(f, g)[0, 1]) < 0.01
    h = oracle.normal_field(870, 2, 250, 400, 0).ravel()        # other iteration
    assert abs(np.corrcoef(f, h)[0, 1]) < 0.01


def test_normal_is_pure_and_partition_free():
    # value at (seed, t+1, i, j, stream) does not depend on the field it is drawn in
    f = oracle.normal_field(5, 3, 9, 13, 0)
    for (i, j) in [(0, 0), (4, 7), (8, 12), (3, 3)]:
        assert oracle.normal(5, 3, i, j, 0) == f[i, j]


# ---------------------------------------------------------------- convolution H and adjoint
def test_conv_spec_examples():
    # [1,2,3,4] * [1,1,1] (same, zero BC) = [3,6,9,7]
    x = np.array([[1.0, 2.0, 3.0, 4.0]])
    k = np.array([[1.0, 1.0, 1.0]])
    assert np.array_equal(oracle.conv_fwd(x, k), [[3, 6, 9, 7]])
    # adjoint of u = [1,0,0,0] is [1,1,0,0]
    assert np.array_equal(oracle.conv_adj(np.array([[1.0, 0, 0, 0]]), k), [[1, 1, 0, 0]])
    # delta kernel -> identity
    d = np.zeros((5, 5)); d[2, 2] = 1
    xr = np.random.default_rng(0).standard_normal((7, 9))
    assert np.array_equal(oracle.conv_fwd(xr, d), xr)


@pytest.mark.parametrize("shape,ks", [((13, 17), (5, 5)), ((16, 11), (9, 9)), ((8, 8), (3, 7))])
def test_conv_matches_scipy(shape, ks):
    rng = np.random.default_rng(1)
    x = rng.standard_normal(shape)
    k = synth.random_kernel(*ks).astype(np.float64)
    ref = scipy.signal.convolve2d(x, k, mode="same", boundary="fill")
    np.testing.assert_allclose(oracle.conv_fwd(x, k), ref, rtol=0, atol=1e-13)
    refa = scipy.signal.correlate2d(x, k, mode="same", boundary="fill")
    np.testing.assert_allclose(oracle.conv_adj(x, k), refa, rtol=0, atol=1e-13)


def test_adjoint_identity():
    rng = np.random.default_rng(2)
    for ks in [(5, 5), (9, 9), (3, 5)]:
        k = synth.random_kernel(*ks).astype(np.float64)
        x = rng.standard_normal((21, 19))
        u = rng.standard_normal((21, 19))
        lhs = np.vdot(oracle.conv_fwd(x, k), u)
        rhs = np.vdot(x, oracle.conv_adj(u, k))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_conv_dense_bruteforce():
    # explicit matrix H built column by column from scipy on unit vectors
    ny, nx = 6, 7
    k = synth.random_kernel(5, 3).astype(np.float64)
    H = np.zeros((ny * nx, ny * nx))
    for n in range(ny * nx):
        e = np.zeros(ny * nx); e[n] = 1
        H[:, n] = scipy.signal.convolve2d(e.reshape(ny, nx), k, mode="same").ravel()
    x = np.random.default_rng(3).standard_normal((ny, nx))
    np.testing.assert_allclose(oracle.conv_fwd(x, k).ravel(), H @ x.ravel(), atol=1e-13)
    np.testing.assert_allclose(oracle.conv_adj(x, k).ravel(), H.T @ x.ravel(), atol=1e-13)


# ---------------------------------------------------------------- CNN residual
def _torch_dncnn(x, w, b, K, P, bf16=False):
    t = torch.from_numpy(np.asarray(x, dtype=np.float64))[None, None]
    rb = (lambda a: a.to(torch.float32).to(torch.bfloat16).to(torch.float64)) if bf16 else (lambda a: a)
    t = rb(t)
    off, boff, cin = 0, 0, 1
    for k in range(1, K + 1):
        cout = 1 if k == K else P
        wk = torch.from_numpy(w[off:off + cout * cin * 9].astype(np.float64)).reshape(cout, cin, 3, 3)
        bk = torch.from_numpy(b[boff:boff + cout].astype(np.float64))
        t = torch.nn.functional.conv2d(t, rb(wk), bk, padding=1)
        if k < K:
            t = rb(torch.relu(t))
        off += cout * cin * 9
        boff += cout
        cin = cout
    return t[0, 0].numpy()


@pytest.mark.parametrize("K,P", [(4, 16), (8, 32), (3, 8)])
def test_dncnn_matches_torch(K, P):
    w, b = synth.dncnn_weights(K, P, seed=11)
    x = synth.ground_truth(19, 23)
    G = oracle.dncnn_residual(x, w, b, K, P)
    np.testing.assert_allclose(G, _torch_dncnn(x, w, b, K, P), rtol=0, atol=1e-12)


def test_dncnn_bf16_emulation_matches_torch():
    K, P = 4, 16
    w, b = synth.dncnn_weights(K, P, seed=12)
    x = synth.ground_truth(17, 15)
    G = oracle.dncnn_residual(x, w, b, K, P, bf16_emulate=True)
    np.testing.assert_allclose(G, _torch_dncnn(x, w, b, K, P, bf16=True), rtol=0, atol=1e-12)


def test_dncnn_zero_weights_is_identity_denoiser():
    K, P = 5, 8
    w, b = synth.dncnn_weights(K, P)
    G = oracle.dncnn_residual(synth.ground_truth(9, 9), np.zeros_like(w), np.zeros_like(b), K, P)
    assert np.all(G == 0.0)          # G = 0  <=>  D_eps = Id


def test_dncnn_linear_construction():
    K, P, theta = 6, 4, 0.37
    w, b = synth.linear_cnn_weights(K, P, theta)
    x = synth.ground_truth(11, 13) * 3 - 1
    np.testing.assert_allclose(oracle.dncnn_residual(x, w, b, K, P), theta * x, atol=1e-12)


def test_param_counts_table1():
    for row in _rows("dncnn_param_counts.txt"):
        if row[0] == "ddfb":
            K, F, C, n = map(int, row[1:])
            assert oracle.ddfb_param_count(K, F, C) == n
            continue
        K, F, C, n = map(int, row)
        assert oracle.dncnn_param_count(K, F, C) == n
    w, b = synth.dncnn_weights(8, 32)
    assert w.size + b.size == oracle.dncnn_param_count(8, 32, 1) == 56097


# ---------------------------------------------------------------- step sizes
def test_stepsize_validator_spec_examples():
    assert oracle.check_stepsizes(1, 0, 1, 1, 2, 1 / 8, 0.03) == 0
    assert oracle.check_stepsizes(1, 0, 1, 1, 2, 1 / 8, 0.04) == 2
    assert oracle.check_stepsizes(1, 0, 0, 1, 0, 1 / 4, 0.01) == 0     # boundary equality is OK
    assert oracle.check_stepsizes(1, 0, 0, 1, 0, 0.26, 0.01) == 1
