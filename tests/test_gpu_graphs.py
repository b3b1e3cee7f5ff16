"""CUDA-graph replay of the iteration (pnpula_host.cpp step(): after one direct iteration, each
single-rank untimed iteration replays a captured graph per x-buffer parity; the iteration
scalars t+1, accumulate, 1/n come from a device IterState advanced in-graph).  The replayed
chain must be bitwise equal to the directly launched one (PNPULA_FLAG_NO_GRAPH) for every
posterior the library runs, across reset (new seed / burn-in), checkpoint load, timing toggles
and a tile grid; and the direct path must still agree with the oracle."""
import numpy as np
import pytest

import oracle
import synth
from gpu_common import make_problem, rel_l2
from paper_2511_00870_b200 import FLAG_NO_GRAPH, Sampler, params

pytestmark = pytest.mark.gpu


def _chain(kw, flags, tiles=(1, 1), plan=((9, 3, 11),)):
    """Runs reset(burn_in, seed) + advance(n) for each (n, burn_in, seed) in plan; returns the
    fields after the last one and the library's launch count."""
    s = Sampler(**kw, tiles=tiles, flags=flags)
    try:
        for n, b, seed in plan:
            s.run(n, b, seed)
        x, z, t = s.state()
        mean, var, cnt = s.moments()
        out = dict(x=x, z=z, mean=mean, var=var)
        if kw.get("op") == "poisson":
            out["z1"] = s.z1()
        if kw.get("tv_beta", 0) > 0:
            out["zh"] = s.tv_zh()
        _, launches = s.kernel_time("all")
        return out, (t, cnt), launches
    finally:
        s.close()


def _assert_same(a, b):
    for k in a[0]:
        np.testing.assert_array_equal(a[0][k], b[0][k], err_msg=k)
    assert a[1] == b[1]


def _poisson_tv_kw(ny, nx):
    ky, kx = synth.gaussian_factors(5, 1.0)
    y = synth.observe_poisson(ny, nx, synth.outer(ky, kx), 250.0)
    hp = params.poisson_pnp(250.0)
    gamma = 0.99 / (250.0 ** 2 / hp["rho1"] + 8.0 / 1e-3)
    return dict(ny=ny, nx=nx, y=y, sigma2=1.0, op="poisson", kernel_sep=(ky, kx), gamma=gamma, eta=250.0,
                rho1=hp["rho1"], kappa1=hp["kappa1"], rho=1e-3, kappa=0.99e-3 / 8, tv_beta=13.0,
                x0=(synth.ground_truth(ny, nx) * 0.8 + 0.1).astype(np.float32))


@pytest.mark.parametrize("case", ["cnn", "mask_z", "poisson_tv", "ddfb"])
def test_graph_replay_bitwise_equals_direct(case):
    if case == "cnn":
        kw, _ = make_problem(150, 170, kernel="gauss9", cnn=(8, 32))
    elif case == "mask_z":
        kw, _ = make_problem(97, 130, op="mask", z=True)
    elif case == "poisson_tv":
        kw = _poisson_tv_kw(120, 136)
    else:
        kw, _ = make_problem(96, 100, kernel="gauss5")
        w, gam, ht = synth.ddfb_weights(4, 32, seed=5)
        kw.update(weights=w, n_layers=4, channels=32, alpha=1.0, eps=0.1, den_kind="ddfb", ddfb_gammas=gam,
                  ht_eps=ht)
    plan = ((7, 2, 11), (10, 4, 12))   # second reset: new seed and burn-in -> graphs re-captured
    g = _chain(kw, 0, plan=plan)
    d = _chain(kw, FLAG_NO_GRAPH, plan=plan)
    _assert_same(g, d)
    # a replay counts the kernels it holds (the t advance rides in the first update kernel)
    assert g[2] == d[2]
    _assert_same(g, _chain(kw, 0, tiles=(2, 2), plan=plan))   # tiled replay: bitwise


def test_graph_replay_matches_oracle_and_survives_checkpoint_and_timing():
    kw, pb = make_problem(130, 150, kernel="random5", z=True)
    s = Sampler(**kw)
    try:
        s.run(5, 3, 77)                 # iterations 2.. replay graphs
        blob = s.save_checkpoint()
        s.advance(4)
        x_a, z_a, _ = s.state()
        s.load_checkpoint(blob)         # t goes back: graphs dropped, device t re-uploaded
        s.set_timing(True)
        s.advance(2)                    # direct (timed)
        s.set_timing(False)
        s.advance(2)                    # replay again from t = 7
        x_b, z_b, t = s.state()
        mean, var, n = s.moments()
    finally:
        s.close()
    assert t == 9 and n == 6
    np.testing.assert_array_equal(x_a, x_b)
    np.testing.assert_array_equal(z_a, z_b)
    o = oracle.run(pb, 9, 3, 77)
    assert rel_l2(x_b, o["x"]) <= 1e-5 and rel_l2(mean, o["mean"]) <= 1e-5 and rel_l2(var, o["var"]) <= 1e-5  # R44


def test_long_chain_graph_replay_and_overlap_agree():
    """3,000 iterations (burn-in 500): graph replays (1 x 1 tile) and direct launches with the
    overlapped NCCL exchange (3 x 1 strips through NCCL self send/recv) stay bitwise equal over a
    long run (iteration-state advance, Welford with large n, noise counters), and stay finite."""
    from paper_2511_00870_b200 import FLAG_HALO_VIA_NCCL
    kw, _ = make_problem(120, 96, kernel="gauss9", cnn=(8, 32), z=True)
    a = _chain(kw, 0, plan=((3000, 500, 99),))
    b = _chain(kw, FLAG_HALO_VIA_NCCL, tiles=(3, 1), plan=((3000, 500, 99),))
    _assert_same(a, b)
    assert a[1] == (3000, 2500)
    for k in ("x", "z", "mean", "var"):
        assert np.isfinite(a[0][k]).all(), k
    assert (a[0]["var"] > 0).all()


@pytest.mark.parametrize("tiles", [(2, 1), (3, 1), (2, 2)])
def test_graph_with_captured_nccl_halo_group_bitwise(tiles):
    """The NCCL halo group captured inside the iteration graph (FLAG_HALO_VIA_NCCL: NCCL self
    send/recv on one GPU, the code path of a multi-rank run), with the comm-stream fork/join of the
    overlapped exchange on row strips: bitwise equal to direct launches and to the untiled chain,
    across a reset with a new seed and burn-in."""
    from paper_2511_00870_b200 import FLAG_HALO_VIA_NCCL
    kw, _ = make_problem(96, 70, kernel="gauss9", cnn=(8, 32), z=True)
    plan = ((7, 2, 11), (10, 4, 12))
    g = _chain(kw, FLAG_HALO_VIA_NCCL, tiles=tiles, plan=plan)
    d = _chain(kw, FLAG_HALO_VIA_NCCL | FLAG_NO_GRAPH, tiles=tiles, plan=plan)
    _assert_same(g, d)
    assert g[2] == d[2]
    _assert_same(g, _chain(kw, 0, plan=plan))


@pytest.mark.parametrize("corrupt", ["magic", "truncated", "geometry"])
def test_rejected_checkpoint_leaves_the_chain_untouched(corrupt):
    """A blob that pnpula_load_checkpoint rejects (wrong magic / truncated / another geometry) must
    not switch the live context's buffers: the chain continues bit for bit as if the
    call had not happened, also when the current x^t lives in buffer 1 (odd t) and graphs replay."""
    kw, _ = make_problem(45, 52, kernel="gauss5", cnn=(4, 16), z=True)
    ref = Sampler(**kw)
    ref.run(9, 2, 5)
    want = ref.state()
    ref.close()
    s = Sampler(**kw)
    try:
        s.reset(2, 5)
        s.advance(5)                 # odd t: x^t in buffer 1
        blob = bytearray(s.save_checkpoint())
        if corrupt == "magic":
            blob[0] ^= 0xFF
        elif corrupt == "truncated":
            blob = blob[:-4]
        else:
            kw2, _ = make_problem(45, 60, kernel="gauss5", cnn=(4, 16), z=True)
            other = Sampler(**kw2)
            other.reset(2, 5)
            blob = bytearray(other.save_checkpoint())
            other.close()
        with pytest.raises(Exception):
            s.load_checkpoint(bytes(blob))
        s.advance(4)
        got = s.state()
    finally:
        s.close()
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    assert got[2] == want[2] == 9
