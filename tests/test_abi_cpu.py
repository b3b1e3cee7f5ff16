"""C-ABI checks that need no GPU: the library builds/loads, exports every symbol that
include/pnpula.h declares, the host-only planning helpers are right, and creating a
context without a usable sm_100 GPU fails loudly (no CPU fallback)."""
import os
import re

import numpy as np
import pytest
import torch

import paper_2511_00870_b200 as pk
from paper_2511_00870_b200 import _lib, build
from conftest import ROOT, golden

build.build()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pnpula.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pnpula_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = _header_functions()
    assert len(names) >= 20
    lib = _lib.load()
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.EXPORTED) == names


def test_version():
    assert "sm_100a" in pk.pnpula_version()


def test_partition_paper_fig1():
    with open(golden("partition_fig1.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    for row in rows:
        n, parts = int(row[0]), int(row[1])
        want = [tuple(int(v) for v in s.split(":")) for s in row[2:]]
        assert [pk.pnpula_partition(n, parts, p) for p in range(parts)] == want


def test_halo_width():
    assert pk.pnpula_halo_width(pk.OP_CONV, 9, 9, 8) == 8
    assert pk.pnpula_halo_width(pk.OP_CONV, 5, 5, 4) == 4
    assert pk.pnpula_halo_width(pk.OP_CONV, 9, 9, 0) == 8
    assert pk.pnpula_halo_width(pk.OP_CONV, 15, 3, 2) == 14
    assert pk.pnpula_halo_width(pk.OP_MASK, 0, 0, 8) == 8
    assert pk.pnpula_halo_width(pk.OP_MASK, 0, 0, 0) == 0


def _ghost_owner_bruteforce(ny, nx, ty, tx, h):
    """For every tile d and every ghost pixel of d inside the image, the tile that owns it."""
    rects = []
    for t in range(ty * tx):
        a, b = pk.pnpula_partition(ny, ty, t // tx)
        c, d = pk.pnpula_partition(nx, tx, t % tx)
        rects.append((a, b, c, d))
    owner = np.zeros((ny, nx), int)
    for t, (a, b, c, d) in enumerate(rects):
        owner[a:b, c:d] = t
    need = {}
    for t, (a, b, c, d) in enumerate(rects):
        for i in range(max(a - h, 0), min(b + h, ny)):
            for j in range(max(c - h, 0), min(d + h, nx)):
                if a <= i < b and c <= j < d:
                    continue
                need.setdefault((owner[i, j], t), set()).add((i, j))
    return need


@pytest.mark.parametrize("ny,nx,ty,tx,h", [(20, 20, 4, 1, 2), (23, 29, 2, 2, 4), (64, 64, 2, 2, 4),
                                           (40, 33, 3, 4, 5), (17, 50, 1, 5, 8)])
def test_plan_halo_matches_bruteforce(ny, nx, ty, tx, h):
    msgs = pk.pnpula_plan_halo(ny, nx, ty, tx, h)
    got = {}
    order = []
    for s, d, (i0, j0, hh, ww) in msgs:
        order.append((s, d))
        got[(s, d)] = {(i, j) for i in range(i0, i0 + hh) for j in range(j0, j0 + ww)}
    assert order == sorted(order)                    # canonical (src, dst) order
    assert got == _ghost_owner_bruteforce(ny, nx, ty, tx, h)


def test_plan_halo_too_fine():
    with pytest.raises(pk.PnpulaError):
        pk.pnpula_plan_halo(20, 20, 8, 1, 4)         # 2-3 row tiles < halo 4


def test_stepsize_check_spec_examples():
    assert pk.pnpula_check_stepsizes(1, 0, 1, 1, 2, 1 / 8, 0.03) == 0
    assert pk.pnpula_check_stepsizes(1, 0, 1, 1, 2, 1 / 8, 0.04) == 2
    assert pk.pnpula_check_stepsizes(1, 0, 0, 1, 0, 1 / 4, 0.01) == 0
    assert pk.pnpula_check_stepsizes(1, 0, 0, 1, 0, 0.26, 0.01) == 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks behaviour without a GPU")
def test_create_without_gpu_fails_loudly():
    y = np.zeros((16, 16), np.float32)
    with pytest.raises(pk.PnpulaError) as e:
        pk.Sampler(ny=16, nx=16, y=y, sigma2=0.1, gamma=0.01, op="mask", mask=np.ones((16, 16), np.uint8))
    assert e.value.status in (7, 8)      # E_CUDA / E_NCCL, never a silent CPU path


def test_create_validates_before_touching_the_gpu():
    y = np.zeros((16, 16), np.float32)
    with pytest.raises(pk.PnpulaError) as e:
        pk.Sampler(ny=16, nx=16, y=y, sigma2=0.1, gamma=0.01, kernel=np.ones((4, 4), np.float32))
    assert e.value.status == 1           # even kernel
    with pytest.raises(pk.PnpulaError) as e:
        pk.Sampler(ny=16, nx=16, y=y, sigma2=0.1, gamma=0.01, op="mask", mask=np.ones((16, 16), np.uint8),
                   rho=1.0, kappa=2.0)
    assert e.value.status == 1
    with pytest.raises(pk.PnpulaError) as e:
        pk.Sampler(ny=16, nx=16, y=y, sigma2=0.1, gamma=0.01, kernel=np.ones((9, 9), np.float32), tiles=(4, 1))
    assert e.value.status == 3           # 4-row tiles < halo 8
    w = np.zeros(100, np.float32)
    with pytest.raises(pk.PnpulaError) as e:
        pk.Sampler(ny=16, nx=16, y=y, sigma2=0.1, gamma=0.01, op="mask", mask=np.ones((16, 16), np.uint8),
                   weights=w, biases=w, n_layers=3, channels=24, alpha=1.0, eps=0.1)
    assert e.value.status == 10          # unsupported channel count


def test_create_validates_colour_and_prior_combinations():
    y3 = np.zeros((3, 16, 16), np.float32)
    m = np.ones((16, 16), np.uint8)
    w = np.zeros(4 * 16 * 3 * 9, np.float32)
    with pytest.raises(pk.PnpulaError) as e:   # colour DDFB needs P = 32 / 64 (N = 48 folded adjoint)
        pk.Sampler(ny=16, nx=16, y=y3, sigma2=0.1, gamma=0.01, op="mask", mask=m, weights=w, n_layers=4,
                   channels=16, alpha=1.0, eps=0.1, den_kind="ddfb", ddfb_gammas=np.ones(4, np.float32), ht_eps=0.05)
    assert e.value.status == 10
    with pytest.raises(pk.PnpulaError) as e:   # img_channels other than 1 / 3
        pk.Sampler(ny=16, nx=16, y=np.zeros((2, 16, 16), np.float32), sigma2=0.1, gamma=0.01, op="mask", mask=m)
    assert e.value.status == 10
    with pytest.raises(pk.PnpulaError) as e:   # TV needs its z block (rho > 0) and no box term
        pk.Sampler(ny=16, nx=16, y=y3, sigma2=0.1, gamma=0.01, op="mask", mask=m, tv_beta=1.0)
    assert e.value.status == 1
