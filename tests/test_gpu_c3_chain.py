"""A BASELINE configs[2]-shaped chain (C3: random-mask inpainting with the box-constraint prox)
against the oracle over 50 iterations, at a size whose CNN pass spans several column strips
and row units: 30 % Bernoulli mask (R24), DnCNN-lite 8 x 32, AXDA z-block on [0, 1] (R21) and the
Moreau box [0, 1], 304 x 400 px (4 column strips of the fused 4-layer chunks, a
ragged last strip).  The CNN grid is run twice: the default (one work unit per CTA) and capped at
3 persistent CTAs (PNPULA_MAX_CTAS, 4 units per CTA), which exercises the tcgen05 pipeline's
cross-unit mbarrier phase bookkeeping; both must agree bitwise, and with the fp64 oracle at
north_star's bf16-denoiser tolerance (2e-2) and with the bf16-emulating oracle at 2e-3."""
import numpy as np
import pytest

import oracle
from gpu_common import gpu_run, make_problem, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3_case():
    kw, pb = make_problem(304, 400, op="mask", cnn=(8, 32), z=True)
    o = oracle.run(pb, 50, 10, 903)
    o16 = oracle.run(pb, 50, 10, 903, bf16_emulate=True)
    return kw, o, o16


def test_c3_chain_50_vs_oracle_and_unit_invariance(c3_case, monkeypatch):
    kw, o, o16 = c3_case
    g = gpu_run(kw, 50, 10, 903)
    monkeypatch.setenv("PNPULA_MAX_CTAS", "3")
    g3 = gpu_run(kw, 50, 10, 903)
    for k in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(g[k], g3[k], err_msg=k)
    for k in ("x", "z", "mean"):
        assert rel_l2(g[k], o[k]) <= 2e-2, k
        assert rel_l2(g[k], o16[k]) <= 2e-3, k
    assert np.all(g["z"] >= 0) and np.all(g["z"] <= 1)
