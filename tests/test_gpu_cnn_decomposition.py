"""The CNN chain's work decomposition (cnn_kernels.cu launch_pn): row-block units
taken round-robin, or one contiguous strip-major range of output rows per CTA (a unit per strip
the range touches) when the launcher's cost model prefers it.  Every output pixel's arithmetic is
independent of the unit it falls in (north_star: bitwise tile invariance), so the two
decompositions -- and different CTA counts, which move the range boundaries across strips and
rows -- must give identical chains, bit for bit."""
import numpy as np
import pytest

from gpu_common import gpu_run, make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    # 3 column strips of the fused 4-layer chunks (ragged last), 230 rows
    kw, _ = make_problem(230, 300, kernel="gauss9", cnn=(8, 32), z=True)
    return kw


@pytest.mark.parametrize("max_ctas", [2, 3, 7, 64])
def test_contiguous_ranges_equal_row_blocks(case, max_ctas, monkeypatch):
    monkeypatch.setenv("PNPULA_MAX_CTAS", str(max_ctas))
    monkeypatch.setenv("PNPULA_CNN_CONTIG", "0")
    a = gpu_run(case, 8, 2, 17)
    monkeypatch.setenv("PNPULA_CNN_CONTIG", "2")   # contiguous ranges forced (the cost model may prefer blocks)
    b = gpu_run(case, 8, 2, 17)
    monkeypatch.delenv("PNPULA_CNN_CONTIG")
    monkeypatch.delenv("PNPULA_MAX_CTAS")
    ref = gpu_run(case, 8, 2, 17)   # default grid
    for k in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
        np.testing.assert_array_equal(a[k], ref[k], err_msg=k)
