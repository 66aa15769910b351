"""Host-side CSR builders of the product (bppsa_csr_*_pattern) against the
oracle's independent builders — bit-exact index work, no GPU needed."""
import numpy as np
import pytest

from oracle import csr as C


@pytest.fixture(scope="module")
def api():
    from paper_1907_10134_b200 import build
    build.build()
    from paper_1907_10134_b200 import api as a
    return a


@pytest.mark.parametrize("ci,co,h,w", [(1, 1, 3, 3), (2, 3, 4, 5), (3, 2, 2, 2), (3, 64, 32, 32), (4, 3, 1, 3)])
def test_conv_pattern_matches_oracle(api, ci, co, h, w):
    rng = np.random.default_rng(ci * 100 + co)
    Wt = rng.standard_normal((co, ci, 3, 3)).astype(np.float32)
    ip, ix, tap = api.csr_conv3x3_pattern(ci, co, h, w)
    ref = C.conv_tjac_exact(ci, co, h, w, Wt)
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    assert np.array_equal(Wt.reshape(-1)[tap].astype(np.float64), ref.data)     # Alg. 4 data via taps
    if ci == 3 and co == 64:
        assert len(ix) == 1696512                                               # Table 1 / P:182


def test_pruned_conv_pattern_matches_oracle(api):
    rng = np.random.default_rng(5)
    Wt = rng.standard_normal((8, 5, 3, 3)).astype(np.float32)
    Wt[rng.random(Wt.shape) < 0.9] = 0.0
    ip, ix, tap = api.csr_conv3x3_pattern(5, 8, 6, 7, Wt, drop_zero=True)
    ref = C.conv_tjac_exact(5, 8, 6, 7, Wt, drop_zero_weights=True)
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    assert np.array_equal(Wt.reshape(-1)[tap].astype(np.float64), ref.data)


def test_maxpool_pattern_matches_oracle(api):
    c, h, w = 3, 6, 4
    pidx = np.zeros((c, h // 2, w // 2), np.int64)
    ip, ix = api.csr_maxpool_pattern(c, h, w)
    ref = C.maxpool_window_tjac(pidx, c, h, w)
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
