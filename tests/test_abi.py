"""C-ABI library on the CPU box: it loads, exports every symbol include/cheb_logdet.h
declares, its host-only coefficient routine matches the oracle, and argument
validation fails before any device work."""
import ctypes

import numpy as np
import pytest

from paper_1503_06394_b200 import _lib
from paper_1503_06394_b200._lib import CLOperator, CLCsr


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build_library()
    return _lib.load()


def test_exports_every_header_symbol(L):
    names = _lib.header_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert L.cheb_version() >= 100


def test_no_python_compute_fallback():
    """The binding holds no arithmetic path of its own: it never imports the oracle."""
    import inspect
    import paper_1503_06394_b200.api as api
    import paper_1503_06394_b200.dist as dd
    for mod in (api, dd, _lib):
        src = inspect.getsource(mod)
        assert "oracle" not in src.replace("oracle/", "")


@pytest.mark.parametrize("a,b,n", [(0.2, 1.8, 30), (6.023626e-4, 8.0, 1000), (0.04, 1.96, 100),
                                   (4.05, 17.0, 50), (0.5, 2.0, 0), (0.5, 2.0, 1)])
def test_host_coefficients_match_oracle(L, orc, a, b, n):
    """The library's fp64 coefficient routine (independent code) agrees with the
    pinned oracle to <= 1e-14 max|c|."""
    c = np.empty(n + 1)
    assert L.cheb_coeffs_log(a, b, n, c.ctypes.data) == 0
    want = orc.coeffs_log(a, b, n)
    assert np.abs(c - want).max() <= 1e-14 * max(1.0, np.abs(want).max()) * max(1, n / 30)


@pytest.mark.parametrize("a,b,n", [(0.0, 1.0, 5), (-1.0, 1.0, 5), (2.0, 1.0, 5), (1.0, 1.0, 5),
                                   (float("nan"), 1.0, 5), (0.1, float("inf"), 5), (0.1, 1.0, -1)])
def test_coefficients_reject_bad_interval(L, a, b, n):
    c = np.empty(8)
    assert L.cheb_coeffs_log(a, b, n, c.ctypes.data) == _lib.CL_EINVAL
    assert L.cheb_last_error()


def _op(kind=0, n=4, m=4, At=None):
    s = CLOperator()
    s.kind = kind
    s.A = CLCsr(n, m, 0, 1, 1, 1)  # dummy non-NULL pointers: validation never dereferences them
    if At:
        s.At = CLCsr(*At, 1, 1, 1)
    return s


def test_validation_before_device_work(L):
    ws = ctypes.c_void_p(256)
    mu = ctypes.c_void_p(512)
    op = _op()
    # bad interval / degree / probe range / k -> CL_EINVAL, no CUDA call made
    assert L.cheb_moments(ctypes.byref(op), 1.0, 0.5, 3, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -1
    assert L.cheb_moments(ctypes.byref(op), 0.5, 1.5, -1, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -1
    assert L.cheb_moments(ctypes.byref(op), 0.5, 1.5, 3, 4, 4, 1, 8, ws, 1 << 20, mu, None) == -1
    assert L.cheb_moments(ctypes.byref(op), 0.5, 1.5, 3, 0, 4, 1, 12, ws, 1 << 20, mu, None) == -1
    # non-square A -> CL_EDIM
    bad = _op(n=4, m=5)
    assert L.cheb_moments(ctypes.byref(bad), 0.5, 1.5, 3, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -2
    # B^T with the wrong shape -> CL_EDIM
    btb = _op(kind=2, n=4, m=4, At=(4, 5, 0))
    assert L.cheb_moments(ctypes.byref(btb), 0.5, 1.5, 3, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -2
    # d >= 2^31 -> CL_EDIM
    huge = _op(n=1 << 31, m=1 << 31)
    assert L.cheb_moments(ctypes.byref(huge), 0.5, 1.5, 3, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -2
    # unknown kind
    assert L.cheb_moments(ctypes.byref(_op(kind=7)), 0.5, 1.5, 3, 0, 4, 1, 8, ws, 1 << 20, mu, None) == -1
    assert L.cheb_workspace_bytes(ctypes.byref(op), 12) == 0
    r = _lib.CLResult()
    assert L.cheb_logdet(ctypes.byref(op), 0.5, 1.5, 3, 0, 1, 0, ctypes.byref(r)) == -1
    assert L.cheb_finalize(None, None, 1, 1, None, None, None) == -1
    assert L.cheb_workspace_status(None, None, None) == -1


def test_schedule_controls_validate(L):
    """Process-wide schedule switches reject out-of-range values and round-trip (no device work)."""
    assert L.cheb_set_doubling(2) == _lib.CL_EINVAL
    assert L.cheb_set_doubling(-1) == _lib.CL_EINVAL
    assert L.cheb_set_doubling(1) == 0 and L.cheb_get_doubling() == 1
    assert L.cheb_set_doubling(0) == 0 and L.cheb_get_doubling() == 0
    assert L.cheb_set_resident(2) == _lib.CL_EINVAL
    assert L.cheb_set_resident(0) == 0 and L.cheb_get_resident() == 0
    assert L.cheb_set_resident(1) == 0 and L.cheb_get_resident() == 1
    assert L.cheb_set_persistent(3) == _lib.CL_EINVAL
    assert L.cheb_set_persistent(1) == 0
    assert L.cheb_set_small_tiles(2) == _lib.CL_EINVAL
    assert L.cheb_set_small_tiles(0) == 0 and L.cheb_get_small_tiles() == 0
    assert L.cheb_set_small_tiles(1) == 0 and L.cheb_get_small_tiles() == 1
    assert L.cheb_release_cache() == 0  # nothing allocated on this thread: a no-op
