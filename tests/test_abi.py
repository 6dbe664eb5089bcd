"""C-ABI library checks that need no GPU: the library loads, exports every symbol declared in
include/sig.h, and its host-side queries and argument validation behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sig.h")


@pytest.fixture(scope="module")
def L():
    import paper_2001_00706_b200 as sb
    if not os.path.exists(sb.LIB_PATH):
        from paper_2001_00706_b200 import build
        build.build()
    return sb.lib()


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sig_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 17, names
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/sig.h but not exported"


def test_sizes(L):
    import paper_2001_00706_b200 as sb
    assert sb.sig_signature_channels(8, 5) == 37448
    assert sb.sig_signature_channels(4, 7) == 21844
    assert sb.sig_signature_channels(0, 3) == -1
    assert sb.sig_signature_channels(2, 70) == -1  # overflow
    assert sb.sig_logsignature_channels(4, 7, "words") == 3304
    assert sb.sig_logsignature_channels(8, 5, "brackets") == 7764
    assert sb.sig_logsignature_channels(3, 6, "expand") == 1092
    assert sb.sig_is_supported(8, 5, True) and sb.sig_is_supported(4, 7, True)
    assert sb.sig_is_supported(3, 6) and sb.sig_is_supported(6, 4) and sb.sig_is_supported(4, 4)
    assert not sb.sig_is_supported(9, 3)


def test_validation_before_launch(L):
    """Invalid arguments return an error code before anything touches the device."""
    s = L.sig_signature(None, 2, 5, 3, 4, 0, 0, None, None, None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_INVALID_ARG"
    s = L.sig_signature(ctypes.c_void_p(16), 2, 1, 3, 4, 0, 0, None, ctypes.c_void_p(16), None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_SHAPE"      # one point, no basepoint
    assert b"2 points" in L.sig_last_error()
    s = L.sig_signature(ctypes.c_void_p(16), 2, 5, 3, 0, 0, 0, None, ctypes.c_void_p(16), None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_INVALID_ARG"  # depth 0
    s = L.sig_signature(ctypes.c_void_p(16), 2, 5, 9, 3, 0, 0, None, ctypes.c_void_p(16), None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_UNSUPPORTED"  # C = 9 not instantiated
    s = L.sig_signature(ctypes.c_void_p(16), 2, 5, 3, 4, 0, 2, None, ctypes.c_void_p(16), None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_INVALID_ARG"  # GIVEN basepoint but NULL


def test_path_query_validation_before_launch(L):
    """Queries outside the stream are rejected on the host (SHAPE), before any device access."""
    import numpy as np
    qs = np.array([0, 4], dtype=np.int64)
    qe = np.array([5, 5], dtype=np.int64)  # [4, 5) is a single point
    vp = ctypes.c_void_p
    s = L.sig_path_query(vp(16), vp(16), 2, 9, 3, 4, qs.ctypes.data_as(vp), qe.ctypes.data_as(vp), 2, vp(16),
                         vp(16), 1 << 20, None)
    assert L.sig_status_string(s) == b"SIG_ERR_SHAPE"
    assert b"query 1" in L.sig_last_error()
    qe = np.array([11, 6], dtype=np.int64)  # 11 > M + 1 = 10 points
    s = L.sig_path_query(vp(16), vp(16), 2, 9, 3, 4, qs.ctypes.data_as(vp), qe.ctypes.data_as(vp), 2, vp(16),
                         vp(16), 1 << 20, None)
    assert L.sig_status_string(s) == b"SIG_ERR_SHAPE"
    s = L.sig_signature_ex(vp(16), 2, 1, 3, 4, 0, 0, None, 1, None, vp(16), None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_SHAPE"  # inverse: same validation as sig_signature


def test_workspace_query(L):
    # a single long path is split into time chunks -> needs workspace; a big batch does not
    assert L.sig_signature_workspace_size(1, 2 ** 22, 3, 6, 0, 0) > 0
    assert L.sig_signature_workspace_size(1024, 128, 8, 5, 0, 0) == 0
    assert L.sig_signature_workspace_size(256, 1024, 6, 4, 1, 0) == 0  # stream mode is never chunked


def test_saved_chunk_pair_host_side(L):
    """sig_signature_save / sig_signature_backward_saved (include/sig.h): sizes are host queries,
    and missing buffers are rejected before any launch."""
    # one long path: the backward is time-chunked, so there is state to save ([2][B, m, S] floats)
    nb = L.sig_signature_saved_bytes(1, 40000, 3, 4, 0)
    S = 120
    assert nb >= 2 * 2 * S * 4 and nb % 256 == 0  # at least two chunks, 256-byte rounded
    assert L.sig_signature_backward_saved_workspace_size(1, 40000, 3, 4, 0) > 0
    # a batch that fills the GPU is never chunked: nothing to save
    assert L.sig_signature_saved_bytes(4096, 64, 3, 4, 0) == 0
    assert L.sig_signature_backward_saved_workspace_size(4096, 64, 3, 4, 0) == 0
    # stream mode / bad shapes have no saved form
    assert L.sig_signature_saved_bytes(1, 40000, 9, 3, 0) == 0
    s = L.sig_signature_save(None, 1, 40000, 3, 4, 0, None, None, None, 0, None, 0, None)
    assert L.sig_status_string(s) == b"SIG_ERR_INVALID_ARG"
    p = ctypes.c_void_p(16)
    s = L.sig_signature_save(p, 1, 40000, 3, 4, 0, None, p, p, 0, p, 1 << 30, None)
    assert L.sig_status_string(s) == b"SIG_ERR_WORKSPACE"  # saved buffer too small
    s = L.sig_signature_backward_saved(p, p, p, None, nb, 1, 40000, 3, 4, 0, None, p, None, p, 1 << 30, None)
    assert L.sig_status_string(s) == b"SIG_ERR_INVALID_ARG"  # saved missing
    s = L.sig_signature_backward_saved(p, p, p, p, nb - 1, 1, 40000, 3, 4, 0, None, p, None, p, 1 << 30, None)
    assert L.sig_status_string(s) == b"SIG_ERR_WORKSPACE"
