"""CPU-side checks of the C-ABI boundary (no GPU needed)."""

import ctypes
import os

import pytest

from paper_2504_17954_b200 import _lib


def test_library_loads_and_exports_header_symbols():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libivrgs.so not built")
    L = ctypes.CDLL(_lib.LIB_PATH)
    declared = _lib.exported_symbols()
    assert "ivr_blend_fwd" in declared and "ivr_bin_sort" in declared
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/ivrgs.h but not exported"
    assert _lib.lib().ivr_version() == 4


def test_argument_validation_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libivrgs.so not built")
    L = _lib.lib()
    # null / bad arguments are rejected before any CUDA call
    assert L.ivr_preprocess_fwd(None, None, None, None, None, None, 0, None) == _lib.IVR_ERR_ARG
    assert L.ivr_bin_sort(-1, None, None, None, 1, 1, 1, None, 0, None, None, None, None) == \
        _lib.IVR_ERR_ARG
    assert L.ivr_vq_assign(None, 10, None, 0, None, None, 0, None) == _lib.IVR_ERR_ARG
    assert b"ivr_vq_assign" in L.ivr_last_error()
    assert L.ivr_bin_sort_workspace_size(1000, 4000, 64) > 0
    assert L.ivr_vq_assign_workspace_size() > 0
    assert L.ivr_sh_eval(10, 4, None, None, None, None, None) == _lib.IVR_ERR_ARG  # degree 4
    assert L.ivr_crc32(None, 10, None, None) == _lib.IVR_ERR_ARG
    assert L.ivr_unpack(None, 10, 3, None, None) == _lib.IVR_ERR_ARG
    assert L.ivr_photometric_loss(None, None, 8, 8, 4, None, 0.0, 0.0, 1, None, None, None, 0,
                                  None) == _lib.IVR_ERR_ARG
    assert L.ivr_photometric_workspace_size(800, 800, 4) > 3 * 790 * 790 * 4 * 8


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libivrgs.so")
    with pytest.raises(_lib.NativeLibraryMissing):
        _lib.lib()
