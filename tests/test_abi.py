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


def test_training_and_inverse_plumbing_validation_without_gpu():
    """The step / inverse / deterministic-backward entry points reject bad
    arguments before any CUDA call."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libivrgs.so not built")
    L = _lib.lib()
    E = _lib.IVR_ERR_ARG
    assert L.ivr_stage2_attrs(-1, None, None, None, None, None, None, None, None, None) == E
    assert L.ivr_step_assemble(None, None) == E
    a = _lib.StepGrads_t()
    a.n, a.k = 10, 4
    a.stat = 1  # stat without its inputs
    assert L.ivr_step_assemble(ctypes.byref(a), None) == E
    assert L.ivr_step_partials(1000) >= 1
    assert L.ivr_loss_finalize(None, None, None, None, None) == E
    assert L.ivr_inverse_update(None, None) == E
    st = _lib.InverseStep_t()
    st.n_scenes, st.n_views = 2000, 1  # > 1024 scenes
    assert L.ivr_inverse_update(ctypes.byref(st), None) == E
    groups = (_lib.AdamGroup_t * 1)()
    assert L.ivr_adam_step_sched(groups, 1, 0.9, 0.999, 1e-15, None, None, None) == E
    assert L.ivr_blend_bwd_det_workspace_size(100, 15) == 100 * 8 * 21 * 4
    assert L.ivr_blend_bwd_det_workspace_size(100, 33) == 0
    assert L.ivr_blend_bwd_deterministic(None, None, 1, 1, None, None, None, 4, 16, 16, None, None,
                                         None, 10, None, None, None, 100, None, 0, None, None,
                                         None, None, None, 0, None) == E
