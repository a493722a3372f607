"""ctypes binding of the C ABI in ``include/ivrgs.h`` (libivrgs.so).

The product path has no CPU fallback: every kernel entry point goes through
``lib()``, which raises ``NativeLibraryMissing`` when the in-tree CUDA library
has not been built (``python -m paper_2504_17954_b200.build``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import CorruptIndex, NonFiniteGradient, ShapeMismatch, VoxSplatError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IVR_LIB_PATH") or os.path.join(PKG, "libivrgs.so")  # override: A/B runs

c_double_p = ctypes.POINTER(ctypes.c_double)
P = ctypes.c_void_p
MAX_ATTRS = 8
BLEND_EXACT = 1
PRE_F64, PRE_EXACT_RGB = 1, 2  # ivr_preprocess_fwd mode bits
BLEND_PRECULLED = 2
BLEND_NO_GEOMETRY = 4
BLEND_DOUT_F64 = 8

IVR_OK, IVR_ERR_ARG, IVR_ERR_SHAPE, IVR_ERR_NONFINITE, IVR_ERR_CORRUPT_INDEX, IVR_ERR_CUDA, \
    IVR_ERR_CAPACITY = 0, -1, -2, -3, -4, -5, -6


class NativeLibraryMissing(VoxSplatError, RuntimeError):
    """The CUDA extension is not built / not loadable: there is no fallback."""


class Camera_t(ctypes.Structure):
    _fields_ = [("position", ctypes.c_double * 3), ("rotation", ctypes.c_double * 9),
                ("focal", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class FrameParams_t(ctypes.Structure):
    _fields_ = [("cam", Camera_t), ("light_dir", ctypes.c_double * 3),
                ("term_scales", ctypes.c_double * 4), ("lam", ctypes.c_double * 4),
                ("b", ctypes.c_double * 4), ("orbital", ctypes.c_int32),
                ("rescale_opacity", ctypes.c_int32), ("dl_dp", ctypes.c_double * 3),
                ("dl_da", ctypes.c_double * 3)]


class Gaussians_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("mu", P), ("q_raw", P), ("log_s", P), ("o_logit", P),
                ("n_raw", P), ("cache", P)]


class Shading_t(ctypes.Structure):
    _fields_ = [("delta_c", P), ("k_a_raw", P), ("k_d_raw", P), ("k_s_raw", P), ("log_beta", P),
                ("palette", P), ("per_splat_palette", ctypes.c_int32), ("orbital", ctypes.c_int32),
                ("light_dir", ctypes.c_double * 3), ("term_scales", ctypes.c_double * 4),
                ("lam", ctypes.c_double * 4), ("b", ctypes.c_double * 4)]


class SeedProblem_t(ctypes.Structure):
    _fields_ = [("values", P), ("order", P), ("n", ctypes.c_int64), ("first", ctypes.c_int64),
                ("u", P), ("centers", P)]


class Edits_t(ctypes.Structure):
    _fields_ = [("scene_id", P), ("opacity_scale", P), ("rescale_opacity", ctypes.c_int32)]


class Layout_t(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("col_color", ctypes.c_int32), ("col_alpha", ctypes.c_int32),
                ("col_depth", ctypes.c_int32), ("col_normal", ctypes.c_int32), ("colors", P),
                ("n_attr", ctypes.c_int32), ("attr", P * MAX_ATTRS),
                ("attr_col", ctypes.c_int32 * MAX_ATTRS), ("attr_width", ctypes.c_int32 * MAX_ATTRS)]


class ProjOut_t(ctypes.Structure):
    _fields_ = [("depth_key", P), ("count", P), ("rect", P), ("rec", P), ("values", P),
                ("rec64", P), ("values64", P), ("mean2d", P), ("conic", P), ("cov2d", P),
                ("depth", P), ("opacity", P), ("rgb", P), ("radius", P), ("valid", P),
                ("depth_minmax", P)]


class AdamGroup_t(ctypes.Structure):
    _fields_ = [("param", P), ("m", P), ("v", P), ("grad", P), ("n", ctypes.c_int64),
                ("lr", ctypes.c_double), ("bc1", ctypes.c_double), ("bc2", ctypes.c_double)]


class Grads_t(ctypes.Structure):
    _fields_ = [("g_values", P), ("g_mean2d", P), ("g_conic", P), ("g_opacity", P),
                ("d_rgb_extra", P), ("d_mu", P), ("d_q_raw", P), ("d_log_s", P), ("d_o_logit", P),
                ("d_n_raw", P), ("d_colors", P), ("d_mean2d", P), ("d_values", P),
                ("d_delta_c", P), ("d_k_a_raw", P), ("d_k_d_raw", P), ("d_k_s_raw", P),
                ("d_log_beta", P), ("d_c_p", P), ("d_scale", P), ("d_globals", P),
                ("per_scene", ctypes.c_int32), ("dl_dp", ctypes.c_double * 3),
                ("dl_da", ctypes.c_double * 3), ("bad", P), ("scratch", P),
                ("scratch_len", ctypes.c_int64)]


class StepGrads_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("k", ctypes.c_int32), ("d_values", P),
                ("col_delta_c", ctypes.c_int32), ("col_k_a", ctypes.c_int32),
                ("col_k_d", ctypes.c_int32), ("col_k_s", ctypes.c_int32),
                ("col_beta", ctypes.c_int32), ("o_logit", P), ("k_a_raw", P), ("k_d_raw", P),
                ("k_s_raw", P), ("log_beta", P), ("d_o_logit", P), ("d_delta_c", P),
                ("d_k_a_raw", P), ("d_k_d_raw", P), ("d_k_s_raw", P), ("d_log_beta", P),
                ("d_mean2d", P), ("d_n_raw", P), ("stat", P), ("w_opacity_l1", ctypes.c_double),
                ("o_partial", P), ("gate", P), ("n_pairs", P), ("pair_capacity", ctypes.c_int64),
                ("stat_sum", P)]


class LossTerms_t(ctypes.Structure):
    _fields_ = [("photo_sums", P), ("l1_weight", ctypes.c_double),
                ("ssim_weight", ctypes.c_double), ("numel", ctypes.c_double),
                ("windows", ctypes.c_double), ("terms", P), ("w_normal", ctypes.c_double),
                ("w_offset", ctypes.c_double), ("w_bil", ctypes.c_double), ("o_partial", P),
                ("n_partial", ctypes.c_int32), ("w_opacity_l1", ctypes.c_double),
                ("n", ctypes.c_double)]


class InverseStep_t(ctypes.Structure):
    _fields_ = [("n_scenes", ctypes.c_int32), ("n_views", ctypes.c_int32),
                ("orbital", ctypes.c_int32), ("learnable", ctypes.c_int32),
                ("iters", ctypes.c_int64), ("view_div", ctypes.c_double), ("x", P), ("m", P),
                ("v", P), ("t", P),
                ("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("grad", P), ("loss_sum", P), ("losses", P),
                ("ctl", P), ("params", P), ("tab", P)]


INV_OVERFLOW, INV_DIVERGED = 1, 2

BAD_IDS = ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors", "d_k_a_raw",
           "d_k_d_raw", "d_k_s_raw", "d_log_beta", "d_delta_c")


_SIGS = {
    "ivr_version": ([], ctypes.c_int),
    "ivr_last_error": ([], ctypes.c_char_p),
    "ivr_preprocess_fwd": ([ctypes.POINTER(Gaussians_t), ctypes.POINTER(Shading_t),
                            ctypes.POINTER(Edits_t), ctypes.POINTER(Camera_t),
                            ctypes.POINTER(Layout_t), ctypes.POINTER(ProjOut_t), ctypes.c_int32, P],
                           ctypes.c_int),
    "ivr_preprocess_fwd_params": ([ctypes.POINTER(Gaussians_t), ctypes.POINTER(Shading_t),
                                   ctypes.POINTER(Edits_t), P, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.POINTER(Layout_t), ctypes.POINTER(ProjOut_t),
                                   ctypes.c_int32, P], ctypes.c_int),
    "ivr_shade_fwd": ([ctypes.POINTER(Gaussians_t), ctypes.POINTER(Shading_t), P,
                       ctypes.POINTER(Camera_t), P, P, P], ctypes.c_int),
    "ivr_bin_sort_workspace_size": ([ctypes.c_int64, ctypes.c_int64, ctypes.c_int32], ctypes.c_size_t),
    "ivr_bin_sort": ([ctypes.c_int64, P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P,
                      ctypes.c_size_t, P, P, P, P], ctypes.c_int),
    "ivr_bin_sort_frame": ([ctypes.c_int64, P, P, P, P, P, ctypes.c_int32, ctypes.c_int32,
                            ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P, ctypes.c_size_t, P,
                            P, P, P, P], ctypes.c_int),
    "ivr_blend_fwd": ([P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, P, ctypes.c_int32,
                       ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, ctypes.c_int32, P],
                      ctypes.c_int),
    "ivr_tile_order": ([P, ctypes.c_int32, P, P], ctypes.c_int),
    "ivr_debug_blend_trace": ([P], None),
    "ivr_debug_mufu_error": ([P, P], ctypes.c_int),
    "ivr_debug_sigma_error": ([ctypes.c_int64, ctypes.c_uint32, P, P], ctypes.c_int),
    "ivr_kmeans_seed_workspace_size": ([ctypes.c_int64], ctypes.c_size_t),
    "ivr_kmeans_seed": ([P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, P, P, P,
                         ctypes.c_size_t, P], ctypes.c_int),
    "ivr_kmeans_lloyd_sorted_workspace_size": ([ctypes.c_int32, ctypes.c_int32], ctypes.c_size_t),
    "ivr_kmeans_lloyd_step_sorted": ([P, ctypes.c_int64, P, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                      ctypes.c_size_t, P], ctypes.c_int),
    "ivr_kmeans_seed_sorted_workspace_size": ([P, ctypes.c_int32], ctypes.c_size_t),
    "ivr_kmeans_seed_sorted": ([P, ctypes.c_int32, ctypes.c_int32, P, ctypes.c_size_t, P],
                               ctypes.c_int),
    "ivr_blend_bwd_det_workspace_size": ([ctypes.c_int64, ctypes.c_int32], ctypes.c_size_t),
    "ivr_blend_bwd_deterministic": ([P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int64, P, P,
                                     P, ctypes.c_int64, P, ctypes.c_size_t, P, P, P, P, P,
                                     ctypes.c_int32, P], ctypes.c_int),
    "ivr_blend_bwd_pairs": ([P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int32,
                             ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int64, P,
                             ctypes.c_size_t, P, P], ctypes.c_int),
    "ivr_blend_bwd": ([P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int32,
                       ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P, P, ctypes.c_int32, P],
                      ctypes.c_int),
    "ivr_preprocess_bwd": ([ctypes.POINTER(Gaussians_t), ctypes.POINTER(Shading_t),
                            ctypes.POINTER(Edits_t), P, ctypes.POINTER(Camera_t),
                            ctypes.POINTER(Layout_t), ctypes.POINTER(Grads_t), ctypes.c_int32, P],
                           ctypes.c_int),
    "ivr_bin_sort_cull": ([ctypes.c_int64, P, P, P, P, ctypes.c_int32, ctypes.c_int32,
                           ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P, ctypes.c_size_t, P,
                           P, P, P], ctypes.c_int),
    "ivr_vq_assign_workspace_size": ([], ctypes.c_size_t),
    "ivr_vq_assign": ([P, ctypes.c_int64, P, ctypes.c_int32, P, P, ctypes.c_size_t, P],
                      ctypes.c_int),
    "ivr_vq_decode": ([P, ctypes.c_int64, P, ctypes.c_int32, P, P, P], ctypes.c_int),
    "ivr_sh_eval": ([ctypes.c_int64, ctypes.c_int32, P, P, ctypes.POINTER(ctypes.c_double), P, P],
                    ctypes.c_int),
    "ivr_sh_bwd": ([ctypes.c_int64, ctypes.c_int32, P, P, ctypes.POINTER(ctypes.c_double), P, P, P,
                    P], ctypes.c_int),
    "ivr_crc32": ([P, ctypes.c_int64, P, P], ctypes.c_int),
    "ivr_unpack": ([P, ctypes.c_int64, ctypes.c_int32, P, P], ctypes.c_int),
    "ivr_pack_f32": ([P, ctypes.c_int64, P, P], ctypes.c_int),
    "ivr_preprocess_static": ([ctypes.POINTER(Gaussians_t), ctypes.POINTER(Shading_t), P, P],
                              ctypes.c_int),
    "ivr_kmeans_lloyd_workspace_size": ([ctypes.c_int32], ctypes.c_size_t),
    "ivr_kmeans_lloyd_step": ([P, ctypes.c_int64, P, ctypes.c_int32, P, P, P, ctypes.c_size_t, P],
                              ctypes.c_int),
    "ivr_concat": ([ctypes.POINTER(P), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                    ctypes.c_int32, P, P, P], ctypes.c_int),
    "ivr_dvr_render": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                        ctypes.POINTER(ctypes.c_double), P, P, P, ctypes.c_int32,
                        ctypes.POINTER(Camera_t), ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                        ctypes.POINTER(ctypes.c_double), ctypes.c_double, P, P], ctypes.c_int),
    "ivr_display_u8": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                        ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, P, P, P], ctypes.c_int),
    "ivr_png_size": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32], ctypes.c_int64),
    "ivr_png_encode": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int64, P, P],
                       ctypes.c_int),
    "ivr_adam_step": ([ctypes.POINTER(AdamGroup_t), ctypes.c_int32, ctypes.c_double,
                       ctypes.c_double, ctypes.c_double, P], ctypes.c_int),
    "ivr_adam_step_sched": ([ctypes.POINTER(AdamGroup_t), ctypes.c_int32, ctypes.c_double,
                             ctypes.c_double, ctypes.c_double, P, P, P], ctypes.c_int),
    "ivr_preprocess_bwd_scratch_len": ([ctypes.c_int64, ctypes.c_int32], ctypes.c_int64),
    "ivr_sh_basis": ([ctypes.c_int64, ctypes.c_int32, P, P, P, P], ctypes.c_int),
    "ivr_stage2_attrs": ([ctypes.c_int64, P, P, P, P, P, P, P, P, P], ctypes.c_int),
    "ivr_step_partials": ([ctypes.c_int64], ctypes.c_int32),
    "ivr_inverse_pack": ([ctypes.POINTER(InverseStep_t), P, ctypes.c_double, ctypes.c_double, P, P,
                          P, P, ctypes.c_int64, P], ctypes.c_int),
    "ivr_inverse_update": ([ctypes.POINTER(InverseStep_t), P], ctypes.c_int),
    "ivr_step_assemble": ([ctypes.POINTER(StepGrads_t), P], ctypes.c_int),
    "ivr_loss_finalize": ([ctypes.POINTER(LossTerms_t), P, P, P, P], ctypes.c_int),
    "ivr_regularize_workspace_size": ([ctypes.c_int32, ctypes.c_int32], ctypes.c_size_t),
    "ivr_regularize": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                        ctypes.c_int32, P, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                        P, P, P, ctypes.c_size_t, P], ctypes.c_int),
    "ivr_photometric_workspace_size": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32],
                                       ctypes.c_size_t),
    "ivr_photometric_loss": ([P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              ctypes.POINTER(ctypes.c_double), ctypes.c_double, ctypes.c_double,
                              ctypes.c_int32, P, P, P, ctypes.c_size_t, P], ctypes.c_int),
    "ivr_photometric_loss_frame": ([P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), P,
                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_double), ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int32, P, P, P, ctypes.c_size_t,
                                    P], ctypes.c_int),
}

_lib = None


def lib():
    """Load libivrgs.so (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is missing: build it with `python -m paper_2504_17954_b200.build` "
            "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {e}") from e
    for name, (argt, rest) in _SIGS.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.argtypes = argt
        fn.restype = rest
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/ivrgs.h (checked by tests)."""
    import re
    hdr = os.path.join(os.path.dirname(PKG), "include", "ivrgs.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(ivr_[a-z0-9_]+)\s*\(", text)))


def check(status, what=""):
    """Map a C-ABI status to the reference's typed exceptions."""
    if status == IVR_OK:
        return
    msg = lib().ivr_last_error().decode(errors="replace")
    if status == IVR_ERR_SHAPE:
        raise ShapeMismatch(msg or what)
    if status == IVR_ERR_NONFINITE:
        raise NonFiniteGradient(what)
    if status == IVR_ERR_CORRUPT_INDEX:
        raise CorruptIndex(msg or what)
    raise VoxSplatError(f"{what}: ivrgs status {status}: {msg}")
