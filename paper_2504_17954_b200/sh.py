"""Stage-1 spherical-harmonics colour on the GPU.

``view_dirs`` + ``eval_sh`` and their backward (gaussians.py:497-529), fused
per Gaussian in csrc/sh.cu (float64): the reference materialises the (N, B)
basis and (N, B, 3) basis-derivative arrays; the kernel rebuilds both in
registers.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .gaussians import ShColor


def _pos(cam_position):
    p = np.ascontiguousarray(np.asarray(cam_position, dtype=np.float64).reshape(3))
    return p, p.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def sh_eval_device(mu, coeffs, degree, cam_position, stream=None):
    """rgb (N,3) float64 device tensor = eval_sh(sh, view_dirs(mu, pos))."""
    n = int(mu.shape[0])
    rgb = torch.empty((n, 3), dtype=torch.float64, device=mu.device)
    keep, pp = _pos(cam_position)
    L.check(L.lib().ivr_sh_eval(n, int(degree), D.ptr(mu), D.ptr(coeffs), pp, D.ptr(rgb),
                                D.stream_handle(stream)), "ivr_sh_eval")
    del keep
    return rgb


def sh_backward_device(mu, coeffs, degree, cam_position, d_rgb, d_mu=None, stream=None):
    """d_coeffs (N, B, 3); adds the view-direction gradient into ``d_mu``
    (N,3 device float64, in place) when given."""
    n = int(mu.shape[0])
    d_coeffs = torch.empty_like(coeffs)
    keep, pp = _pos(cam_position)
    L.check(L.lib().ivr_sh_bwd(n, int(degree), D.ptr(mu), D.ptr(coeffs), pp,
                               D.ptr(d_rgb.contiguous()), D.ptr(d_coeffs),
                               D.ptr(d_mu) if d_mu is not None else None,
                               D.stream_handle(stream)), "ivr_sh_bwd")
    del keep
    return d_coeffs


def sh_colors(geom, sh: ShColor, cam):
    """Host rgb of ``view_dirs`` + ``eval_sh`` for one camera
    (render_model's base-stage branch, trainer.py:639-641)."""
    mu = D.to_dev(np.asarray(geom.mu, np.float64))
    c = D.to_dev(np.asarray(sh.coefficients, np.float64))
    return sh_eval_device(mu, c, sh.degree, cam.position).cpu().numpy()


def sh_colors_backward(geom, sh: ShColor, cam, d_rgb):
    """(d_coeffs, d_mu) of ``sh_colors`` for an upstream d_rgb (N,3)."""
    mu = D.to_dev(np.asarray(geom.mu, np.float64))
    c = D.to_dev(np.asarray(sh.coefficients, np.float64))
    d_mu = torch.zeros_like(mu)
    d_c = sh_backward_device(mu, c, sh.degree, cam.position, D.to_dev(np.asarray(d_rgb)), d_mu)
    return d_c.cpu().numpy(), d_mu.cpu().numpy()
