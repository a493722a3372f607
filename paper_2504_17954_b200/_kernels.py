"""Drop-in for ``voxsplat._kernels`` -- the reference's plugin point
(selected by ``voxsplat/_accel.py:12-26``; called only by rasterize_forward /
rasterize_backward, rasterizer.py:127, 154-157, 229-234).

Same positional numpy signatures and in-place output semantics as
_kernels.py:19-135, executed on the GPU through the C ABI:

* ``fill_pairs``: the splat-major pair emission, on the device;
* ``composite_forward``: K3 in EXACT mode (the reference's float64 per-pair
  arithmetic, float32 accumulation rounding when ``values`` are float32);
* ``composite_backward``: K4a writing per-list-entry gradients
  (``ivr_blend_bwd_pairs``), same decisions as the forward.

A voxsplat maintainer swaps the backend with
``from paper_2504_17954_b200 import _kernels as K`` in ``_accel.py``.  The
tile size must be 16 (rasterizer.py:24), as in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import ShapeMismatch

TILE = 16


def _t(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(D.cuda_device(), dtype)


def fill_pairs(offsets, tx0, tx1, ty0, ty1, ntx, pair_tile, pair_splat):
    """Emit every (tile, splat) pair splat-major, then ty, then tx
    (_kernels.py:19-28) into the caller's int64 arrays."""
    counts = (np.asarray(tx1) - tx0 + 1) * (np.asarray(ty1) - ty0 + 1)
    n = counts.shape[0]
    P = pair_tile.shape[0]
    if P == 0 or n == 0:
        return
    dev = D.cuda_device()
    c = _t(np.maximum(counts, 0), torch.int64)
    splat = torch.repeat_interleave(torch.arange(n, device=dev), c, output_size=P)
    q = torch.arange(P, device=dev) - _t(offsets, torch.int64)[splat]
    w = (_t(tx1, torch.int64) - _t(tx0, torch.int64) + 1)[splat]
    ty = _t(ty0, torch.int64)[splat] + q // w
    tx = _t(tx0, torch.int64)[splat] + q % w
    pair_tile[:] = D.to_host(ty * int(ntx) + tx)
    pair_splat[:] = D.to_host(splat)


def _records(mean2d, conic, opacity, values):
    """Blend records without K1's float32 skip bounds (hi = +inf, thr = -inf):
    every pair is decided by the reference's float64 arithmetic."""
    f64 = np.asarray(values).dtype == np.float64
    n = mean2d.shape[0]
    rec = np.zeros((n, 8), dtype=np.float32)
    rec[:, 0:2] = np.asarray(mean2d, np.float32)
    rec[:, 2] = np.asarray(opacity, np.float32)
    rec[:, 3] = np.inf
    c32 = np.asarray(conic, np.float32)
    rec[:, 4], rec[:, 5], rec[:, 6] = 0.5 * c32[:, 0], c32[:, 1], 0.5 * c32[:, 2]
    rec[:, 7] = -np.inf
    dev = {"rec": _t(rec, torch.float32),
           "values": _t(np.asarray(values, np.float32), torch.float32)}
    if f64:
        r64 = np.zeros((n, 8), dtype=np.float64)
        r64[:, 0:2], r64[:, 2:5], r64[:, 5] = mean2d, conic, opacity
        dev["rec64"] = _t(r64, torch.float64)
        dev["values64"] = _t(np.asarray(values, np.float64), torch.float64)
    return f64, dev


def _check_tile(tile_size):
    if int(tile_size) != TILE:
        raise ShapeMismatch(f"tile size {tile_size}: the GPU kernels use {TILE}x{TILE} tiles")


def _forward(tile_ranges, pair_splat, mean2d, conic, opacity, values, width, height, ntx):
    W, H = int(width), int(height)
    nty = (H + TILE - 1) // TILE
    K = int(np.asarray(values).shape[1])
    f64, R = _records(mean2d, conic, opacity, values)
    dev = D.cuda_device()
    tr, ps = _t(tile_ranges, torch.int32), _t(pair_splat, torch.int32)
    out = torch.empty((H, W, K), dtype=torch.float32, device=dev)
    out64 = torch.empty((H, W, K), dtype=torch.float64, device=dev) if f64 else None
    cnt = torch.empty((H, W), dtype=torch.int32, device=dev)
    last = torch.empty((H, W), dtype=torch.int32, device=dev)
    tf = torch.empty((H, W), dtype=torch.float64, device=dev)
    L.check(L.lib().ivr_blend_fwd(D.ptr(tr), D.ptr(ps), int(ntx), nty, D.ptr(R["rec"]),
                                  D.ptr(R["values"]), D.ptr(R.get("rec64")),
                                  D.ptr(R.get("values64")), K, W, H,
                                  None if f64 else D.ptr(out), D.ptr(out64), D.ptr(cnt),
                                  D.ptr(last), D.ptr(tf), None, L.BLEND_EXACT,
                                  D.stream_handle()), "ivr_blend_fwd")
    if f64:
        out = out64.float()
    return tr, ps, R, out, out64, cnt, last, tf, K, nty


def composite_forward(tile_ranges, pair_splat, mean2d, conic, opacity, values, width, height,
                      tile_size, ntx, out, contrib, last_pos, t_final):
    """Front-to-back compositing per tile (_kernels.py:31-72); fills ``out``
    (H,W,K), ``contrib``, ``last_pos`` and ``t_final`` in place."""
    _check_tile(tile_size)
    tr, ps, R, o32, o64, cnt, last, tf, K, nty = _forward(
        tile_ranges, pair_splat, mean2d, conic, opacity, values, width, height, ntx)
    out[...] = D.to_host(o64 if o64 is not None else o32).astype(out.dtype, copy=False)
    contrib[...] = D.to_host(cnt)
    last_pos[...] = D.to_host(last)
    t_final[...] = D.to_host(tf)


def composite_backward(tile_ranges, pair_splat, mean2d, conic, opacity, values, width, height,
                       tile_size, ntx, d_out, last_pos, t_final,
                       pair_dv, pair_dmean, pair_dconic, pair_dopac):
    """Per-pair gradients of composite_forward (_kernels.py:75-135) into the
    caller's (zeroed) pair_dv (P,K), pair_dmean (P,2), pair_dconic (P,3),
    pair_dopac (P,).  The forward is re-run on the device (EXACT, identical
    decisions) for the blend records; the walk starts from the caller's
    t_final, back to front like the reference."""
    _check_tile(tile_size)
    tr, ps, R, o32, o64, cnt, last, tf, K, nty = _forward(
        tile_ranges, pair_splat, mean2d, conic, opacity, values, width, height, ntx)
    if not np.array_equal(last.cpu().numpy(), np.asarray(last_pos)):
        raise ShapeMismatch("last_pos does not come from composite_forward on these inputs")
    P = int(np.asarray(pair_splat).shape[0])
    if P == 0:
        return
    d = _t(np.asarray(d_out, np.float64).reshape(int(height), int(width), K), torch.float32)
    nb = int(L.lib().ivr_blend_bwd_det_workspace_size(P, K))
    ws = torch.empty(max(nb, 8), dtype=torch.uint8, device=d.device)
    g = torch.empty((P, K + 6), dtype=torch.float32, device=d.device)
    tfd = _t(np.asarray(t_final, np.float64).reshape(int(height), int(width)), torch.float64)
    L.check(L.lib().ivr_blend_bwd_pairs(D.ptr(tr), D.ptr(ps), int(ntx), nty, D.ptr(R["rec"]),
                                        D.ptr(R["values"]), D.ptr(R.get("rec64")), K,
                                        int(width), int(height), D.ptr(tfd), D.ptr(last), D.ptr(d),
                                        P, D.ptr(ws), nb, D.ptr(g),
                                        D.stream_handle()), "ivr_blend_bwd_pairs")
    h = D.to_host(g.double())
    pair_dv += h[:, :K]
    pair_dmean += h[:, K:K + 2]
    pair_dconic += h[:, K + 2:K + 5]
    pair_dopac += h[:, K + 5]
