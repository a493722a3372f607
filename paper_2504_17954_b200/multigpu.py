"""Multi-GPU units of the hot path that need no data-path collective
(SURVEY.md 8(e)): one process per GPU, ``torch.distributed`` only to hand
results to rank 0.

* ``render_views`` -- batched render (BASELINE configs[1] with many views):
  camera views round-robin over the ranks, a full scene replica per GPU, each
  rank's views replayed through one captured ``FrameGraph``; with
  ``gather`` rank 0 receives every view's RGBA in the callers' order.
* ``train_per_rank`` -- basic-model training (BASELINE configs[2]): rank r
  trains ``datasets[r]`` (``train_base`` then ``train_editable``) with no
  communication; with ``gather`` rank 0 receives every rank's model.

The inverse exploration, whose views are sharded with one all-reduce per
iteration, lives in ``inverse.InverseGraph`` (``dist=``).  ``render_fn`` /
``train_fn`` replace the per-rank work (used by the CPU tests of the sharding
and gathering logic).
"""

from __future__ import annotations

import numpy as np


def dist_info(dist=None, group=None):
    """(rank, world) of ``dist`` (a ``torch.distributed`` module with an
    initialised process group), or (0, 1)."""
    if dist is None:
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard(n, rank, world):
    """Indices of the items of rank ``rank`` among ``n``: round-robin
    (i % world == rank), so neighbouring views land on different GPUs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"shard: bad rank {rank} of {world}")
    return list(range(rank, int(n), world))


def _default_render(scene, cams):
    import torch
    from .scene import DeviceScene, FrameGraph
    ds = DeviceScene(scene)
    out, fg, host = [], None, None
    for cam in cams:
        if fg is None or (cam.width, cam.height) != (fg.W, fg.H):
            fg = FrameGraph(ds, cam.width, cam.height, warm_cam=cam)
            host = torch.empty((cam.height, cam.width, 4), dtype=torch.float32, pin_memory=True)
        fg.render_host(cam, host)  # replay, D2H, re-capture if the pair capacity overflowed
        out.append(host.numpy().copy())
    return out


def render_views(scene, cams, dist=None, group=None, gather=True, render_fn=None):
    """Render ``cams`` (RGBA float32, the FAST FrameGraph path) split over the
    ranks (see module docstring).  Returns this rank's [(view index, RGBA)]
    list, or on rank 0 with ``gather`` the list of every view's RGBA in the
    order of ``cams`` (other ranks: None)."""
    rank, world = dist_info(dist, group)
    mine = shard(len(cams), rank, world)
    fn = render_fn or (lambda cs: _default_render(scene, cs))
    imgs = fn([cams[i] for i in mine]) if mine else []
    local = list(zip(mine, imgs))
    if not gather:
        return local
    if world == 1:
        return [img for _, img in sorted(local, key=lambda t: t[0])]
    parts = [None] * world if rank == 0 else None
    dist.gather_object(local, parts, dst=0, group=group)
    if rank != 0:
        return None
    allv = [None] * len(cams)
    for part in parts:
        for i, img in part:
            allv[i] = np.asarray(img)
    return allv


def _default_train(dataset, cfg):
    from .trainer import train_base, train_editable
    base, log1 = train_base(dataset, cfg)
    editable, log2 = train_editable(base, dataset, cfg)
    return {"base": base, "editable": editable, "log": (log1, log2)}


def train_per_rank(datasets, cfg=None, dist=None, group=None, gather=True, train_fn=None):
    """One basic transfer function per GPU (see module docstring): rank r
    trains ``datasets[r]``; ``len(datasets)`` must equal the world size.
    Returns this rank's result, or on rank 0 with ``gather`` the list of
    every rank's result in rank order (other ranks: None)."""
    rank, world = dist_info(dist, group)
    if len(datasets) != world:
        raise ValueError(f"train_per_rank: {len(datasets)} datasets for {world} ranks")
    fn = train_fn or _default_train
    res = fn(datasets[rank], cfg)
    if not gather:
        return res
    if world == 1:
        return [res]
    parts = [None] * world if rank == 0 else None
    dist.gather_object(res, parts, dst=0, group=group)
    return parts if rank == 0 else None
