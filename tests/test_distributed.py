"""World-size-2 gloo tests (CPU) of the multi-GPU paths' host logic.

* inverse exploration with views sharded over ranks: one all-reduce of the
  packed (4S+10)+1 vector per iteration gives every rank the mean over ALL
  views and therefore identical Adam updates (inverse.reduce_views /
  transform_step);
* bench/render and training shard independent units: no collective.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

S = 3
NP = 4 * S + 10


def _fake_view_grads(view):
    rng = np.random.default_rng(100 + view)
    return rng.normal(size=NP), float(rng.uniform(0.1, 1.0))


def _run_fit(views, iters, dist_mod=None, n_views=None):
    from paper_2504_17954_b200.inverse import Adam, TransformParams, reduce_views, transform_step
    p = TransformParams(np.full((S, 3), 0.5), np.zeros(S), np.ones(4), np.zeros(4), 0.1, 0.2,
                        "orbital")
    adam = Adam(eps=1e-15)
    angles = np.array([p.polar, p.azimuth])
    losses = []
    for it in range(iters):
        total = torch.zeros(NP, dtype=torch.float64)
        lsum = torch.zeros(1, dtype=torch.float64)
        for v in views:
            g, l = _fake_view_grads(v * 10 + it)
            total += torch.from_numpy(g)
            lsum += l
        mean, loss = reduce_views(total, lsum, n_views or len(views), dist_mod)
        losses.append(loss)
        unpack = {"c_p": mean[:3 * S].reshape(S, 3), "opacity_raw": mean[3 * S:4 * S],
                  "lam": mean[4 * S:4 * S + 4], "b": mean[4 * S + 4:4 * S + 8],
                  "angles": mean[4 * S + 8:]}
        transform_step(p, unpack, adam, 0.01, ("c_p", "opacity_raw", "lam", "b", "angles"), angles)
    return np.concatenate([p.c_p.ravel(), p.opacity_raw, p.lam, p.b, [p.polar, p.azimuth]]), losses


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = [v for v in range(4) if v % world == rank]  # views sharded round-robin
    vec, losses = _run_fit(mine, 3, dist, n_views=4)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([vec, losses]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_views_equal_single_process(tmp_path):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1), "ranks diverged"
    vec, losses = _run_fit([0, 1, 2, 3], 3)
    np.testing.assert_allclose(r0, np.concatenate([vec, losses]), rtol=1e-12, atol=1e-15)


def _fake_render(cams):
    return [np.full((2, 3, 4), float(c), np.float32) for c in cams]


def _fake_train(dataset, cfg):
    return {"tf": dataset, "n": len(dataset)}


def _units_worker(rank, world, port, out_dir):
    import pickle
    from paper_2504_17954_b200.multigpu import render_views, shard, train_per_rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cams = list(range(7))  # "cameras": the fake render paints the view index
    imgs = render_views(None, cams, dist=dist, render_fn=_fake_render)
    local = render_views(None, cams, dist=dist, gather=False, render_fn=_fake_render)
    models = train_per_rank([f"tf{r}" for r in range(world)], dist=dist, train_fn=_fake_train)
    with open(os.path.join(out_dir, f"u{rank}.pkl"), "wb") as f:
        pickle.dump({"imgs": imgs, "local": [i for i, _ in local], "models": models,
                     "shard": shard(7, rank, world)}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_render_views_and_train_per_rank_gather_in_order(tmp_path):
    """multigpu.render_views / train_per_rank: views round-robin over the ranks,
    one training unit per rank, no data-path collective; rank 0 gathers
    every view in the callers' order and every rank's model in rank order."""
    import pickle
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_units_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    u0 = pickle.load(open(tmp_path / "u0.pkl", "rb"))
    u1 = pickle.load(open(tmp_path / "u1.pkl", "rb"))
    assert u0["local"] == [0, 2, 4, 6] and u1["local"] == [1, 3, 5]
    assert u0["shard"] == [0, 2, 4, 6] and u1["shard"] == [1, 3, 5]
    assert u1["imgs"] is None and u1["models"] is None
    assert [float(img[0, 0, 0]) for img in u0["imgs"]] == [float(v) for v in range(7)]
    assert [m["tf"] for m in u0["models"]] == ["tf0", "tf1"]


def test_single_process_units():
    from paper_2504_17954_b200.multigpu import render_views, shard, train_per_rank
    imgs = render_views(None, [3, 1, 2], render_fn=_fake_render)
    assert [float(i[0, 0, 0]) for i in imgs] == [3.0, 1.0, 2.0]
    assert train_per_rank(["a"], train_fn=_fake_train) == [{"tf": "a", "n": 1}]
    with pytest.raises(ValueError):
        train_per_rank(["a", "b"], train_fn=_fake_train)
    with pytest.raises(ValueError):
        shard(4, 2, 2)
