"""The voxsplat._kernels drop-in (paper_2504_17954_b200._kernels): the
reference's plugin-point signatures, in-place outputs, against the oracle's C
restatement of the same three functions."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _state(dtype):
    import oracle as O
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    n = 3000
    a = editable_arrays(21, n, density=n)
    cam = bench_camera(72, 56, azimuth=0.9)
    colors = np.random.default_rng(21).uniform(0, 1, (n, 3))
    return O.rasterize(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"], colors, cam,
                       channels=("color", "alpha", "depth", "normal"), dtype=dtype), cam


def test_fill_pairs_order():
    from paper_2504_17954_b200._kernels import fill_pairs
    rng = np.random.default_rng(3)
    n, ntx = 50, 9
    tx0 = rng.integers(0, ntx, n)
    tx1 = np.minimum(tx0 + rng.integers(0, 3, n), ntx - 1)
    ty0 = rng.integers(0, 6, n)
    ty1 = ty0 + rng.integers(0, 3, n)
    counts = (tx1 - tx0 + 1) * (ty1 - ty0 + 1)
    offsets = np.concatenate([[0], np.cumsum(counts)[:-1]])
    P = int(counts.sum())
    pt, ps = np.empty(P, np.int64), np.empty(P, np.int64)
    fill_pairs(offsets, tx0, tx1, ty0, ty1, ntx, pt, ps)
    et, es = [], []
    for i in range(n):  # splat-major, then ty, then tx (_kernels.py:22-28)
        for ty in range(ty0[i], ty1[i] + 1):
            for tx in range(tx0[i], tx1[i] + 1):
                et.append(ty * ntx + tx)
                es.append(i)
    assert np.array_equal(pt, et) and np.array_equal(ps, es)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_composite_forward_matches_oracle(dtype):
    from paper_2504_17954_b200._kernels import composite_forward
    st, cam = _state(dtype)
    km, kc, ko, kv = st["kmean2d"], st["kconic"], st["kopacity"], st["values"]
    H, W, K = cam.height, cam.width, kv.shape[1]
    out = np.zeros((H, W, K), dtype=dtype)
    contrib = np.zeros((H, W), np.int32)
    last = np.zeros((H, W), np.int64)
    tf = np.zeros((H, W))
    composite_forward(st["tile_ranges"], st["pair_splat"], km, kc, ko, kv, W, H, 16, st["ntx"],
                      out, contrib, last, tf)
    assert np.array_equal(contrib, st["contrib"])
    assert np.array_equal(last, st["last_pos"])
    assert np.abs(out - st["out"]).max() <= 1e-6
    assert np.abs(tf - st["t_final"]).max() <= 1e-6


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_composite_backward_matches_oracle(dtype):
    from oracle.port import _p, lib
    from paper_2504_17954_b200._kernels import composite_backward
    st, cam = _state(dtype)
    km, kc, ko, kv = st["kmean2d"], st["kconic"], st["kopacity"], st["values"]
    H, W, K = cam.height, cam.width, kv.shape[1]
    P = st["pair_splat"].size
    d_out = np.random.default_rng(5).normal(size=(H, W, K))
    got = [np.zeros((P, K)), np.zeros((P, 2)), np.zeros((P, 3)), np.zeros(P)]
    composite_backward(st["tile_ranges"], st["pair_splat"], km, kc, ko, kv, W, H, 16, st["ntx"],
                       d_out, st["last_pos"], st["t_final"], *got)
    ref = [np.zeros((P, K)), np.zeros((P, 2)), np.zeros((P, 3)), np.zeros(P)]
    f = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    lib().orc_composite_backward(
        _p(st["tile_ranges"]), st["ntx"] * st["nty"], _p(st["pair_splat"]), _p(f(km)),
        _p(f(kc)), _p(f(ko)), _p(f(kv)), K, W, H, 16, st["ntx"], _p(f(d_out)),
        _p(st["last_pos"]), _p(st["t_final"]), *(_p(r) for r in ref), 0)
    for g, r in zip(got, ref):
        err = np.linalg.norm(g - r)
        assert err <= 1e-3 * max(np.linalg.norm(r), 1e-12), (err, np.linalg.norm(r))
