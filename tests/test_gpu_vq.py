"""GPU VQ (K5 assign / K6 decode / device k-means) vs the reference."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_assign_bit_exact_vs_reference():
    """searchsorted(mids, v, 'left') incl. exact ties, NaN, +-1e300."""
    from paper_2504_17954_b200.vq import assign_nearest
    d = golden("vq")
    assert np.array_equal(assign_nearest(d["values"], d["centroids"]), d["indices"])


def test_assign_large_vs_oracle():
    import oracle as O
    from paper_2504_17954_b200.vq import assign_nearest
    rng = np.random.default_rng(0)
    for k in (2, 17, 256, 4096, 9000):  # 9000: midpoints beyond the smem table
        c = np.sort(rng.normal(size=k))
        v = rng.normal(size=200_000) * 1.5
        assert np.array_equal(assign_nearest(v, c), O.vq_assign(v, c)), k


def test_assign_bucket_table_corner_cases():
    """Clustered codebooks, values exactly on midpoints and bucket edges, a
    huge offset with tiny spacing (bucket index rounding), +-inf and NaN."""
    import oracle as O
    from paper_2504_17954_b200.vq import assign_nearest
    rng = np.random.default_rng(3)
    cases = []
    c = np.sort(np.concatenate([rng.normal(0, 1e-6, 3000), rng.normal(5, 2, 1000)]))
    mids = 0.5 * (c[1:] + c[:-1])
    v = np.concatenate([rng.normal(0, 1e-6, 50_000), rng.normal(5, 3, 50_000), mids,
                        np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf),
                        [np.inf, -np.inf, np.nan, 1e300, -1e300, 0.0, -0.0]])
    cases.append((c, v))
    c2 = np.sort(1e6 + np.arange(4096) * 1e-9 + rng.uniform(0, 1e-10, 4096))
    m2 = 0.5 * (c2[1:] + c2[:-1])
    lo, hi = m2[0], m2[-1]
    edges = lo + np.arange(8192) * ((hi - lo) / 8192)
    v2 = np.concatenate([m2, edges, np.nextafter(edges, np.inf), np.nextafter(edges, -np.inf),
                         rng.uniform(c2[0] - 1e-6, c2[-1] + 1e-6, 100_000)])
    cases.append((c2, v2))
    c3 = np.array([-1.0, -1.0, 0.0, 0.0, 0.0, 3.0])  # duplicate centroids
    cases.append((c3, np.array([-2.0, -1.0, -0.5, 0.0, 1.5, 3.0, 9.0])))
    for c, v in cases:
        assert np.array_equal(assign_nearest(v, c), O.vq_assign(v, c))


def test_decode_and_corrupt_index():
    from paper_2504_17954_b200 import CorruptIndex
    from paper_2504_17954_b200.vq import Codebook
    cb = Codebook("x", np.array([-1.0, 0.25, 3.0]))
    idx = np.array([[0, 2], [1, 1]], dtype=np.uint8)
    assert np.array_equal(cb.decode(idx), cb.centroids[idx.astype(np.int64)])
    with pytest.raises(CorruptIndex):
        cb.decode(np.array([0, 3], dtype=np.uint8))
    with pytest.raises(CorruptIndex):  # wider types: checked before the uint16 upload
        cb.decode(np.array([0, 65536 + 1], dtype=np.int64))
    # signed indices follow numpy indexing, as the reference's centroids[indices]
    assert np.array_equal(cb.decode(np.array([-1, -3, 2])), cb.centroids[[-1, -3, 2]])
    with pytest.raises(IndexError):
        cb.decode(np.array([0, -4]))


def test_kmeans_matches_reference():
    from paper_2504_17954_b200.vq import kmeans
    d = golden("vq")
    got = kmeans(d["samples"], 16, seed=1)
    ref = d["kmeans16"]
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-12)


def test_kmeans_distinct_shortcut_and_separable():
    from paper_2504_17954_b200.vq import kmeans
    assert np.array_equal(kmeans(np.array([3.0, 1.0, 2.0, 1.0, 3.0]), 8), [1.0, 2.0, 3.0])
    assert np.array_equal(kmeans(np.array([0.0, 0.0, 10.0, 10.0]), 2), [0.0, 10.0])


def test_quantize_dequantize_round_trip():
    from paper_2504_17954_b200 import dequantize_model, quantize_model
    from paper_2504_17954_b200.synthetic import editable_model
    m = editable_model(4, 3000)
    q = quantize_model(m, k=64, seed=0)
    assert q.is_quantized and q.shading is None
    for name, (cb, idx) in q.quantized.items():
        assert cb.k <= 64 and idx.dtype == np.uint8
    for name in ("q_raw", "log_s", "o_logit"):  # the model's dequantized views
        cb, idx = q.quantized[name]
        got = getattr(q.geometry, name)
        assert got.shape == idx.shape and np.array_equal(got, cb.decode(idx)), name
    d = dequantize_model(q)
    for name, (cb, idx) in q.quantized.items():
        owner = d.geometry if name in ("q_raw", "log_s", "o_logit") else d.shading
        assert np.array_equal(getattr(owner, name), cb.centroids[idx.astype(np.int64)])
    assert np.array_equal(d.geometry.mu, m.geometry.mu)


def test_seed_plusplus_follows_the_reference_stream():
    """Fused device k-means++ (ivr_kmeans_seed) picks the same centres as the
    reference's _seed_plusplus (vq.py:60-72) from the same numpy stream."""
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.vq import _seed_plusplus
    x = np.random.default_rng(11).normal(size=50_000) ** 3
    k = 300
    rng = np.random.default_rng(3)
    ref = np.empty(k)
    ref[0] = x[rng.integers(x.size)]
    d2 = (x - ref[0]) ** 2
    for i in range(1, k):
        ref[i] = x[rng.choice(x.size, p=d2 / d2.sum())]
        d2 = np.minimum(d2, (x - ref[i]) ** 2)
    got = _seed_plusplus(to_dev(x), k, np.random.default_rng(3)).cpu().numpy()
    assert np.array_equal(got, ref)


def _seed_full_pass(x, k, rng):
    """ivr_kmeans_seed (every sample every step) with the same draws."""
    import torch
    from paper_2504_17954_b200 import _lib as L
    from paper_2504_17954_b200 import device as D
    n = x.numel()
    first = int(rng.integers(n))
    u = torch.from_numpy(rng.random(k - 1)).to(x.device)
    c = torch.empty(k, dtype=torch.float64, device=x.device)
    nb = int(L.lib().ivr_kmeans_seed_workspace_size(n))
    ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    L.check(L.lib().ivr_kmeans_seed(D.ptr(x), n, int(k), first, D.ptr(u), D.ptr(c), D.ptr(ws), nb,
                                    D.stream_handle()), "ivr_kmeans_seed")
    return c.cpu().numpy()


@pytest.mark.parametrize("case", ["cubed", "ties", "clusters", "tiny", "exhausted", "large"])
def test_sorted_seeding_equals_full_pass(case):
    """ivr_kmeans_seed_sorted (d2 lowered only between the adjacent chosen
    centres in value order) picks the same centres as the full-pass seeding
    from the same draws: heavy ties, clustered values, n < one block, more
    centres than distinct values (the all-mass-chosen fill), 3M values."""
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.vq import _seed_plusplus
    g = np.random.default_rng(5)
    k = 256
    if case == "cubed":
        x = g.normal(size=200_000) ** 3
    elif case == "ties":
        x = g.integers(0, 3000, size=150_000).astype(np.float64) * 0.25
    elif case == "clusters":
        x = np.concatenate([g.normal(m, 1e-3, size=40_000) for m in (-5.0, 0.0, 0.1, 7.0)])
        g.shuffle(x)
    elif case == "tiny":
        x, k = g.normal(size=23), 9
    elif case == "exhausted":
        x, k = g.integers(0, 40, size=5_000).astype(np.float64), 64
    else:
        x, k = g.standard_t(3, size=3_000_000), 1024
    xd = to_dev(x)
    got = _seed_plusplus(xd, k, np.random.default_rng(8)).cpu().numpy()
    ref = _seed_full_pass(xd, k, np.random.default_rng(8))
    assert np.array_equal(got, ref)
    if case == "exhausted":  # the remaining centres repeat the first one, as the reference
        assert len(np.unique(got)) == 40 and np.all(got[40:] == got[0])


@pytest.mark.parametrize("n,k,restarts", [(120_000, 300, 5), (5_000, 64, 8), (40_000, 500, 3),
                                          (3_000, 40, 11), (2_000, 1, 3)])
def test_batched_restart_seedings_equal_sequential(n, k, restarts):
    """k-means' restarts seeded in one launch (all draws taken up front in the
    reference's order) == the restarts seeded one after the other; more than
    8 restarts take two launches; k = 1 draws only the first centres."""
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.vq import _seed_restarts
    g = np.random.default_rng(n)
    x = np.concatenate([g.normal(size=n - n // 4) ** 3, g.integers(0, 50, size=n // 4) * 0.5])
    g.shuffle(x)
    xd = to_dev(x)
    got = _seed_restarts(xd, k, np.random.default_rng(2), restarts).cpu().numpy()
    rng = np.random.default_rng(2)
    for r in range(restarts):
        assert np.array_equal(got[r], _seed_full_pass(xd, k, rng)), r


def test_quantize_attributes_indices_equal_codebook_encode():
    """quantize_attributes' device-side encode (one upload per attribute,
    uint16 straight into the index dtype) == Codebook.encode (the reference's
    assign_nearest path), shapes and dtypes included."""
    from paper_2504_17954_b200.vq import quantize_attributes
    g = np.random.default_rng(4)
    arrays = {"a": g.normal(size=(3000, 4)), "b": g.standard_t(2, size=5000),
              "c": np.repeat(g.normal(size=7), 100)}
    for k in (64, 300):
        q = quantize_attributes(arrays, k=k, seed=1)
        for name, arr in arrays.items():
            cb, idx = q[name]
            ref = cb.encode(arr)
            assert idx.dtype == ref.dtype == cb.index_dtype and idx.shape == arr.shape
            assert np.array_equal(idx, ref), (k, name)


def test_lloyd_sets_match_per_restart_lloyd():
    """The restarts' Lloyd runs in one loop on the sorted values (segment sums
    between midpoints, ivr_kmeans_lloyd_step_sorted) == each restart's own
    loop with the atomic accumulation (ivr_kmeans_lloyd_step), up to the
    float64 summation order."""
    import torch
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.vq import _lloyd, _lloyd_sets, _seed_restarts
    g = np.random.default_rng(6)
    x = np.concatenate([g.normal(size=60_000) ** 3, g.integers(0, 30, size=20_000) * 0.1])
    g.shuffle(x)
    xd = to_dev(x)
    seeds = _seed_restarts(xd, 128, np.random.default_rng(1), 4)
    got = _lloyd_sets(xd, torch.sort(xd).values, seeds).cpu().numpy()
    for r in range(4):
        ref = _lloyd(xd, seeds[r].clone()).cpu().numpy()
        np.testing.assert_allclose(got[r], ref, rtol=1e-9, atol=1e-12, err_msg=str(r))


def test_quantize_attributes_batched_seedings_equal_per_attribute_kmeans():
    """All attributes' restart seedings in one launch (quantize_attributes) ==
    each attribute's own kmeans call (vq.py:137-147: a fresh default_rng(seed)
    per attribute), codebook for codebook."""
    from paper_2504_17954_b200.vq import kmeans, quantize_attributes
    g = np.random.default_rng(9)
    arrays = {"q": g.normal(size=(20_000, 4)), "s": g.standard_t(3, size=(15_000, 3)),
              "o": g.normal(size=9_000) ** 3, "few": np.repeat([0.5, -1.0, 2.0], 50)}
    q = quantize_attributes(arrays, k=200, seed=3)
    for name, arr in arrays.items():
        assert np.array_equal(q[name][0].centroids, kmeans(arr.reshape(-1), 200, seed=3)), name


def test_sorted_lloyd_step_ties_empty_buckets_and_sets():
    """One ivr_kmeans_lloyd_step_sorted step == vq.py:75-87's step in numpy
    (searchsorted on the midpoints, bincount means, empty buckets keep their
    centroid) for values exactly on midpoints, empty buckets and 3 sets."""
    import torch
    from paper_2504_17954_b200 import _lib as L
    from paper_2504_17954_b200 import device as D
    g = np.random.default_rng(12)
    x = np.concatenate([g.normal(size=5000), [0.5, 2.0, 2.0, -7.0, 11.0]])
    sets = np.array([[0.0, 1.0, 3.0, 4.0, 50.0], [-9.0, -8.0, 0.0, 0.25, 0.3],
                     [-1.0, -1.0, 0.0, 1.0, 1.0]])
    xs = D.to_dev(np.sort(x))
    c = D.to_dev(sets.reshape(-1))
    new = torch.empty_like(c)
    shift = torch.empty(3, dtype=torch.float64, device=c.device)
    k = sets.shape[1]
    nb = int(L.lib().ivr_kmeans_lloyd_sorted_workspace_size(k, 3))
    ws = torch.empty(nb, dtype=torch.uint8, device=c.device)
    L.check(L.lib().ivr_kmeans_lloyd_step_sorted(D.ptr(xs), xs.numel(), D.ptr(c), k, 3,
                                                 D.ptr(new), D.ptr(shift), D.ptr(ws), nb,
                                                 D.stream_handle()), "lloyd sorted")
    got = new.cpu().numpy().reshape(3, k)
    for r in range(3):
        cen = sets[r]
        idx = np.searchsorted(0.5 * (cen[1:] + cen[:-1]), x)
        sums = np.bincount(idx, weights=x, minlength=k)
        cnt = np.bincount(idx, minlength=k)
        ref = np.where(cnt > 0, sums / np.maximum(cnt, 1), cen)
        np.testing.assert_allclose(got[r], ref, rtol=1e-13, atol=1e-15, err_msg=str(r))
        assert shift[r].item() == pytest.approx(np.abs(ref - cen).max(), rel=1e-12)


@pytest.mark.parametrize("n,k,dist", [(200_000, 1000, "t2"), (120_000, 2048, "mixture")])
def test_seed_plusplus_follows_the_reference_stream_at_scale(n, k, dist):
    """The sorted seeding against the reference's own _seed_plusplus loop
    (vq.py:60-72, numpy rng.choice) on heavier inputs: every centre equal."""
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.vq import _seed_plusplus
    g = np.random.default_rng(n)
    if dist == "t2":
        x = g.standard_t(2, size=n)
    else:
        x = np.concatenate([g.normal(-3, 0.1, n // 3), g.exponential(2.0, n // 3),
                            g.integers(0, 500, n - 2 * (n // 3)) * 0.01])
        g.shuffle(x)
    rng = np.random.default_rng(7)
    ref = np.empty(k)
    ref[0] = x[rng.integers(x.size)]
    d2 = (x - ref[0]) ** 2
    for i in range(1, k):
        ref[i] = x[rng.choice(x.size, p=d2 / d2.sum())]
        d2 = np.minimum(d2, (x - ref[i]) ** 2)
    got = _seed_plusplus(to_dev(x), k, np.random.default_rng(7)).cpu().numpy()
    assert np.array_equal(got, ref)
