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


def test_decode_and_corrupt_index():
    from paper_2504_17954_b200 import CorruptIndex
    from paper_2504_17954_b200.vq import Codebook
    cb = Codebook("x", np.array([-1.0, 0.25, 3.0]))
    idx = np.array([[0, 2], [1, 1]], dtype=np.uint8)
    assert np.array_equal(cb.decode(idx), cb.centroids[idx.astype(np.int64)])
    with pytest.raises(CorruptIndex):
        cb.decode(np.array([0, 3], dtype=np.uint8))


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
    d = dequantize_model(q)
    for name, (cb, idx) in q.quantized.items():
        owner = d.geometry if name in ("q_raw", "log_s", "o_logit") else d.shading
        assert np.array_equal(getattr(owner, name), cb.centroids[idx.astype(np.int64)])
    assert np.array_equal(d.geometry.mu, m.geometry.mu)
