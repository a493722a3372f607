"""Host logic of the device k-means (no GPU): the up-front restart draws
follow the reference's random stream, and the C-ABI rejects bad seeding /
Lloyd arguments before touching the device."""
import ctypes

import numpy as np
import pytest


def test_draw_seeds_follow_the_reference_stream():
    """vq._draw_seeds == the reference's consumption (vq.py:47-72): per restart
    rng.integers(n), then one rng.random() per rng.choice call."""
    from paper_2504_17954_b200.vq import _draw_seeds
    n, k, restarts = 12345, 17, 5
    got = _draw_seeds(n, k, np.random.default_rng(42), restarts)
    rng = np.random.default_rng(42)
    for first, u in got:
        assert first == int(rng.integers(n))
        assert np.array_equal(u, np.array([rng.random() for _ in range(k - 1)]))


def test_draw_seeds_k1_draws_only_the_first_centres():
    from paper_2504_17954_b200.vq import _draw_seeds
    got = _draw_seeds(100, 1, np.random.default_rng(1), 3)
    rng = np.random.default_rng(1)
    assert [f for f, _ in got] == [int(rng.integers(100)) for _ in range(3)]
    assert all(u.size == 0 for _, u in got)


def test_seed_and_lloyd_entry_points_reject_bad_arguments():
    """Argument checks run before any device work (count, k, n, first, null
    pointers, workspace size)."""
    from paper_2504_17954_b200 import _lib as L
    lib = L.lib()
    fake = 256  # never dereferenced: every call below fails validation
    arr = (L.SeedProblem_t * 1)()
    arr[0].values, arr[0].order, arr[0].n, arr[0].first = fake, fake, 1000, 3
    arr[0].u, arr[0].centers = fake, fake
    big = 1 << 40
    assert lib.ivr_kmeans_seed_sorted(arr, 0, 16, fake, big, None) != 0      # no seeding
    assert lib.ivr_kmeans_seed_sorted(arr, 65, 16, fake, big, None) != 0     # > 64 per launch
    assert lib.ivr_kmeans_seed_sorted(arr, 1, 0, fake, big, None) != 0       # k < 1
    assert lib.ivr_kmeans_seed_sorted(arr, 1, 40000, fake, big, None) != 0   # k > 32768
    assert lib.ivr_kmeans_seed_sorted(arr, 1, 16, fake, 8, None) != 0        # workspace
    arr[0].first = 1000
    assert lib.ivr_kmeans_seed_sorted(arr, 1, 16, fake, big, None) != 0      # first >= n
    arr[0].first, arr[0].u = 3, None
    assert lib.ivr_kmeans_seed_sorted(arr, 1, 16, fake, big, None) != 0      # no draws
    assert "ivr_kmeans_seed_sorted" in lib.ivr_last_error().decode()
    ws = lib.ivr_kmeans_lloyd_sorted_workspace_size(16, 2)
    assert ws >= 8 * 17 * 2
    assert lib.ivr_kmeans_lloyd_step_sorted(fake, 1000, fake, 1, 1, fake, fake, fake, ws,
                                            None) != 0  # k < 2
    assert lib.ivr_kmeans_lloyd_step_sorted(fake, 1000, fake, 16, 2, fake, fake, fake, ws - 1,
                                            None) != 0  # workspace
    assert lib.ivr_kmeans_lloyd_step_sorted(fake, 0, fake, 16, 2, fake, fake, fake, ws,
                                            None) != 0  # n < 1
