"""Fused L1 + SSIM kernels (csrc/ssim.cu) vs the oracle restatement of
losses.ssim / losses.photometric_loss (float64, tolerance 1e-12 relative on
values, 1e-10 on gradients: only the summation order differs)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("shape", [(11, 11, 1), (11, 30, 4), (37, 53, 4), (64, 48, 3), (40, 33)])
def test_ssim_matches_oracle(shape):
    import oracle as O
    from paper_2504_17954_b200.losses import ssim
    rng = np.random.default_rng(sum(shape))
    x = rng.uniform(0, 1, shape)
    y = np.clip(x + rng.normal(0, 0.1, shape), 0, 1)
    v, d = ssim(x, y)
    rv, rd = O.ssim(x, y)
    assert abs(v - rv) <= 1e-12 * abs(rv)
    assert d.shape == rd.shape
    np.testing.assert_allclose(d, rd, rtol=1e-9, atol=1e-14 * np.abs(rd).max())


@pytest.mark.parametrize("w", [(0.8, 0.2), (1.0, 0.0), (0.0, 1.0)])
def test_photometric_loss_matches_oracle(w):
    import oracle as O
    from paper_2504_17954_b200.losses import LossWeights, photometric_loss
    rng = np.random.default_rng(7)
    pred = rng.uniform(0, 1, (45, 70, 4))
    gt = rng.uniform(0, 1, (45, 70, 4))
    gt[:5] = pred[:5]  # exact zeros of pred - gt: sign(0) = 0
    loss, d = photometric_loss(pred, gt, LossWeights(l1_weight=w[0], ssim_weight=w[1]))
    rl, rd = O.photometric_loss(pred, gt, l1_w=w[0], ssim_w=w[1])
    assert abs(loss - rl) <= 1e-12 * abs(rl)
    np.testing.assert_allclose(d, rd, rtol=1e-9, atol=1e-14 * np.abs(rd).max())


def test_small_image_errors():
    from paper_2504_17954_b200 import ShapeMismatch
    from paper_2504_17954_b200.losses import LossWeights, photometric_loss, ssim
    x = np.zeros((10, 20, 4))
    with pytest.raises(ShapeMismatch):
        ssim(x, x)
    with pytest.raises(ShapeMismatch):
        photometric_loss(x, x)
    loss, d = photometric_loss(x, x + 0.5, LossWeights(ssim_weight=0.0))  # L1 only: fine
    assert abs(loss - 0.4) < 1e-15 and np.allclose(d, -0.8 / x.size)
