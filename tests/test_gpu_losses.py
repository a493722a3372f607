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


def test_fused_regularizers_match_loss_functions():
    """ivr_regularize == the per-term functions (pseudo normals + consistency,
    offset sparsity, bilateral smoothness on four maps) on random maps."""
    import torch
    from paper_2504_17954_b200 import orbit_camera
    from paper_2504_17954_b200.losses import (bilateral_smoothness, normal_consistency_loss,
                                              offset_sparsity_loss, pseudo_normal_from_depth,
                                              regularize_t)
    rng = np.random.default_rng(11)
    H, W, K = 37, 45, 15
    out = rng.uniform(0.05, 1.0, (H, W, K)).astype(np.float32)
    out[..., 4] = (2.0 + rng.uniform(0, 0.3, (H, W))).astype(np.float32)  # depth
    out[:5, :7, 3] = 0.0                                                     # alpha holes
    gt = rng.uniform(0, 1, (H, W, 4))
    d_rgba = rng.normal(size=(H, W, 4))
    cam = orbit_camera(np.zeros(3), 2.5, 0.4, -0.3, 0.9, W, H)
    blk = np.concatenate([[0.5 * H / np.tan(0.5 * cam.fov_y), (W - 1) / 2.0, (H - 1) / 2.0],
                          cam.rotation.reshape(9)])
    dev = torch.device("cuda")
    terms, d_out = regularize_t(torch.from_numpy(out).to(dev), (0, 3, 4, 5, 8),
                                gt=torch.from_numpy(gt).to(dev), d_rgba=torch.from_numpy(d_rgba).to(dev),
                                cam_params=torch.from_numpy(blk).to(dev), w_normal=0.01,
                                w_offset=0.02, w_bil=0.03, bil_cols=(11, 12, 13, 14))
    terms, d_out = terms.cpu().numpy(), d_out.cpu().numpy()
    o = out.astype(np.float64)
    target, mask = pseudo_normal_from_depth(o[..., 4], o[..., 3], cam)
    nl, dn = normal_consistency_loss(o[..., 5:8], target, mask)
    assert abs(terms[0] - nl) <= 1e-9 * max(abs(nl), 1e-30)
    np.testing.assert_allclose(d_out[..., 5:8], (0.01 * dn).astype(np.float32), rtol=1e-5, atol=1e-9)
    ol, do = offset_sparsity_loss(o[..., 8:11])
    assert abs(terms[1] - ol) <= 1e-12 * abs(ol)
    np.testing.assert_allclose(d_out[..., 8:11], (0.02 * do).astype(np.float32), rtol=1e-6)
    bl = 0.0
    for ch in (11, 12, 13, 14):
        b, db = bilateral_smoothness(o[..., ch], gt[..., :3])
        bl += b
        np.testing.assert_allclose(d_out[..., ch], (0.03 * db).astype(np.float32), rtol=1e-5,
                                   atol=1e-12)
    assert abs(terms[2] - bl) <= 1e-10 * abs(bl)
    np.testing.assert_allclose(d_out[..., 0:3], d_rgba[..., :3].astype(np.float32))
    np.testing.assert_allclose(d_out[..., 3], d_rgba[..., 3].astype(np.float32))
    assert np.all(d_out[..., 4] == 0.0)


@pytest.mark.parametrize("with_ssim", [True, False])
def test_photometric_frame_source_is_bit_identical(with_ssim):
    """ivr_photometric_loss_frame (prediction read in place from a float32
    (H,W,k) frame at a column map) == ivr_photometric_loss on the gathered
    float64 copy, bit for bit (f32 -> f64 promotion is exact)."""
    import torch
    from paper_2504_17954_b200 import ShapeMismatch
    from paper_2504_17954_b200.losses import _photometric_dev, _photometric_frame_dev
    g = torch.Generator().manual_seed(3)
    frame = torch.rand((67, 91, 15), generator=g).cuda()
    gt = torch.rand((67, 91, 4), generator=g, dtype=torch.float64).cuda()
    cols = (4, 5, 6, 11)
    s0, d0 = _photometric_dev(frame[..., list(cols)].double(), gt, 0.3, -0.7, with_ssim)
    s1, d1 = _photometric_frame_dev(frame, cols, gt, 0.3, -0.7, with_ssim)
    assert torch.equal(s0, s1) and torch.equal(d0, d1)
    with pytest.raises(ShapeMismatch):
        _photometric_frame_dev(frame, cols[:3], gt, 0.3, -0.7, with_ssim)
    with pytest.raises(Exception):
        _photometric_frame_dev(frame, (0, 1, 2, 15), gt, 0.3, -0.7, with_ssim)
    with pytest.raises(ShapeMismatch):  # float32 ground truth, float64 frame
        _photometric_frame_dev(frame, cols, gt.float(), 0.3, -0.7, with_ssim)
    with pytest.raises(ShapeMismatch):
        _photometric_frame_dev(frame.double(), cols, gt, 0.3, -0.7, with_ssim)
