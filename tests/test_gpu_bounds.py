"""The instruction error bounds FAST mode's certified decisions rest on,
measured on the device (VERDICT r01 "what's weak" 1): K3/K4 budget the
ex2.approx.ftz.f32 of alpha = o 2^(-sigma log2 e) at 2 ulp (csrc/blend.cu,
`rel = E + 1.2e-7 sigma + 3.6e-7`: 2.4e-7 of it for the instruction) and the
rcp.approx.ftz.f32 of the tile cull / T error bound at 2^-22."""

import pytest

pytestmark = pytest.mark.gpu


def test_mufu_approx_errors_within_the_certified_budget():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_17954_b200 import _lib as L
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    L.check(L.lib().ivr_debug_mufu_error(out.data_ptr(), None), "ivr_debug_mufu_error")
    torch.cuda.synchronize()
    ex2, rcp = (float(v) for v in out.cpu())
    print(f"max relative error: ex2.approx {ex2:.3g} ({ex2 / 2 ** -23:.2f} ulp), "
          f"rcp.approx {rcp:.3g} ({rcp / 2 ** -23:.2f} ulp)")
    assert 0.0 < ex2 <= 2 * 2 ** -23
    assert 0.0 < rcp <= 2 * 2 ** -23


def test_float32_exponent_error_within_ksigmaerr():
    """kSigmaErr = 4e-7 (csrc/blend.cu:48-51) bounds |sigma32 - sigma_ref| per
    unit of |a/2 dx^2| + |b dx dy| + |c/2 dy^2|; 2^26 random samples."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_17954_b200 import _lib as L
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    L.check(L.lib().ivr_debug_sigma_error(1 << 26, 12345, out.data_ptr(), None),
            "ivr_debug_sigma_error")
    torch.cuda.synchronize()
    worst = float(out.item())
    print(f"max |sigma32 - sigma_ref| / terms = {worst:.3g} (kSigmaErr 4e-7)")
    assert 0.0 < worst <= 4e-7
