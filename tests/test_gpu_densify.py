"""Densify / prune vs the reference (golden from voxsplat.trainer.densify_and_prune,
trainer.py:241-261 -> _densify_params :135-193).

The split offsets come from the same numpy stream as the reference's
(``rng.standard_normal((2*ns, 3))``), so the surviving rows, their order and
every copied attribute are identical; the split children's positions
(mu + R @ offsets, a 3-term einsum) agree to rounding."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
SHADE = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _models(d):
    from paper_2504_17954_b200 import (BasicSceneModel, GaussianGeometry, Palette, ShadingAttributes,
                                       ShColor)
    geom = GaussianGeometry(*(d[k] for k in GEOM))
    edit = BasicSceneModel("editable", geom, shading=ShadingAttributes(*(d[k] for k in SHADE)),
                           palette=Palette(d["palette"]))
    base = BasicSceneModel("base", geom, sh=ShColor(d["sh"], 1))
    return edit, base


@pytest.mark.parametrize("tag,seed,maxp,extent", [("edit", 3, 500, 30.0),
                                                   ("nobudget", 4, 400, 0.8),
                                                   ("base", 5, 120000, 40.0)])
def test_densify_and_prune_matches_reference(tag, seed, maxp, extent):
    from paper_2504_17954_b200.trainer import TrainConfig, densify_and_prune
    d = golden("densify")
    edit, base = _models(d)
    model = base if tag == "base" else edit
    cfg = TrainConfig(max_primitives=maxp, seed=seed)
    new, info = densify_and_prune(model, d["stats"], cfg, extent=extent,
                                  rng=np.random.default_rng(seed))
    for k in ("cloned", "split", "pruned", "count"):
        assert info[k] == int(d[f"{tag}_info_{k}"]), (k, info)
    for k in GEOM:
        got, ref = np.asarray(getattr(new.geometry, k)), d[f"{tag}_{k}"]
        assert got.shape == ref.shape, k
        if k == "mu":  # split children: mu + R @ (offs * s), summation order may differ
            np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15, err_msg=k)
        else:
            assert np.array_equal(got, ref), k
    if tag == "base":
        assert np.array_equal(new.sh.coefficients, d["base_sh"])
    else:
        for k in SHADE:
            assert np.array_equal(getattr(new.shading, k), d[f"{tag}_{k}"]), k


def test_densify_all_pruned_returns_empty_model():
    from paper_2504_17954_b200 import BasicSceneModel, GaussianGeometry, Palette, ShadingAttributes
    from paper_2504_17954_b200.trainer import TrainConfig, densify_and_prune
    d = golden("densify")
    o = np.full(400, -9.0)
    geom = GaussianGeometry(d["mu"], d["q_raw"], d["log_s"], o, d["n_raw"])
    m = BasicSceneModel("editable", geom, shading=ShadingAttributes(*(d[k] for k in SHADE)),
                        palette=Palette(d["palette"]))
    new, info = densify_and_prune(m, d["stats"], TrainConfig(), extent=0.8,
                                  rng=np.random.default_rng(0))
    assert len(new.geometry.mu) == int(d["empty_count"]) == 0
    for k in ("cloned", "split", "pruned", "count"):
        assert info[k] == int(d[f"empty_info_{k}"]), (k, info)
