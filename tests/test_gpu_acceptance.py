"""The reference's desk-scale acceptance pipeline on the GPU path
(pkg/tests/test_acceptance.py:170-310): two basic transfer functions on the
64^3 nested-shells volume, ground truth from the DVR ray march, both training
stages (3000 + 1000 iterations, densify / prune, the captured step) at 128^2,
then the PSNR, composition, VQ and relighting gates at the reference's
thresholds.

The reference picks each scene's view count from an entropy score
(viewsampler.py, out of scope here); this port trains on a fixed 42-view
Fibonacci rig and evaluates on 20 other directions.  On that rig the
reference's own editable stage lands ~2 dB under its base stage (its
"editable within 1 dB" gate is rig-dependent), so the quality gate here is
the reference's own result on the same data (tests/golden/desk_reference.json,
written by make_desk_reference.py running voxsplat): the base stage within
0.5 dB of it, the editable stage within 1 dB, plus the reference's absolute
24 dB floor.  The editable stage's trajectory depends on the order of the
blend backward's float32 atomics: six runs of scene 0 gave 34.54-35.65 dB
(reference 35.45; IVR_DETERMINISTIC=1 gives 34.96 every run), the base
stage 37.46-37.55 dB (reference 37.48).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RES = 128
STAGE1, STAGE2 = 3000, 1000


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_17954_b200 import _lib
    _lib.lib()


def psnr(a, b):
    """metrics.psnr (metrics.py:18-29): rgb channels, capped at 99 dB."""
    a, b = np.asarray(a, np.float64)[..., :3], np.asarray(b, np.float64)[..., :3]
    mse = np.mean((a - b) ** 2)
    return 99.0 if mse <= 0.0 else min(10.0 * np.log10(1.0 / mse), 99.0)


def fibonacci_dirs(n, offset=0.5):
    """Unit directions on a golden-angle lattice."""
    i = np.arange(n, dtype=np.float64) + offset
    z = 1.0 - 2.0 * i / n
    r = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def cameras(dirs, radius):
    from paper_2504_17954_b200 import Camera
    return [Camera.look_at(radius * d, np.zeros(3), 0.8, RES, RES) for d in dirs]


@pytest.fixture(scope="module")
def desk_pipeline(tmp_path_factory):
    from paper_2504_17954_b200 import LightConfig
    from paper_2504_17954_b200 import dvr
    from paper_2504_17954_b200.trainer import TrainConfig, ViewDataset, train_base, train_editable
    vol = dvr.make_shells_volume((64, 64, 64))
    tfs = [dvr.TransferFunction1D.basic_bump(0.35, 0.55, (0.2, 0.5, 0.9), 0.8),
           dvr.TransferFunction1D.basic_bump(0.60, 0.80, (0.9, 0.4, 0.15), 0.8)]
    assert dvr.transfer_functions_disjoint(tfs)
    light = LightConfig()
    lo, hi = vol.bbox
    radius = 1.1 * float(np.linalg.norm(np.asarray(hi) - np.asarray(lo)))
    train_cams = cameras(fibonacci_dirs(42), radius)
    held_cams = cameras(fibonacci_dirs(20, offset=0.25), radius)
    scenes = []
    for tf in tfs:
        imgs = [dvr.render_view(vol, tf, c, light) for c in train_cams]
        ds = ViewDataset(list(train_cams), imgs, light, {"volume": vol.descriptor(), "cameras": []})
        cfg = TrainConfig(stage1_iters=STAGE1, stage2_iters=STAGE2, seed=0)
        base, log1 = train_base(ds, cfg)
        editable, log2 = train_editable(base, ds, cfg)
        held_gt = [dvr.render_view(vol, tf, c, light) for c in held_cams]
        scenes.append({"tf": tf, "base": base, "editable": editable, "held_gt": held_gt,
                       "log": (log1, log2)})
    return {"volume": vol, "light": light, "held_cams": held_cams, "scenes": scenes,
            "dir": tmp_path_factory.mktemp("desk")}


def _held_out_psnrs(model, cams, gts, light=None):
    from paper_2504_17954_b200 import render_model
    return np.array([psnr(render_model(model, cam, light, dtype=np.float64), gt)
                     for cam, gt in zip(cams, gts)])


def test_end_to_end_training_matches_the_reference_quality(desk_pipeline):
    import json
    import os
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "desk_reference.json")))
    p = desk_pipeline
    for s, r in zip(p["scenes"], ref["scenes"]):
        base = _held_out_psnrs(s["base"], p["held_cams"], s["held_gt"])
        edit = _held_out_psnrs(s["editable"], p["held_cams"], s["held_gt"], p["light"])
        print(f"held-out PSNR base {base.mean():.2f} dB (reference {r['base_psnr']:.2f}), "
              f"editable {edit.mean():.2f} dB (reference {r['editable_psnr']:.2f}); "
              f"{len(s['base'])} / {len(s['editable'])} Gaussians "
              f"(reference {r['base_count']} / {r['editable_count']})")
        assert base.mean() >= 24.0 and edit.mean() >= 24.0
        assert base.mean() >= r["base_psnr"] - 0.5
        assert edit.mean() >= r["editable_psnr"] - 1.0  # run-to-run spread, see module doc


def test_composition_reaches_22db_against_volume_oracle(desk_pipeline):
    from paper_2504_17954_b200 import ComposedScene, dvr, render_composed
    p = desk_pipeline
    union = dvr.union_transfer_functions([s["tf"] for s in p["scenes"]])
    scene = ComposedScene.compose([s["editable"] for s in p["scenes"]], p["light"])
    vals = []
    for cam in p["held_cams"]:
        gt = dvr.render_view(p["volume"], union, cam, p["light"])
        out = render_composed(scene, cam, dtype=np.float64)
        vals.append(psnr(np.concatenate([out.color, out.alpha[..., None]], axis=-1), gt))
    assert np.mean(vals) >= 22.0


def test_compose_then_render_bit_equals_union_list_render(desk_pipeline):
    from paper_2504_17954_b200 import (ComposedScene, apply_edits, rasterize_forward,
                                       render_composed, shade_gaussians)
    p = desk_pipeline
    scene = ComposedScene.compose([s["editable"] for s in p["scenes"]], p["light"])
    cam = p["held_cams"][0]
    composed = render_composed(scene, cam, dtype=np.float64, sequential=True)
    eff = apply_edits(scene)
    rgb, _, _ = shade_gaussians(eff.geometry, eff.shading, eff.palette_rgb, p["light"], cam)
    union, _ = rasterize_forward(eff.geometry, rgb, cam, channels=("color", "alpha"),
                                 dtype=np.float64, sequential=True)
    assert np.array_equal(composed.color, union.color)
    assert np.array_equal(composed.alpha, union.alpha)


def test_vq_k256_psnr_drop(desk_pipeline):
    """PSNR gate of the reference's VQ acceptance test; its whole-file 3x
    ratio bar fails in the reference itself (positions and normals stay
    unquantized: ~2.15x, test_acceptance.py:283-288) and is reported here."""
    import os
    from paper_2504_17954_b200 import dequantize_model, quantize_model
    from paper_2504_17954_b200.ivrg import save_model
    p = desk_pipeline
    model = p["scenes"][0]["editable"]
    quant = quantize_model(model, k=256, seed=0)
    plain = _held_out_psnrs(model, p["held_cams"], p["scenes"][0]["held_gt"], p["light"])
    qpsnr = _held_out_psnrs(dequantize_model(quant), p["held_cams"], p["scenes"][0]["held_gt"],
                            p["light"])
    assert plain.mean() - qpsnr.mean() <= 0.5
    raw, q = str(p["dir"] / "raw.ivrg"), str(p["dir"] / "quant.ivrg")
    save_model(model, raw)
    save_model(quant, q)
    print(f"whole-file compression ratio {os.path.getsize(raw) / os.path.getsize(q):.2f}x")


def test_relighting_changes_terms_but_not_ambient(desk_pipeline):
    from paper_2504_17954_b200 import LightConfig, rasterize_forward, shade_gaussians
    p = desk_pipeline
    model = p["scenes"][0]["editable"]  # trained with a headlight
    cam = p["held_cams"][0]
    rotated = LightConfig("orbital", polar=np.pi / 4, azimuth=0.0)

    def term_maps(light):
        _, terms, _ = shade_gaussians(model.geometry, model.shading, model.palette, light, cam)
        out = {}
        for name in ("ambient", "diffuse", "specular"):
            m, _ = rasterize_forward(model.geometry, terms[name], cam, channels=("color",),
                                     dtype=np.float64)
            out[name] = m.color
        return out

    before, after = term_maps(p["light"]), term_maps(rotated)
    assert np.array_equal(before["ambient"], after["ambient"])
    assert not np.array_equal(before["diffuse"], after["diffuse"])
    assert not np.array_equal(before["specular"], after["specular"])
