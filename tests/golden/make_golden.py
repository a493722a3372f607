"""Generate golden vectors from the REAL reference (voxsplat) for parity tests.

Run in the container that has the read-only reference mounted:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Writes small ``*.npz`` fixtures next to this script.  Nothing at test or bench
time reads /root/reference; the fixtures are the pin.  Every case below calls
the reference's own public functions (rasterize_forward / backward,
shade_gaussians / shade_backward, render_composed, inverse._step, vq.kmeans /
assign_nearest, losses.photometric_loss).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
for p in ("/root/reference/pkg/src", "/root/reference/pkg/tests"):
    if p not in sys.path:
        sys.path.insert(0, p)

from voxsplat import inverse as ref_inverse  # noqa: E402
from voxsplat.gaussians import GaussianGeometry, orbit_camera  # noqa: E402
from voxsplat.losses import photometric_loss  # noqa: E402
from voxsplat.rasterizer import rasterize_backward, rasterize_forward  # noqa: E402
from voxsplat.scene import ComposedScene, EditState, apply_edits, render_composed  # noqa: E402
from voxsplat.shading import LightConfig, Palette, ShadingAttributes, shade_backward, shade_gaussians  # noqa: E402
from voxsplat.vq import assign_nearest, kmeans  # noqa: E402
from voxsplat.scene import STAGE_EDITABLE, BasicSceneModel  # noqa: E402
from oracles import random_editable_model  # noqa: E402

from paper_2504_17954_b200.synthetic import editable_arrays, GEOM_KEYS, SHADE_KEYS  # noqa: E402


def model_from(a):
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    attrs = ShadingAttributes(*(a[k] for k in SHADE_KEYS))
    return BasicSceneModel(STAGE_EDITABLE, geom, shading=attrs, palette=Palette(a["palette"]))


def cam_dict(cam, prefix="cam_"):
    return {prefix + "position": cam.position, prefix + "rotation": cam.rotation,
            prefix + "fov_y": np.float64(cam.fov_y), prefix + "width": np.int64(cam.width),
            prefix + "height": np.int64(cam.height), prefix + "focal": np.float64(cam.focal)}


def check_generator():
    """Our seeded generator reproduces the reference fixture bit-for-bit."""
    for seed, n in ((0, 50), (3, 7)):
        ref = random_editable_model(np.random.default_rng(seed), n)
        ours = editable_arrays(seed, n)
        for k in GEOM_KEYS:
            assert np.array_equal(getattr(ref.geometry, k), ours[k]), k
        for k in SHADE_KEYS:
            assert np.array_equal(getattr(ref.shading, k), ours[k]), k
        assert np.array_equal(ref.palette.c_p, ours["palette"])


def render_case(name, seed, n, W, H, density=None, light=None, azimuth=0.8, dtype=np.float32):
    a = editable_arrays(seed, n, density=density)
    m = model_from(a)
    cam = orbit_camera(np.zeros(3), 3.0, 0.3, azimuth, np.pi / 3, W, H)
    light = light or LightConfig()
    scene = ComposedScene.compose([m], light)
    rgb, _, _ = shade_gaussians(m.geometry, m.shading, m.palette, light, cam)
    out, st = rasterize_forward(m.geometry, rgb, cam, dtype=dtype)
    comp = render_composed(scene, cam, dtype=dtype)
    assert np.array_equal(comp.color, out.color)
    proj = st["proj"]
    d = dict(a)
    d.update(cam_dict(cam))
    d.update(light_mode=np.array(light.mode), light_polar=np.float64(light.polar),
             light_azimuth=np.float64(light.azimuth), light_ts=light.term_scales,
             rgb=rgb, depth=proj["depth"], mean2d=proj["mean2d"], conic=proj["conic"],
             cov2d=proj["cov2d"], valid=proj["valid"],
             pair_splat=st["pair_splat"].astype(np.int32),
             tile_ranges=st["tile_ranges"].astype(np.int32),
             kmean2d=st["kmean2d"], kconic=st["kconic"], kopacity=st["kopacity"],
             values=st["values"], color=out.color, alpha=out.alpha,
             contrib=out.per_pixel_contrib_count,
             last_pos=st["last_pos"].astype(np.int32), t_final=st["t_final"])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
    print(name, "N", n, "P", st["pair_splat"].size, "img", (H, W))


def composed_case():
    parts = [editable_arrays(s, 1500) for s in (1, 2, 3)]
    models = [model_from(a) for a in parts]
    light = LightConfig("orbital", 0.45, 0.9, np.array([1.2, 0.8, 1.0, 1.0]))
    scene = ComposedScene.compose(models, light)
    scene.edits[1] = EditState(palette_override=np.array([0.2, 0.6, 0.9]))
    scene.edits[2] = EditState(opacity_scale=0.5)
    cam = orbit_camera(np.zeros(3), 3.0, 0.3, 0.8, np.pi / 3, 96, 80)
    eff = apply_edits(scene)
    rgb, _, _ = shade_gaussians(eff.geometry, eff.shading, eff.palette_rgb, eff.light, cam)
    o32 = render_composed(scene, cam, dtype=np.float32)
    o64 = render_composed(scene, cam, dtype=np.float64)
    d = {}
    for i, a in enumerate(parts):
        for k, v in a.items():
            d[f"m{i}_{k}"] = v
    d.update(cam_dict(cam))
    d.update(eff_o_logit=eff.geometry.o_logit, rgb=rgb, color32=o32.color, alpha32=o32.alpha,
             contrib32=o32.per_pixel_contrib_count, color64=o64.color, alpha64=o64.alpha,
             contrib64=o64.per_pixel_contrib_count)
    np.savez_compressed(os.path.join(HERE, "composed_edit.npz"), **d)
    print("composed_edit", eff.geometry.mu.shape[0])


def backward_case():
    a = editable_arrays(11, 40, spread=0.5)
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    rng = np.random.default_rng(5)
    colors = rng.uniform(0.1, 0.9, (40, 3))
    attrs = {"ka": rng.uniform(0.1, 0.9, 40)}
    cam = orbit_camera(np.zeros(3), 2.5, 0.3, 0.8, 0.9, 24, 24)
    w = {"color": rng.normal(size=(24, 24, 3)), "alpha": rng.normal(size=(24, 24)),
         "depth": rng.normal(size=(24, 24)) * 0.1, "normal": rng.normal(size=(24, 24, 3)),
         "ka": rng.normal(size=(24, 24))}
    out, st = rasterize_forward(geom, colors, cam, channels=("color", "alpha", "depth", "normal"),
                                attrs=attrs, dtype=np.float64)
    g = rasterize_backward(st, w)
    d = dict(a)
    d.update(cam_dict(cam))
    d.update(colors=colors, attr_ka=attrs["ka"], **{"w_" + k: v for k, v in w.items()})
    for k in ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors", "d_mean2d"):
        d[k] = g[k]
    d["d_attr_ka"] = g["d_attrs"]["ka"]
    d["color"], d["alpha"], d["depth_map"], d["normal_map"] = out.color, out.alpha, out.depth, out.normal
    d["attr_map"] = out.attr["ka"]
    np.savez_compressed(os.path.join(HERE, "backward_small.npz"), **d)
    print("backward_small")


def shade_case():
    a = editable_arrays(21, 500)
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    attrs = ShadingAttributes(*(a[k] for k in SHADE_KEYS))
    cam = orbit_camera(np.zeros(3), 3.0, 0.3, 0.8, np.pi / 3, 64, 64)
    rng = np.random.default_rng(7)
    d_rgb = rng.normal(size=(500, 3))
    pal = rng.uniform(0.1, 0.9, (500, 3))
    d = dict(a)
    d.update(cam_dict(cam), d_rgb=d_rgb, palette_ps=pal)
    lam, b = np.array([1.2, 0.8, 1.1, 0.9]), np.array([0.01, -0.02, 0.03, 0.2])
    for tag, light, ct, palette in (
            ("head", LightConfig(), None, Palette(a["palette"])),
            ("orb", LightConfig("orbital", 0.45, 0.9, np.array([1.2, 0.8, 1.0, 1.1])), (lam, b), pal)):
        rgb, terms, cache = shade_gaussians(geom, attrs, palette, light, cam, coeff_transform=ct)
        g = shade_backward(cache, d_rgb)
        d[tag + "_rgb"] = rgb
        for k, v in g.items():
            d[tag + "_" + k] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "shade.npz"), **d)
    print("shade")


def vq_case():
    rng = np.random.default_rng(3)
    samples = np.concatenate([rng.normal(size=1500), rng.normal(3.0, 0.2, 500)])
    cents = kmeans(samples, 16, seed=1)
    c4096 = np.sort(rng.normal(size=4096) * 2.0)
    vals = rng.normal(size=50000) * 2.5
    mids = 0.5 * (c4096[1:] + c4096[:-1])
    vals[:64] = mids[rng.integers(0, mids.size, 64)]  # exact ties -> lower index
    vals[64] = np.nan
    vals[65], vals[66] = -1e300, 1e300
    idx = assign_nearest(vals, c4096)
    np.savez_compressed(os.path.join(HERE, "vq.npz"), samples=samples, kmeans16=cents,
                        centroids=c4096, values=vals, indices=idx.astype(np.int32))
    print("vq")


def loss_case():
    rng = np.random.default_rng(4)
    pred = rng.uniform(0, 1, (32, 40, 4))
    gt = rng.uniform(0, 1, (32, 40, 4))
    loss, d = photometric_loss(pred, gt)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), pred=pred, gt=gt, loss=np.float64(loss), d=d)
    print("loss")


def inverse_case():
    parts = [editable_arrays(s, 60, spread=0.5) for s in (31, 32)]
    scene = ComposedScene.compose([model_from(a) for a in parts], LightConfig())
    cam = orbit_camera(np.zeros(3), 2.5, 0.3, 0.8, 0.9, 40, 40)
    gt = scene.copy()
    gt.edits[0] = EditState(palette_override=np.array([0.2, 0.6, 0.9]))
    gt.edits[1] = EditState(opacity_scale=0.5)
    gp = ref_inverse.init_transform(gt)
    gp.lam = np.array([1.2, 0.8, 1.0, 1.0])
    ref = ref_inverse.render_with_transform(gt, gp, cam, dtype=np.float64)
    p0 = ref_inverse.init_transform(scene)
    loss, grads = ref_inverse._step(ref_inverse._frozen_parts(scene), scene.light, p0, cam, ref)
    fitted, losses = ref_inverse.optimize_to_reference(scene, p0, ref, cam, iters=5, lr=0.01)
    d = {}
    for i, a in enumerate(parts):
        for k, v in a.items():
            d[f"m{i}_{k}"] = v
    d.update(cam_dict(cam), reference=ref, loss0=np.float64(loss),
             fit_losses=np.array(losses), fit_c_p=fitted.c_p, fit_opacity_raw=fitted.opacity_raw,
             fit_lam=fitted.lam, fit_b=fitted.b)
    for k, v in grads.items():
        d["g_" + k] = v
    np.savez_compressed(os.path.join(HERE, "inverse.npz"), **d)
    print("inverse")


def stage2_case():
    """One trainer._stage2_step (trainer.py:397-444) with all regularizers."""
    from voxsplat import trainer as ref_trainer
    from voxsplat.losses import LossWeights
    a = editable_arrays(41, 300, spread=0.5)
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    attrs = ShadingAttributes(*(a[k] for k in SHADE_KEYS))
    cam = orbit_camera(np.zeros(3), 2.5, 0.3, 0.8, 0.9, 40, 32)
    rng = np.random.default_rng(8)
    gt = rng.uniform(0, 1, (32, 40, 4))
    light = LightConfig("orbital", 0.3, -0.7, np.array([1.0, 1.1, 0.9, 1.0]))
    loss, grads, stat = ref_trainer._stage2_step(geom, attrs, Palette(a["palette"]), light, cam, gt,
                                                 LossWeights())
    d = dict(a)
    d.update(cam_dict(cam), gt=gt, loss=np.float64(loss), stat=stat)
    for k, v in grads.items():
        d["g_" + k] = v
    np.savez_compressed(os.path.join(HERE, "stage2.npz"), **d)
    print("stage2", loss)


def sh_case():
    """view_dirs + eval_sh / eval_sh_backward + view_dirs_backward
    (gaussians.py:497-529) for degrees 0..3, including clamped channels."""
    from voxsplat.gaussians import ShColor, eval_sh, eval_sh_backward, view_dirs, view_dirs_backward
    rng = np.random.default_rng(12)
    d = {}
    n = 400
    mu = rng.uniform(-1, 1, (n, 3))
    pos = np.array([0.3, -2.2, 1.1])
    d["mu"], d["pos"] = mu, pos
    for deg in range(4):
        coeffs = rng.normal(0, 0.6, (n, (deg + 1) ** 2, 3))
        dirs = view_dirs(mu, pos)
        rgb, cache = eval_sh(ShColor(coeffs, deg), dirs)
        d_rgb = rng.normal(size=(n, 3))
        d_c, d_dir = eval_sh_backward(cache, d_rgb)
        d_mu = view_dirs_backward(mu, pos, d_dir)
        d.update({f"coeffs{deg}": coeffs, f"rgb{deg}": rgb, f"drgb{deg}": d_rgb,
                  f"dcoeffs{deg}": d_c, f"dmu{deg}": d_mu})
    np.savez_compressed(os.path.join(HERE, "sh.npz"), **d)
    print("sh")


def stage1_case():
    """One trainer._stage1_step (trainer.py:375-394): SH colour, colour/alpha/
    depth/normal channels, L1+SSIM + normal consistency."""
    from voxsplat import trainer as ref_trainer
    from voxsplat.gaussians import ShColor
    from voxsplat.losses import LossWeights
    a = editable_arrays(43, 300, spread=0.5)
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    rng = np.random.default_rng(9)
    sh = ShColor(rng.normal(0, 0.5, (300, 9, 3)), 2)
    cam = orbit_camera(np.zeros(3), 2.5, 0.35, -0.6, 0.9, 40, 32)
    gt = rng.uniform(0, 1, (32, 40, 4))
    loss, grads, stat = ref_trainer._stage1_step(geom, sh, cam, gt, LossWeights())
    d = {k: a[k] for k in GEOM_KEYS}
    d.update(cam_dict(cam), sh=sh.coefficients, gt=gt, loss=np.float64(loss), stat=stat)
    for k, v in grads.items():
        d["g_" + k] = v
    np.savez_compressed(os.path.join(HERE, "stage1.npz"), **d)
    print("stage1", loss)


def ivrg_case():
    """IVRG files written by the reference save_model (scene.py:286-329) plus
    the arrays its load_model returns (scene.py:349-436)."""
    from voxsplat.gaussians import ShColor
    from voxsplat.scene import STAGE_BASE, load_model, save_model
    from voxsplat.vq import quantize_model
    out_dir = os.path.join(HERE, "ivrg")
    os.makedirs(out_dir, exist_ok=True)
    ed = model_from(editable_arrays(50, 300))
    ed.metadata = {"name": "editable", "seed": 50}
    a = editable_arrays(51, 200)
    sh = ShColor(np.random.default_rng(51).normal(0, 0.5, (200, 9, 3)), 2)
    base = BasicSceneModel(STAGE_BASE, GaussianGeometry(*(a[k] for k in GEOM_KEYS)), sh=sh,
                           metadata={"stage1_iters": 7})
    quant = quantize_model(model_from(editable_arrays(52, 400)), k=16, seed=3)
    quant_wide = quantize_model(model_from(editable_arrays(53, 600)), k=300, seed=4)
    comp = ComposedScene.compose([model_from(editable_arrays(54 + i, 150 + 50 * i)) for i in range(3)],
                                 LightConfig("orbital", 0.4, -1.1, np.array([1.1, 0.9, 1.0, 1.2])))
    comp.edits[1] = EditState(np.array([0.1, 0.7, 0.3]), 0.5)
    comp.edits[2] = EditState(None, 1.5)
    comp.transform = {"c_p": [[0.2, 0.6, 0.9]], "note": "fit"}
    for name, obj in (("editable", ed), ("base", base), ("quantized", quant),
                      ("quantized_wide", quant_wide), ("composed", comp)):
        path = os.path.join(out_dir, name + ".ivrg")
        save_model(obj, path)
        back = load_model(path)
        models = back.models if isinstance(back, ComposedScene) else [back]
        d = {}
        for i, m in enumerate(models):
            for k in GEOM_KEYS:
                d[f"m{i}_{k}"] = getattr(m.geometry, k)
            if m.sh is not None:
                d[f"m{i}_sh"] = m.sh.coefficients
            if m.shading is not None:
                for k in SHADE_KEYS:
                    d[f"m{i}_{k}"] = getattr(m.shading, k)
            if m.palette is not None:
                d[f"m{i}_palette"] = m.palette.c_p
            if m.quantized is not None:
                for k, (cb, idx) in m.quantized.items():
                    d[f"m{i}_cb_{k}"] = cb.centroids
                    d[f"m{i}_idx_{k}"] = idx
        np.savez_compressed(os.path.join(out_dir, name + ".npz"), **d)
    print("ivrg")


def display_case():
    """render_modes.render_mode_image for every mode on a composed scene with
    edits (render_modes.py:31-72) and a base-stage model."""
    from voxsplat.gaussians import ShColor
    from voxsplat.render_modes import RENDER_MODES, render_mode_image, to_uint8
    from voxsplat.scene import STAGE_BASE
    sc = ComposedScene.compose([model_from(editable_arrays(70 + i, 1500, spread=0.5, density=3000))
                                for i in range(2)],
                               LightConfig("orbital", 0.3, 0.7, np.array([1.1, 0.9, 1.0, 1.2])))
    sc.edits[1] = EditState(np.array([0.2, 0.7, 0.4]), 0.6)
    cam = orbit_camera(np.zeros(3), 2.4, 0.35, 0.5, 0.9, 40, 32)
    d = cam_dict(cam)
    for mode in RENDER_MODES:
        img = render_mode_image(sc, cam, mode)
        d["img_" + mode] = img
        d["u8_" + mode] = to_uint8(img)
    a = editable_arrays(75, 1200, spread=0.5, density=3000)
    sh = ShColor(np.random.default_rng(75).normal(0, 0.4, (1200, 4, 3)), 1)
    base = BasicSceneModel(STAGE_BASE, GaussianGeometry(*(a[k] for k in GEOM_KEYS)), sh=sh)
    for mode in ("shaded", "alpha", "normal", "depth"):
        d["base_" + mode] = render_mode_image(base, cam, mode)
    np.savez_compressed(os.path.join(HERE, "display.npz"), **d)
    print("display")


def dvr_case():
    """dvr.render_view (dvr.py:424-452) for the three synthetic volumes,
    headlight and orbital light, a union of two transfer-function bumps."""
    from voxsplat.dvr import Material, TransferFunction1D, make_volume, render_view, union_transfer_functions
    tf = union_transfer_functions([TransferFunction1D.basic_bump(0.2, 0.45, (0.9, 0.3, 0.2), 0.8),
                                   TransferFunction1D.basic_bump(0.55, 0.8, (0.2, 0.5, 0.9), 0.6)])
    d = {}
    cam = orbit_camera(np.zeros(3), 3.0 * 16.0, 0.4, 0.7, 0.8, 24, 20)
    for kind in ("shells", "lobes", "swirl"):
        vol = make_volume(kind, (24, 20, 28))
        d[kind + "_head"] = render_view(vol, tf, cam, LightConfig())
        d[kind + "_orb"] = render_view(vol, tf, cam, LightConfig("orbital", 0.3, -0.8),
                                       Material(0.3, 0.5, 0.4, 8.0), step_scale=0.35)
    d.update(cam_dict(cam))
    np.savez_compressed(os.path.join(HERE, "dvr.npz"), **d)
    print("dvr")


def densify_case():
    """trainer.densify_and_prune (trainer.py:241-261 -> _densify_params
    :135-193): clone small / split large over-threshold primitives (offsets
    from the numpy stream), budget cap, opacity prune; plus the all-pruned
    round (empty model) and a stage-1 (SH) model."""
    from voxsplat import trainer as ref_trainer
    from voxsplat.gaussians import ShColor
    d = {}
    a = editable_arrays(51, 400, spread=0.5)
    a["o_logit"][::7] = -9.0  # below the prune threshold
    rng = np.random.default_rng(13)
    stats = rng.uniform(0.0, 4e-4, 400)
    m = model_from(a)
    cases = {"edit": (m, ref_trainer.TrainConfig(max_primitives=500, seed=3), 30.0),
             "nobudget": (m, ref_trainer.TrainConfig(max_primitives=400, seed=4), 0.8)}
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    sh = ShColor(rng.normal(0, 0.5, (400, 4, 3)), 1)
    cases["base"] = (BasicSceneModel("base", geom, sh=sh), ref_trainer.TrainConfig(seed=5), 40.0)
    for tag, (model, cfg, extent) in cases.items():
        new, info = ref_trainer.densify_and_prune(model, stats, cfg, extent=extent,
                                                  rng=np.random.default_rng(cfg.seed))
        for k in GEOM_KEYS:
            d[f"{tag}_{k}"] = getattr(new.geometry, k)
        if new.shading is not None:
            for k in SHADE_KEYS:
                d[f"{tag}_{k}"] = getattr(new.shading, k)
        if new.sh is not None:
            d[f"{tag}_sh"] = new.sh.coefficients
        for k, v in info.items():
            d[f"{tag}_info_{k}"] = np.int64(v)
    b = dict(a)
    b["o_logit"] = np.full(400, -9.0)
    new, info = ref_trainer.densify_and_prune(model_from(b), stats, ref_trainer.TrainConfig(),
                                              extent=0.8, rng=np.random.default_rng(0))
    d["empty_count"] = np.int64(len(new.geometry.mu))
    for k, v in info.items():
        d[f"empty_info_{k}"] = np.int64(v)
    d.update({k: a[k] for k in a}, stats=stats, sh=sh.coefficients)
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **d)
    print("densify", {k: int(v) for k, v in d.items() if "_info_" in k})


if __name__ == "__main__":
    import sys as _sys
    if len(_sys.argv) > 1:  # regenerate selected cases only
        for name in _sys.argv[1:]:
            globals()[name]()
        _sys.exit(0)
    check_generator()
    # C1 (bench config 0): 10k density-scaled, 128^2
    render_case("render_c1", 0, 10_000, 128, 128, density=10_000)
    # unmodified fixture scales: large overlapping splats, early termination
    render_case("render_fixture", 1, 2000, 64, 64)
    # non-multiple-of-16 frame, orbital light with term scales
    render_case("render_ragged", 2, 3000, 72, 50, density=3000,
                light=LightConfig("orbital", -0.3, 2.0, np.array([0.9, 1.3, 1.0, 0.7])), azimuth=-2.1)
    composed_case()
    backward_case()
    shade_case()
    vq_case()
    loss_case()
    inverse_case()
    stage2_case()
    sh_case()
    stage1_case()
    ivrg_case()
    display_case()
    dvr_case()
    densify_case()
