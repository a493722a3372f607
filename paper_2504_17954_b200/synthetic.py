"""Seeded synthetic editable-Gaussian scenes (host numpy).

``editable_arrays`` draws exactly the random stream of the reference test
fixture ``random_editable_model`` (pkg/tests/oracles.py:86-126: q, mu, log_s,
opacity, normal, then delta_c, k_a, k_d, k_s, log_beta, palette), so that a
seeded scene is identical to the reference's fixture.  ``density`` replaces the
fixture's log-scales with the density-matched scales of SURVEY.md 8(d):
``log_s = ln(0.55 * (1.728 / density)^(1/3)) + N(0, 0.3)`` per axis, drawn
after the fixture stream, which gives realistic footprints at 1M Gaussians.
"""

from __future__ import annotations

import numpy as np

GEOM_KEYS = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
SHADE_KEYS = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")


def editable_arrays(seed, n, spread=0.6, density=None, f32=False):
    """``seed`` is an int or a numpy Generator (drawn in place, like the
    reference fixtures that draw several models from one stream)."""
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    mu = rng.uniform(-spread, spread, size=(n, 3))
    log_s = rng.uniform(-2.2, -0.7, size=(n, 3))
    u = rng.uniform(0.15, 0.85, size=n)
    o_logit = np.log(u / (1 - u))
    n_raw = rng.normal(size=(n, 3))
    delta_c = rng.uniform(-0.2, 0.2, (n, 3))
    k_a = rng.normal(0.0, 1.0, n)
    k_d = rng.normal(0.0, 1.0, n)
    k_s = rng.normal(0.0, 1.0, n)
    log_beta = rng.uniform(0.5, 2.5, n)
    palette = rng.uniform(0.2, 0.8, 3)
    if density is not None:
        log_s = np.log(0.55 * (1.728 / float(density)) ** (1.0 / 3.0)) + rng.normal(0.0, 0.3, (n, 3))
    out = {"mu": mu, "q_raw": q, "log_s": log_s, "o_logit": o_logit, "n_raw": n_raw,
           "delta_c": delta_c, "k_a_raw": k_a, "k_d_raw": k_d, "k_s_raw": k_s,
           "log_beta": log_beta, "palette": palette}
    if f32:
        out = {k: v.astype(np.float32).astype(np.float64) for k, v in out.items()}
    return out


def editable_model(seed, n, spread=0.6, density=None, f32=False):
    """A BasicSceneModel (editable stage) built from ``editable_arrays``."""
    from .gaussians import GaussianGeometry
    from .scene import STAGE_EDITABLE, BasicSceneModel
    from .shading import Palette, ShadingAttributes

    a = editable_arrays(seed, n, spread, density, f32)
    geom = GaussianGeometry(*(a[k] for k in GEOM_KEYS))
    attrs = ShadingAttributes(*(a[k] for k in SHADE_KEYS))
    return BasicSceneModel(STAGE_EDITABLE, geom, shading=attrs, palette=Palette(a["palette"]),
                           metadata={"name": f"synthetic-{seed}"})


# C2 edit sequence applied per frame
C2_PALETTE_OVERRIDE = (0.2, 0.6, 0.9)


def c2_scene(per_model=200_000, n_models=5, density=1_000_000, light=True):
    """Composed C2 scene: ``n_models`` basic models (seeds 0..n-1) with the
    survey's edit sequence (palette override on scene 1, opacity 0.5 on scene
    2, orbital light (0.45, 0.9), term scales (1.2, 0.8, 1, 1))."""
    from .scene import ComposedScene, EditState
    from .shading import LightConfig

    models = [editable_model(s, per_model, density=density) for s in range(n_models)]
    lc = LightConfig("orbital", 0.45, 0.9, np.array([1.2, 0.8, 1.0, 1.0])) if light else LightConfig()
    scene = ComposedScene.compose(models, lc)
    if n_models > 1:
        scene.edits[1] = EditState(palette_override=np.array(C2_PALETTE_OVERRIDE))
    if n_models > 2:
        scene.edits[2] = EditState(opacity_scale=0.5)
    return scene


def bench_camera(width=800, height=800, azimuth=0.8):
    """orbit_camera(0, r=3, polar=0.3, azimuth, fov=pi/3)."""
    from .gaussians import orbit_camera
    return orbit_camera(np.zeros(3), 3.0, 0.3, azimuth, np.pi / 3, width, height)
