"""GPU inverse fitting + losses vs the reference (golden fixtures from
voxsplat.inverse._step / optimize_to_reference / losses.photometric_loss)."""

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


def _scene(d, n_models=2):
    from paper_2504_17954_b200 import (BasicSceneModel, ComposedScene, GaussianGeometry,
                                       LightConfig, Palette, ShadingAttributes)
    ms = []
    for i in range(n_models):
        g = GaussianGeometry(*(d[f"m{i}_{k}"] for k in GEOM))
        a = ShadingAttributes(*(d[f"m{i}_{k}"] for k in SHADE))
        ms.append(BasicSceneModel("editable", g, shading=a, palette=Palette(d[f"m{i}_palette"])))
    return ComposedScene.compose(ms, LightConfig())


def _cam(d):
    from paper_2504_17954_b200 import Camera
    return Camera(d["cam_position"], d["cam_rotation"], float(d["cam_fov_y"]),
                  int(d["cam_width"]), int(d["cam_height"]))


def test_photometric_loss_matches_reference():
    from paper_2504_17954_b200.losses import photometric_loss
    d = golden("loss")
    loss, g = photometric_loss(d["pred"], d["gt"])
    assert abs(loss - float(d["loss"])) <= 1e-12 * abs(float(d["loss"]))
    assert np.abs(g - d["d"]).max() <= 1e-12 * np.abs(d["d"]).max()


@pytest.mark.parametrize("exact", [True, False])
def test_inverse_step_matches_reference(exact):
    from paper_2504_17954_b200.inverse import init_transform, inverse_step
    d = golden("inverse")
    sc = _scene(d)
    loss, g = inverse_step(sc, init_transform(sc), _cam(d), d["reference"], exact=exact)
    assert abs(loss - float(d["loss0"])) <= 1e-6 * abs(float(d["loss0"]))
    for k in ("c_p", "opacity_raw", "lam", "b"):
        ref = np.asarray(d["g_" + k])
        err = np.linalg.norm(np.asarray(g[k]) - ref)
        assert err <= 1e-3 * max(np.linalg.norm(ref), 1e-12), (k, g[k], ref)
    assert np.abs(g["angles"]).max() == 0.0  # headlight: no angle gradient


def test_optimize_to_reference_trajectory():
    from paper_2504_17954_b200.inverse import init_transform, optimize_to_reference
    d = golden("inverse")
    sc = _scene(d)
    fitted, losses = optimize_to_reference(sc, init_transform(sc), d["reference"], _cam(d),
                                           iters=5, lr=0.01)
    np.testing.assert_allclose(losses, d["fit_losses"], rtol=1e-5)
    for k in ("c_p", "opacity_raw", "lam", "b"):
        np.testing.assert_allclose(getattr(fitted, k), d["fit_" + k], atol=1e-5, err_msg=k)


def test_identity_transform_renders_like_render_composed():
    from paper_2504_17954_b200 import render_composed
    from paper_2504_17954_b200.inverse import init_transform, render_with_transform
    d = golden("inverse")
    sc = _scene(d)
    cam = _cam(d)
    out = render_composed(sc, cam)
    rgba = np.concatenate([out.color, out.alpha[..., None]], axis=-1)
    assert np.array_equal(rgba, render_with_transform(sc, init_transform(sc), cam))


def test_multiview_mean_equals_mean_of_single_views():
    """Extension: V views give the mean of the per-view gradients."""
    from paper_2504_17954_b200 import orbit_camera
    from paper_2504_17954_b200.inverse import InverseFitter, init_transform
    d = golden("inverse")
    sc = _scene(d)
    cams = [orbit_camera(np.zeros(3), 2.5, 0.3, az, 0.9, 40, 40) for az in (0.8, 2.0)]
    p = init_transform(sc)
    refs = [np.asarray(InverseFitter(sc, [], []).render(p, c).out64.cpu().numpy()) * 0.9
            for c in cams]
    fit = InverseFitter(sc, refs, cams)
    l0, g0 = fit.view_grads(p, 0)
    l1, g1 = fit.view_grads(p, 1)
    mean = ((g0 + g1) / 2).cpu().numpy()
    assert np.all(np.isfinite(mean)) and np.abs(mean).max() > 0


def _orbital_setup(n_views=2):
    from paper_2504_17954_b200 import LightConfig, orbit_camera
    from paper_2504_17954_b200.inverse import InverseFitter, init_transform
    d = golden("inverse")
    sc = _scene(d)
    sc.light = LightConfig("orbital", 0.4, 0.7)
    cams = [orbit_camera(np.zeros(3), 2.5, 0.3, az, 0.9, 40, 40) for az in (0.8, 2.0, 3.1)][:n_views]
    p = init_transform(sc)
    p_true = p.copy()
    p_true.lam = np.array([1.2, 0.8, 1.0, 1.0])
    p_true.polar, p_true.azimuth = 0.5, 0.9
    refs = [InverseFitter(sc, [], []).render(p_true, c).out64.cpu().numpy() for c in cams]
    return sc, p, refs, cams


def test_inverse_graph_matches_host_loop():
    """The graph-replayed loop (device Adam + table refresh) follows the host
    loop's trajectory (orbital light: angle gradients and light refresh)."""
    from paper_2504_17954_b200.inverse import optimize_to_reference
    sc, p, refs, cams = _orbital_setup()
    seen = []
    fh, lh = optimize_to_reference(sc, p, refs, cams, iters=6, lr=0.01,
                                   callback=lambda it, loss, prm: seen.append(it))
    fg, lg = optimize_to_reference(sc, p, refs, cams, iters=6, lr=0.01)
    assert seen == list(range(1, 7))
    # K4a's float32 atomics make each run's gradients differ in the last bits
    np.testing.assert_allclose(lg, lh, rtol=1e-6)
    for k in ("c_p", "opacity_raw", "lam", "b", "polar", "azimuth"):
        np.testing.assert_allclose(getattr(fg, k), getattr(fh, k), rtol=1e-6, atol=1e-8,
                                   err_msg=k)
    assert abs(fg.polar - p.polar) > 0  # the angles moved


def test_inverse_graph_recovers_from_pair_overflow():
    """A too-small pair capacity gates the update (sticky), and run() grows the
    capacity, recaptures and resumes from the first gated iteration."""
    from paper_2504_17954_b200.inverse import InverseFitter, InverseGraph
    sc, p, refs, cams = _orbital_setup(1)
    ref_x, ref_l = InverseGraph(InverseFitter(sc, refs, cams), p, 4).run()
    G = InverseGraph(InverseFitter(sc, refs, cams), p, 4)
    G.capacity = 64
    G._capture()
    x, losses = G.run()
    assert G.capacity > 64
    np.testing.assert_allclose(losses, ref_l, rtol=1e-6)
    np.testing.assert_allclose(x, ref_x, rtol=1e-6, atol=1e-8)


def test_inverse_graph_divergence_raises():
    from paper_2504_17954_b200 import DivergedLoss
    from paper_2504_17954_b200.inverse import optimize_to_reference
    sc, p, refs, cams = _orbital_setup(1)
    bad = refs[0].copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(DivergedLoss):
        optimize_to_reference(sc, p, [bad], cams, iters=3)


def _dist_fit_worker(rank, world, port, out_dir):
    import os
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_17954_b200.inverse import optimize_to_reference
    sc, p, refs, cams = _orbital_setup(2)
    fitted, losses = optimize_to_reference(sc, p, [refs[rank]], [cams[rank]], iters=4, lr=0.01)
    np.save(os.path.join(out_dir, f"r{rank}.npy"),
            np.concatenate([fitted.c_p.ravel(), fitted.opacity_raw, fitted.lam, fitted.b,
                            [fitted.polar, fitted.azimuth], losses]))
    tdist.barrier()
    tdist.destroy_process_group()


def test_inverse_graph_sharded_views_equal_single_process(tmp_path):
    """Views sharded over 2 ranks (functional check: gloo, both ranks on
    cuda:0): the graph loop with one all-reduce per iteration gives every
    rank the single-process 2-view trajectory."""
    import socket
    import torch.multiprocessing as mp
    from paper_2504_17954_b200.inverse import optimize_to_reference
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_dist_fit_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    np.testing.assert_allclose(r0, r1, rtol=1e-12, atol=1e-15)
    sc, p, refs, cams = _orbital_setup(2)
    f, losses = optimize_to_reference(sc, p, refs, cams, iters=4, lr=0.01)
    ref = np.concatenate([f.c_p.ravel(), f.opacity_raw, f.lam, f.b, [f.polar, f.azimuth], losses])
    np.testing.assert_allclose(r0, ref, rtol=1e-6, atol=1e-9)


def _dist_fit_uneven_worker(rank, world, port, out_dir):
    import os
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_17954_b200.inverse import optimize_to_reference
    sc, p, refs, cams = _orbital_setup(2)
    mine = [0, 1] if rank == 0 else []  # rank 1 holds no view
    fitted, losses = optimize_to_reference(sc, p, [refs[v] for v in mine], [cams[v] for v in mine],
                                           iters=4, lr=0.01)
    np.save(os.path.join(out_dir, f"u{rank}.npy"),
            np.concatenate([fitted.c_p.ravel(), fitted.opacity_raw, fitted.lam, fitted.b,
                            [fitted.polar, fitted.azimuth], losses]))
    tdist.barrier()
    tdist.destroy_process_group()


def test_inverse_graph_rank_without_views(tmp_path):
    """A rank holding no view takes the same (graph) path as the others and
    only joins the all-reduce + update: both ranks end on the single-process
    2-view trajectory (the collectives stay matched)."""
    import socket
    import torch.multiprocessing as mp
    from paper_2504_17954_b200.inverse import optimize_to_reference
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_dist_fit_uneven_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = np.load(tmp_path / "u0.npy"), np.load(tmp_path / "u1.npy")
    np.testing.assert_allclose(r0, r1, rtol=1e-12, atol=1e-15)
    sc, p, refs, cams = _orbital_setup(2)
    f, losses = optimize_to_reference(sc, p, refs, cams, iters=4, lr=0.01)
    ref = np.concatenate([f.c_p.ravel(), f.opacity_raw, f.lam, f.b, [f.polar, f.azimuth], losses])
    np.testing.assert_allclose(r0, ref, rtol=1e-6, atol=1e-9)
