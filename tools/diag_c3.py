"""C3 gradient diagnostics: per-tensor relative errors of the stage-2 step
at 300k vs the oracle, including K4a's per-Gaussian accumulators
(d_mean2d / d_conic / d_opacity / d_values) in atomic and deterministic mode."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2504_17954_b200 import LightConfig, device as D  # noqa: E402
from paper_2504_17954_b200.device import to_dev  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays  # noqa: E402
from paper_2504_17954_b200.trainer import EditableTrainer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
a = editable_arrays(0, n, density=n)
cam = bench_camera(800, 800, 1.1)
gt = np.random.default_rng(7).uniform(0.0, 1.0, (800, 800, 4))
ts = np.array([1.0, 1.1, 0.9, 1.0])
keys = ("mu", "q_raw", "log_s", "o_logit", "n_raw", "delta_c", "k_a_raw", "k_d_raw", "k_s_raw",
        "log_beta")
aux = {}
r_loss, r_g, r_stat = O.stage2_step({k: a[k] for k in keys}, a["palette"], ("orbital", 0.45, 0.9, ts),
                                    cam, gt, aux=aux)
rg = aux["raster"]
cap = {}
orig = D.blend_backward


def hook(F, d_out, **kw):
    g = orig(F, d_out, **kw)
    cap["g"] = g
    cap["d_out"] = d_out.detach().double().cpu().numpy()
    cap["out"] = F.out.double().cpu().numpy()
    return g


D.blend_backward = hook


def rel(x, y):
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


for det in ("0",):
    os.environ["IVR_DETERMINISTIC"] = det
    tr = EditableTrainer({k: a[k] for k in keys}, a["palette"], LightConfig("orbital", 0.45, 0.9, ts))
    tr.exact = os.environ.get("EXACT", "0") == "1"
    loss, grads, stat = tr.step(cam, to_dev(gt))
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy().astype(np.float64) for k, v in cap["g"].items()}
    print(f"deterministic={det} loss rel {abs(float(loss) - r_loss) / abs(r_loss):.3g}")
    print("  K4a d_mean2d", rel(g["mean2d"].reshape(n, 2), rg["d_mean2d"]),
          "d_conic", rel(g["conic"].reshape(n, 3), rg["d_conic"]),
          "d_opacity", rel(g["opacity"], rg["d_opacity"]),
          "d_values", rel(g["values"].reshape(n, -1), rg["d_values"]))
    st = aux["state"]
    lay = st["layout"]
    col = 0
    for name, w in lay:
        ref = np.asarray(aux["d_maps"].get(name, np.zeros((800, 800, w)))).reshape(800, 800, w)
        got = cap["d_out"][:, :, col:col + w]
        ro = st["out"][:, :, col:col + w]
        go = cap["out"][:, :, col:col + w]
        nd = int(np.sum(np.abs(got - ref) > 1e-3 * np.abs(ref).max()))
        print(f"  d_out[{name}] rel {rel(got, ref):.3g}  big diffs {nd}  "
              f"out maxdiff {np.abs(go - ro).max():.3g}")
        col += w
    for k in keys:
        print(f"  {k:9s} {rel(grads[k].cpu().numpy().reshape(r_g[k].shape), r_g[k]):.3g}")
    print("  stat", rel(stat.cpu().numpy(), r_stat))
