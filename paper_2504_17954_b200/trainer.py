"""Two-stage training on the GPU (trainer.py:375-626 semantics).

Stage 1 (base, ``train_base``): SH colour (csrc/sh.cu) -> K1 (K=8 channels:
colour, alpha, depth, normal) -> K2 -> K3 -> L1+SSIM + normal consistency ->
K4a -> K4b -> SH / view-direction backward (_stage1_step, trainer.py:375-394).

Stage 2 (editable, ``train_editable``): K1 with fused shading (K=15 channels:
colour, alpha, depth, normal, Δc, k_a, k_d, k_s, β) -> K2 -> K3 -> L1+SSIM and
the four regularizers in torch (losses.py) -> K4a -> K4b (projection +
shading backward fused) -> the attribute chain rules of _stage2_step
(trainer.py:433-442).

Both stages: all parameters, Adam moments and the per-step work stay on the
device; Adam with the reference's learning-rate schedules and periodic
densify / prune (torch) run in the shared loop ``_run_stage``
(trainer.py:463-526).

One training view per iteration (reference semantics, trainer.py:485).  Runs
for independent basic transfer functions shard one per GPU with no
communication.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import DatasetEmpty, DivergedLoss, OutOfRange, ShapeMismatch
from .gaussians import GaussianGeometry, ShColor
from .losses import SSIM_RADIUS, LossWeights, _photometric_frame_dev, regularize_t
from .rasterizer import _channel_layout, _cols
from .scene import STAGE_BASE, STAGE_EDITABLE, BasicSceneModel, DeviceScene
from .shading import LightConfig, Palette, ShadingAttributes

PSNR_CAP = 99.0


@dataclass
class TrainConfig:
    """Hyper-parameters (trainer.py:46-94)."""

    stage1_iters: int = 30000
    stage2_iters: int = 10000
    adam_eps: float = 1e-15
    adam_betas: tuple = (0.9, 0.999)
    lr_mu: float = 1.6e-4
    lr_mu_final: float = 1.6e-6
    lr_q: float = 1e-3
    lr_log_s: float = 5e-3
    lr_o: float = 0.05
    lr_sh: float = 2.5e-3
    lr_normal: float = 0.01
    lr_shading: float = 0.01
    lr_decay_floor: float = 0.1
    densify_interval: int = 100
    densify_start_iter: int = 500
    densify_until_iter: int = None
    densify_grad_threshold: float = 2e-4
    prune_opacity_threshold: float = 0.005
    max_primitives: int = 120000
    init_count: int = 5000
    init_opacity: float = 0.1
    sh_degree: int = 2
    silhouette_carve: bool = False
    seed: int = 0
    log_interval: int = 50
    weights: LossWeights = field(default_factory=LossWeights)

    def __post_init__(self):
        if self.stage1_iters < 0 or self.stage2_iters < 0:
            raise OutOfRange("iteration counts must be >= 0")
        for name in ("densify_grad_threshold", "prune_opacity_threshold", "densify_interval",
                     "init_count", "max_primitives"):
            if getattr(self, name) <= 0:
                raise OutOfRange(f"{name} must be > 0")

    def until_iter(self, stage_iters):
        return self.densify_until_iter if self.densify_until_iter is not None else stage_iters // 2


class Adam:
    """trainer.Adam (trainer.py:100-128): per-parameter Adam on host float64
    arrays (in place), moments surviving densification.  The training loops
    use DeviceAdam / the captured Adam kernel; this is the reference's host
    optimizer object (also driving the small transform vector of the
    multi-rank inverse host loop)."""

    def __init__(self, eps=1e-15, betas=(0.9, 0.999)):
        self.eps = eps
        self.b1, self.b2 = betas
        self.state = {}

    def step(self, name, param, grad, lr):
        st = self.state.setdefault(name, {"m": np.zeros_like(param), "v": np.zeros_like(param),
                                          "t": 0})
        st["t"] += 1
        st["m"] = self.b1 * st["m"] + (1.0 - self.b1) * grad
        st["v"] = self.b2 * st["v"] + (1.0 - self.b2) * grad * grad
        mhat = st["m"] / (1.0 - self.b1 ** st["t"])
        vhat = st["v"] / (1.0 - self.b2 ** st["t"])
        param -= lr * mhat / (np.sqrt(vhat) + self.eps)
        return param

    def remap(self, parents, is_new):
        for st in self.state.values():
            for key in ("m", "v"):
                arr = st[key][parents].copy()
                arr[is_new] = 0.0
                st[key] = arr


class DeviceAdam:
    """trainer.Adam on device tensors (one fused launch for all parameter
    groups, csrc/adam.cu); moments survive densification (remap)."""

    def __init__(self, eps=1e-15, betas=(0.9, 0.999)):
        self.eps, (self.b1, self.b2), self.state = eps, betas, {}

    def step(self, name, param, grad, lr):
        self.step_all([(name, param, grad, lr)])

    @torch.no_grad()
    def step_all(self, items):
        """Update every (name, param, grad, lr) of one training step."""
        arr = (L.AdamGroup_t * len(items))()
        keep = []
        for k, (name, param, grad, lr) in enumerate(items):
            st = self.state.get(name)
            if st is None:
                st = self.state[name] = {"m": torch.zeros_like(param), "v": torch.zeros_like(param),
                                         "t": 0}
            st["t"] += 1
            t = st["t"]
            g = grad.to(torch.float64).contiguous()
            keep.append(g)
            if not param.is_contiguous():
                raise ValueError(f"parameter {name} must be contiguous")
            a = arr[k]
            a.param, a.m, a.v, a.grad = (param.data_ptr(), st["m"].data_ptr(), st["v"].data_ptr(),
                                         g.data_ptr())
            a.n = param.numel()
            a.lr = float(lr)
            a.bc1 = 1.0 - self.b1 ** t
            a.bc2 = 1.0 - self.b2 ** t
        L.check(L.lib().ivr_adam_step(arr, len(items), self.b1, self.b2, self.eps,
                                      D.stream_handle()), "ivr_adam_step")
        del keep

    def groups(self, items):
        """ivr_adam_group array for (name, param, grad) items (state created
        on first use); the pointers stay valid while the tensors live."""
        arr = (L.AdamGroup_t * len(items))()
        for k, (name, param, grad) in enumerate(items):
            st = self.state.get(name)
            if st is None:
                st = self.state[name] = {"m": torch.zeros_like(param), "v": torch.zeros_like(param),
                                         "t": 0}
            if not (param.is_contiguous() and grad.is_contiguous() and grad.dtype == torch.float64):
                raise ValueError(f"parameter {name}: contiguous float64 param and gradient required")
            a = arr[k]
            a.param, a.m, a.v, a.grad = (param.data_ptr(), st["m"].data_ptr(), st["v"].data_ptr(),
                                         grad.data_ptr())
            a.n = param.numel()
        return arr

    def ensure(self, named_params):
        for name, param in named_params:
            if name not in self.state:
                self.state[name] = {"m": torch.zeros_like(param), "v": torch.zeros_like(param),
                                    "t": 0}

    def schedule(self, names_lrs):
        """Advance each group's step count; returns [lr, bc1, bc2] per group."""
        out = []
        for name, lr in names_lrs:
            st = self.state[name]
            st["t"] += 1
            out += [float(lr), 1.0 - self.b1 ** st["t"], 1.0 - self.b2 ** st["t"]]
        return out

    def remap(self, parents, is_new):
        for st in self.state.values():
            for key in ("m", "v"):
                arr = st[key][parents].clone()
                arr[is_new] = 0.0
                st[key] = arr


_LR = {"mu": "lr_mu", "q_raw": "lr_q", "log_s": "lr_log_s", "o_logit": "lr_o", "n_raw": "lr_normal",
       "sh": "lr_sh",
       "delta_c": "lr_shading", "k_a_raw": "lr_shading", "k_d_raw": "lr_shading",
       "k_s_raw": "lr_shading", "log_beta": "lr_shading"}
GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
SHADE = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")
ATTR_NAMES = ("delta_c", "k_a", "k_d", "k_s", "beta")


def _psnr_t(a, b):
    mse = float(((a[..., :3] - b[..., :3]) ** 2).mean())
    return PSNR_CAP if mse <= 0.0 else min(10.0 * math.log10(1.0 / mse), PSNR_CAP)


class _StageTrainer:
    """Device state of one training stage: row-aligned float64 parameter
    tensors, Adam moments, the render workspace (the reference's ``params``
    dict + Adam of _run_stage, trainer.py:463-474)."""

    KEYS = GEOM

    def __init__(self, params, cfg=None, device=None):
        self.dev = device or D.cuda_device()
        self.p = {k: D.to_dev(params[k], device=self.dev) for k in self.KEYS}
        self.cfg = cfg or TrainConfig()
        self.adam = DeviceAdam(self.cfg.adam_eps, self.cfg.adam_betas)
        self.ws = D.Workspace(self.dev)
        self._bad = None
        self._first_bad = None
        # blend mode of the training forward: FAST (certified float32, the
        # default) or EXACT (the reference's float64 arithmetic, bit-faithful
        # maps: the loss terms built on sign() / normalisation then see the
        # reference's exact inputs)
        self.exact = False

    @property
    def n(self):
        return int(self.p["mu"].shape[0])

    def lr(self, name, it, iters, decay_extra=()):
        """The reference's per-group learning-rate schedule (trainer.py:491-499)."""
        cfg = self.cfg
        frac = it / max(iters, 1)
        lr = getattr(cfg, _LR[name])
        if name == "mu" and cfg.lr_mu > 0.0:
            lr = cfg.lr_mu * (cfg.lr_mu_final / cfg.lr_mu) ** frac
        elif _LR[name] in ("lr_shading", "lr_normal") or name in decay_extra:
            lr = lr * cfg.lr_decay_floor ** frac
        return lr

    def step_views(self, cams, gts, weights=None):
        """Batch-of-views step (BASELINE configs[2]; an extension of the
        reference's one view per iteration, SURVEY.md finding 6): the mean
        over the views of the per-view loss and gradients of ``step`` (the
        per-view densify statistics are summed), to be applied with one
        ``apply``.  Its parity is the mean of the reference's per-view step
        gradients; with one view it is ``step``."""
        cams, gts = list(cams), list(gts)
        if not cams or len(cams) != len(gts):
            raise ValueError("step_views: need one ground-truth image per camera")
        loss_acc = grads_acc = stat_acc = None
        for cam, gt in zip(cams, gts):
            loss, grads, stat = self.step(cam, gt, weights)
            if grads_acc is None:  # step reuses its buffers: keep copies
                loss_acc = loss.clone()
                grads_acc = {k: g.clone() for k, g in grads.items()}
                stat_acc = stat.clone()
            else:
                loss_acc += loss
                for k, g in grads.items():
                    grads_acc[k] += g
                stat_acc += stat
        inv = 1.0 / len(cams)
        for g in grads_acc.values():
            g.mul_(inv)
        return loss_acc * inv, grads_acc, stat_acc

    def apply(self, grads, it, iters, decay_extra=()):
        """Adam on every group with the reference schedules (trainer.py:491-499)."""
        items = [(name, self.p[name], grad, self.lr(name, it, iters, decay_extra))
                 for name, grad in grads.items()]
        self.adam.step_all(items)

    @torch.no_grad()
    def densify(self, mean_stat, extent, rng, keep_if_empty=True):
        """_densify_params (trainer.py:135-193) on the device.  The split
        offsets are drawn on the host from the reference's numpy stream
        (``rng.standard_normal((2*ns, 3))``, trainer.py:176), the same
        Generator that picks each iteration's view, and uploaded, so a seeded
        run follows the reference's view sequence through every split.
        keep_if_empty: when every row would be pruned, keep the current
        parameters (the reference's _run_stage guard, trainer.py:510-513);
        otherwise apply (densify_and_prune returns the empty model)."""
        cfg, p = self.cfg, self.p
        n = self.n
        over = mean_stat >= cfg.densify_grad_threshold
        budget = cfg.max_primitives - n
        if budget <= 0:
            over[:] = False
        else:
            cand = torch.nonzero(over).flatten()
            if cand.numel() > budget:
                order = torch.argsort(-mean_stat[cand], stable=True)
                over = torch.zeros_like(over)
                over[cand[order[:budget]]] = True
        scales = torch.exp(p["log_s"])
        big = scales.max(dim=1).values >= 0.01 * extent
        clone, split = over & ~big, over & big
        keep = torch.nonzero(~split).flatten()
        c_idx = torch.nonzero(clone).flatten()
        s_idx = torch.nonzero(split).flatten()
        parents = torch.cat([keep, c_idx, s_idx, s_idx])
        out = {k: v[parents].clone() for k, v in p.items()}
        ns = s_idx.numel()
        if ns:
            sp = torch.cat([s_idx, s_idx])
            q = p["q_raw"][sp]
            q = q / torch.clamp(torch.linalg.norm(q, dim=1, keepdim=True), min=1e-12)
            R = _quat_rot_t(q)
            offs = torch.from_numpy(rng.standard_normal((2 * ns, 3))).to(self.dev) * scales[sp]
            out["mu"][-2 * ns:] = p["mu"][sp] + torch.einsum("nij,nj->ni", R, offs)
            out["log_s"][-2 * ns:] = p["log_s"][sp] - math.log(1.6)
        alive = torch.sigmoid(out["o_logit"]) >= cfg.prune_opacity_threshold
        is_new = torch.arange(parents.numel(), device=self.dev) >= keep.numel()
        info = {"cloned": int(c_idx.numel()), "split": int(ns),
                "pruned": int((~alive).sum()), "count": int(alive.sum())}
        if info["count"] == 0 and keep_if_empty:
            return info
        self.p = {k: v[alive].contiguous() for k, v in out.items()}
        self.adam.remap(parents[alive], is_new[alive])
        return info

    def _rgba(self, out):
        c = {name: c for name, c, w in _cols_named(self.layout)}
        return torch.cat([out[..., c["color"]:c["color"] + 3], out[..., c["alpha"]:c["alpha"] + 1]],
                         dim=-1)

    def _cam_params(self, cam):
        """Device block (focal, cx, cy, rotation[9]) for the pseudo-normal
        term, staged through pinned memory (no host synchronisation)."""
        if getattr(self, "_cam_pin", None) is None:
            self._cam_pin = torch.empty(12, dtype=torch.float64, pin_memory=True)
            self._cam_dev = torch.empty(12, dtype=torch.float64, device=self.dev)
            self._cam_ev = None
        if self._cam_ev is not None:
            self._cam_ev.synchronize()
        h = self._cam_pin.numpy()
        h[0] = 0.5 * cam.height / np.tan(0.5 * cam.fov_y)
        h[1], h[2] = (cam.width - 1) / 2.0, (cam.height - 1) / 2.0
        h[3:] = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
        self._cam_dev.copy_(self._cam_pin, non_blocking=True)
        self._cam_ev = torch.cuda.Event()
        self._cam_ev.record()
        return self._cam_dev

    def _map_terms(self, F, cam, gt, weights, offset=False, bilateral=False, cam_dev=None):
        """Photometric L1+SSIM (K7) and the map regularizers (fused kernel):
        returns (loss terms for ivr_loss_finalize, tensors they point to,
        d_out float32 (H,W,K), column map).  No host synchronisation."""
        c = {name: c for name, c, w in _cols_named(self.layout)}
        rgba_cols = (c["color"], c["color"] + 1, c["color"] + 2, c["alpha"])
        h, w, nc = F.out.shape[0], F.out.shape[1], len(rgba_cols)
        if (h, w, nc) != tuple(gt.shape):
            raise ShapeMismatch(f"prediction {(h, w, nc)} vs ground truth {tuple(gt.shape)}")
        win = 2 * SSIM_RADIUS + 1
        with_ssim = weights.ssim_weight > 0.0
        if with_ssim and (h < win or w < win):
            raise ShapeMismatch(f"image {h}x{w} smaller than the {win}x{win} ssim window")
        numel = h * w * nc
        # K7 reads the rgba columns of the float32 frame in place (exact f64
        # promotion; same values as frame[..., cols].double())
        sums, d_rgba = _photometric_frame_dev(F.out, rgba_cols, gt.to(torch.float64),
                                              weights.l1_weight / numel, -weights.ssim_weight,
                                              with_ssim)
        wn = weights.normal_consistency
        wo = weights.offset_sparsity if offset else 0.0
        wb = weights.bilateral_smoothness if bilateral else 0.0
        bil = tuple(c[n] for n in ("k_a", "k_d", "k_s", "beta")) if wb > 0.0 else ()
        cols = (c["color"], c["alpha"], c.get("depth", -1), c.get("normal", -1),
                c.get("delta_c", -1))
        terms, d_out = regularize_t(F.out, cols, gt=gt, d_rgba=d_rgba,
                                    cam_params=(cam_dev if cam_dev is not None else
                                                self._cam_params(cam)) if wn > 0.0 else None,
                                    w_normal=wn, w_offset=wo, w_bil=wb, bil_cols=bil)
        lt = L.LossTerms_t()
        lt.photo_sums = sums.data_ptr()
        lt.l1_weight, lt.ssim_weight = weights.l1_weight, weights.ssim_weight
        lt.numel = float(numel)
        lt.windows = float((h - win + 1) * (w - win + 1) * nc)
        lt.terms = terms.data_ptr()
        lt.w_normal, lt.w_offset, lt.w_bil = wn, wo, wb
        return lt, (sums, terms), d_out, c

    def _assemble(self, gr, c=None, weights=None, shading=False, graph=None):
        """ivr_step_assemble (value-channel chain rule, opacity L1, densify
        statistic) in place on K4b's outputs; returns (stat, o partials).
        ``graph`` (a StepGraph being captured): the kernel also updates the
        sticky overflow gate and adds the statistic into graph.stat_sum."""
        n, p = self.n, self.p
        A = L.StepGrads_t()
        if graph is not None:
            A.gate, A.n_pairs = graph.gate.data_ptr(), graph.n_pairs.data_ptr()
            A.pair_capacity, A.stat_sum = int(graph.capacity), graph.stat_sum.data_ptr()
        A.n, A.k = n, self.K
        A.col_delta_c = A.col_k_a = A.col_k_d = A.col_k_s = A.col_beta = -1
        stat = torch.empty(n, dtype=torch.float64, device=self.dev)
        A.d_mean2d, A.d_n_raw, A.stat = gr["d_mean2d"].data_ptr(), gr["d_n_raw"].data_ptr(), \
            stat.data_ptr()
        part = None
        if shading:
            A.d_values = gr["d_values"].data_ptr()
            A.col_delta_c, A.col_k_a, A.col_k_d = c["delta_c"], c["k_a"], c["k_d"]
            A.col_k_s, A.col_beta = c["k_s"], c["beta"]
            for k in ("k_a_raw", "k_d_raw", "k_s_raw", "log_beta"):
                setattr(A, k, p[k].data_ptr())
            for k in ("d_delta_c", "d_k_a_raw", "d_k_d_raw", "d_k_s_raw", "d_log_beta"):
                setattr(A, k, gr[k].data_ptr())
            A.o_logit, A.d_o_logit = p["o_logit"].data_ptr(), gr["d_o_logit"].data_ptr()
            A.w_opacity_l1 = weights.opacity_l1
            part = torch.empty(int(L.lib().ivr_step_partials(n)), dtype=torch.float64,
                               device=self.dev)
            A.o_partial = part.data_ptr()
        L.check(L.lib().ivr_step_assemble(ctypes.byref(A), D.stream_handle()), "ivr_step_assemble")
        return stat, part

    def _finalize(self, lt, part=None, w_opacity_l1=0.0):
        """ivr_loss_finalize: the step's loss (device scalar) + the device-side
        DivergedLoss bookkeeping (first non-finite photometric loss)."""
        if self._first_bad is None:
            self._first_bad = torch.tensor([0, -1], dtype=torch.int64, device=self.dev)
            self._last_bad_loss = torch.zeros((), dtype=torch.float64, device=self.dev)
        if part is not None:
            lt.o_partial, lt.n_partial = part.data_ptr(), part.numel()
            lt.w_opacity_l1, lt.n = w_opacity_l1, float(self.n)
        loss = torch.empty((), dtype=torch.float64, device=self.dev)
        L.check(L.lib().ivr_loss_finalize(ctypes.byref(lt), loss.data_ptr(),
                                          self._first_bad.data_ptr(),
                                          self._last_bad_loss.data_ptr(), D.stream_handle()),
                "ivr_loss_finalize")
        return loss

    def check_finite(self):
        """Raise DivergedLoss if any step so far had a non-finite loss."""
        if self._first_bad is not None:
            step_no, first = (int(x) for x in self._first_bad.cpu())
            if first >= 0:
                raise DivergedLoss(f"loss became {float(self._last_bad_loss)} at step {first}")


class BaseTrainer(_StageTrainer):
    """Stage-1 state: geometry + SH coefficients (trainer.py:375-394, 532-560)."""

    KEYS = GEOM + ("sh",)

    def __init__(self, params, degree, cfg=None, device=None):
        super().__init__(params, cfg, device)
        self.degree = int(degree)
        self.layout = _channel_layout(("color", "alpha", "depth", "normal"), None)
        self.cols, self.attr_cols, self.K = _cols(self.layout)

    def _dg(self):
        return D.DeviceGaussians({k: self.p[k] for k in GEOM}, None, None, self.dev)

    def forward(self, cam, want_state=True):
        from .sh import sh_eval_device
        dg = self._dg()
        rgb = sh_eval_device(self.p["mu"], self.p["sh"], self.degree, cam.position)
        F = D.rasterize_device(dg, cam, self.K, self.cols, self.ws, colors=rgb, f64=False,
                               want_state=want_state, exact=self.exact)
        return F, dg

    def step(self, cam, gt, weights=None):
        """One _stage1_step (trainer.py:375-394): (loss, grads, densify stat)."""
        from .sh import sh_backward_device
        weights = weights or self.cfg.weights
        F, dg = self.forward(cam)
        lt, keep, d_out, _ = self._map_terms(F, cam, gt, weights)
        loss = self._finalize(lt)
        g = D.blend_backward(F, d_out)
        want = ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors", "d_mean2d")
        gr, bad = D.preprocess_backward(dg, cam, self.K, self.cols, g=g, geometry=True, want=want)
        n = self.n
        d_mu = gr["d_mu"].view(n, 3)
        d_sh = sh_backward_device(self.p["mu"], self.p["sh"], self.degree, cam.position,
                                  gr["d_colors"].view(n, 3), d_mu=d_mu)
        grads = {"mu": d_mu, "q_raw": gr["d_q_raw"].view(n, 4), "log_s": gr["d_log_s"].view(n, 3),
                 "o_logit": gr["d_o_logit"], "n_raw": gr["d_n_raw"].view(n, 3), "sh": d_sh}
        stat, _ = self._assemble(gr)
        self._bad = bad
        return loss, grads, stat

    def render_rgba(self, cam):
        F, _ = self.forward(cam, want_state=False)
        return self._rgba(F.out.double())

    def model(self, metadata=None):
        h = {k: D.to_host(v) for k, v in self.p.items()}
        geom = GaussianGeometry(*(h[k] for k in GEOM))
        return BasicSceneModel(STAGE_BASE, geom, sh=ShColor(h["sh"], self.degree),
                               metadata=metadata or {})


class EditableTrainer(_StageTrainer):
    """Stage-2 state on the device: params (float64 tensors), palette, light."""

    KEYS = GEOM + SHADE

    def __init__(self, params, palette, light, cfg=None, device=None):
        super().__init__(params, cfg, device)
        self.palette = D.to_dev(np.asarray(palette, np.float64).reshape(1, 3), device=self.dev)
        self.light = light
        self.layout = _channel_layout(("color", "alpha", "depth", "normal"),
                                      {"delta_c": np.zeros((1, 3)), "k_a": np.zeros(1),
                                       "k_d": np.zeros(1), "k_s": np.zeros(1), "beta": np.zeros(1)})
        self.cols, self.attr_cols, self.K = _cols(self.layout)
        self.colmap = {name: (c, w) for name, c, w in self.attr_cols}

    def _dg(self):
        return D.DeviceGaussians({k: self.p[k] for k in GEOM}, {k: self.p[k] for k in SHADE},
                                 None, self.dev)

    def forward(self, cam, want_state=True, dg=None, graph=None):
        dg = dg or self._dg()
        S = D.shading_struct(dg, self.palette, False, self.light)
        p = self.p
        n = self.n
        buf = getattr(self, "_attr_buf", None)
        if buf is None or buf.shape[1] != n:
            buf = self._attr_buf = torch.empty((4, n), dtype=torch.float64, device=self.dev)
        L.check(L.lib().ivr_stage2_attrs(n, p["k_a_raw"].data_ptr(), p["k_d_raw"].data_ptr(),
                                         p["k_s_raw"].data_ptr(), p["log_beta"].data_ptr(),
                                         buf[0].data_ptr(), buf[1].data_ptr(), buf[2].data_ptr(),
                                         buf[3].data_ptr(), D.stream_handle()), "ivr_stage2_attrs")
        attrs = {"delta_c": p["delta_c"], "k_a": buf[0], "k_d": buf[1], "k_s": buf[2],
                 "beta": buf[3]}
        attrs_dev = [(attrs[name].reshape(self.n, w).contiguous(), c, w)
                     for name, c, w in self.attr_cols]
        F = D.rasterize_device(dg, cam, self.K, self.cols, graph.ws if graph else self.ws,
                               shading=S, attrs=attrs_dev, f64=False, want_state=want_state,
                               exact=self.exact, params_dev=graph.params_dev if graph else None,
                               capacity=graph.capacity if graph else None)
        return F, S, attrs, dg

    def step(self, cam, gt, weights=None, graph=None, events=None):
        """One _stage2_step (trainer.py:397-444): (loss, grads, densify stat),
        all device tensors.  ``graph``: the StepGraph being captured (camera
        and pseudo-normal block from its device buffers, no host sync).
        ``events``: 6 CUDA events recorded around forward (K14 attrs + K1-K3),
        losses (K7 + K10), K4a, K4b and assembly/loss (K14) -- the bench's
        per-kernel split."""
        weights = weights or self.cfg.weights
        rec = (lambda j: events[j].record()) if events else (lambda j: None)
        rec(0)
        F, S, attrs, dg = self.forward(cam, graph=graph)
        rec(1)
        lt, keep, d_out, c = self._map_terms(F, cam, gt, weights, offset=True, bilateral=True,
                                             cam_dev=graph.cam_dev if graph else None)
        rec(2)
        g = D.blend_backward(F, d_out)
        rec(3)
        want = ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_mean2d", "d_values",
                "d_delta_c", "d_k_a_raw", "d_k_d_raw", "d_k_s_raw", "d_log_beta")
        gr, bad = D.preprocess_backward(dg, cam, self.K, self.cols, g=g, shading=S, geometry=True,
                                        want=want, light=self.light,
                                        params_dev=graph.params_dev if graph else None)
        rec(4)
        if graph is not None:
            graph.n_pairs = F.n_pairs
        n = self.n
        stat, part = self._assemble(gr, c, weights, shading=True, graph=graph)
        loss = self._finalize(lt, part, weights.opacity_l1)
        rec(5)
        self._last_pairs = F.n_pairs
        grads = {"mu": gr["d_mu"].view(n, 3), "q_raw": gr["d_q_raw"].view(n, 4),
                 "log_s": gr["d_log_s"].view(n, 3), "o_logit": gr["d_o_logit"],
                 "n_raw": gr["d_n_raw"].view(n, 3), "delta_c": gr["d_delta_c"].view(n, 3),
                 "k_a_raw": gr["d_k_a_raw"], "k_d_raw": gr["d_k_d_raw"],
                 "k_s_raw": gr["d_k_s_raw"], "log_beta": gr["d_log_beta"]}
        self._bad = bad
        return loss, grads, stat

    def render_rgba(self, cam):
        F, _, _, _ = self.forward(cam, want_state=False)
        return self._rgba(F.out.double())

    def model(self, palette, metadata=None):
        h = {k: D.to_host(v) for k, v in self.p.items()}
        geom = GaussianGeometry(*(h[k] for k in GEOM))
        attrs = ShadingAttributes(*(h[k] for k in SHADE))
        return BasicSceneModel(STAGE_EDITABLE, geom, shading=attrs, palette=Palette(palette),
                               metadata=metadata or {})


def _cols_named(layout):
    c = 0
    for name, w in layout:
        yield name, c, w
        c += w


def _quat_rot_t(q):
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = torch.empty((q.shape[0], 3, 3), dtype=q.dtype, device=q.device)
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def scene_extent(mu):
    """Half the bounding-box diagonal (trainer.py:233-238)."""
    mu = np.asarray(mu)
    if mu.size == 0:
        return 1.0
    return max(0.5 * float(np.linalg.norm(mu.max(axis=0) - mu.min(axis=0))), 1e-6)


def foreground_mean_color(dataset):
    """Alpha-weighted mean rgb over the training images (trainer.py:331-341)."""
    num, den = np.zeros(3), 0.0
    for img in dataset.images:
        img = np.asarray(img, np.float64)
        a = img[..., 3]
        num += (img[..., :3] * a[..., None]).sum(axis=(0, 1))
        den += a.sum()
    return np.full(3, 0.5) if den <= 0.0 else num / den


@dataclass
class ViewDataset:
    """Multi-view RGBA images with their cameras and light (the fields of
    dvr.VolumeDataset the trainer reads, dvr.py:459-482)."""

    cameras: list
    images: list
    light: LightConfig = field(default_factory=LightConfig)
    manifest: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.cameras)

    def bbox(self):
        """Volume bounds from the manifest, else a cube inside the camera
        orbit (dvr.py:471-482)."""
        vol = self.manifest.get("volume")
        if vol is not None:
            half = (np.asarray(vol["dims"], dtype=np.float64) - 1.0) \
                * np.asarray(vol["spacing"], dtype=np.float64) / 2.0
            return -half, half
        pos = np.array([c.position for c in self.cameras])
        r = 0.5 * float(np.min(np.linalg.norm(pos, axis=1)))
        half = np.full(3, max(r, 1e-6))
        return -half, half


def _project_px(points, cam):
    rel = (points - cam.position[None, :]) @ cam.rotation.T
    z = rel[:, 2]
    ok = z > 1e-6
    zs = np.where(ok, z, 1.0)
    px = (cam.focal * rel[:, 0] / zs + cam.center_px[0]).astype(np.int64)
    py = (cam.focal * rel[:, 1] / zs + cam.center_px[1]).astype(np.int64)
    ok &= (px >= 0) & (px < cam.width) & (py >= 0) & (py < cam.height)
    return np.nonzero(ok)[0], px, py


class StepGraph:
    """One stage-2 training step -- K1-K3, L1+SSIM, map regularizers, K4a/K4b,
    gradient assembly, loss, Adam on every group -- captured once as a CUDA
    graph for the trainer's current Gaussian count (recapture after densify).

    Per step the host writes the view's ``ivr_frame_params``, its
    pseudo-normal camera block and the Adam schedule (lr, bias corrections)
    into a pinned ring slot, copies them and the view's ground truth into the
    graph's fixed device buffers, and replays: one launch instead of ~43 and
    no host synchronisation.  The pair capacity learned at capture (+30%) is
    verified when a step retires (its pair count is copied back
    asynchronously); an overflowed step and every later one are gated on the
    device (Adam and the densify statistic skip them), and the host then
    recaptures with a larger capacity and replays the gated steps in order,
    so the update sequence is exactly the eager one."""

    RING = 4

    def __init__(self, tr, cam, gt, weights=None, decay_extra=(), headroom=1.3):
        if not isinstance(tr, EditableTrainer):
            raise OutOfRange("StepGraph captures the stage-2 (EditableTrainer) step")
        self.tr, self.weights, self.decay_extra = tr, weights or tr.cfg.weights, decay_extra
        self.headroom = headroom
        dev = tr.dev
        self.W, self.H = int(cam.width), int(cam.height)
        self.nb = ctypes.sizeof(L.FrameParams_t)
        self.names = list(tr.p.keys())
        G = len(self.names)
        # own workspace: eager renders between replays (holdout logging) must
        # never reallocate a buffer the graph captured
        self.ws = D.Workspace(dev)
        # one device staging block (one H2D per step): frame params | camera
        # block for the pseudo normals | Adam schedule
        slot_bytes = self.nb + 12 * 8 + 3 * G * 8
        self.stage_dev = torch.empty(slot_bytes, dtype=torch.uint8, device=dev)
        self.params_dev = self.stage_dev[:self.nb]
        self.cam_dev = self.stage_dev[self.nb:self.nb + 96].view(torch.float64)
        self.sched_dev = self.stage_dev[self.nb + 96:].view(torch.float64)
        self.gt_dev = torch.empty((self.H, self.W, 4), dtype=torch.float64, device=dev)
        self.gate = torch.zeros(1, dtype=torch.int32, device=dev)
        self.stat_sum = torch.zeros(tr.n, dtype=torch.float64, device=dev)
        self._pin = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True)
                     for _ in range(self.RING)]
        self._np = [torch.zeros(1, dtype=torch.int32, pin_memory=True) for _ in range(self.RING)]
        self._pending = []  # (slot, event, it, iters, cam, gt, t-before per group)
        self._k = 0
        # pair capacity from one synchronising forward of this view
        F, _, _, _ = tr.forward(cam, want_state=False)
        self.capacity = max(int(int(F.n_pairs.item()) * headroom) + 4096, tr.ws.pair_capacity)
        self._capture(cam, gt)

    # -- staging -------------------------------------------------------------
    def _stage(self, cam, gt, it, iters):
        k = self._k
        self._k = (k + 1) % self.RING
        while any(p[0] == k for p in self._pending):  # reuse a slot once its step retired
            self._retire_oldest()
        tr = self.tr
        h = self._pin[k].numpy()
        P = D.frame_params(cam, tr.light)
        ctypes.memmove(h.ctypes.data, ctypes.addressof(P), self.nb)
        f = np.frombuffer(h, dtype=np.float64, offset=self.nb)
        f[0] = 0.5 * cam.height / np.tan(0.5 * cam.fov_y)
        f[1], f[2] = (cam.width - 1) / 2.0, (cam.height - 1) / 2.0
        f[3:12] = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
        t_before = {n: tr.adam.state[n]["t"] for n in self.names}
        f[12:] = tr.adam.schedule([(n, tr.lr(n, it, iters, self.decay_extra)) for n in self.names])
        pin = self._pin[k]
        self.stage_dev.copy_(pin, non_blocking=True)
        self.gt_dev.copy_(gt, non_blocking=True)
        return k, t_before

    def _capture(self, cam, gt):
        tr = self.tr
        self._cam0 = cam
        tr.adam.ensure([(n, tr.p[n]) for n in self.names])
        saved_t = {n: tr.adam.state[n]["t"] for n in self.names}
        self._stage(cam, gt, 1, 1)
        self._body(capturing=False)  # sizes every buffer before capture
        torch.cuda.synchronize()
        # undo the warm-up step: parameters, moments, step counts, statistics
        for n in self.names:
            tr.adam.state[n]["t"] = saved_t[n]
        self._restore()
        self.g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g):
            self._body(capturing=True)
        torch.cuda.synchronize()

    def _snapshot(self):
        tr = self.tr
        self._snap = ({n: v.clone() for n, v in tr.p.items()},
                      {n: (st["m"].clone(), st["v"].clone()) for n, st in tr.adam.state.items()})

    def _restore(self):
        tr = self.tr
        p, mv = self._snap
        for n, v in p.items():
            tr.p[n].copy_(v)
        for n, (m, v) in mv.items():
            tr.adam.state[n]["m"].copy_(m)
            tr.adam.state[n]["v"].copy_(v)
        self.stat_sum.zero_()
        self.gate.zero_()

    def _body(self, capturing):
        tr = self.tr
        if not capturing:
            self._snapshot()
        # the step's assembly kernel also raises the sticky gate (this step's
        # pair list overflowed, or an earlier one did) and adds the densify
        # statistic of ungated steps into stat_sum
        loss, grads, stat = tr.step(self._cam0, self.gt_dev, self.weights, graph=self)
        items = [(n, tr.p[n], grads[n]) for n in self.names]
        self._groups = tr.adam.groups(items)
        self._keep = grads
        L.check(L.lib().ivr_adam_step_sched(self._groups, len(items), tr.adam.b1, tr.adam.b2,
                                            tr.adam.eps, self.sched_dev.data_ptr(),
                                            self.gate.data_ptr(), D.stream_handle()),
                "ivr_adam_step_sched")
        self.loss = loss

    # -- running ---------------------------------------------------------------
    def step(self, cam, gt, it, iters):
        """Stage and replay one step; returns the step's loss (device scalar,
        overwritten by the next replay)."""
        k, t_before = self._stage(cam, gt, it, iters)
        self.g.replay()
        self._np[k].copy_(self.n_pairs[:1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pending.append((k, ev, it, iters, cam, gt, t_before))
        return self.loss

    def _retire_oldest(self):
        """Retire the oldest pending step; on an overflow, recapture with a
        larger capacity and replay the gated steps."""
        k, ev = self._pending[0][:2]
        ev.synchronize()
        if int(self._np[k][0]) > self.capacity:
            self._redo()
        else:
            self._pending.pop(0)

    def _redo(self):
        """The oldest pending step overflowed: every pending step was gated."""
        torch.cuda.synchronize()
        redo = self._pending
        self._pending = []
        tr = self.tr
        for n in self.names:
            tr.adam.state[n]["t"] = redo[0][6][n]
        peak = max(int(self._np[r[0]][0]) for r in redo)
        self.capacity = max(int(peak * self.headroom) + 4096, 2 * self.capacity)
        stat_sum = self.stat_sum.clone()
        self._capture(redo[0][4], redo[0][5])
        self.stat_sum.copy_(stat_sum)
        for r in redo:
            self.step(r[4], r[5], r[2], r[3])

    def flush(self):
        """Retire every pending step (host synchronisation point)."""
        while self._pending:
            self._retire_oldest()


def densify_and_prune(model, grad_stats, cfg, extent=None, rng=None):
    """One round of adaptive density control on a scene model
    (trainer.py:241-261): clone / split (at scale / 1.6) the primitives whose
    mean gradient statistic exceeds the threshold, prune low opacity; on the
    GPU (the trainers' ``densify``).  Split offsets come from ``rng``
    exactly as in the reference.  Returns (new model, info); an all-pruned
    round returns the empty model with count 0."""
    rng = rng if rng is not None else np.random.default_rng(cfg.seed)
    extent = extent if extent is not None else scene_extent(np.asarray(model.geometry.mu))
    g = model.geometry
    params = {k: getattr(g, k) for k in GEOM}
    if model.stage == STAGE_EDITABLE:
        params.update({k: getattr(model.shading, k) for k in SHADE})
        tr = EditableTrainer(params, model.palette.c_p, LightConfig(), cfg)
    else:
        params["sh"] = np.asarray(model.sh.coefficients, np.float64)
        tr = BaseTrainer(params, model.sh.degree, cfg)
    stats = np.asarray(grad_stats, np.float64)
    if stats.shape != (len(model),):
        raise OutOfRange(f"grad stats must be ({len(model)},), got {stats.shape}")
    info = tr.densify(D.to_dev(stats), extent, rng, keep_if_empty=False)
    if model.stage == STAGE_EDITABLE:
        new = tr.model(model.palette.c_p, dict(model.metadata))
    else:
        new = tr.model(dict(model.metadata))
    return new, info


def _dc_colors_from_view(points, cam, image):
    """rgb of the training pixel each point projects to, else mid grey
    (trainer.py:264-279)."""
    rgb = np.full((points.shape[0], 3), 0.5)
    idx, px, py = _project_px(points, cam)
    rgb[idx] = np.asarray(image)[py[idx], px[idx], :3]
    return rgb


def _inside_any_silhouette(points, dataset):
    """trainer.py:282-294."""
    keep = np.zeros(points.shape[0], dtype=bool)
    for cam, img in zip(dataset.cameras, dataset.images):
        idx, px, py = _project_px(points, cam)
        keep[idx] |= np.asarray(img)[py[idx], px[idx], 3] > 0.0
    return keep


def initialize_base(dataset, cfg, rng):
    """Uniform in-box seeding, 3-NN scales, DC colours from the first view
    (trainer.py:297-328).  Host-side, once per run."""
    from scipy.spatial import cKDTree
    lo, hi = dataset.bbox()
    pts = rng.uniform(lo, hi, (cfg.init_count, 3))
    if cfg.silhouette_carve:
        for _ in range(20):
            keep = _inside_any_silhouette(pts, dataset)
            if keep.all():
                break
            fresh = rng.uniform(lo, hi, (int(np.count_nonzero(~keep)), 3))
            pts = np.concatenate([pts[keep], fresh])
        pts = pts[:cfg.init_count]
    n = pts.shape[0]
    if n > 1:
        dists, _ = cKDTree(pts).query(pts, k=min(4, n))
        nn = np.maximum(dists[:, 1:].mean(axis=1), 1e-6)
    else:
        nn = np.full(n, 0.1 * scene_extent(np.stack([lo, hi])))
    log_s = np.log(nn)[:, None].repeat(3, axis=1)
    q_raw = np.zeros((n, 4))
    q_raw[:, 0] = 1.0
    o_logit = np.full(n, np.log(cfg.init_opacity / (1.0 - cfg.init_opacity)))
    first = dataset.cameras[0]
    v = first.position[None, :] - pts
    n_raw = v / np.maximum(np.linalg.norm(v, axis=-1, keepdims=True), 1e-12)
    geom = GaussianGeometry(pts, q_raw, log_s, o_logit, n_raw)
    sh = ShColor.from_dc(_dc_colors_from_view(pts, first, dataset.images[0]), degree=cfg.sh_degree)
    return geom, sh


def _run_stage(tr, dataset, cfg, iters, rng, densify_start=None, decay_extra=()):
    """The shared optimisation loop (trainer.py:463-526) over a device
    trainer: one random view per iteration, Adam with the schedules,
    densify/prune on the trailing interval's mean statistic, holdout PSNR
    logged every ``log_interval``."""
    if len(dataset) < 2:
        raise DatasetEmpty("training needs at least two views")
    extent = scene_extent(np.stack(dataset.bbox()))
    until = cfg.until_iter(iters)
    start = cfg.densify_start_iter if densify_start is None else densify_start
    holdout = len(dataset) - 1
    gts = [D.to_dev(np.asarray(im, np.float64)) for im in dataset.images]
    stats_sum = torch.zeros(tr.n, dtype=torch.float64, device=tr.dev)
    stats_iters = 0
    log = []
    # stage 2: whole steps replay as a CUDA graph (recaptured after densify)
    use_graph = isinstance(tr, EditableTrainer) and os.environ.get("IVR_TRAIN_GRAPH", "1") != "0"
    G = None
    for it in range(1, iters + 1):
        view = int(rng.integers(len(dataset)))
        if use_graph:
            if G is None:
                G = StepGraph(tr, dataset.cameras[view], gts[view], decay_extra=decay_extra)
            loss = G.step(dataset.cameras[view], gts[view], it, iters)
            if it % cfg.log_interval == 0:
                G.flush()
                tr.check_finite()
                D.raise_if_bad(tr._bad, tr.n, ("d_mu", "d_q_raw", "d_log_s", "d_o_logit",
                                               "d_n_raw", "d_colors"))
        else:
            loss, grads, stat = tr.step(dataset.cameras[view], gts[view])
            if it % cfg.log_interval == 0:
                tr.check_finite()
                D.raise_if_bad(tr._bad, tr.n, ("d_mu", "d_q_raw", "d_log_s", "d_o_logit",
                                               "d_n_raw", "d_colors"))
            tr.apply(grads, it, iters, decay_extra)
            stats_sum += stat
        stats_iters += 1
        if it % cfg.densify_interval == 0:
            if G is not None:
                G.flush()
                stats_sum = G.stat_sum
            if start <= it <= until:
                tr.densify(stats_sum / max(stats_iters, 1), extent, rng)
                G = None  # parameter tensors replaced: recapture on the next step
            elif G is not None:
                G.stat_sum.zero_()
            stats_sum = torch.zeros(tr.n, dtype=torch.float64, device=tr.dev)
            stats_iters = 0
        if it % cfg.log_interval == 0 or it == iters:
            if G is not None:
                G.flush()
            tr.check_finite()
            lv = float(loss)
            if not np.isfinite(lv):
                raise DivergedLoss(f"loss became {lv} at iteration {it}")
            img = tr.render_rgba(dataset.cameras[holdout])
            log.append({"iteration": it, "loss": lv, "count": tr.n,
                        "psnr": _psnr_t(img, gts[holdout])})
    return log


def train_base(dataset, cfg=None, init=None):
    """Stage 1 on the GPU (trainer.py:532-560): returns (base model, log).
    ``init`` optionally supplies a (geometry, ShColor) starting point."""
    cfg = cfg or TrainConfig()
    if len(dataset) < 2:
        raise DatasetEmpty("training needs at least two views")
    rng = np.random.default_rng(cfg.seed)
    geom, sh = init if init is not None else initialize_base(dataset, cfg, rng)
    params = {k: getattr(geom, k) for k in GEOM}
    params["sh"] = np.asarray(sh.coefficients, np.float64)
    tr = BaseTrainer(params, sh.degree, cfg)
    log = _run_stage(tr, dataset, cfg, cfg.stage1_iters, rng)
    return tr.model({"stage1_iters": cfg.stage1_iters, "seed": cfg.seed}), log


def _stage2_init(n):
    """trainer.py:562-577: neutral start."""
    return {"delta_c": np.zeros((n, 3)), "k_a_raw": np.zeros(n), "k_d_raw": np.zeros(n),
            "k_s_raw": np.zeros(n), "log_beta": np.full(n, np.log(9.0))}


def train_editable(base, dataset, cfg=None):
    """Stage 2 on the GPU (trainer.py:580-626): returns (editable model, log)."""
    cfg = cfg or TrainConfig()
    if base.stage != STAGE_BASE:
        raise OutOfRange("stage-2 training expects a base-stage model")
    rng = np.random.default_rng(cfg.seed + 1)
    if len(dataset) < 2:
        raise DatasetEmpty("training needs at least two views")
    palette = foreground_mean_color(dataset)
    light = dataset.light
    g = base.geometry
    params = {k: getattr(g, k) for k in GEOM}
    params.update(_stage2_init(len(g)))
    tr = EditableTrainer(params, palette, light, cfg)
    log = _run_stage(tr, dataset, cfg, cfg.stage2_iters, rng,
                     densify_start=cfg.densify_interval, decay_extra=("o_logit",))
    model = tr.model(palette, {"stage2_iters": cfg.stage2_iters, "seed": cfg.seed,
                               "light": light.to_dict(),
                               "transfer_function": getattr(dataset, "manifest", {}).get(
                                   "transfer_function")})
    return model, log


def render_model(model, cam, light=None, dtype=np.float32):
    """RGBA image of one basic model of either stage (trainer.py:633-647)."""
    from .vq import dequantize_model
    if model.is_quantized:
        model = dequantize_model(model)
    if model.stage == STAGE_BASE:
        from .rasterizer import rasterize_forward
        from .sh import sh_colors
        rgb = sh_colors(model.geometry, model.sh, cam)
        out, _ = rasterize_forward(model.geometry, rgb, cam, channels=("color", "alpha"),
                                   dtype=dtype)
    else:
        from .scene import ComposedScene
        sc = ComposedScene.compose([model], light or LightConfig())
        out = DeviceScene(sc).render(cam, dtype=dtype)
    return np.concatenate([np.asarray(out.color, np.float64), np.asarray(out.alpha, np.float64)[..., None]],
                          axis=-1)


def write_training_log(path, records):
    with open(path, "w") as f:
        for rec in records:
            f.write(json.dumps(rec, sort_keys=True) + "\n")
