"""Inverse appearance fitting on the GPU (drop-in for voxsplat/inverse.py).

The scene's primitives stay frozen and resident in HBM (a DeviceScene); each
iteration renders with the transform (K1-K3, float64 semantics), evaluates
the L1+SSIM loss on the device, runs K4 with only the transform gradients
requested (per-scene palette and opacity scale, global (lam, b), light
angles -- inverse.py:161-190), and applies the reference's Adam on the
(4S+10)-float parameter vector.

Multi-view extension: ``optimize_to_reference``
accepts lists of references/cameras and minimises the MEAN per-view loss;
under torch.distributed each rank owns a slice of the views and the packed
gradient vector (4S+10 floats + loss) is summed with ONE NCCL all-reduce per
iteration, so every rank applies the identical Adam step.  One view reproduces
the reference exactly.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .errors import DivergedLoss, OutOfRange, ShapeMismatch
from .losses import _photometric_dev, photometric_loss_t
from .scene import ComposedScene, DeviceScene
from .shading import ORBITAL, LightConfig


def softplus(x):
    return np.logaddexp(0.0, np.asarray(x, dtype=np.float64))


def inv_softplus(y):
    y = np.asarray(y, dtype=np.float64)
    if np.any(y <= 0.0):
        raise OutOfRange("softplus output must be positive")
    return y + np.log1p(-np.exp(-y))


def _sigmoid(x):
    """_mathutil.sigmoid (branch on sign)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


@dataclass
class TransformParams:
    """Per-scene palette (S,3) and opacity softplus pre-image (S,), global
    (lam, b) on (k_a, k_d, k_s, beta), orbital light angles (inverse.py:35-88)."""

    c_p: np.ndarray
    opacity_raw: np.ndarray
    lam: np.ndarray
    b: np.ndarray
    polar: float = 0.0
    azimuth: float = 0.0
    light_mode: str = "headlight"

    def __post_init__(self):
        self.c_p = np.atleast_2d(np.asarray(self.c_p, dtype=np.float64))
        s = self.c_p.shape[0]
        if self.c_p.shape != (s, 3):
            raise ShapeMismatch(f"c_p must be (S, 3), got {self.c_p.shape}")
        self.opacity_raw = np.asarray(self.opacity_raw, dtype=np.float64).reshape(s)
        self.lam = np.asarray(self.lam, dtype=np.float64).reshape(4)
        self.b = np.asarray(self.b, dtype=np.float64).reshape(4)
        self.polar = float(self.polar)
        self.azimuth = float(self.azimuth)

    @property
    def opacity_scale(self):
        return softplus(self.opacity_raw)

    def copy(self):
        return TransformParams(self.c_p.copy(), self.opacity_raw.copy(), self.lam.copy(),
                               self.b.copy(), self.polar, self.azimuth, self.light_mode)

    def to_dict(self):
        return {"c_p": self.c_p.tolist(), "opacity_scale": self.opacity_scale.tolist(),
                "lam": self.lam.tolist(), "b": self.b.tolist(), "polar": self.polar,
                "azimuth": self.azimuth, "light_mode": self.light_mode}

    @classmethod
    def from_dict(cls, d):
        return cls(np.asarray(d["c_p"]), inv_softplus(np.asarray(d["opacity_scale"])),
                   np.asarray(d["lam"]), np.asarray(d["b"]), d["polar"], d["azimuth"],
                   d["light_mode"])


def init_transform(scene: ComposedScene) -> TransformParams:
    """Identity transform for the scene's current edits (inverse.py:91-101)."""
    c_p = np.stack([e.palette_override if e.palette_override is not None else m.palette.c_p
                    for m, e in zip(scene.models, scene.edits)])
    scales = np.array([max(e.opacity_scale, 1e-6) for e in scene.edits])
    return TransformParams(c_p, inv_softplus(scales), np.ones(4), np.zeros(4),
                           scene.light.polar, scene.light.azimuth, scene.light.mode)


from .trainer import Adam  # noqa: E402  (trainer.Adam, trainer.py:100-128)


def _light(scene, params):
    return LightConfig(scene.light.mode, params.polar, params.azimuth,
                       term_scales=scene.light.term_scales.copy())


class InverseFitter:
    """Frozen scene resident on the device + per-view references."""

    def __init__(self, scene, references, cams, exact=False, ds=None):
        self.scene = scene
        self.ds = ds or DeviceScene(scene)
        self.cams = list(cams)
        self.refs = [D.to_dev(np.asarray(r, dtype=np.float64)) if not isinstance(r, torch.Tensor)
                     else r.to(self.ds.dg.device, torch.float64) for r in references]
        self.exact = exact
        self.S = self.ds.n_scenes

    def render(self, params, cam, dtype=np.float64, want_state=False):
        return self.ds.render_frame(cam, ("color", "alpha"), None, dtype, want_state=want_state,
                                    light=_light(self.scene, params), lam=params.lam, b=params.b,
                                    palettes=params.c_p, opacity_scales=params.opacity_scale,
                                    exact=self.exact)

    def view_grads(self, params, v, events=None):
        """(loss, packed gradient (4S+10,) float64 device tensor) for view v.
        ``events``: 5 CUDA events around render (K1-K3), loss (K7), K4a, K4b."""
        rec = (lambda j: events[j].record()) if events else (lambda j: None)
        cam, ref = self.cams[v], self.refs[v]
        rec(0)
        F = self.render(params, cam, want_state=True)
        rec(1)
        rgba = F.out64 if F.f64 else F.out.double()
        loss, d = photometric_loss_t(rgba, ref)
        rec(2)
        g = D.blend_backward(F, d, geometry=False)
        rec(3)
        self._last_pairs = F.n_pairs
        shading, edits = F._keep_tabs
        light = _light(self.scene, params)
        out, _ = D.preprocess_backward(self.ds.dg, cam, 4, (0, 3, -1, -1), g=g, shading=shading,
                                       edits=edits, geometry=False, want=("d_c_p", "d_scale", "d_globals"),
                                       per_scene=self.S, light=light)
        rec(4)
        S = self.S
        sig = torch.from_numpy(_sigmoid(params.opacity_raw)).to(out["d_scale"].device)
        gl = out["d_globals"]
        packed = torch.cat([out["d_c_p"][:3 * S], out["d_scale"][:S] * sig, gl[0:4], gl[4:8],
                            gl[8:10] if light.mode == ORBITAL else torch.zeros_like(gl[8:10])])
        return loss, packed

    def unpack(self, packed):
        S = self.S
        p = packed.cpu().numpy() if isinstance(packed, torch.Tensor) else packed
        return {"c_p": p[:3 * S].reshape(S, 3), "opacity_raw": p[3 * S:4 * S],
                "lam": p[4 * S:4 * S + 4], "b": p[4 * S + 4:4 * S + 8],
                "angles": p[4 * S + 8:4 * S + 10]}


def _frozen_fingerprint(scene):
    h = hashlib.sha256()
    for m in scene.models:
        for arr in (m.geometry.mu, m.geometry.q_raw, m.geometry.log_s, m.geometry.o_logit,
                    m.geometry.n_raw, m.shading.delta_c, m.shading.k_a_raw, m.shading.k_d_raw,
                    m.shading.k_s_raw, m.shading.log_beta, m.palette.c_p):
            h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def render_with_transform(scene, params, cam, dtype=np.float32):
    """RGBA render of a composed scene under an appearance transform
    (inverse.py:154-158)."""
    fit = InverseFitter(scene, [], [], exact=True)
    F = fit.render(params, cam, dtype=dtype)
    return D.to_host(F.out64 if F.f64 else F.out).astype(dtype, copy=False)


def reduce_views(total, loss_sum, n_views, dist=None, group=None):
    """Mean over ALL views of the packed gradient and loss: one all-reduce
    (sum) of (4S+10)+1 float64 values when distributed (NCCL on GPU ranks,
    gloo in the CPU tests).  Returns (host gradient vector, loss)."""
    buf = torch.cat([total.reshape(-1), loss_sum.reshape(-1).to(total.dtype)])
    if dist is not None:
        dist.all_reduce(buf, group=group)
    host = (buf / n_views).cpu().numpy()
    return host[:-1], float(host[-1])


def transform_step(params, grads, adam, lr, learnable, angles):
    """The reference's per-iteration update (inverse.py:229-238): Adam on each
    learnable group whose gradient exceeds the 1e-12 floor."""
    floor = 1e-12
    for name in ("c_p", "opacity_raw", "lam", "b"):
        if name in learnable and np.abs(grads[name]).max() > floor:
            adam.step(name, getattr(params, name), grads[name], lr)
    if params.light_mode == ORBITAL and "angles" in learnable and \
            np.abs(grads["angles"]).max() > floor:
        adam.step("angles", angles, grads["angles"], lr)
        params.polar, params.azimuth = float(angles[0]), float(angles[1])


_LEARN_BITS = {"c_p": 1, "opacity_raw": 2, "lam": 4, "b": 8, "angles": 16}


class InverseGraph:
    """Whole inverse iterations replayed as one CUDA graph: every view's
    render (K1-K3), L1+SSIM, K4a, transform-only K4b and gradient pack, then
    the device Adam + table refresh (csrc/inverse.cu).  The transform state
    (x, Adam moments, per-group step counts) and the frame tables live in HBM,
    so an iteration needs no host round trip; ``run`` replays and checks the
    sticky overflow / divergence gate once at the end (growing the pair
    capacity and resuming from the first gated iteration if needed).

    With ``dist`` (views sharded over ranks) an iteration is two graphs: the
    views' compute + pack, then -- after one stream-ordered all-reduce of the
    packed gradient, loss and overflow count (4S+12 float64) -- the update,
    so every rank applies the identical step and gates the same iterations;
    ``view_div`` is the global view count."""

    def __init__(self, fit, params, iters, lr=0.01, learnable=None, headroom=1.3, dist=None,
                 group=None, view_div=None):
        from . import _lib as L
        self.fit, self.L = fit, L
        self.dist, self.group = dist, group
        ds = fit.ds
        dev = ds.dg.device
        self.ws = D.Workspace(dev)
        S, V = fit.S, len(fit.cams)
        N = 4 * S + 10
        self.S, self.V, self.N, self.iters = S, V, N, int(iters)
        learnable = learnable or ("c_p", "opacity_raw", "lam", "b", "angles")
        self.light = _light(fit.scene, params)
        self.orbital = self.light.mode == ORBITAL  # angle gradients packed (view_grads)
        if params.light_mode != ORBITAL:  # ... but only stepped for an orbital transform
            learnable = tuple(k for k in learnable if k != "angles")
        x0 = np.concatenate([params.c_p.reshape(-1), params.opacity_raw, params.lam, params.b,
                             [params.polar, params.azimuth]]).astype(np.float64)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.from_numpy(x0).to(dev)
        self.m, self.v = torch.zeros(N, **f64), torch.zeros(N, **f64)
        self.t = torch.zeros(5, dtype=torch.int64, device=dev)
        self.acc = torch.zeros(N + 2, **f64)  # grad (N), loss sum, overflow count
        self.losses = torch.zeros(self.iters, **f64)
        self.ctl = torch.tensor([0, -1, 0], dtype=torch.int64, device=dev)
        self.nb = nb = ctypes.sizeof(L.FrameParams_t)
        scales = softplus(params.opacity_raw)
        host = bytearray()
        for cam in fit.cams:
            P = D.frame_params(cam, self.light, params.lam, params.b,
                               rescale_opacity=not np.all(scales == 1.0))
            host += bytes(P)
        if not host:  # a rank without views still runs the update
            host = bytearray(nb)
        self.params_dev = torch.frombuffer(host, dtype=torch.uint8).to(dev)
        self.tab = torch.from_numpy(np.concatenate([params.c_p.reshape(-1), scales])).to(dev)
        self._init = [t.clone() for t in (self.x, self.params_dev, self.tab)]
        st = L.InverseStep_t()
        st.n_scenes, st.n_views = S, V
        st.orbital = 1 if self.orbital else 0
        st.learnable = sum(_LEARN_BITS[k] for k in learnable)
        st.iters = self.iters
        st.view_div = float(view_div) if view_div else 0.0
        st.x, st.m, st.v, st.t = (self.x.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                  self.t.data_ptr())
        st.lr, st.beta1, st.beta2, st.eps = float(lr), 0.9, 0.999, 1e-15
        st.grad, st.loss_sum = self.acc.data_ptr(), self.acc[N:].data_ptr()
        st.losses, st.ctl = self.losses.data_ptr(), self.ctl.data_ptr()
        st.params, st.tab = self.params_dev.data_ptr(), self.tab.data_ptr()
        self.st = st
        self.shading = D.shading_struct(ds.dg, self.tab[:3 * S], False, self.light, params.lam,
                                        params.b)
        self.edits = L.Edits_t()
        self.edits.scene_id = ds.dg.scene_id.data_ptr()
        self.edits.opacity_scale = self.tab[3 * S:].data_ptr()
        # pair capacity from one synchronous render per view (+ headroom)
        peak = 0
        for cam in fit.cams:
            F = fit.render(params, cam, want_state=False)
            peak = max(peak, int(F.n_pairs.item()))
        self.capacity = max(int(peak * headroom) + 4096, 1 << 16)
        self._capture()

    def _views(self, events=None):
        """Every view: render, loss, backward, pack into self.acc.  ``events``
        (eager diagnostics, outside capture): 7 CUDA events recorded around
        K1, K2, K3, K7, K4a, K4b + pack of the first view."""
        L, fit, ds = self.L, self.fit, self.fit.ds
        ws = self.ws  # owned: eager renders on ds.ws cannot move captured buffers
        for v, cam in enumerate(fit.cams):
            rec = (lambda j: events[j].record()) if events and v == 0 else (lambda j: None)
            pdev = self.params_dev[v * self.nb:(v + 1) * self.nb]
            rec(0)
            F = D.preprocess(ds.dg, cam, 4, (0, 3, -1, -1), ws, self.shading, self.edits, None, (),
                             True, params_dev=pdev)
            rec(1)
            D.bin_sort(F, ws, capacity=self.capacity)
            rec(2)
            D.blend(F, ws, want_state=True, exact=fit.exact)
            rec(3)
            h, w, nc = F.out64.shape
            win = 11
            sums, d = _photometric_dev(F.out64, fit.refs[v], 0.8 / F.out64.numel(), -0.2, True)
            rec(4)
            g = D.blend_backward(F, d, geometry=False)
            rec(5)
            self._last_pairs = F.n_pairs
            out, _ = D.preprocess_backward(ds.dg, cam, 4, (0, 3, -1, -1), g=g, shading=self.shading,
                                           edits=self.edits, params_dev=pdev, geometry=False,
                                           want=("d_c_p", "d_scale", "d_globals"), per_scene=self.S,
                                           light=self.light)
            L.check(L.lib().ivr_inverse_pack(
                ctypes.byref(self.st), sums.data_ptr(), float(h * w * nc),
                float((h - win + 1) * (w - win + 1) * nc), out["d_c_p"].data_ptr(),
                out["d_scale"].data_ptr(), out["d_globals"].data_ptr(), F.n_pairs.data_ptr(),
                self.capacity, D.stream_handle()), "ivr_inverse_pack")
            rec(6)

    def _update(self):
        L = self.L
        L.check(L.lib().ivr_inverse_update(ctypes.byref(self.st), D.stream_handle()),
                "ivr_inverse_update")

    def _reduce(self):
        """Sum the packed gradient, loss and overflow count over the ranks
        (stream-ordered, no host synchronisation)."""
        if self.dist is not None:
            self.dist.all_reduce(self.acc, group=self.group)

    def _capture(self):
        saved = [t.clone() for t in (self.x, self.m, self.v, self.t, self.acc, self.losses,
                                     self.ctl, self.params_dev, self.tab)]
        self._views()  # sizes every workspace buffer before capture
        self._reduce()
        self._update()
        torch.cuda.synchronize()
        for t, s0 in zip((self.x, self.m, self.v, self.t, self.acc, self.losses, self.ctl,
                          self.params_dev, self.tab), saved):
            t.copy_(s0)
        torch.cuda.synchronize()
        self.g = torch.cuda.CUDAGraph()
        if self.dist is None:
            with torch.cuda.graph(self.g):
                self._views()
                self._update()
        else:  # the collective stays outside the graphs
            self.g2 = torch.cuda.CUDAGraph()
            if self.V:
                with torch.cuda.graph(self.g):
                    self._views()
            with torch.cuda.graph(self.g2):
                self._update()
        torch.cuda.synchronize()

    def replay(self):
        """One iteration (a rank without views only joins the all-reduce)."""
        if self.dist is None:
            self.g.replay()
            return
        if self.V:
            self.g.replay()
        self._reduce()
        self.g2.replay()

    def run(self):
        """All iterations; returns (TransformParams fields as numpy, losses)."""
        start = 0
        while True:
            for _ in range(self.iters - start):
                self.replay()
            ctl = self.ctl.cpu().numpy()
            first, reason = int(ctl[1]), int(ctl[2])
            if first < 0:
                break
            if reason & self.L.INV_OVERFLOW:
                self.capacity *= 2
                self.ctl.copy_(torch.tensor([first, -1, 0], dtype=torch.int64))
                self._capture()
                start = first
                continue
            raise DivergedLoss(f"loss became {float(self.losses[first])}")
        return self.x.cpu().numpy(), self.losses.cpu().numpy().tolist()


def optimize_to_reference(scene, params, reference_rgba, reference_cam, iters=1000, lr=0.01,
                          callback=None, learnable=None, group=None, exact=False):
    """Fit the transform to reference image(s) with Adam on L1 + SSIM
    (inverse.py:205-244).  Returns (fitted params, per-iteration losses).

    ``reference_rgba`` / ``reference_cam`` may be lists (multi-view mean loss).
    With torch.distributed initialised (or ``group`` given) and more than one
    rank, each rank passes ITS views; gradients are all-reduced (sum) once per
    iteration and divided by the global view count."""
    refs = reference_rgba if isinstance(reference_rgba, (list, tuple)) else [reference_rgba]
    cams = reference_cam if isinstance(reference_cam, (list, tuple)) else [reference_cam]
    if len(refs) != len(cams):
        raise ShapeMismatch("one camera per reference image required")
    params = params.copy()
    before = _frozen_fingerprint(scene)
    learnable = learnable or ("c_p", "opacity_raw", "lam", "b", "angles")
    fit = InverseFitter(scene, refs, cams, exact=exact)
    dist = None
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        if torch.distributed.get_world_size(group) > 1:
            dist = torch.distributed
    n_views = torch.tensor([float(len(refs))], dtype=torch.float64, device=fit.ds.dg.device)
    if dist:
        dist.all_reduce(n_views, group=group)
    n_views = float(n_views.item())
    use_graph = os.environ.get("IVR_INVERSE_GRAPH", "1") != "0" and callback is None and iters > 0
    if dist:  # one decision for all ranks: the two paths issue different collectives
        flag = torch.tensor([1.0 if use_graph else 0.0], dtype=torch.float64,
                            device=fit.ds.dg.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        use_graph = bool(flag.item() > 0.5)
    if use_graph:
        # whole iterations replay as CUDA graphs (no host round trip); sharded
        # views add one stream-ordered all-reduce per iteration
        G = InverseGraph(fit, params, iters, lr, learnable, dist=dist, group=group,
                         view_div=n_views)
        x, losses = G.run()
        S = fit.S
        params.c_p = x[:3 * S].reshape(S, 3).copy()
        params.opacity_raw = x[3 * S:4 * S].copy()
        params.lam, params.b = x[4 * S:4 * S + 4].copy(), x[4 * S + 4:4 * S + 8].copy()
        if params.light_mode == ORBITAL:
            params.polar, params.azimuth = float(x[4 * S + 8]), float(x[4 * S + 9])
        after = _frozen_fingerprint(scene)
        assert before == after, "primitive attributes changed during inverse fitting"
        return params, losses
    adam = Adam(eps=1e-15)
    angles = np.array([params.polar, params.azimuth])
    losses = []
    for it in range(1, iters + 1):
        total = None
        loss_sum = torch.zeros(1, dtype=torch.float64, device=fit.ds.dg.device)
        for v in range(len(refs)):
            loss, packed = fit.view_grads(params, v)
            total = packed if total is None else total + packed
            loss_sum = loss_sum + loss
        if total is None:
            total = torch.zeros(4 * fit.S + 10, dtype=torch.float64, device=fit.ds.dg.device)
        mean, loss = reduce_views(total, loss_sum, n_views, dist, group)
        if not np.isfinite(loss):
            raise DivergedLoss(f"loss became {loss}")
        losses.append(loss)
        transform_step(params, fit.unpack(mean), adam, lr, learnable, angles)
        if callback is not None:
            callback(it, loss, params)
    after = _frozen_fingerprint(scene)
    assert before == after, "primitive attributes changed during inverse fitting"
    return params, losses


def inverse_step(scene, params, cam, reference, exact=False):
    """One inverse._step (inverse.py:161-190): (loss, grads dict)."""
    fit = InverseFitter(scene, [reference], [cam], exact=exact)
    loss, packed = fit.view_grads(params, 0)
    return float(loss), fit.unpack(packed)
