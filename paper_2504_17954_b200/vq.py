"""Scalar-codebook vector quantization (drop-in for voxsplat/vq.py).

Assignment (K5) and decode (K6) run on the GPU; both are HBM-bound kernels
(1-D codebooks: nearest codeword = binary search over float64 midpoints,
bit-identical to np.searchsorted(mids, v, 'left'), vq.py:90-96).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import CorruptIndex, EmptyInput, OutOfRange

DEFAULT_CODEBOOK_SIZE = 256
KMEANS_MAX_ITERS = 50
KMEANS_SHIFT_TOL = 1e-6

QUANTIZED_ATTRIBUTES = (
    ("q_raw", "geometry"), ("log_s", "geometry"), ("o_logit", "geometry"),
    ("delta_c", "shading"), ("k_a_raw", "shading"), ("k_d_raw", "shading"),
    ("k_s_raw", "shading"), ("log_beta", "shading"),
)


def assign_device(values_dev, centroids_dev):
    """GPU nearest-centroid index (uint16 stored in int16 tensor)."""
    n = values_dev.numel()
    k = centroids_dev.numel()
    out = torch.empty(n, dtype=torch.int16, device=values_dev.device)
    nb = L.lib().ivr_vq_assign_workspace_size()
    ws = _WS.get(values_dev.device)
    if ws is None:
        ws = _WS[values_dev.device] = torch.empty(nb, dtype=torch.uint8, device=values_dev.device)
    L.check(L.lib().ivr_vq_assign(D.ptr(values_dev), n, D.ptr(centroids_dev), k, D.ptr(out),
                                  D.ptr(ws), nb, D.stream_handle()), "ivr_vq_assign")
    return out


_WS = {}


def decode_device(idx_dev, centroids_dev):
    """GPU codebook gather; raises CorruptIndex on an out-of-range index."""
    n = idx_dev.numel()
    k = centroids_dev.numel()
    out = torch.empty(n, dtype=torch.float64, device=idx_dev.device)
    bad = torch.full((1,), -1, dtype=torch.int64, device=idx_dev.device)
    L.check(L.lib().ivr_vq_decode(D.ptr(idx_dev), n, D.ptr(centroids_dev), k, D.ptr(out),
                                  D.ptr(bad), D.stream_handle()), "ivr_vq_decode")
    return out, bad


def assign_nearest(values, centroids):
    """Index of the nearest sorted centroid for each value (vq.py:90-96)."""
    values = np.asarray(values, dtype=np.float64)
    centroids = np.asarray(centroids, dtype=np.float64).reshape(-1)
    if centroids.size == 1:
        return np.zeros(values.shape, dtype=np.int64)
    if centroids.size > 65536:
        raise OutOfRange("codebooks above 65536 entries are not supported")
    if values.size == 0:
        return np.zeros(values.shape, dtype=np.int64)
    idx = assign_device(D.to_dev(values.reshape(-1)), D.to_dev(centroids))
    return D.to_host(idx).view(np.uint16).astype(np.int64).reshape(values.shape)


def _index_dtype(k):
    return np.uint8 if k <= 256 else np.uint16


@dataclass
class Codebook:
    """Sorted scalar centroids for one attribute (shared by its components)."""

    name: str
    centroids: np.ndarray

    def __post_init__(self):
        self.centroids = np.asarray(self.centroids, dtype=np.float64).reshape(-1)
        if self.centroids.size < 1:
            raise EmptyInput(f"codebook {self.name!r} is empty")
        if np.any(np.diff(self.centroids) < 0):
            raise OutOfRange(f"codebook {self.name!r} centroids must be sorted")

    @property
    def k(self):
        return self.centroids.size

    @property
    def index_dtype(self):
        return _index_dtype(self.k)

    def encode(self, values):
        return assign_nearest(values, self.centroids).astype(self.index_dtype)

    def decode(self, indices):
        indices = np.asarray(indices)
        if indices.size == 0:
            return np.zeros(indices.shape)
        if indices.dtype not in (np.uint8, np.uint16) and int(indices.max()) >= self.k:
            # wider or signed index types: a value >= 2^16 would wrap below
            raise CorruptIndex(f"codebook {self.name!r}: index {int(indices.max())} >= K={self.k}")
        if indices.dtype not in (np.uint8, np.uint16) and int(indices.min()) < 0:
            # the reference indexes centroids[indices] with numpy semantics:
            # -k <= i < 0 counts from the end, below that numpy's IndexError
            if int(indices.min()) < -self.k:
                raise IndexError(f"index {int(indices.min())} is out of bounds for axis 0 "
                                 f"with size {self.k}")
            indices = np.where(indices < 0, indices + self.k, indices)
        flat = np.ascontiguousarray(indices.reshape(-1)).astype(np.uint16, copy=False)
        idx = D.to_dev(flat.view(np.int16), torch.int16)  # out-of-range: the device check
        out, bad = decode_device(idx, D.to_dev(self.centroids))
        if int(bad.item()) >= 0:
            raise CorruptIndex(f"codebook {self.name!r}: index {int(bad.item())} >= K={self.k}")
        return D.to_host(out).reshape(indices.shape)


def kmeans(samples, k, seed=0, restarts=5):
    """Scalar k-means: k-means++ restarts + Lloyd, lowest SSE wins
    (vq.py:31-87).  Returns sorted distinct centroids."""
    samples = np.asarray(samples, dtype=np.float64).reshape(-1)
    if samples.size == 0:
        raise EmptyInput("kmeans needs at least one sample")
    if k < 1:
        raise OutOfRange("codebook size must be >= 1")
    return _kmeans_dev(D.to_dev(samples), k, seed, restarts)


def _kmeans_dev(x, k, seed=0, restarts=5):
    """kmeans on a float64 device vector (numpy centroids out)."""
    distinct = torch.unique(x)  # sorted
    if distinct.numel() <= k:
        return distinct.cpu().numpy()
    rng = np.random.default_rng(seed)
    n = x.numel()
    if not _sorted_seeding(n, k):
        best, best_sse = None, np.inf
        for _ in range(restarts):
            c = _lloyd(x, _seed_plusplus(x, k, rng))
            sse = _sse(x, c)
            if sse < best_sse:
                best, best_sse = c, sse
        return torch.unique(best).cpu().numpy()
    order = _value_order(x)  # shared by the restarts' seedings
    seeds = _seed_batch([(x, order, f, u) for f, u in _draw_seeds(n, k, rng, restarts)], k)
    return _kmeans_finish(x, order, seeds)


def _sse(x, c):
    idx = _assign_idx(x, c)
    return float(((x - c[idx]) ** 2).sum())


def _kmeans_finish(x, order, seeds):
    """Lloyd for every restart's seeding (one loop, sorted values), then the
    lowest-SSE restart (the first on ties), as vq.py:47-57."""
    fitted = _lloyd_sets(x, x[order.long()], torch.stack(list(seeds)))
    best, best_sse = None, np.inf
    for r in range(fitted.shape[0]):
        sse = _sse(x, fitted[r])
        if sse < best_sse:
            best, best_sse = fitted[r], sse
    return torch.unique(best).cpu().numpy()


SEED_SORTED_MAX_K = 32768
SEED_SORTED_MAX_P = 64  # seedings per ivr_kmeans_seed_sorted launch


def _value_order(x):
    """int32 permutation sorting x ascending (the value order the sorted
    seeding walks), or None where that path does not apply."""
    if x.numel() >= 2 ** 31:
        return None
    return torch.argsort(x).to(torch.int32)


def _sorted_seeding(n, k):
    return k <= SEED_SORTED_MAX_K and n < 2 ** 31


def _draw_seeds(n, k, rng, restarts):
    """The restarts' draws in the reference's order: per restart rng.integers
    for the first centre, then k - 1 rng.random() (one per rng.choice).  They
    do not depend on the data, and the distinct-value shortcut in kmeans means
    no seeding runs out of mass early (which would leave draws unconsumed in
    the reference)."""
    out = []
    for _ in range(restarts):
        first = int(rng.integers(n))
        out.append((first, rng.random(k - 1)))  # k == 1: no draw, as the reference
    return out


def _seed_batch(problems, k):
    """ivr_kmeans_seed_sorted over independent seedings: problems = [(x, order,
    first, u_host)] (values on the device, int32 value order); up to 64 per
    launch.  Returns one (k,) centre tensor per problem."""
    out = []
    for p0 in range(0, len(problems), SEED_SORTED_MAX_P):
        chunk = problems[p0:p0 + SEED_SORTED_MAX_P]
        dev = chunk[0][0].device
        u = torch.from_numpy(np.concatenate([p[3] for p in chunk] + [np.zeros(1)])).to(dev)
        cents = torch.empty((len(chunk), k), dtype=torch.float64, device=dev)
        arr = (L.SeedProblem_t * len(chunk))()
        for i, (x, order, first, _) in enumerate(chunk):
            arr[i].values, arr[i].order, arr[i].n = D.ptr(x), D.ptr(order), x.numel()
            arr[i].first, arr[i].centers = first, D.ptr(cents[i])
            arr[i].u = u.data_ptr() + 8 * (k - 1) * i
        nb = int(L.lib().ivr_kmeans_seed_sorted_workspace_size(arr, len(chunk)))
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        L.check(L.lib().ivr_kmeans_seed_sorted(arr, len(chunk), int(k), D.ptr(ws), nb,
                                               D.stream_handle()), "ivr_kmeans_seed_sorted")
        out.extend(cents.unbind(0))
    return out


def _seed_restarts(x, k, rng, restarts, order=None):
    """All of k-means' restart seedings of one attribute in one
    ivr_kmeans_seed_sorted launch.  Returns (restarts, k) centres, or None
    where the sorted seeding does not apply."""
    n = x.numel()
    if not _sorted_seeding(n, k):
        return None
    if order is None:
        order = _value_order(x)
    return torch.stack(_seed_batch([(x, order, f, u) for f, u in _draw_seeds(n, k, rng, restarts)],
                                   k))


def _seed_plusplus(x, k, rng, order=None):
    """k-means++ seeding on the device (vq.py:60-72) with the reference's
    random stream: rng.integers for the first centre, then one rng.random()
    per rng.choice(p = d2 / sum d2) -- the first index (in sample order) whose
    cumulative d2 exceeds u * sum d2.  ivr_kmeans_seed_sorted (one
    cooperative kernel; d2 lowered only between the adjacent chosen centres
    in value order) when k <= 32768 and n < 2^31, else ivr_kmeans_seed (two
    kernels per centre over every sample)."""
    n = x.numel()
    if _sorted_seeding(n, k):
        return _seed_restarts(x, k, rng, 1, order)[0]
    first = int(rng.integers(n))
    u = torch.from_numpy(rng.random(k - 1)).to(x.device)  # k == 1: no draw, as the reference
    c = torch.empty(k, dtype=torch.float64, device=x.device)
    nb = int(L.lib().ivr_kmeans_seed_workspace_size(n))
    ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    L.check(L.lib().ivr_kmeans_seed(D.ptr(x), n, int(k), first, D.ptr(u), D.ptr(c), D.ptr(ws), nb,
                                    D.stream_handle()), "ivr_kmeans_seed")
    return c


def _assign_idx(x, c):
    if c.numel() == 1:
        return torch.zeros(x.numel(), dtype=torch.int64, device=x.device)
    return assign_device(x, c.contiguous()).view(torch.uint16).to(torch.int64)


def _lloyd(x, c):
    """Lloyd iterations on the device (vq.py:75-87): assign with K5, centroid
    update with bincount sums (float64)."""
    scale = max(float(x.abs().max()), 1e-12)
    k = c.numel()
    fused = 2 <= k <= 4097
    if fused:
        nb = L.lib().ivr_kmeans_lloyd_workspace_size(k)
        ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
        shift_d = torch.empty(1, dtype=torch.float64, device=x.device)
    for _ in range(KMEANS_MAX_ITERS):
        c = torch.sort(c).values
        if fused:  # assign + sums + counts + update in one pass (csrc/vq.cu)
            new = torch.empty_like(c)
            L.check(L.lib().ivr_kmeans_lloyd_step(D.ptr(x), x.numel(), D.ptr(c), k, D.ptr(new),
                                                  D.ptr(shift_d), D.ptr(ws), nb,
                                                  D.stream_handle()), "ivr_kmeans_lloyd_step")
            shift = float(shift_d.item()) / scale
        else:
            idx = _assign_idx(x, c)
            sums = torch.bincount(idx, weights=x, minlength=k)
            cnt = torch.bincount(idx, minlength=k)
            new = torch.where(cnt > 0, sums / torch.clamp(cnt, min=1).to(torch.float64), c)
            shift = float((new - c).abs().max()) / scale
        c = new
        if shift < KMEANS_SHIFT_TOL:
            break
    return torch.sort(c).values


def _lloyd_sets(x, xs, seeds):
    """Lloyd iterations (vq.py:75-87) of every restart at once on the sorted
    values xs (ivr_kmeans_lloyd_step_sorted: segment sums between the
    midpoints, all sets in one launch, one host read of the shifts per
    iteration); each set stops at its own convergence or after
    KMEANS_MAX_ITERS, exactly as its own loop would.  Returns (R, k) sorted
    centroids."""
    R, k = seeds.shape
    scale = max(float(x.abs().max()), 1e-12)
    c = torch.sort(seeds, dim=1).values
    if k < 2:
        return c
    nb = int(L.lib().ivr_kmeans_lloyd_sorted_workspace_size(k, R))
    ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    shift = torch.empty(R, dtype=torch.float64, device=x.device)
    active = list(range(R))
    for _ in range(KMEANS_MAX_ITERS):
        cur = c[active].contiguous() if len(active) < R else c
        cur = torch.sort(cur, dim=1).values
        new = torch.empty_like(cur)
        na = len(active)
        L.check(L.lib().ivr_kmeans_lloyd_step_sorted(D.ptr(xs), xs.numel(), D.ptr(cur), k, na,
                                                     D.ptr(new), D.ptr(shift), D.ptr(ws), nb,
                                                     D.stream_handle()),
                "ivr_kmeans_lloyd_step_sorted")
        sh = shift[:na].cpu().numpy() / scale
        c[active] = new
        active = [r for r, v in zip(active, sh) if not v < KMEANS_SHIFT_TOL]
        if not active:
            break
    return torch.sort(c, dim=1).values


def quantize_attributes(arrays, k=DEFAULT_CODEBOOK_SIZE, seed=0, restarts=5):
    """vq.py:137-147: per attribute, kmeans over all its components, then the
    indices (Codebook.encode's values).  One upload per attribute; every
    attribute's restart seedings share one ivr_kmeans_seed_sorted launch (each
    attribute draws from its own default_rng(seed), as the reference's
    per-attribute kmeans call); indices come back in the index dtype."""
    if k < 1:
        raise OutOfRange("codebook size must be >= 1")
    prep, problems = [], []
    for name, arr in arrays.items():
        arr = np.asarray(arr, dtype=np.float64)
        if arr.size == 0:
            raise EmptyInput("kmeans needs at least one sample")
        x = D.to_dev(arr.reshape(-1))
        distinct = torch.unique(x)
        if distinct.numel() <= k:
            prep.append((name, arr, x, distinct.cpu().numpy(), None, 0))
        elif not _sorted_seeding(x.numel(), k):
            prep.append((name, arr, x, _kmeans_dev(x, k, seed, restarts), None, 0))
        else:
            order = _value_order(x)
            draws = _draw_seeds(x.numel(), k, np.random.default_rng(seed), restarts)
            prep.append((name, arr, x, None, order, len(problems)))
            problems.extend((x, order, f, u) for f, u in draws)
    seeds = _seed_batch(problems, k) if problems else []
    out = {}
    for name, arr, x, cents, order, p0 in prep:
        if cents is None:
            cents = _kmeans_finish(x, order, seeds[p0:p0 + restarts])
        cb = Codebook(name, cents)
        if cb.k == 1:
            idx = np.zeros(arr.shape, dtype=cb.index_dtype)
        else:
            idx = D.to_host(assign_device(x, D.to_dev(cb.centroids))).view(np.uint16)
            idx = idx.astype(cb.index_dtype, copy=False).reshape(arr.shape)
        out[name] = (cb, idx)
    return out


def quantize_model(model, k=DEFAULT_CODEBOOK_SIZE, seed=0):
    """Codebook-compress an editable model (vq.py:150-176)."""
    from .scene import STAGE_EDITABLE, BasicSceneModel
    if model.stage != STAGE_EDITABLE:
        raise OutOfRange("only editable-stage models are quantized")
    if model.quantized is not None:
        return model.copy()
    arrays = {name: np.asarray(getattr(getattr(model, owner), name))
              for name, owner in QUANTIZED_ATTRIBUTES}
    quant = quantize_attributes(arrays, k=k, seed=seed)
    geom = model.geometry.copy()
    geom.q_raw = quant["q_raw"][0].decode(quant["q_raw"][1])
    geom.log_s = quant["log_s"][0].decode(quant["log_s"][1])
    geom.o_logit = quant["o_logit"][0].decode(quant["o_logit"][1])
    return BasicSceneModel(stage=STAGE_EDITABLE, geometry=geom, shading=None,
                           palette=model.palette.copy(), quantized=quant,
                           metadata=dict(model.metadata))


def dequantize_model(model):
    """Materialise a plain editable model from a quantized one (vq.py:179-210)."""
    from .scene import STAGE_EDITABLE, BasicSceneModel
    from .shading import ShadingAttributes
    if model.quantized is None:
        return model.copy()
    q = model.quantized

    def dec(name):
        cb, idx = q[name]
        return cb.decode(idx)

    geom = model.geometry.copy()
    geom.q_raw, geom.log_s, geom.o_logit = dec("q_raw"), dec("log_s"), dec("o_logit")
    shading = ShadingAttributes(dec("delta_c"), dec("k_a_raw"), dec("k_d_raw"), dec("k_s_raw"),
                                dec("log_beta"))
    return BasicSceneModel(stage=STAGE_EDITABLE, geometry=geom, shading=shading,
                           palette=model.palette.copy(), quantized=None,
                           metadata=dict(model.metadata))
