"""Render entry points: the drop-in for render.py of the reference.

``render_frame`` / ``render_reference`` / ``render_pagetable_only`` /
``render_classic_octree`` keep the reference signatures (``render.py:236-262``) and return the same ``FrameOutput`` (numpy image,
ordered brick / metadata request lists, usage mask, level histogram,
per-pixel brick switches, stats).  Underneath, one call is:

  host: pack channels + LOD/step tables (render.py:101-122, µs)
  GPU : k_raycast (kernel 1), then request ordering + budget (kernel 3a)
  D2H : image, usage mask, histogram, counters, <= budget request entries

``render_frame_device`` is the same pass without the host copies; the
Session uses it so the usage mask feeds ``note_sampled`` on the device.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .camera import Camera, ray_basis
from .octree import ResidencyOctree
from .paging import MultiChannelPaging
from .transfer import TransferFunction

MODE_RESIDENCY = N.RO_MODE_RESIDENCY
MODE_REFERENCE = N.RO_MODE_REFERENCE
MODE_PAGETABLE = N.RO_MODE_PAGETABLE
MODE_CLASSIC = N.RO_MODE_CLASSIC


class RenderError(ValueError):
    pass


@dataclass(frozen=True)
class ChannelSettings:
    """One active channel; list order is importance order."""
    slot: int
    tf: TransferFunction
    level_range: tuple = (0, 15)

    def __post_init__(self):
        if self.level_range[0] > self.level_range[1]:
            raise RenderError(f"level range {self.level_range} inverted")


@dataclass(frozen=True)
class RenderConfig:
    image_dims: tuple = (256, 256)
    base_step: float = 1.0 / 256.0
    lod_reference_distance: float = 1.0
    early_term_alpha: float = 0.99
    max_requests_per_frame: int = 256
    traversal_start_level: int = 2
    homogeneity_eps: float = 0.0

    def __post_init__(self):
        if self.base_step <= 0.0:
            raise RenderError("base step must be positive")
        if self.lod_reference_distance <= 0.0:
            raise RenderError("lod reference distance must be positive")
        if not 0.0 < self.early_term_alpha <= 1.0:
            raise RenderError("early termination alpha outside (0, 1]")
        if self.max_requests_per_frame < 1:
            raise RenderError("request budget must be positive")
        if self.traversal_start_level < 0:
            raise RenderError("traversal start level must be >= 0")


@dataclass
class FrameStats:
    traversal_steps: int = 0
    samples_evaluated: int = 0
    samples_skipped: int = 0
    skip_violations: int = 0
    required_bricks: int = 0
    required_bytes: int = 0
    requests_issued: int = 0
    render_ms: float = 0.0
    livelocked_rays: int = 0


@dataclass
class FrameOutput:
    image: np.ndarray
    brick_requests: list
    metadata_requests: list
    stats: FrameStats
    required_mask: np.ndarray = field(repr=False, default=None)
    level_histogram: np.ndarray = field(repr=False, default=None)
    pixel_required: np.ndarray = field(repr=False, default=None)
    required_mask_device: torch.Tensor = field(repr=False, default=None)


# ---------------------------------------------------------------------------
# host tables
# ---------------------------------------------------------------------------

_LOD_THRESHOLDS = None


def lod_thresholds() -> list:
    """T[L] = smallest ratio >= 1 with floor(log2(ratio)) >= L, found with
    the platform libm log2 -- the function kernels.py:49 calls."""
    global _LOD_THRESHOLDS
    if _LOD_THRESHOLDS is None:
        out = [1.0]
        for L in range(1, N.RO_MAX_LEVELS):
            r = float(2 ** L)
            if math.floor(math.log2(r)) < L:
                raise RuntimeError("libm log2 is not exact at powers of two")
            while True:
                p = math.nextafter(r, 0.0)
                if math.floor(math.log2(p)) >= L:
                    r = p
                else:
                    break
            out.append(r)
        out.append(float("inf"))
        _LOD_THRESHOLDS = out
    return _LOD_THRESHOLDS


def traversal_depth(step: float, max_depth: int) -> int:
    """kernels.py:57-66"""
    if step >= 1.0:
        return 0
    d = int(math.floor(math.log2(1.0 / step)))
    return min(max(d, 0), max_depth)


def choose_resolution_level(t, t0, lo=0, hi=15) -> int:
    """kernels.py:43-54 (host mirror)."""
    ratio = t / t0
    lev = 0 if ratio < 1.0 else int(math.floor(math.log2(ratio)))
    return min(max(lev, lo), hi)


def choose_traversal_depth(step, max_depth) -> int:
    return traversal_depth(step, max_depth)


@functools.lru_cache(maxsize=256)
def _channel_block(slot: int, lo: int, hi: int, tf: TransferFunction) -> N.Channel:
    """ro_channel of one visible channel (render.py:101-122 packing), built
    once per (slot, level range, transfer function)."""
    ch = N.Channel()
    ch.slot, ch.lo, ch.hi = slot, lo, hi
    ch.npoints = len(tf.points)
    xs = np.zeros(N.RO_MAX_TF_POINTS, dtype=np.float64)
    rgba = np.zeros((N.RO_MAX_TF_POINTS, 4), dtype=np.float64)
    for j, (x, c) in enumerate(tf.points):
        xs[j] = float(x)
        rgba[j] = [float(v) for v in c]
    C.memmove(ch.tf_x, xs.ctypes.data, xs.nbytes)
    C.memmove(ch.tf_rgba, rgba.ctypes.data, rgba.nbytes)
    eb = np.ascontiguousarray(tf.empty_below(), dtype=np.uint16)
    C.memmove(ch.empty_below, eb.ctypes.data, eb.nbytes)
    ch.zero_upto = tf.zero_upto()
    # kernel TF search start: first segment whose right knot is >= j
    n = len(tf.points)
    seg = np.searchsorted(xs[1:max(n - 1, 1)], np.arange(256, dtype=np.float64), side="left")
    seg = np.minimum(seg, max(n - 2, 0)).astype(np.uint8)
    C.memmove(ch.tf_seg, seg.ctypes.data, seg.nbytes)
    return ch


@functools.lru_cache(maxsize=256)
def _channel_descs(key) -> "C.Array":
    """ro_channel_desc[] of a channel list, built once per list."""
    descs = (N.ChannelDesc * len(key))()
    for i, (slot, (lo, hi), tf) in enumerate(key):
        d = descs[i]
        d.slot, d.level_lo, d.level_hi = slot, lo, hi
        d.npoints = len(tf.points)
        for j, (x, rgba) in enumerate(tf.points):
            d.x[j] = float(x)
            for q in range(4):
                d.rgba[j][q] = float(rgba[q])
    return descs


def _pack_frame(mode, paging: MultiChannelPaging, channels, camera: Camera,
                config: RenderConfig, depth: int, eps_h: float,
                reference_paging: MultiChannelPaging | None = None,
                partition=(1, 0, 8), classic: "ClassicMetadata | None" = None) -> N.Frame:
    """The product packing: ro_pack_frame (csrc/pack.cu) fills the frame in
    native code (camera basis, LOD thresholds, step / depth tables, channel
    blocks); _pack_frame_py below is its Python restatement, kept byte-equal
    by tests/test_host_logic.py."""
    if not channels:
        raise RenderError("need at least one active channel")
    if len(channels) > N.RO_MAX_CH:
        raise RenderError(f"at most {N.RO_MAX_CH} active channels")
    for c in channels:
        if not 0 <= c.slot < paging.config.m:
            raise RenderError(f"channel slot {c.slot} out of range")
        if len(c.tf.points) > N.RO_MAX_TF_POINTS:
            raise RenderError(f"transfer function with > {N.RO_MAX_TF_POINTS} points")
    w, h = config.image_dims
    cam = N.CameraDesc((C.c_double * 3)(*camera.position), (C.c_double * 3)(*camera.target),
                       (C.c_double * 3)(*camera.up), float(camera.fov_deg))
    rc = N.RenderConfigDesc(int(w), int(h), float(config.base_step),
                            float(config.lod_reference_distance),
                            float(config.early_term_alpha), int(config.traversal_start_level), 0)
    descs = _channel_descs(tuple((c.slot, tuple(c.level_range), c.tf) for c in channels))
    F = N.Frame()
    N.check(N.lib().ro_pack_frame(paging.config.k, paging.config.m, depth, mode, C.byref(cam),
                                  C.byref(rc), descs, len(channels), float(eps_h), C.byref(F)))
    F.n_parts, F.part, F.tile_rows = partition
    if reference_paging is not None:
        F.check_skips = 1
        F.ref_pt = reference_paging.pt.data_ptr()
        F.ref_cache = reference_paging.cache_dev.data_ptr()
    if classic is not None:
        F.cls_depth = classic.depth
        F.cls_min = classic.min_arr.data_ptr()
        F.cls_max = classic.max_arr.data_ptr()
    return F


def _pack_frame_py(mode, paging: MultiChannelPaging, channels, camera: Camera,
                   config: RenderConfig, depth: int, eps_h: float,
                   reference_paging: MultiChannelPaging | None = None,
                   partition=(1, 0, 8), classic: "ClassicMetadata | None" = None) -> N.Frame:
    """Python restatement of ro_pack_frame (render.py:101-122 packing)."""
    if not channels:
        raise RenderError("need at least one active channel")
    if len(channels) > N.RO_MAX_CH:
        raise RenderError(f"at most {N.RO_MAX_CH} active channels")
    k = paging.config.k
    w, h = config.image_dims
    F = N.Frame()
    F.mode = mode
    F.n_ch = len(channels)
    F.width, F.height = int(w), int(h)
    b = ray_basis(camera, w, h)
    for a in range(3):
        F.cam_pos[a] = b.pos[a]
        F.cam_fwd[a] = b.fwd[a]
        F.cam_right[a] = b.right[a]
        F.cam_up[a] = b.up[a]
    F.tan_half, F.aspect = b.tan_half, b.aspect
    F.base_step = config.base_step
    F.t0 = config.lod_reference_distance
    F.early_alpha = config.early_term_alpha
    F.eps_h = eps_h
    F.start_level = config.traversal_start_level
    for i, t in enumerate(lod_thresholds()):
        F.lod_threshold[i] = t
    los, his = [], []
    for i, c in enumerate(channels):
        if not 0 <= c.slot < paging.config.m:
            raise RenderError(f"channel slot {c.slot} out of range")
        lo = max(0, min(c.level_range[0], k - 1))
        hi = max(0, min(c.level_range[1], k - 1))
        los.append(lo)
        his.append(hi)
        if len(c.tf.points) > N.RO_MAX_TF_POINTS:
            raise RenderError(f"transfer function with > {N.RO_MAX_TF_POINTS} points")
        F.ch[i] = _channel_block(c.slot, lo, hi, c.tf)
    for raw in range(N.RO_MAX_LEVELS):
        maxlev = 0
        for lo, hi in zip(los, his):
            lev = min(max(raw, lo), hi)
            maxlev = max(maxlev, lev)
        step = config.base_step * (1 << maxlev)
        F.maxlev_tab[raw] = maxlev
        F.step_tab[raw] = step
        F.dt_tab[raw] = traversal_depth(step, depth)
    F.n_parts, F.part, F.tile_rows = partition
    if reference_paging is not None:
        F.check_skips = 1
        F.ref_pt = reference_paging.pt.data_ptr()
        F.ref_cache = reference_paging.cache_dev.data_ptr()
    if classic is not None:
        F.cls_depth = classic.depth
        F.cls_min = classic.min_arr.data_ptr()
        F.cls_max = classic.max_arr.data_ptr()
    return F


# ---------------------------------------------------------------------------
# device frame
# ---------------------------------------------------------------------------

class DeviceFrame:
    """Device-side results of one pass (plus the host feedback lists)."""

    def __init__(self, paging, n_ch, k, npix_local, budget):
        dev = paging.device
        self.image = torch.empty((npix_local, 4), dtype=torch.float32, device=dev)
        self.required = torch.empty(paging.total_entries, dtype=torch.uint8, device=dev)
        self.pix_required = torch.empty(npix_local, dtype=torch.int32, device=dev)
        # histogram, counters, the four feedback lists and the feedback counts
        # share one int64 block so a frame's small results come back in one copy
        nh, nc, nb = n_ch * k, N.RO_NUM_COUNTERS, max(budget, 1)
        self.small = torch.empty(nh + nc + 4 * nb + 4, dtype=torch.int64, device=dev)
        self.hist = self.small[:nh].view(n_ch, k)
        self.counters = self.small[nh:nh + nc]
        self.fb = self.small[nh + nc:nh + nc + 4 * nb].view(4, nb)
        self.counts_dev = self.small[nh + nc + 4 * nb:]
        self.budget = budget
        self.counts = np.zeros(4, dtype=np.int64)
        self.outputs = N.Outputs(self.image.data_ptr(), self.required.data_ptr(),
                                 self.pix_required.data_ptr(), self.hist.data_ptr(),
                                 self.counters.data_ptr())
        # synchronous form (host counts) and the asynchronous one (device counts only)
        self.feedback = N.Feedback(self.fb[0].data_ptr(), self.fb[1].data_ptr(),
                                   self.fb[2].data_ptr(), self.fb[3].data_ptr(),
                                   self.counts.ctypes.data, self.counts_dev.data_ptr())
        self.feedback_async = N.Feedback(self.fb[0].data_ptr(), self.fb[1].data_ptr(),
                                         self.fb[2].data_ptr(), self.fb[3].data_ptr(),
                                         None, self.counts_dev.data_ptr())

    @property
    def n_bricks(self) -> int:
        return int(self.counts[2])

    @property
    def n_metas(self) -> int:
        return int(self.counts[3])


def _buffers(paging, n_ch, npix_local, budget) -> DeviceFrame:
    key = (n_ch, npix_local, budget)
    cache = paging.__dict__.setdefault("_frame_buffers", {})
    buf = cache.get(key)
    if buf is None:
        if len(cache) > 4:
            cache.clear()
        buf = DeviceFrame(paging, n_ch, paging.config.k, npix_local, budget)
        cache[key] = buf
    return buf


class FramePass:
    """A packed frame bound to its state and output buffers: ``render()``
    launches kernel 1, ``collect()`` orders/truncates the requests (kernel
    3a, synchronising).  Reusable across frames with the same camera."""

    def __init__(self, mode, paging: MultiChannelPaging, octree: ResidencyOctree | None,
                 channels, camera: Camera, config: RenderConfig, reference_paging=None,
                 partition=(1, 0, 8), bricks_first: bool = True, classic=None,
                 max_samples: int = 0):
        N.require_cuda()
        if mode == MODE_RESIDENCY:
            if octree is None:
                raise RenderError("residency mode needs the octree")
            depth, eps_h = octree.config.depth, octree.config.homogeneity_eps
        else:
            depth, eps_h = 0, config.homogeneity_eps
        if mode == MODE_CLASSIC:
            if classic is None:
                raise RenderError("classic mode needs ClassicMetadata")
            cp = classic.paging
            if (cp is not paging and (cp.config.m != paging.config.m
                                      or not np.array_equal(cp.level_grids,
                                                            paging.level_grids))):
                raise RenderError("classic metadata built for another volume layout")
        self.paging = paging
        self.config = config
        self.bricks_first = bricks_first
        self.classic = classic  # keeps the metadata buffers alive
        self.frame = _pack_frame(mode, paging, channels, camera, config, depth, eps_h,
                                 reference_paging, partition, classic)
        self.frame.max_samples = int(max_samples)
        w, h = config.image_dims
        self.local_rows = N.lib().ro_local_rows(h, *partition)
        self.buf = _buffers(paging, len(channels), self.local_rows * w,
                            config.max_requests_per_frame)
        self.state = paging.state(with_words=(mode == MODE_RESIDENCY))

    def render(self, outputs: N.Outputs | None = None):
        out = outputs if outputs is not None else self.buf.outputs
        N.check(N.lib().ro_render(self.paging.ctx, C.byref(self.frame), C.byref(self.state),
                                  C.byref(out), N.stream_ptr()))

    def collect(self, asynchronous: bool = False):
        """Order + truncate the requests on the device.  Synchronous: the
        counts are in ``buf.counts`` on return.  Asynchronous: nothing waits;
        the counts are in ``buf.counts_dev`` (part of ``buf.small``)."""
        fb = self.buf.feedback_async if asynchronous else self.buf.feedback
        N.check(N.lib().ro_feedback_collect(self.paging.ctx,
                                            self.config.max_requests_per_frame,
                                            1 if self.bricks_first else 0,
                                            C.byref(fb), N.stream_ptr()))


def render_frame_device(mode, paging: MultiChannelPaging, octree: ResidencyOctree | None,
                        channels, camera: Camera, config: RenderConfig,
                        reference_paging=None, partition=(1, 0, 8),
                        bricks_first: bool = True, collect: bool = True,
                        classic=None) -> DeviceFrame:
    """One ray-cast pass + feedback ordering, results left on the device.

    Not re-entrant per paging: the returned buffers are reused by the next
    call with the same shape."""
    fp = FramePass(mode, paging, octree, channels, camera, config, reference_paging,
                   partition, bricks_first, classic)
    fp.render()
    if collect:
        fp.collect()
    return fp.buf


class _ResultPool:
    """Page-locked host buffers for frame results, with explicit ownership.

    A frame's four result buffers (image, per-pixel counts, usage mask, the
    small int64 block) form one *set*.  The ray caster stores the image and
    per-pixel counts straight into a set over PCIe (zero-copy) and the rest is
    copied behind it; the numpy arrays handed to the caller are views of the
    set, and a ``weakref.finalize`` on each returns the set to the pool once
    every view (including any slice the caller kept) is gone.  At most
    ``depth`` sets exist per shape: when the caller holds all of them (e.g. a
    Session keeping its frame history) the frame lands in a private staging
    set and is copied out into ordinary numpy arrays -- page-locked memory
    is never allocated per frame (cudaHostAlloc of a 1080p frame costs
    ~15 ms) and never grows without bound."""

    def __init__(self, depth: int = 4, pin: bool = True):
        self.depth = depth
        self.pin = pin
        self._free: dict = {}      # key -> [set, ...]
        self._count: dict = {}     # key -> sets created (handed out or free)
        self._staging: dict = {}   # key -> the private set

    def _make(self, shapes):
        return tuple(torch.empty(shp, dtype=dt, pin_memory=self.pin) for shp, dt in shapes)

    def reserve(self, shapes, n: int = 1):
        """Create up to n free sets (and the staging set) ahead of the first frame."""
        key = tuple(shapes)
        free = self._free.setdefault(key, [])
        while len(free) < n and self._count.get(key, 0) < self.depth:
            free.append(self._make(shapes))
            self._count[key] = self._count.get(key, 0) + 1
        if key not in self._staging:
            self._staging[key] = self._make(shapes)

    def acquire(self, shapes):
        """(set, owned): owned = handed out (release on finalize) or not
        (the staging set: copy the results out)."""
        key = tuple(shapes)
        free = self._free.setdefault(key, [])
        if free:
            return free.pop(), True
        if self._count.get(key, 0) < self.depth:
            self._count[key] = self._count.get(key, 0) + 1
            return self._make(shapes), True
        if key not in self._staging:
            self._staging[key] = self._make(shapes)
        return self._staging[key], False

    def handout(self, shapes, bufset, tensors) -> list:
        """numpy arrays over ``tensors`` (members of bufset); bufset returns
        to the pool when every one of them, and every view derived from
        them, is garbage.  Each array's memory owner is a fresh lease object
        (numpy keeps a view's chain of bases alive up to it), so the lease's
        finalizer is the exact "no view left" signal."""
        key = tuple(shapes)
        state = {"left": len(tensors)}
        free = self._free.setdefault(key, [])

        def done():
            state["left"] -= 1
            if state["left"] == 0:
                free.append(bufset)
        out = []
        for t in tensors:
            lease = _Lease(t)
            weakref.finalize(lease, done)
            out.append(np.asarray(lease))
        return out


class _Lease:
    """Memory owner of the numpy views handed out from one pooled buffer."""

    def __init__(self, t: torch.Tensor):
        self.t = t
        self.__array_interface__ = {"data": (t.data_ptr(), False), "shape": tuple(t.shape),
                                    "typestr": np.dtype(str(t.dtype).split(".")[-1]).str,
                                    "version": 3}


_RESULTS = _ResultPool()


def _result_shapes(buf) -> tuple:
    return ((tuple(buf.image.shape), torch.float32), (tuple(buf.pix_required.shape), torch.int32),
            (tuple(buf.required.shape), torch.uint8), (tuple(buf.small.shape), torch.int64))


def _run(mode, paging, channels, camera, config, octree=None,
         reference_paging=None, classic=None, partition=(1, 0, 8),
         max_samples: int = 0) -> FrameOutput:
    start = time.perf_counter()
    fp = FramePass(mode, paging, octree, channels, camera, config, reference_paging,
                   partition=partition, classic=classic, max_samples=max_samples)
    buf = fp.buf
    # Zero-copy image: the ray caster stores each pixel's RGBA and brick
    # count straight into pinned host memory (UVA-mapped), so the 20 B/pixel
    # device->host transfer rides PCIe while the kernel runs instead of
    # after it.  Usage mask, histogram and counters stay in HBM (scattered
    # writes / atomics) and are copied once the kernel is done.
    shapes = _result_shapes(buf)
    (img, pixr, req, small), owned = _RESULTS.acquire(shapes)
    nh = buf.hist.numel()
    fp.render(N.Outputs(img.data_ptr(), buf.required.data_ptr(), pixr.data_ptr(),
                        buf.hist.data_ptr(), buf.counters.data_ptr()))
    fp.collect(asynchronous=True)
    # usage mask (E bytes) and the histogram / counters / ordered requests /
    # counts block: two copies behind the request ordering, one
    # synchronisation for the whole frame (the kernel's host stores included)
    main = torch.cuda.current_stream()
    req.copy_(buf.required, non_blocking=True)
    small.copy_(buf.small, non_blocking=True)
    main.synchronize()
    m = paging.config.m
    sm = small.numpy()
    buf.counts[:] = sm[-4:]
    nb, nm = buf.n_bricks, buf.n_metas
    elapsed_ms = (time.perf_counter() - start) * 1000.0
    hist = sm[:nh].reshape(buf.hist.shape).copy()
    counters = sm[nh:nh + N.RO_NUM_COUNTERS]
    fb = sm[nh + N.RO_NUM_COUNTERS:-4].reshape(4, -1)
    bricks = fb[1][:nb].tolist()
    metas = [divmod(v, m) for v in fb[3][:nm].tolist()]
    required = req.numpy()
    nreq = int(required.sum())
    sx, sy, sz = paging.config.brick_size
    stats = FrameStats(traversal_steps=int(counters[0]), samples_evaluated=int(counters[1]),
                       samples_skipped=int(counters[2]), skip_violations=int(counters[3]),
                       required_bricks=nreq, required_bytes=nreq * sx * sy * sz,
                       requests_issued=len(bricks) + len(metas), render_ms=elapsed_ms,
                       livelocked_rays=int(counters[4]))
    w, h = config.image_dims
    rows = buf.image.shape[0] // w  # local rows of a partition (h for a full frame)
    if owned:
        image, pixel_required, required = _RESULTS.handout(
            shapes, (img, pixr, req, small), (img, pixr, req))
    else:   # every pooled set is still held by the caller: copy out of staging
        image, pixel_required, required = img.numpy().copy(), pixr.numpy().copy(), req.numpy().copy()
    image = image.reshape(rows, w, 4)
    return FrameOutput(image=image, brick_requests=bricks,
                       metadata_requests=metas, stats=stats, required_mask=required,
                       level_histogram=hist, pixel_required=pixel_required,
                       required_mask_device=buf.required)


def render_frame(paging: MultiChannelPaging, octree: ResidencyOctree,
                 channels, camera: Camera, config: RenderConfig,
                 reference_paging: MultiChannelPaging | None = None) -> FrameOutput:
    """Residency-octree renderer (render.py:236-243); pass reference paging to
    audit every skip."""
    return _run(MODE_RESIDENCY, paging, channels, camera, config, octree=octree,
                reference_paging=reference_paging)


def render_frame_part(paging: MultiChannelPaging, octree: ResidencyOctree, channels,
                      camera: Camera, config: RenderConfig, partition) -> FrameOutput:
    """render_frame for the rows of one sort-first part.  ``partition`` =
    (n_parts, part, tile_rows): rows are cut in blocks of tile_rows and block
    b belongs to part b % n_parts.  The image / pixel_required hold only this
    part's rows (in order); requests, usage and histogram are this part's,
    with the bricks-first budget applied to them -- the per-GPU frame of a
    capacity-mode Session (distributed.gather_image assembles the frame)."""
    return _run(MODE_RESIDENCY, paging, channels, camera, config, octree=octree,
                partition=tuple(partition))


@dataclass
class SampleProbe:
    """What one sample resolved through the shared residency cursor leaves
    behind -- the observable part of the reference's TraversalResult
    (render.py traverse_sample, checked by tests/test_render_units.py:194-269)."""
    steps: int                 # octree node visits over all channels
    brick_requests: list       # BrickIDs in first-seen order
    metadata_requests: list    # (node index, slot) in first-seen order
    sampled_levels: list       # per channel: the level sampled, None if none
    skippable: bool            # resolved ZERO / CONST / MISSU for every channel
    rgba: tuple                # the sample composited over nothing
    output: FrameOutput


def probe_sample(paging: MultiChannelPaging, octree: ResidencyOctree, channels,
                 position, levels, depth: int, start_depth: int = 0,
                 direction=(1.0, 0.0, 0.0)) -> SampleProbe:
    """Resolve ONE sample at ``position`` on the GPU, the way the ray caster
    resolves every sample (kernels.py:431-558): a 1x1 frame whose ray starts
    inside the volume at ``position`` (t = 0), with channel i's desired level
    pinned to ``levels[i]``, the traversal depth to ``depth`` (step
    2^-depth) and the cursor starting at ``start_depth``; the ray stops after
    that sample (ro_frame.max_samples = 1; a skippable sample still runs its
    skip loop, which is how ``skippable`` is observed: skipped samples, or
    more than one constant-composited sample, and so the skip region must
    span more than one step for a CONST outcome to read as skippable)."""
    if len(levels) != len(channels):
        raise RenderError("one desired level per channel")
    chans = [ChannelSettings(slot=c.slot, tf=c.tf, level_range=(int(lv), int(lv)))
             for c, lv in zip(channels, levels)]
    base = 2.0 ** -int(depth) / (1 << max(int(v) for v in levels))
    cfg = RenderConfig(image_dims=(1, 1), base_step=base, max_requests_per_frame=4096,
                       traversal_start_level=int(start_depth) + 1)
    pos = tuple(float(v) for v in position)
    cam = Camera(position=pos, target=tuple(p + float(d) for p, d in zip(pos, direction)),
                 up=(0.0, 1.0, 0.0) if abs(direction[1]) < 0.9 else (1.0, 0.0, 0.0))
    out = _run(MODE_RESIDENCY, paging, chans, cam, cfg, octree=octree, max_samples=1)
    st = out.stats
    hist = out.level_histogram
    sampled = [int(np.flatnonzero(hist[i])[0]) if hist[i].any() else None
               for i in range(len(chans))]
    return SampleProbe(steps=st.traversal_steps, brick_requests=list(out.brick_requests),
                       metadata_requests=list(out.metadata_requests), sampled_levels=sampled,
                       skippable=st.samples_skipped > 0 or st.samples_evaluated > 1,
                       rgba=tuple(float(v) for v in out.image[0, 0]), output=out)


def render_reference(paging: MultiChannelPaging, channels, camera: Camera,
                     config: RenderConfig) -> FrameOutput:
    """In-core oracle mode (render.py:246-250): every sample translated and
    evaluated, no skipping or substitution."""
    return _run(MODE_REFERENCE, paging, channels, camera, config)


def render_pagetable_only(paging: MultiChannelPaging, channels, camera: Camera,
                          config: RenderConfig) -> FrameOutput:
    """Page-table-only baseline (render.py:253-256, kernels.py:316-357):
    desired-level translation per sample; EMPTY entries skip to their brick
    exit, unmapped ones are requested."""
    return _run(MODE_PAGETABLE, paging, channels, camera, config)


def render_classic_octree(paging: MultiChannelPaging, classic: "ClassicMetadata",
                          channels, camera: Camera, config: RenderConfig) -> FrameOutput:
    """Classic-octree baseline (render.py:259-262, kernels.py:359-429): one
    root-to-target descent per channel per sample over per-node min / max,
    falling back to the deepest resident ancestor when a brick is missing."""
    return _run(MODE_CLASSIC, paging, channels, camera, config, classic=classic)


# ---------------------------------------------------------------------------
# classic-octree baseline metadata
# ---------------------------------------------------------------------------

class ClassicMetadata:
    """Per-node min / max of the classic one-node-one-brick octree
    (render.py:271-315), kept in HBM as u8[n_nodes, m] (``min_arr`` /
    ``max_arr``, unfilled slots = (0, 255)).

    Node depth d corresponds to resolution level (depth - d); every level's
    brick grid must be 2^(depth - level) bricks per axis, so each node owns
    exactly one brick.  ``build_from_volume`` reduces a slot's level-0 volume
    bottom-up on the device (exact block min / max, no dilation)."""

    def __init__(self, paging: MultiChannelPaging):
        k = paging.config.k
        self.depth = k - 1
        for lev in range(k):
            g = [int(v) for v in paging.level_grids[lev]]
            want = 1 << (self.depth - lev)
            if not g[0] == g[1] == g[2] == want:
                raise RenderError("classic octree needs power-of-two brick grids "
                                  f"(level {lev} grid {tuple(g)}, expected {want}^3)")
        if self.depth > 8:
            raise RenderError("classic octree depth > 8 (brick coordinates are 8-bit)")
        self.paging = paging
        m = paging.config.m
        n_nodes = ((1 << (3 * k)) - 1) // 7
        dev = paging.device
        self.min_arr = torch.zeros((n_nodes, m), dtype=torch.uint8, device=dev)
        self.max_arr = torch.full((n_nodes, m), 255, dtype=torch.uint8, device=dev)
        self.lvl_off = np.array([((1 << (3 * d)) - 1) // 7 for d in range(k)],
                                dtype=np.int64)

    def build_from_volume(self, slot: int, volume):
        """Fill a slot's metadata column from its full-resolution volume
        (z, y, x), numpy or torch."""
        if not 0 <= slot < self.paging.config.m:
            raise RenderError(f"channel slot {slot} out of range")
        from .metadata import node_minmax
        vol = torch.as_tensor(volume)
        if vol.dtype != torch.uint8:
            raise RenderError("classic metadata volumes are u8 (normalised level 0)")
        vol = vol.to(self.min_arr.device).contiguous()
        g = 1 << self.depth
        nz, ny, nx = vol.shape
        if nz % g or ny % g or nx % g:
            raise RenderError("volume dims must divide the leaf node grid")
        # every depth's exact block min / max straight from level 0
        # (ro_node_minmax with no dilation: the windows are the blocks)
        for d in range(self.depth, -1, -1):
            off = int(self.lvl_off[d])
            lo, hi = node_minmax(vol, d, 0)
            self.min_arr[off:off + lo.numel(), slot] = lo
            self.max_arr[off:off + hi.numel(), slot] = hi
