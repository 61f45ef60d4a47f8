"""ctypes driver for the C oracle -- TEST INFRASTRUCTURE ONLY.

Restates the host half of a frame the way the reference does it:
* ray generation, ``camera.py:32-51`` (fp64 numpy, same operation order);
* channel / transfer-function packing, ``render.py:101-122`` with the TF
  tables of ``transfer.py:38-120``;
* output allocation and the bricks-first request budget,
  ``render.py:176-215``.

State is passed in the REFERENCE layout (``pt_status`` i8 + ``pt_slot`` i32,
``words`` u32[N, m], ``cache`` u8[S, bz, by, bx]).
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from .build import build, lib_path

INF = float("inf")
MODE_RESIDENCY = 0
MODE_REFERENCE = 1
MODE_PAGETABLE = 2
MODE_CLASSIC = 3

_P = C.c_void_p


class _Frame(C.Structure):
    _fields_ = [
        ("mode", C.c_int64), ("npix", C.c_int64), ("origins", _P), ("dirs", _P),
        ("n_ch", C.c_int64), ("ch_slot", _P), ("ch_lo", _P), ("ch_hi", _P),
        ("npoints", C.c_int64), ("tf_x", _P), ("tf_rgba", _P), ("tf_np", _P),
        ("tf_f", _P), ("tf_op", _P),
        ("base_step", C.c_double), ("t0", C.c_double),
        ("early_alpha", C.c_double), ("eps_h", C.c_double),
        ("start_level", C.c_int64), ("depth_d", C.c_int64), ("k", C.c_int64),
        ("m", C.c_int64),
        ("lvl_off", _P), ("words", _P), ("dims", _P), ("grids", _P),
        ("bx", C.c_int64), ("by", C.c_int64), ("bz", C.c_int64),
        ("pt_offsets", _P), ("pt_status", _P), ("pt_slot", _P), ("cache", _P),
        ("check_skips", C.c_int64), ("ref_status", _P), ("ref_slot", _P),
        ("ref_cache", _P),
        ("cls_min", _P), ("cls_max", _P), ("cls_depth", C.c_int64),
        ("cls_lvl_off", _P),
        ("image", _P), ("brick_req", _P), ("brick_req_n", _P),
        ("meta_req", _P), ("meta_req_n", _P), ("req_cap", C.c_int64),
        ("seen_brick", _P), ("seen_meta", _P), ("required", _P),
        ("pix_required", _P), ("hist", _P), ("counters", _P),
        ("pix_begin", C.c_int64), ("pix_end", C.c_int64), ("touched", C.c_void_p),
    ]


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.oracle_raycast.argtypes = [C.POINTER(_Frame)]
        lib.oracle_raycast.restype = C.c_int
        lib.oracle_raycast_parallel.argtypes = [C.POINTER(_Frame), C.c_int64,
                                                C.c_int64, C.c_int64]
        lib.oracle_raycast_parallel.restype = C.c_int
        _LIB = lib
    return _LIB


# ---------------------------------------------------------------------------
# transfer-function tables (transfer.py:38-120, restated)
# ---------------------------------------------------------------------------

def tf_evaluate(points, scalar):
    if scalar < points[0][0] or scalar > points[-1][0]:
        return (0.0, 0.0, 0.0, 0.0)
    for i in range(len(points) - 1):
        x0, c0 = points[i]
        x1, c1 = points[i + 1]
        if x0 <= scalar <= x1:
            t = 0.0 if x1 == x0 else (scalar - x0) / (x1 - x0)
            return tuple(c0[j] + (c1[j] - c0[j]) * t for j in range(4))
    return (0.0, 0.0, 0.0, 0.0)


def _support_intervals(points):
    out = []
    for i in range(len(points) - 1):
        (x0, c0), (x1, c1) = points[i], points[i + 1]
        if c0[3] > 0.0 or c1[3] > 0.0:
            end_closed = c1[3] > 0.0
            if out and x0 <= out[-1][1]:
                out[-1][1] = x1
                out[-1][2] = end_closed
            else:
                out.append([x0, x1, end_closed])
    return out


def _first_support_at_or_after(points, a):
    if tf_evaluate(points, a)[3] > 0.0:
        return a
    best = INF
    for s, e, end_closed in _support_intervals(points):
        if e > a or (e == a and end_closed):
            best = min(best, max(s, a))
    return best


def tf_tables(points):
    f = np.empty(256, dtype=np.float64)
    op = np.empty(256, dtype=np.float64)
    for v in range(256):
        f[v] = _first_support_at_or_after(points, float(v))
        op[v] = tf_evaluate(points, float(v))[3]
    f[~np.isfinite(f)] = 1e30
    return f, op


# ---------------------------------------------------------------------------
# rays (camera.py:32-51, restated)
# ---------------------------------------------------------------------------

def generate_rays(position, target, up, fov_deg, width, height):
    pos = np.array(position, dtype=np.float64)
    fwd = np.array(target, dtype=np.float64) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.array(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    upv = np.cross(right, fwd)
    tan_half = math.tan(math.radians(fov_deg) / 2.0)
    aspect = width / height
    js, is_ = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    u = ((is_ + 0.5) / width * 2.0 - 1.0) * tan_half * aspect
    v = (1.0 - (js + 0.5) / height * 2.0) * tan_half
    dirs = (fwd[None, None, :] + u[..., None] * right[None, None, :]
            + v[..., None] * upv[None, None, :])
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    origins = np.broadcast_to(pos, dirs.reshape(-1, 3).shape).copy()
    return origins, np.ascontiguousarray(dirs.reshape(-1, 3))


# ---------------------------------------------------------------------------
# frame driver (render.py:125-233, restated)
# ---------------------------------------------------------------------------

@dataclass
class OracleState:
    """Reference-layout render state."""
    m: int
    k: int
    brick_size: tuple
    level_dims: np.ndarray      # int32 (k,3) x,y,z
    level_grids: np.ndarray     # int32 (k,3)
    pt_offsets: np.ndarray      # int64 (m*k+1)
    pt_status: np.ndarray       # int8 (E)
    pt_slot: np.ndarray         # int32 (E)
    cache: np.ndarray           # uint8 (S,bz,by,bx)
    words: np.ndarray | None = None   # uint32 (N,m)
    depth: int = 0
    eps_h: float = 0.0


@dataclass
class OracleChannel:
    slot: int
    points: tuple               # ((x, (r,g,b,a)), ...)
    level_range: tuple = (0, 15)


@dataclass
class OracleOutput:
    image: np.ndarray
    brick_requests: list
    metadata_requests: list
    required_mask: np.ndarray
    level_histogram: np.ndarray
    pixel_required: np.ndarray
    counters: np.ndarray
    all_brick_requests: list = field(default_factory=list)
    all_metadata_requests: list = field(default_factory=list)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def render(state: OracleState, channels, camera, image_dims, base_step,
           t0=1.0, early_alpha=0.99, budget=256, start_level=2,
           mode=MODE_RESIDENCY, reference_state: OracleState | None = None,
           rows=None, threads=1, rays=None, classic=None, touched=None) -> OracleOutput:
    """One oracle frame.

    camera: (position, target, up, fov_deg).  ``classic`` = (min u8[n, m],
    max u8[n, m], depth) for MODE_CLASSIC (render.py:271-315).  ``rows`` = (row_begin,
    row_end) renders only those scanlines (the other pixels stay zero);
    ``threads`` > 1 uses the band-parallel driver (identical results).
    ``touched``: optional u8 array shaped like the cache; every voxel a
    trilinear fetch reads is set to 1 (fixture generation only).
    """
    lib = _lib()
    k, m = state.k, state.m
    n_ch = len(channels)
    npoints = max(len(c.points) for c in channels)
    ch_slot = np.array([c.slot for c in channels], dtype=np.int64)
    ch_lo = np.array([max(0, min(c.level_range[0], k - 1)) for c in channels],
                     dtype=np.int64)
    ch_hi = np.array([max(0, min(c.level_range[1], k - 1)) for c in channels],
                     dtype=np.int64)
    tf_x = np.zeros((n_ch, npoints))
    tf_rgba = np.zeros((n_ch, npoints, 4))
    tf_np = np.zeros(n_ch, dtype=np.int64)
    tf_f = np.zeros((n_ch, 256))
    tf_op = np.zeros((n_ch, 256))
    for i, c in enumerate(channels):
        for j, (x, rgba) in enumerate(c.points):
            tf_x[i, j] = x
            tf_rgba[i, j] = rgba
        tf_np[i] = len(c.points)
        tf_f[i], tf_op[i] = tf_tables(c.points)

    w, h = image_dims
    if rays is None:
        origins, dirs = generate_rays(*camera, w, h)
    else:
        origins, dirs = rays
    npix = w * h
    if mode == MODE_RESIDENCY:
        depth = state.depth
        words = np.ascontiguousarray(state.words, dtype=np.uint32)
        num_nodes = words.shape[0]
    else:
        depth = 0
        words = np.zeros((1, 1), dtype=np.uint32)
        num_nodes = 1
    lvl_off = np.array([((1 << (3 * d)) - 1) // 7 for d in range(depth + 1)],
                       dtype=np.int64)
    total = int(state.pt_offsets[-1])
    cap = max(4 * budget, 1024)
    image = np.zeros((npix, 4), dtype=np.float32)
    brick_req = np.zeros(cap, dtype=np.int64)
    brick_n = np.zeros(1, dtype=np.int64)
    meta_req = np.zeros(cap, dtype=np.int64)
    meta_n = np.zeros(1, dtype=np.int64)
    seen_brick = np.zeros(total, dtype=np.uint8)
    seen_meta = np.zeros(num_nodes * m, dtype=np.uint8)
    required = np.zeros(total, dtype=np.uint8)
    pix_required = np.zeros(npix, dtype=np.int32)
    hist = np.zeros((n_ch, k), dtype=np.int64)
    counters = np.zeros(5, dtype=np.int64)
    dims = np.ascontiguousarray(state.level_dims, dtype=np.int32)
    grids = np.ascontiguousarray(state.level_grids, dtype=np.int32)
    pt_offsets = np.ascontiguousarray(state.pt_offsets, dtype=np.int64)
    pt_status = np.ascontiguousarray(state.pt_status, dtype=np.int8)
    pt_slot = np.ascontiguousarray(state.pt_slot, dtype=np.int32)
    cache = np.ascontiguousarray(state.cache, dtype=np.uint8)
    if reference_state is not None:
        ref = (np.ascontiguousarray(reference_state.pt_status, dtype=np.int8),
               np.ascontiguousarray(reference_state.pt_slot, dtype=np.int32),
               np.ascontiguousarray(reference_state.cache, dtype=np.uint8))
    else:
        ref = (None, None, None)
    if mode == MODE_CLASSIC:
        cmin = np.ascontiguousarray(classic[0], dtype=np.uint8)
        cmax = np.ascontiguousarray(classic[1], dtype=np.uint8)
        cdepth = int(classic[2])
    else:
        cmin = cmax = np.zeros((1, m), dtype=np.uint8)
        cdepth = 0
    cls_off = np.array([((1 << (3 * d)) - 1) // 7 for d in range(cdepth + 1)],
                       dtype=np.int64)
    r0, r1 = (0, h) if rows is None else rows
    fr = _Frame(
        mode=mode, npix=npix, origins=_ptr(origins), dirs=_ptr(dirs),
        n_ch=n_ch, ch_slot=_ptr(ch_slot), ch_lo=_ptr(ch_lo), ch_hi=_ptr(ch_hi),
        npoints=npoints, tf_x=_ptr(tf_x), tf_rgba=_ptr(tf_rgba),
        tf_np=_ptr(tf_np), tf_f=_ptr(tf_f), tf_op=_ptr(tf_op),
        base_step=base_step, t0=t0, early_alpha=early_alpha, eps_h=state.eps_h,
        start_level=start_level, depth_d=depth, k=k, m=m,
        lvl_off=_ptr(lvl_off), words=_ptr(words), dims=_ptr(dims),
        grids=_ptr(grids), bx=state.brick_size[0], by=state.brick_size[1],
        bz=state.brick_size[2], pt_offsets=_ptr(pt_offsets),
        pt_status=_ptr(pt_status), pt_slot=_ptr(pt_slot), cache=_ptr(cache),
        check_skips=1 if reference_state is not None else 0,
        ref_status=_ptr(ref[0]), ref_slot=_ptr(ref[1]), ref_cache=_ptr(ref[2]),
        cls_min=_ptr(cmin), cls_max=_ptr(cmax), cls_depth=cdepth,
        cls_lvl_off=_ptr(cls_off),
        image=_ptr(image), brick_req=_ptr(brick_req), brick_req_n=_ptr(brick_n),
        meta_req=_ptr(meta_req), meta_req_n=_ptr(meta_n), req_cap=cap,
        seen_brick=_ptr(seen_brick), seen_meta=_ptr(seen_meta),
        required=_ptr(required), pix_required=_ptr(pix_required),
        hist=_ptr(hist), counters=_ptr(counters),
        pix_begin=r0 * w, pix_end=r1 * w, touched=_ptr(touched))
    if threads <= 1:
        rc = lib.oracle_raycast(C.byref(fr))
    else:
        rc = lib.oracle_raycast_parallel(C.byref(fr), total, num_nodes * m,
                                         threads)
    if rc != 0:
        raise RuntimeError(f"oracle_raycast failed ({rc})")
    all_b = [int(v) for v in brick_req[:int(brick_n[0])]]
    all_m = [(int(v) // m, int(v) % m) for v in meta_req[:int(meta_n[0])]]
    bricks = all_b[:budget]
    metas = all_m[:budget - len(bricks)]
    return OracleOutput(image=image.reshape(h, w, 4), brick_requests=bricks,
                        metadata_requests=metas, required_mask=required,
                        level_histogram=hist, pixel_required=pix_required,
                        counters=counters, all_brick_requests=all_b,
                        all_metadata_requests=all_m)
