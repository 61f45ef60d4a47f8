"""Scene builders shared by the tests (restated ingest, see volume.py)."""

from __future__ import annotations

import functools
import hashlib

import numpy as np

from paper_2309_04393_b200 import volume as V


@functools.lru_cache(maxsize=None)
def store(kind: str) -> V.VolumeStore:
    if kind == "mc64":
        return V.VolumeStore(V.sparse_multichannel(64, channels=4), (16, 16, 16), 3,
                             (2, 2, 2))
    if kind == "shell64":
        return V.VolumeStore([V.shell_volume(64)], (16, 16, 16), 3, (2, 2, 2))
    if kind == "vessel256":
        return V.VolumeStore([V.vessel_volume(256)], (32, 32, 32), 4, (2, 2, 2))
    if kind == "sparse256x4":
        return V.VolumeStore(V.sparse_multichannel(256, channels=4), (32, 32, 32), 4,
                             (2, 2, 2))
    raise KeyError(kind)


def pyramid_sha(st: V.VolumeStore, channels) -> str:
    hh = hashlib.sha256()
    for c in channels:
        for l in range(len(st.manifest.levels)):
            hh.update(np.ascontiguousarray(st.level_array(c, l)).tobytes())
    return hh.hexdigest()


def full_cache_slots(st, m):
    """bench.py:41-71: smallest cube of slots holding every brick of m channels."""
    import math
    total = m * sum(math.prod(l.brick_grid_dims) for l in st.manifest.levels)
    side = 1
    while side ** 3 < total:
        side += 1
    return (side, side, side)


def keep_partial(slot, lev, x, y, z, k=4):
    """Partial-residency rule of the baselines fixtures (make_golden.py
    _keep): the coarsest level always, otherwise 3 of 4 bricks."""
    return lev == k - 1 or (x * 7 + y * 13 + z * 29 + lev * 3 + slot * 5) % 4 != 0


def paging_hashes(st) -> dict:
    """make_golden.paging_hashes over an oracle state."""
    from oracle.session import state_hashes
    d = state_hashes(st)
    d.pop("words")
    return d


def oracle_render_state(st, with_words=False):
    from oracle import raycast as orc
    return orc.OracleState(m=st.m, k=st.k, brick_size=st.brick_size,
                           level_dims=st.level_dims, level_grids=st.level_grids,
                           pt_offsets=st.pt_offsets, pt_status=st.pt_status,
                           pt_slot=st.pt_slot, cache=st.cache,
                           words=st.words if with_words else None, depth=st.depth)


def tf_points(js):
    return tuple((float(x), tuple(float(v) for v in c)) for x, c in js)


def oracle_channels(meta_channels):
    from oracle.raycast import OracleChannel
    return [OracleChannel(slot=c["slot"], points=tf_points(c["tf"]),
                          level_range=tuple(c["level_range"])) for c in meta_channels]


def product_channels(meta_channels):
    from paper_2309_04393_b200 import ChannelSettings, TransferFunction
    return [ChannelSettings(slot=c["slot"], tf=TransferFunction(points=tf_points(c["tf"])),
                            level_range=tuple(c["level_range"])) for c in meta_channels]


def render_kw(meta_render):
    return dict(image_dims=tuple(meta_render["image_dims"]),
                base_step=meta_render["base_step"], t0=meta_render["t0"],
                early_alpha=meta_render["early_alpha"], budget=meta_render["budget"],
                start_level=meta_render["start_level"])


def render_config(meta_render):
    from paper_2309_04393_b200 import RenderConfig
    return RenderConfig(image_dims=tuple(meta_render["image_dims"]),
                        base_step=meta_render["base_step"],
                        lod_reference_distance=meta_render["t0"],
                        early_term_alpha=meta_render["early_alpha"],
                        max_requests_per_frame=meta_render["budget"],
                        traversal_start_level=meta_render["start_level"])


def check_frame(rec, prefix, image, bricks, metas, required, hist, pixreq, counters,
                image_atol=0.0):
    """Compare one frame against a golden record; returns list of problems."""
    bad = []
    gi = rec[prefix + "image"].reshape(image.shape)
    if image_atol == 0.0:
        if not np.array_equal(gi, image):
            bad.append(f"image: {int((gi != image).sum())} components differ, "
                       f"max {float(np.abs(gi - image).max()):.3g}")
    elif not np.allclose(gi, image, atol=image_atol, rtol=0):
        bad.append(f"image max diff {float(np.abs(gi - image).max()):.3g}")
    if list(rec[prefix + "bricks"]) != list(bricks):
        bad.append("brick requests differ")
    gm = [tuple(int(v) for v in r) for r in rec[prefix + "metas"]]
    if gm != [tuple(int(v) for v in r) for r in metas]:
        bad.append("metadata requests differ")
    if not np.array_equal(rec[prefix + "required"], required):
        bad.append("usage mask differs")
    if not np.array_equal(rec[prefix + "hist"], hist):
        bad.append("level histogram differs")
    if not np.array_equal(rec[prefix + "pixreq"], pixreq):
        bad.append("pixel_required differs")
    if list(rec[prefix + "counters"]) != list(counters)[:4]:
        bad.append(f"counters {list(counters)[:4]} != {list(rec[prefix + 'counters'])}")
    return bad
