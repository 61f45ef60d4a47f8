"""Oracle frame loop -- TEST INFRASTRUCTURE ONLY.

Restates ``Session.step_frame`` (session.py:65-103) over the oracle state
(``oracle.state.OracleResidency``) and the C ray-cast oracle, fetching from
an in-memory store (``service.py:71-115`` semantics).  Also restates the
bulk ``prepare_engine`` path (bench.py:49-61, engine.py:138-179).
"""

from __future__ import annotations

import hashlib

import numpy as np

from . import raycast as orc
from .state import OracleResidency


def _h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def state_hashes(st: OracleResidency) -> dict:
    return {"words": _h(st.words), "pt_status": _h(st.pt_status),
            "pt_slot": _h(st.pt_slot), "slot_brick": _h(st.slot_brick),
            "slot_last_used": _h(st.slot_last_used), "cache": _h(st.cache),
            "free": _h(np.array(st.free, dtype=np.int64))}


def metadata_box(level0_dims, d, x, y, z, pad):
    """engine.py:109-127"""
    side = 1 << d
    node = (x, y, z)
    lo, hi = [], []
    for a in range(3):
        v0 = (node[a] * level0_dims[a]) // side - pad
        v1 = -((-(node[a] + 1) * level0_dims[a]) // side) + pad
        lo.append(max(0, v0))
        hi.append(min(level0_dims[a], v1))
    return lo, hi


def node_from_index(index):
    d = 0
    while ((1 << (3 * (d + 1))) - 1) // 7 <= index:
        d += 1
    rem = index - ((1 << (3 * d)) - 1) // 7
    side = 1 << d
    return d, rem & (side - 1), (rem >> d) & (side - 1), rem >> (2 * d)


class OracleSession:
    """store: object with brick(c, l, coord), region_min_max(c, l, box) and
    manifest.levels[i].dims / brick_grid_dims, manifest.brick_size."""

    def __init__(self, store, m, depth, cache_slots, channels, render_kw, pad):
        man = store.manifest
        self.store = store
        self.k = len(man.levels)
        self.st = OracleResidency(m, self.k, man.brick_size,
                                  [l.dims for l in man.levels],
                                  [l.brick_grid_dims for l in man.levels],
                                  cache_slots, depth)
        self.channels = channels
        self.render_kw = dict(render_kw)
        self.pad = pad
        self.frame = 0
        self.mapping = list(range(m))
        self.level0 = man.levels[0].dims

    def oracle_state(self) -> orc.OracleState:
        s = self.st
        return orc.OracleState(m=s.m, k=s.k, brick_size=s.brick_size,
                               level_dims=s.level_dims, level_grids=s.level_grids,
                               pt_offsets=s.pt_offsets, pt_status=s.pt_status,
                               pt_slot=s.pt_slot, cache=s.cache, words=s.words,
                               depth=s.depth, eps_h=0.0)

    def render(self, camera, **kw):
        args = dict(self.render_kw)
        args.update(kw)
        return orc.render(self.oracle_state(), self.channels, camera, **args)

    def step_frame(self, camera):
        self.frame += 1
        out = self.render(camera)
        self.st.note_sampled(out.required_mask, self.frame)
        for bid in out.brick_requests:
            pt = (bid >> 24) & 0xFF
            slot, lev = pt // self.k, pt % self.k
            coord = (bid & 0xFF, (bid >> 8) & 0xFF, (bid >> 16) & 0xFF)
            payload = self.store.brick(self.mapping[slot], lev, coord)
            self.st.apply_brick(bid, payload, self.frame)
        for nidx, slot in out.metadata_requests:
            d, x, y, z = node_from_index(nidx)
            lo, hi = metadata_box(self.level0, d, x, y, z, self.pad)
            mn, mx = self.store.region_min_max(self.mapping[slot], 0,
                                               (lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]))
            self.st.set_node_metadata(nidx, slot, mn, mx)
        return out

    def swap_channel(self, slot, channel):
        self.st.swap_channel(slot)
        self.mapping[slot] = channel


def prepare_full(store, slots_to_channels, m, depth, cache_slots, pad,
                 box_minmax_grid):
    """bench.prepare_engine: prefill every brick of the mapped channels in
    (slot, level, z, y, x) order at frame 0, then exact metadata."""
    man = store.manifest
    k = len(man.levels)
    st = OracleResidency(m, k, man.brick_size, [l.dims for l in man.levels],
                         [l.brick_grid_dims for l in man.levels], cache_slots, depth)
    for slot in sorted(slots_to_channels):
        ch = slots_to_channels[slot]
        for lev in range(k):
            gx, gy, gz = man.levels[lev].brick_grid_dims
            for z in range(gz):
                for y in range(gy):
                    for x in range(gx):
                        bid = ((slot * k + lev) << 24) | (z << 16) | (y << 8) | x
                        st.apply_brick(bid, store.brick(ch, lev, (x, y, z)), 0)
    for slot, ch in slots_to_channels.items():
        vol = store.level_array(ch, 0)
        for d in range(depth + 1):
            side = 1 << d
            mins, maxs = box_minmax_grid(vol, side, pad)
            base = ((1 << (3 * d)) - 1) // 7
            w = (mins.astype(np.uint32) << 16) | (maxs.astype(np.uint32) << 24)
            masks = st.words[base:base + side ** 3, slot] & np.uint32(0xFFFF)
            st.words[base:base + side ** 3, slot] = masks | w.ravel()
    return st


def prepare_paging(store, slots_to_channels, m, depth, cache_slots, keep=None,
                   zero_as_empty=False):
    """Paging-only prefill in (slot, level, z, y, x) order at frame 0.

    ``zero_as_empty`` restates bench.py:74-95 (prepare_pagetable_engine):
    all-zero payloads are entered EMPTY instead of taking a cache slot.
    ``keep(slot, level, x, y, z)`` (optional) selects the bricks inserted,
    for partially resident baselines; the octree is left untouched."""
    man = store.manifest
    k = len(man.levels)
    st = OracleResidency(m, k, man.brick_size, [l.dims for l in man.levels],
                         [l.brick_grid_dims for l in man.levels], cache_slots, depth)
    for slot in sorted(slots_to_channels):
        ch = slots_to_channels[slot]
        for lev in range(k):
            gx, gy, gz = man.levels[lev].brick_grid_dims
            for z in range(gz):
                for y in range(gy):
                    for x in range(gx):
                        payload = store.brick(ch, lev, (x, y, z))
                        bid = ((slot * k + lev) << 24) | (z << 16) | (y << 8) | x
                        if zero_as_empty and int(payload.max()) == 0:
                            st.mark_empty(bid)
                        elif keep is None or keep(slot, lev, x, y, z):
                            st.insert_brick(bid, payload, 0)
    return st


def classic_metadata(level0_volumes, m, k):
    """Per-node min / max of the classic one-node-one-brick octree
    (render.py:271-315, ClassicMetadata.build_from_volume): node depth d
    holds the exact min / max of its (dims / 2^d)-voxel block of the level-0
    volume, depth = k - 1.  Unfilled slots keep (min 0, max 255).
    Returns (min u8[n, m], max u8[n, m], depth)."""
    depth = k - 1
    n_nodes = ((1 << (3 * k)) - 1) // 7
    mins = np.zeros((n_nodes, m), dtype=np.uint8)
    maxs = np.full((n_nodes, m), 255, dtype=np.uint8)
    for slot, vol in level0_volumes.items():
        g = 1 << depth
        nz, ny, nx = vol.shape
        blocks = vol.reshape(g, nz // g, g, ny // g, g, nx // g)
        lo = blocks.min(axis=(1, 3, 5))
        hi = blocks.max(axis=(1, 3, 5))
        for d in range(depth, -1, -1):
            base = ((1 << (3 * d)) - 1) // 7
            side = 1 << d
            mins[base:base + side ** 3, slot] = lo.reshape(-1)
            maxs[base:base + side ** 3, slot] = hi.reshape(-1)
            if d:
                h = side // 2
                lo = lo.reshape(h, 2, h, 2, h, 2).min(axis=(1, 3, 5))
                hi = hi.reshape(h, 2, h, 2, h, 2).max(axis=(1, 3, 5))
    return mins, maxs, depth
