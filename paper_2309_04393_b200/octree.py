"""Device-resident residency octree (octree.py:19-406 of the reference).

One u32 word per (node, channel slot), node-major, in HBM as
``words_dev`` int32[N, m] (bit pattern = the reference's uint32): bits 0-15
residency mask per level, 16-23 min, 24-31 max; 0x00FF0000 = INVALID.
Nodes are pointerless: depth d starts at (8^d - 1)/7 and is z-major.

Updates after uploads/evictions run in libresoct.so (residency.cu, kernel
2).  The host-side geometry here (integer form of the reference's exact
``fractions.Fraction`` overlap tests, octree.py:126-189) serves tests and
introspection.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .paging import MAPPED, MultiChannelPaging

INVALID_WORD = np.uint32(0x00FF0000)


class OctreeError(ValueError):
    pass


@dataclass(frozen=True)
class OctreeConfig:
    depth: int
    channel_slots: int
    homogeneity_eps: float = 0.0
    min_metadata_voxels: int = 1

    def __post_init__(self):
        if not 0 <= self.depth <= 15:
            raise OctreeError("depth must be in [0, 15]")
        if self.min_metadata_voxels < 1:
            raise OctreeError("minMetadataVoxels must be positive")
        if not 0.0 <= self.homogeneity_eps <= 255.0:
            raise OctreeError("homogeneity epsilon outside [0, 255]")


@dataclass(frozen=True)
class NodeAddress:
    d: int
    x: int
    y: int
    z: int

    def __post_init__(self):
        side = 1 << self.d
        if not (0 <= self.x < side and 0 <= self.y < side and 0 <= self.z < side):
            raise OctreeError(f"node coord outside level {self.d} grid")

    @property
    def index(self) -> int:
        return level_offset(self.d) + ((self.z << self.d) + self.y << self.d) + self.x

    @property
    def parent(self):
        if self.d == 0:
            return None
        return NodeAddress(self.d - 1, self.x >> 1, self.y >> 1, self.z >> 1)

    def children(self):
        d = self.d + 1
        return [NodeAddress(d, 2 * self.x + i, 2 * self.y + j, 2 * self.z + k)
                for k in (0, 1) for j in (0, 1) for i in (0, 1)]


def level_offset(d: int) -> int:
    return ((1 << (3 * d)) - 1) // 7


def total_nodes(depth: int) -> int:
    return ((1 << (3 * (depth + 1))) - 1) // 7


def node_from_index(index: int) -> NodeAddress:
    if index < 0:
        raise OctreeError(f"negative node index {index}")
    d = 0
    while level_offset(d + 1) <= index:
        d += 1
    rem = index - level_offset(d)
    side = 1 << d
    return NodeAddress(d, rem & (side - 1), (rem >> d) & (side - 1), rem >> (2 * d))


def _floor_div(a, b):
    return a // b


def _ceil_div(a, b):
    return -((-a) // b)


class ResidencyOctree:
    def __init__(self, config: OctreeConfig, paging: MultiChannelPaging):
        self.config = config
        self.paging = paging
        self.k = paging.config.k
        if config.channel_slots != paging.config.m:
            raise OctreeError("octree and paging disagree on channel slots")
        self.num_nodes = total_nodes(config.depth)
        self.words_dev = torch.full((self.num_nodes, config.channel_slots),
                                    int(INVALID_WORD), dtype=torch.int32,
                                    device=paging.device)
        paging._attach_octree(self.words_dev, config.depth)

    # -- host snapshot ------------------------------------------------------

    @property
    def words(self) -> np.ndarray:
        return self.words_dev.cpu().numpy().view(np.uint32)

    def upload_words(self, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint32).view(np.int32)
        self.words_dev.copy_(torch.from_numpy(w).reshape(self.words_dev.shape))

    def _word(self, addr: NodeAddress, slot: int) -> int:
        return int(self.words_dev[addr.index, slot].item()) & 0xFFFFFFFF

    # -- geometry (exact, integer) ------------------------------------------

    def leaf_range(self, level, coord):
        D = self.config.depth
        side = 1 << D
        B = self.paging.config.brick_size
        out = []
        for a in range(3):
            dim = int(self.paging.level_dims[level][a])
            lo = max(0, _floor_div(coord[a] * B[a] * side, dim))
            hi = min(side - 1, _ceil_div((coord[a] + 1) * B[a] * side, dim) - 1)
            if lo > hi:
                return None
            out.append((lo, hi))
        return out

    def leaves_for_brick(self, level, coord):
        r = self.leaf_range(level, coord)
        if r is None:
            return []
        D = self.config.depth
        return [NodeAddress(D, x, y, z) for z in range(r[2][0], r[2][1] + 1)
                for y in range(r[1][0], r[1][1] + 1) for x in range(r[0][0], r[0][1] + 1)]

    def bricks_overlapping(self, addr: NodeAddress, level):
        dims = self.paging.level_dims[level]
        grid = self.paging.level_grids[level]
        B = self.paging.config.brick_size
        side = 1 << addr.d
        node = (addr.x, addr.y, addr.z)
        ranges = []
        for a in range(3):
            lo = max(0, _floor_div(node[a] * int(dims[a]), side * B[a]))
            hi = min(int(grid[a]) - 1, _ceil_div((node[a] + 1) * int(dims[a]), side * B[a]) - 1)
            if lo > hi:
                return []
            ranges.append((lo, hi))
        return [(x, y, z) for z in range(ranges[2][0], ranges[2][1] + 1)
                for y in range(ranges[1][0], ranges[1][1] + 1)
                for x in range(ranges[0][0], ranges[0][1] + 1)]

    # -- metadata from bricks (octree.py:275-329) ----------------------------

    def _voxel_ranges(self, addr: NodeAddress, level: int) -> list:
        """Half-open voxel ranges of `level` whose open cells meet the node's
        open extent (octree.py:316-329, exact integer form)."""
        dims = self.paging.level_dims[level]
        side = 1 << addr.d
        node = (addr.x, addr.y, addr.z)
        out = []
        for a in range(3):
            n = int(dims[a])
            v0 = max(0, _floor_div(node[a] * n, side))
            v1 = min(n, _ceil_div((node[a] + 1) * n, side))
            out.append((v0, v1))
        return out

    def choose_metadata_level(self, addr: NodeAddress) -> int:
        """Coarsest level whose footprint in the node meets
        min_metadata_voxels (octree.py:307-314)."""
        for level in range(self.paging.config.k - 1, -1, -1):
            count = 1
            for v0, v1 in self._voxel_ranges(addr, level):
                count *= max(0, v1 - v0)
            if count >= self.config.min_metadata_voxels:
                return level
        return 0

    def compute_node_metadata_from_bricks(self, addr: NodeAddress, slot: int, fetch):
        """Min / max over the node's extent at choose_metadata_level, from the
        overlapping bricks (octree.py:275-306).  fetch(slot, level, coord)
        returns a payload (numpy or torch); it may raise, leaving the node
        INVALID.  The reduction runs on the device (ro_bricks_box_minmax)."""
        level = self.choose_metadata_level(addr)
        dims = [int(v) for v in self.paging.level_dims[level]]
        B = self.paging.config.brick_size
        vr = self._voxel_ranges(addr, level)
        coords, boxes = [], []
        for coord in self.bricks_overlapping(addr, level):
            box = []
            for a in range(3):
                c0 = coord[a] * B[a]
                box.append((max(vr[a][0], c0) - c0, min(vr[a][1], c0 + B[a], dims[a]) - c0))
            if any(lo >= hi for lo, hi in box):
                continue
            coords.append(coord)
            boxes.append([box[0][0], box[1][0], box[2][0], box[0][1], box[1][1], box[2][1]])
        if not coords:
            return 0, 0  # the extent met no in-volume voxels
        dev = self.paging.device
        pays = torch.stack([torch.as_tensor(fetch(slot, level, c)).to(dev).reshape(
            B[2], B[1], B[0]) for c in coords]).contiguous()
        bx_ = torch.as_tensor(np.array(boxes, dtype=np.int32)).to(dev)
        mins = torch.empty(len(coords), dtype=torch.uint8, device=dev)
        maxs = torch.empty(len(coords), dtype=torch.uint8, device=dev)
        N.check(N.lib().ro_bricks_box_minmax(pays.data_ptr(), bx_.data_ptr(), len(coords),
                                             B[0], B[1], B[2], mins.data_ptr(),
                                             maxs.data_ptr(), N.stream_ptr()))
        return int(mins.min().item()), int(maxs.max().item())

    # -- residency updates (native) -----------------------------------------

    def update_for_bricks(self, brick_ids):
        """Recompute the masks of every leaf the bricks overlap, then OR up.

        Serves both on_brick_inserted and on_brick_evicted: masks are a pure
        function of the resident set (octree.py:355-395)."""
        ids = np.ascontiguousarray(np.asarray(brick_ids, dtype=np.int64).reshape(-1))
        if len(ids) == 0:
            return
        p = self.paging
        p._ids_array(ids)
        st = p.state()
        N.check(N.lib().ro_octree_update(p.ctx, C.byref(st), ids.ctypes.data, len(ids),
                                         N.stream_ptr()))

    def on_brick_inserted(self, brick_id: int):
        self.update_for_bricks([brick_id])

    def on_brick_evicted(self, brick_id: int):
        """Call after the page entry is UNMAPPED (octree.py:204-219)."""
        self.update_for_bricks([brick_id])

    def rebuild_masks(self):
        p = self.paging
        st = p.state()
        N.check(N.lib().ro_rebuild_masks(p.ctx, C.byref(st), N.stream_ptr()))

    # -- metadata -----------------------------------------------------------

    def residency_mask(self, addr: NodeAddress, slot: int) -> int:
        return self._word(addr, slot) & 0xFFFF

    def metadata(self, addr: NodeAddress, slot: int):
        w = self._word(addr, slot)
        mn, mx = (w >> 16) & 0xFF, (w >> 24) & 0xFF
        if mn == 255 and mx == 0:
            return None
        return mn, mx

    def is_valid(self, addr, slot) -> bool:
        return self.metadata(addr, slot) is not None

    def is_empty(self, addr: NodeAddress, slots, tfs: dict) -> bool:
        """octree.py:333-342: every slot has valid metadata whose range maps
        to zero opacity under that slot's transfer function."""
        for slot in slots:
            meta = self.metadata(addr, slot)
            if meta is None or tfs[slot].interval_max_opacity(meta[0], meta[1]) != 0.0:
                return False
        return True

    def is_homogeneous(self, addr: NodeAddress, slots) -> bool:
        """octree.py:344-351"""
        for slot in slots:
            meta = self.metadata(addr, slot)
            if meta is None or meta[1] - meta[0] > self.config.homogeneity_eps:
                return False
        return True

    def overlapping_leaves(self, box_lo, box_hi) -> list:
        """octree.py:126-147: leaves whose open extent meets the open box
        (coordinates as Fractions, ints or floats; exact)."""
        from fractions import Fraction
        import math
        side = 1 << self.config.depth
        ranges = []
        for a in range(3):
            lo = Fraction(box_lo[a]) * side
            hi = Fraction(box_hi[a]) * side
            i_lo = max(0, math.floor(lo))
            i_hi = min(side - 1, math.ceil(hi) - 1)
            if i_lo > i_hi:
                return []
            ranges.append((i_lo, i_hi))
        D = self.config.depth
        return [NodeAddress(D, x, y, z) for z in range(ranges[2][0], ranges[2][1] + 1)
                for y in range(ranges[1][0], ranges[1][1] + 1)
                for x in range(ranges[0][0], ranges[0][1] + 1)]

    def set_node_metadata(self, addr: NodeAddress, slot: int, min_val: int, max_val: int):
        self.set_metadata_batch([addr.index], [slot], [min_val], [max_val])

    def set_metadata_batch(self, node_idx, slots, mins, maxs):
        node_idx = np.ascontiguousarray(node_idx, dtype=np.int64)
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        mins = np.ascontiguousarray(mins, dtype=np.int32)
        maxs = np.ascontiguousarray(maxs, dtype=np.int32)
        n = len(node_idx)
        if n == 0:
            return
        bad = ~((0 <= mins) & (mins <= maxs) & (maxs <= 255))
        if bad.any():
            i = int(np.flatnonzero(bad)[0])
            raise OctreeError(f"need 0 <= min <= max <= 255, got ({mins[i]},{maxs[i]})")
        p = self.paging
        st = p.state()
        N.check(N.lib().ro_apply_metadata(p.ctx, C.byref(st), node_idx.ctypes.data,
                                          slots.ctypes.data, mins.ctypes.data,
                                          maxs.ctypes.data, n, N.stream_ptr()))

    def write_level_metadata(self, slot: int, d: int, mins: torch.Tensor, maxs: torch.Tensor):
        """Bulk metadata for every node of depth d (device u8 grids, z,y,x)."""
        side = 1 << d
        mins = mins.to(device=self.words_dev.device, dtype=torch.uint8).contiguous()
        maxs = maxs.to(device=self.words_dev.device, dtype=torch.uint8).contiguous()
        if mins.numel() != side ** 3 or maxs.numel() != side ** 3:
            raise OctreeError("metadata grid size mismatch")
        p = self.paging
        st = p.state()
        N.check(N.lib().ro_write_level_metadata(p.ctx, C.byref(st), slot, d,
                                                mins.data_ptr(), maxs.data_ptr(),
                                                N.stream_ptr()))

    def invalidate_channel(self, slot: int):
        self.words_dev[:, slot] = int(INVALID_WORD)

    # -- full-scan invariants (host) ----------------------------------------

    def check_mask_consistency(self):
        w = self.words.astype(np.int64) & 0xFFFF
        for d in range(self.config.depth):
            side = 1 << d
            cs = side * 2
            child = w[level_offset(d + 1):level_offset(d + 2)].reshape(cs, cs, cs, -1)
            ored = np.zeros((side, side, side, w.shape[1]), dtype=np.int64)
            for dz in (0, 1):
                for dy in (0, 1):
                    for dx in (0, 1):
                        ored |= child[dz::2, dy::2, dx::2]
            got = w[level_offset(d):level_offset(d + 1)].reshape(side, side, side, -1)
            if not np.array_equal(got, ored):
                raise AssertionError(f"depth {d}: mask != OR(children)")

    def check_leaf_ground_truth(self):
        p = self.paging
        sb = p.slot_brick
        resident = {}
        for b in sb[sb >= 0]:
            slot, level, coord = p.decode(int(b))
            resident.setdefault((slot, level), set()).add(coord)
        D = self.config.depth
        side = 1 << D
        w = self.words
        for slot in range(self.config.channel_slots):
            for level in range(self.k):
                truth = np.zeros((side, side, side), dtype=bool)
                for coord in resident.get((slot, level), ()):
                    r = self.leaf_range(level, coord)
                    if r is not None:
                        truth[r[2][0]:r[2][1] + 1, r[1][0]:r[1][1] + 1,
                              r[0][0]:r[0][1] + 1] = True
                got = (w[level_offset(D):level_offset(D + 1), slot] >> level) & 1
                if not np.array_equal(got.reshape(side, side, side).astype(bool), truth):
                    raise AssertionError(f"slot {slot} level {level}: leaf masks differ")
