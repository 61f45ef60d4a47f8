"""Pure-Python restatement of the residency state updates -- TEST INFRASTRUCTURE ONLY.

Sequential, exactly as the reference mutates its state between frames:

* ``insert_brick`` LRU: LIFO free list, victim = occupied slot with minimum
  (last_used, slot)  -- ``paging.py:187-218``, ``_release_slot`` 236-239;
* ``set_channel_mapping`` -- ``paging.py:263-284``; ``mark_empty`` 228-234;
* octree residency masks: insert/evict with OR propagation --
  ``octree.py:193-246`` (exact open-box overlap via integer arithmetic that
  equals the reference's ``fractions.Fraction`` form, ``octree.py:126-189``);
* ``set_node_metadata`` / ``invalidate_channel`` -- ``octree.py:263-273``;
* ``Engine.note_sampled`` / ``apply_brick`` / ``swap_channel`` --
  ``engine.py:72-105``.

Arrays use the reference layout (pt_status/pt_slot, words u32[N, m]).
"""

from __future__ import annotations

import numpy as np

UNMAPPED, MAPPED, EMPTY = 0, 1, 2
INVALID_WORD = 0x00FF0000


def level_offset(d: int) -> int:
    return ((1 << (3 * d)) - 1) // 7


def decode(bid: int, k: int):
    return (((bid >> 24) & 0xFF) // k, ((bid >> 24) & 0xFF) % k,
            (bid & 0xFF, (bid >> 8) & 0xFF, (bid >> 16) & 0xFF))


def encode(slot: int, level: int, coord, k: int) -> int:
    x, y, z = coord
    return ((slot * k + level) << 24) | (z << 16) | (y << 8) | x


def _floor_div(a, b):
    return a // b


def _ceil_div(a, b):
    return -((-a) // b)


class OracleResidency:
    """Reference-semantics paging + octree over numpy arrays."""

    def __init__(self, m, k, brick_size, level_dims, level_grids, cache_slots,
                 depth, with_payloads=True):
        self.m, self.k, self.depth = m, k, depth
        self.brick_size = tuple(brick_size)
        self.level_dims = np.array(level_dims, dtype=np.int32)
        self.level_grids = np.array(level_grids, dtype=np.int32)
        sizes = [int(np.prod(self.level_grids[pt % k])) for pt in range(m * k)]
        self.pt_offsets = np.zeros(m * k + 1, dtype=np.int64)
        np.cumsum(sizes, out=self.pt_offsets[1:])
        total = int(self.pt_offsets[-1])
        self.pt_status = np.zeros(total, dtype=np.int8)
        self.pt_slot = np.full(total, -1, dtype=np.int32)
        self.num_slots = int(np.prod(cache_slots))
        sx, sy, sz = self.brick_size
        self.cache = (np.zeros((self.num_slots, sz, sy, sx), dtype=np.uint8)
                      if with_payloads else None)
        self.slot_brick = np.full(self.num_slots, -1, dtype=np.int64)
        self.slot_last_used = np.zeros(self.num_slots, dtype=np.int64)
        self.free = list(range(self.num_slots - 1, -1, -1))
        self.num_nodes = level_offset(depth + 1)
        self.words = np.full((self.num_nodes, m), INVALID_WORD, dtype=np.uint32)

    # -- addressing ---------------------------------------------------------
    def entry(self, slot, level, coord):
        gx, gy, _ = (int(v) for v in self.level_grids[level])
        x, y, z = coord
        return int(self.pt_offsets[slot * self.k + level]) + (z * gy + y) * gx + x

    def leaf_range(self, level, coord):
        """Leaves overlapping the brick's open box (octree.py:126-159)."""
        D = self.depth
        side = 1 << D
        out = []
        for a in range(3):
            B = self.brick_size[a]
            dim = int(self.level_dims[level][a])
            lo = max(0, _floor_div(coord[a] * B * side, dim))
            hi = min(side - 1, _ceil_div((coord[a] + 1) * B * side, dim) - 1)
            if lo > hi:
                return None
            out.append((lo, hi))
        return out

    def brick_range(self, d, node, level):
        """Bricks of `level` overlapping the node's open box (octree.py:161-189)."""
        side = 1 << d
        out = []
        for a in range(3):
            B = self.brick_size[a]
            dim = int(self.level_dims[level][a])
            grid = int(self.level_grids[level][a])
            lo = max(0, _floor_div(node[a] * dim, side * B))
            hi = min(grid - 1, _ceil_div((node[a] + 1) * dim, side * B) - 1)
            if lo > hi:
                return None
            out.append((lo, hi))
        return out

    def node_index(self, d, x, y, z):
        return level_offset(d) + ((z << d) + y << d) + x

    # -- paging -------------------------------------------------------------
    def insert_brick(self, bid, payload, frame):
        slot, level, coord = decode(bid, self.k)
        idx = self.entry(slot, level, coord)
        if self.pt_status[idx] == MAPPED:
            return int(self.pt_slot[idx]), None
        evicted = None
        if self.free:
            lin = self.free.pop()
        else:
            occupied = np.flatnonzero(self.slot_brick >= 0)
            lin = int(occupied[np.argmin(self.slot_last_used[occupied])])
            evicted = int(self.slot_brick[lin])
            es, el, ec = decode(evicted, self.k)
            e_idx = self.entry(es, el, ec)
            self.pt_status[e_idx] = UNMAPPED
            self.pt_slot[e_idx] = -1
        if self.cache is not None and payload is not None:
            self.cache[lin] = payload
        self.slot_brick[lin] = bid
        self.slot_last_used[lin] = frame
        self.pt_status[idx] = MAPPED
        self.pt_slot[idx] = lin
        return lin, evicted

    def release_slot(self, lin):
        self.slot_brick[lin] = -1
        self.slot_last_used[lin] = 0
        self.free.append(lin)

    def mark_empty(self, bid):
        slot, level, coord = decode(bid, self.k)
        idx = self.entry(slot, level, coord)
        if self.pt_status[idx] == MAPPED:
            self.release_slot(int(self.pt_slot[idx]))
        self.pt_status[idx] = EMPTY
        self.pt_slot[idx] = -1

    def set_channel_mapping(self, channel_slot):
        for level in range(self.k):
            pt = channel_slot * self.k + level
            lo, hi = int(self.pt_offsets[pt]), int(self.pt_offsets[pt + 1])
            self.pt_status[lo:hi] = UNMAPPED
            self.pt_slot[lo:hi] = -1
        for lin in np.flatnonzero(self.slot_brick >= 0):
            slot, _, _ = decode(int(self.slot_brick[lin]), self.k)
            if slot == channel_slot:
                self.release_slot(int(lin))

    # -- octree -------------------------------------------------------------
    def _leaf_backed(self, leaf, slot, level):
        r = self.brick_range(self.depth, leaf, level)
        if r is None:
            return False
        for z in range(r[2][0], r[2][1] + 1):
            for y in range(r[1][0], r[1][1] + 1):
                for x in range(r[0][0], r[0][1] + 1):
                    if self.pt_status[self.entry(slot, level, (x, y, z))] == MAPPED:
                        return True
        return False

    def _leaves(self, level, coord):
        r = self.leaf_range(level, coord)
        if r is None:
            return []
        return [(x, y, z) for z in range(r[2][0], r[2][1] + 1)
                for y in range(r[1][0], r[1][1] + 1)
                for x in range(r[0][0], r[0][1] + 1)]

    def on_brick_inserted(self, bid):
        slot, level, coord = decode(bid, self.k)
        bit = np.uint32(1 << level)
        changed = []
        for leaf in self._leaves(level, coord):
            li = self.node_index(self.depth, *leaf)
            w = self.words[li, slot]
            if not w & bit:
                self.words[li, slot] = w | bit
                changed.append(leaf)
        self._propagate_up(changed, slot)

    def on_brick_evicted(self, bid):
        slot, level, coord = decode(bid, self.k)
        bit = np.uint32(1 << level)
        changed = []
        for leaf in self._leaves(level, coord):
            li = self.node_index(self.depth, *leaf)
            w = self.words[li, slot]
            if not w & bit:
                continue
            if not self._leaf_backed(leaf, slot, level):
                self.words[li, slot] = w & ~bit
                changed.append(leaf)
        self._propagate_up(changed, slot)

    def _propagate_up(self, changed, slot):
        frontier = set(changed)
        d = self.depth
        while d > 0 and frontier:
            parents = {(x >> 1, y >> 1, z >> 1) for x, y, z in frontier}
            frontier = set()
            for px, py, pz in parents:
                mask = np.uint32(0)
                for kz in (0, 1):
                    for jy in (0, 1):
                        for ix in (0, 1):
                            ci = self.node_index(d, 2 * px + ix, 2 * py + jy,
                                                 2 * pz + kz)
                            mask |= self.words[ci, slot] & np.uint32(0xFFFF)
                pi = self.node_index(d - 1, px, py, pz)
                w = self.words[pi, slot]
                new = (w & np.uint32(0xFFFF0000)) | mask
                if new != w:
                    self.words[pi, slot] = new
                    frontier.add((px, py, pz))
            d -= 1

    def set_node_metadata(self, node_index, slot, mn, mx):
        w = int(self.words[node_index, slot])
        self.words[node_index, slot] = np.uint32((w & 0xFFFF) | (mn << 16) | (mx << 24))

    def invalidate_channel(self, slot):
        self.words[:, slot] = INVALID_WORD

    # -- engine -------------------------------------------------------------
    def apply_brick(self, bid, payload, frame):
        lin, evicted = self.insert_brick(bid, payload, frame)
        if evicted is not None:
            self.on_brick_evicted(evicted)
        self.on_brick_inserted(bid)
        return lin, evicted

    def note_sampled(self, required_mask, frame):
        for e in np.flatnonzero(required_mask):
            if self.pt_status[e] == MAPPED:
                self.slot_last_used[int(self.pt_slot[e])] = frame

    def swap_channel(self, channel_slot):
        self.set_channel_mapping(channel_slot)
        self.invalidate_channel(channel_slot)

    def masks_from_scratch(self):
        """Leaf ground truth + OR closure (octree.py:355-395) as one array."""
        out = self.words & np.uint32(0xFFFF0000)
        side = 1 << self.depth
        for s in range(self.m):
            for level in range(self.k):
                for z in range(side):
                    for y in range(side):
                        for x in range(side):
                            if self._leaf_backed((x, y, z), s, level):
                                li = self.node_index(self.depth, x, y, z)
                                out[li, s] |= np.uint32(1 << level)
        for d in range(self.depth - 1, -1, -1):
            sd = 1 << d
            for z in range(sd):
                for y in range(sd):
                    for x in range(sd):
                        pi = self.node_index(d, x, y, z)
                        for s in range(self.m):
                            mask = np.uint32(0)
                            for kz in (0, 1):
                                for jy in (0, 1):
                                    for ix in (0, 1):
                                        ci = self.node_index(d + 1, 2 * x + ix,
                                                             2 * y + jy, 2 * z + kz)
                                        mask |= out[ci, s] & np.uint32(0xFFFF)
                            out[pi, s] |= mask
        return out
