"""Device-resident page tables + LRU brick cache (paging.py:23-312 of the reference).

Layout in HBM (torch tensors owned here, borrowed by libresoct.so):

* ``pt``          int32[E]   packed page-table entry: cache slot if MAPPED,
                             -1 UNMAPPED, -2 EMPTY (one 4-byte probe per
                             lookup instead of the reference's i8 + i32 pair)
* ``cache_dev``   uint8[S, bz, by, bx]  the brick cache
* ``slot_brick_dev``, ``slot_last_used_dev``  int64[S]
* ``free_stack``  int32[S] LIFO free list (top at free_count-1) + ``free_count``

Reference-named attributes (``pt_status``, ``pt_slot``, ``cache``,
``slot_brick``, ``slot_last_used``, ``_free``) are host snapshots for tests
and introspection; all mutation goes through the native calls.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N

UNMAPPED = 0
MAPPED = 1
EMPTY = 2

_STATUS_NAMES = {UNMAPPED: "UNMAPPED", MAPPED: "MAPPED", EMPTY: "EMPTY"}


class PagingError(ValueError):
    pass


@dataclass(frozen=True)
class PagingConfig:
    brick_size: tuple
    cache_slots: tuple
    m: int
    k: int

    def __post_init__(self):
        if self.m * self.k > 256:
            raise PagingError("m*k must be <= 256 (8-bit page table ID)")
        if math.prod(self.cache_slots) < 1:
            raise PagingError("cache must have at least one slot")
        if self.m < 1 or self.k < 1:
            raise PagingError("m and k must be >= 1")


def encode_brick_id(channel_slot, level, coord, k, m) -> int:
    x, y, z = coord
    if not (0 <= channel_slot < m and 0 <= level < k):
        raise PagingError(f"slot/level out of range: ({channel_slot},{level})")
    if not all(0 <= v < 256 for v in (x, y, z)):
        raise PagingError(f"brick coord out of 8-bit range: {coord}")
    return ((channel_slot * k + level) << 24) | (z << 16) | (y << 8) | x


def decode_brick_id(brick_id: int, k: int):
    if not (0 <= brick_id < 1 << 32):
        raise PagingError(f"brick id out of 32-bit range: {brick_id}")
    x = brick_id & 0xFF
    y = (brick_id >> 8) & 0xFF
    z = (brick_id >> 16) & 0xFF
    pt = (brick_id >> 24) & 0xFF
    return pt // k, pt % k, (x, y, z)


@dataclass(frozen=True)
class VirtualAddress:
    level: int
    channel_slot: int
    position: tuple


@dataclass(frozen=True)
class Translation:
    status: int
    cache_slot: tuple | None = None
    local_coord: tuple | None = None

    @property
    def status_name(self) -> str:
        return _STATUS_NAMES[self.status]


class PinnedBrickBuffer:
    """Recycled page-locked host buffer that a frame's fetched bricks are
    stacked into, so ro_apply_bricks DMAs them straight to the device on its
    upload stream (no second host copy through the staging buffer).  The
    returned view is valid until the next ``stack`` call; apply_bricks has
    finished reading it when it returns."""

    def __init__(self, brick_shape_zyx):
        self.brick_shape = tuple(brick_shape_zyx)
        self._buf = None

    def reserve(self, n: int):
        """Page-locked room for n bricks ahead of the first batch."""
        need = n * math.prod(self.brick_shape)
        if self._buf is None or self._buf.numel() < need:
            self._buf = torch.empty(need, dtype=torch.uint8, pin_memory=True)

    def stack(self, payloads):
        n = len(payloads)
        for i, p in enumerate(payloads):   # insert_brick's check (paging.py:196-197)
            if np.shape(p) != self.brick_shape:
                raise PagingError(f"payload shape {np.shape(p)} != brick size "
                                  f"(payload {i} of {n})")
        if any(np.asarray(p).dtype != np.uint8 for p in payloads):
            return np.stack(payloads)   # insert_bricks converts / reports it
        need = n * math.prod(self.brick_shape)
        if self._buf is None or self._buf.numel() < need:
            cap = max(need, 2 * (0 if self._buf is None else self._buf.numel()))
            self._buf = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        view = self._buf[:need].view(n, *self.brick_shape)
        np.stack(payloads, out=view.numpy())
        return view


class MultiChannelPaging:
    """m channel slots x k levels of page tables over one device brick cache.

    Single writer: mutate only between render passes (paging.py:84-87)."""

    def __init__(self, config: PagingConfig, level_dims, level_grids,
                 device=None):
        N.require_cuda()
        if len(level_dims) != config.k or len(level_grids) != config.k:
            raise PagingError("need dims and grid per level")
        self.config = config
        self.device = torch.device(device if device is not None else "cuda")
        self.level_dims = np.array(level_dims, dtype=np.int32)
        self.level_grids = np.array(level_grids, dtype=np.int32)
        if (self.level_grids > 256).any():
            raise PagingError("brick grid exceeds 256 per axis")
        n_pt = config.m * config.k
        sizes = [int(np.prod(self.level_grids[pt % config.k])) for pt in range(n_pt)]
        self.pt_offsets = np.zeros(n_pt + 1, dtype=np.int64)
        np.cumsum(sizes, out=self.pt_offsets[1:])
        self.total_entries = int(self.pt_offsets[-1])
        sx, sy, sz = config.brick_size
        self.num_slots = math.prod(config.cache_slots)
        dev = self.device
        self.pt = torch.full((self.total_entries,), N.RO_PT_UNMAPPED,
                             dtype=torch.int32, device=dev)
        # one brick of tail padding: the ray caster may read (never use) the
        # byte after a brick's last tap (resoct.h, ro_state.cache)
        self._cache_storage = torch.zeros((self.num_slots + 1, sz, sy, sx),
                                          dtype=torch.uint8, device=dev)
        self.cache_dev = self._cache_storage[:self.num_slots]
        self.slot_brick_dev = torch.full((self.num_slots,), -1, dtype=torch.int64,
                                         device=dev)
        self.slot_last_used_dev = torch.zeros(self.num_slots, dtype=torch.int64,
                                              device=dev)
        self.free_stack = torch.arange(self.num_slots - 1, -1, -1, dtype=torch.int32,
                                       device=dev)
        self.free_count = torch.tensor([self.num_slots], dtype=torch.int32, device=dev)
        # dilated 8^3 sub-block maxima per slot (resoct.h ro_state.sub_max),
        # maintained by every insert; 255 = unknown
        if min(sx, sy, sz) >= N.RO_SUB_EDGE:
            e = N.RO_SUB_EDGE_ALLOC
            nsb = (sx // e) * (sy // e) * (sz // e)
            self.sub_max = torch.full((self.num_slots * nsb,), 255, dtype=torch.uint8,
                                      device=dev)
        else:
            self.sub_max = None
        self.channel_mapping = list(range(config.m))
        self._octree_words = None
        self._depth = 0
        self._ctx = None

    # -- native context -----------------------------------------------------

    def _attach_octree(self, words: torch.Tensor, depth: int):
        self._octree_words = words
        if self._ctx is not None and self._depth != depth:
            N.lib().ro_destroy(self._ctx)
            self._ctx = None
        self._depth = depth

    def layout(self) -> N.Layout:
        L = N.Layout()
        L.m, L.k, L.depth = self.config.m, self.config.k, self._depth
        for a in range(3):
            L.brick[a] = self.config.brick_size[a]
        for lev in range(self.config.k):
            for a in range(3):
                L.level_dims[lev][a] = int(self.level_dims[lev][a])
                L.level_grids[lev][a] = int(self.level_grids[lev][a])
        for i, v in enumerate(self.pt_offsets):
            L.pt_offsets[i] = int(v)
        L.num_slots = self.num_slots
        return L

    @property
    def ctx(self):
        if self._ctx is None:
            lib = N.lib()
            with torch.cuda.device(self.device):
                h = C.c_void_p()
                lay = self.layout()
                N.check(lib.ro_create(C.byref(lay), C.byref(h)))
            self._ctx = h
        return self._ctx

    def state(self, with_words: bool = True) -> N.State:
        st = N.State()
        st.words = (self._octree_words.data_ptr()
                    if (with_words and self._octree_words is not None) else None)
        st.pt = self.pt.data_ptr()
        st.cache = self.cache_dev.data_ptr()
        st.slot_brick = self.slot_brick_dev.data_ptr()
        st.slot_last_used = self.slot_last_used_dev.data_ptr()
        st.free_stack = self.free_stack.data_ptr()
        st.free_count = self.free_count.data_ptr()
        st.sub_max = self.sub_max.data_ptr() if self.sub_max is not None else None
        return st

    def __del__(self):
        try:
            if self._ctx is not None and N._LIB is not None:
                N._LIB.ro_destroy(self._ctx)
                self._ctx = None
        except Exception:
            pass

    # -- addressing ---------------------------------------------------------

    def _pt_index(self, channel_slot, level) -> int:
        if not (0 <= channel_slot < self.config.m and 0 <= level < self.config.k):
            raise PagingError(f"bad slot/level ({channel_slot},{level})")
        return channel_slot * self.config.k + level

    def _entry_index(self, channel_slot, level, coord) -> int:
        pt = self._pt_index(channel_slot, level)
        gx, gy, gz = (int(v) for v in self.level_grids[level])
        x, y, z = coord
        if not (0 <= x < gx and 0 <= y < gy and 0 <= z < gz):
            raise PagingError(f"brick coord {coord} outside grid {(gx, gy, gz)}")
        return int(self.pt_offsets[pt]) + (z * gy + y) * gx + x

    def slot_triple(self, linear: int):
        cx, cy, _ = self.config.cache_slots
        return (linear % cx, (linear // cx) % cy, linear // (cx * cy))

    def slot_linear(self, triple) -> int:
        cx, cy, cz = self.config.cache_slots
        x, y, z = triple
        if not (0 <= x < cx and 0 <= y < cy and 0 <= z < cz):
            raise PagingError(f"cache slot {triple} out of range")
        return (z * cy + y) * cx + x

    def brick_coord_of(self, level, position):
        dims = self.level_dims[level]
        grid = self.level_grids[level]
        out = []
        for a in range(3):
            c = int(position[a] * dims[a] // self.config.brick_size[a])
            out.append(min(max(c, 0), int(grid[a]) - 1))
        return tuple(out)

    def encode(self, channel_slot, level, coord) -> int:
        self._entry_index(channel_slot, level, coord)
        return encode_brick_id(channel_slot, level, coord, self.config.k, self.config.m)

    def decode(self, brick_id):
        return decode_brick_id(brick_id, self.config.k)

    # -- host snapshots (reference attribute names) -------------------------

    @property
    def pt_status(self) -> np.ndarray:
        p = self.pt.cpu().numpy()
        out = np.zeros(p.shape, dtype=np.int8)
        out[p >= 0] = MAPPED
        out[p == N.RO_PT_EMPTY] = EMPTY
        return out

    @property
    def pt_slot(self) -> np.ndarray:
        p = self.pt.cpu().numpy()
        return np.where(p >= 0, p, -1).astype(np.int32)

    @property
    def cache(self) -> np.ndarray:
        return self.cache_dev.cpu().numpy()

    @property
    def slot_brick(self) -> np.ndarray:
        return self.slot_brick_dev.cpu().numpy()

    @property
    def slot_last_used(self) -> np.ndarray:
        return self.slot_last_used_dev.cpu().numpy()

    @property
    def _free(self) -> list:
        n = int(self.free_count.item())
        return [int(v) for v in self.free_stack[:n].cpu().numpy()]

    # -- lookup -------------------------------------------------------------

    def translate(self, addr: VirtualAddress) -> Translation:
        coord = self.brick_coord_of(addr.level, addr.position)
        idx = self._entry_index(addr.channel_slot, addr.level, coord)
        v = int(self.pt[idx].item())
        if v < 0:
            return Translation(status=EMPTY if v == N.RO_PT_EMPTY else UNMAPPED)
        dims = self.level_dims[addr.level]
        local = tuple(float(addr.position[a] * dims[a] - coord[a] * self.config.brick_size[a])
                      for a in range(3))
        return Translation(status=MAPPED, cache_slot=self.slot_triple(v), local_coord=local)

    def resident_slot(self, brick_id):
        slot, level, coord = self.decode(brick_id)
        v = int(self.pt[self._entry_index(slot, level, coord)].item())
        return v if v >= 0 else None

    # -- mutation -----------------------------------------------------------

    def _ids_array(self, brick_ids) -> np.ndarray:
        """Validate a list of brick ids (vectorised decode_brick_id +
        _entry_index range checks); raises PagingError on the first bad one."""
        ids = np.ascontiguousarray(np.asarray(brick_ids, dtype=np.int64).reshape(-1))
        if len(ids) == 0:
            return ids
        k, m = self.config.k, self.config.m
        pt = (ids >> 24) & 0xFF
        slot, level = pt // k, pt % k
        xyz = np.stack([ids & 0xFF, (ids >> 8) & 0xFF, (ids >> 16) & 0xFF], axis=1)
        grids = np.asarray(self.level_grids, dtype=np.int64)[np.minimum(level, k - 1)]
        ok = (ids >= 0) & (ids < (1 << 32)) & (slot < m) & (xyz < grids).all(axis=1)
        if not ok.all():
            b = int(ids[int(np.flatnonzero(~ok)[0])])
            slot_b, level_b, coord_b = self.decode(b)
            self._entry_index(slot_b, level_b, coord_b)  # raises with the reason
            raise PagingError(f"bad brick id {b:#x}")
        return ids

    def _payload_arg(self, payloads, n):
        sx, sy, sz = self.config.brick_size
        if payloads is None:
            return None, 0, None
        if isinstance(payloads, torch.Tensor):
            t = payloads.reshape(n, sz, sy, sx)
            if t.dtype != torch.uint8:
                raise PagingError("payloads must be uint8")
            if t.is_cuda:
                t = t.contiguous()
                return t.data_ptr(), 1, t
            t = t.contiguous()
            return t.data_ptr(), 0, t
        arr = np.asarray(payloads)
        if arr.size != n * sx * sy * sz:
            raise PagingError(f"payload shape {arr.shape} != {n} bricks of {(sz, sy, sx)}")
        arr = np.ascontiguousarray(arr, dtype=np.uint8)
        return arr.ctypes.data, 0, arr

    def insert_bricks(self, brick_ids, payloads, frame: int,
                      update_octree: bool = False, return_slots: bool = True):
        """Batched insert_brick (paging.py:187-218) for an ordered id list.

        Returns (slots, evicted) as numpy arrays (evicted = -1 where none)
        when return_slots, else None."""
        ids = self._ids_array(brick_ids)
        n = len(ids)
        if n == 0:
            return (np.zeros(0, np.int32), np.zeros(0, np.int64)) if return_slots else None
        pptr, on_dev, keep = self._payload_arg(payloads, n)
        slots = np.zeros(n, dtype=np.int32) if return_slots else None
        evicted = np.zeros(n, dtype=np.int64) if return_slots else None
        st = self.state(with_words=update_octree)
        N.check(N.lib().ro_apply_bricks(
            self.ctx, C.byref(st), ids.ctypes.data, n, pptr, on_dev, int(frame),
            1 if update_octree else 0,
            slots.ctypes.data if return_slots else None,
            evicted.ctypes.data if return_slots else None, N.stream_ptr()))
        del keep
        return (slots, evicted) if return_slots else None

    def insert_bricks_lz4(self, brick_ids, frames, frame: int, update_octree: bool = False,
                          return_slots: bool = True):
        """insert_bricks with LZ4-framed payloads (the wire format,
        ingest.py:114-117), decoded on the GPU into the cache.  ``frames``:
        list of bytes or (uint8 buffer, int64 offsets[n+1]); a torch CUDA
        buffer is decoded in place.  Nothing is inserted if a frame is bad."""
        from .ingest import pack_frames
        ids = self._ids_array(brick_ids)
        n = len(ids)
        if n == 0:
            return (np.zeros(0, np.int32), np.zeros(0, np.int64)) if return_slots else None
        buf, offs = frames if isinstance(frames, tuple) else pack_frames(list(frames))
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        if len(offs) != n + 1:
            raise PagingError(f"{len(offs) - 1} frames for {n} bricks")
        on_dev = isinstance(buf, torch.Tensor) and buf.is_cuda
        if isinstance(buf, torch.Tensor) and not on_dev:
            buf = buf.numpy()
        if not on_dev:
            buf = np.ascontiguousarray(buf, dtype=np.uint8)
        # host frames are indexed from frames + offs[0]
        ptr = buf.data_ptr() if on_dev else buf.ctypes.data
        slots = np.zeros(n, dtype=np.int32) if return_slots else None
        evicted = np.zeros(n, dtype=np.int64) if return_slots else None
        st = self.state(with_words=update_octree)
        N.check(N.lib().ro_apply_bricks_lz4(
            self.ctx, C.byref(st), ids.ctypes.data, n, ptr, offs.ctypes.data,
            1 if on_dev else 0, int(frame), 1 if update_octree else 0,
            slots.ctypes.data if return_slots else None,
            evicted.ctypes.data if return_slots else None, N.stream_ptr()))
        return (slots, evicted) if return_slots else None

    def insert_brick(self, brick_id, payload, frame):
        """Returns (cache slot triple, evicted brick id or None)."""
        sx, sy, sz = self.config.brick_size
        if tuple(np.shape(payload)) != (sz, sy, sx):
            raise PagingError(f"payload shape {np.shape(payload)} != brick size")
        slots, evicted = self.insert_bricks([brick_id], [payload], frame)
        ev = int(evicted[0])
        return self.slot_triple(int(slots[0])), (None if ev < 0 else ev)

    def mark_used(self, slot, frame):
        lin = self.slot_linear(slot)
        if int(self.slot_brick_dev[lin].item()) < 0:
            raise PagingError(f"slot {slot} is not occupied")
        if frame < int(self.slot_last_used_dev[lin].item()):
            raise PagingError("frame counter must be monotone")
        self.slot_last_used_dev[lin] = frame

    def mark_empty(self, brick_id):
        """paging.py:228-234: release the brick's slot if mapped, enter EMPTY."""
        self.mark_empty_many([brick_id])

    def mark_empty_many(self, brick_ids):
        """mark_empty over an ordered id list (one launch)."""
        ids = self._ids_array(brick_ids)
        if len(ids) == 0:
            return
        st = self.state(with_words=False)
        N.check(N.lib().ro_mark_empty(self.ctx, C.byref(st), ids.ctypes.data, len(ids),
                                      N.stream_ptr()))

    def evict_bricks(self, brick_ids, update_octree: bool = False):
        """Explicit eviction: unmap, release the slot (verify.py:110-121)."""
        ids = self._ids_array(brick_ids)
        if len(ids) == 0:
            return
        st = self.state(with_words=update_octree)
        N.check(N.lib().ro_evict_bricks(self.ctx, C.byref(st), ids.ctypes.data, len(ids),
                                        1 if update_octree else 0, N.stream_ptr()))

    def sample(self, slot, local_coord) -> float:
        """paging.py:241-261: trilinear value of one cache slot at a
        brick-local coordinate (query helper; reads that slot's brick)."""
        brick = self.cache_dev[self.slot_linear(slot)].double().cpu().numpy()
        sx, sy, sz = self.config.brick_size
        lx = min(max(local_coord[0] - 0.5, 0.0), sx - 1.0)
        ly = min(max(local_coord[1] - 0.5, 0.0), sy - 1.0)
        lz = min(max(local_coord[2] - 0.5, 0.0), sz - 1.0)
        x0, y0, z0 = int(lx), int(ly), int(lz)
        x1, y1, z1 = min(x0 + 1, sx - 1), min(y0 + 1, sy - 1), min(z0 + 1, sz - 1)
        fx, fy, fz = lx - x0, ly - y0, lz - z0

        def lerp(a, b, t):
            return a + (b - a) * t
        c00 = lerp(brick[z0, y0, x0], brick[z0, y0, x1], fx)
        c10 = lerp(brick[z0, y1, x0], brick[z0, y1, x1], fx)
        c01 = lerp(brick[z1, y0, x0], brick[z1, y0, x1], fx)
        c11 = lerp(brick[z1, y1, x0], brick[z1, y1, x1], fx)
        return float(lerp(lerp(c00, c10, fy), lerp(c01, c11, fy), fz))

    def set_channel_mapping(self, channel_slot, dataset_channel, channel_count=None,
                            _invalidate_octree: bool = False):
        if not 0 <= channel_slot < self.config.m:
            raise PagingError(f"channel slot {channel_slot} out of range")
        if channel_count is not None and not 0 <= dataset_channel < channel_count:
            raise PagingError(f"dataset channel {dataset_channel} >= n ({channel_count})")
        st = self.state(with_words=_invalidate_octree)
        N.check(N.lib().ro_swap_channel(self.ctx, C.byref(st), channel_slot,
                                        1 if _invalidate_octree else 0, N.stream_ptr()))
        self.channel_mapping[channel_slot] = dataset_channel

    # -- introspection ------------------------------------------------------

    def resident_brick_ids(self) -> list:
        sb = self.slot_brick
        return [int(b) for b in sb if b >= 0]

    def occupied_slot_count(self) -> int:
        return int((self.slot_brick_dev >= 0).sum().item())

    def load_reference_state(self, pt_status, pt_slot, cache, slot_brick, slot_last_used,
                             free_list, words=None):
        """Adopt a reference-layout host state (paging.py:95-112 arrays, and
        octree.py:116-118 words if given) through ro_upload_state."""
        arr = dict(
            pt_status=np.ascontiguousarray(pt_status, dtype=np.int8),
            pt_slot=np.ascontiguousarray(pt_slot, dtype=np.int32),
            cache=np.ascontiguousarray(cache, dtype=np.uint8),
            slot_brick=np.ascontiguousarray(slot_brick, dtype=np.int64),
            slot_last_used=np.ascontiguousarray(slot_last_used, dtype=np.int64),
            free_list=np.ascontiguousarray(free_list, dtype=np.int32))
        if arr["pt_status"].size != self.total_entries or arr["slot_brick"].size != self.num_slots:
            raise PagingError("reference state does not match this layout")
        w = None if words is None else np.ascontiguousarray(words, dtype=np.uint32)
        h = N.HostState(arr["pt_status"].ctypes.data, arr["pt_slot"].ctypes.data,
                        w.ctypes.data if w is not None else None, arr["cache"].ctypes.data,
                        arr["slot_brick"].ctypes.data, arr["slot_last_used"].ctypes.data,
                        arr["free_list"].ctypes.data if arr["free_list"].size else None,
                        int(arr["free_list"].size))
        st = self.state(with_words=w is not None)
        N.check(N.lib().ro_upload_state(self.ctx, C.byref(h), C.byref(st), N.stream_ptr()))

    def check_bijection(self):
        p = self.pt.cpu().numpy()
        sb = self.slot_brick
        mapped = np.flatnonzero(p >= 0)
        lins = p[mapped]
        if len(np.unique(lins)) != len(lins):
            raise AssertionError("two entries share a cache slot")
        if set(int(v) for v in lins) != set(int(i) for i in np.flatnonzero(sb >= 0)):
            raise AssertionError("MAPPED entries and occupied slots differ")
        for e, lin in zip(mapped, lins):
            slot, level, coord = self.decode(int(sb[lin]))
            if self._entry_index(slot, level, coord) != int(e):
                raise AssertionError("resident brick does not decode to its entry")
