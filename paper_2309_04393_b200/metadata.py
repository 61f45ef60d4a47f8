"""Culling-metadata producer on the GPU.

A node's metadata is the min / max of the level-0 volume over its extent
dilated by ``pad`` voxels (``engine.py:109-127`` metadata_box).  The
reference computes it on the server per request (``service.py:102-115``
region_min_max, one numpy reduction per node, requested by
``session.py:140-158``) or per tree level with ``_box_minmax_grid``
(``engine.py:138-152, 186-219``).  Here ``ro_node_minmax`` reduces a
device-resident volume for a whole tree level in three separable passes, and
``MetadataPyramid`` keeps every node of every depth so metadata requests
become lookups -- the same numbers, bit for bit.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N


def _device_u8(volume, device=None) -> torch.Tensor:
    t = torch.as_tensor(volume)
    if t.dtype != torch.uint8:
        raise ValueError("metadata volumes are u8 (normalised level 0)")
    dev = device if device is not None else (t.device if t.is_cuda else torch.device("cuda"))
    return t.to(dev).contiguous()


def node_minmax(volume, d: int, pad: int, ctx=None):
    """(mins, maxs) u8[8^d] on the device for every depth-d node, (z, y, x)
    order -- exactly ``_box_minmax_grid(volume, 2^d, pad)`` (engine.py:186-219)."""
    from .ingest import _ctx
    vol = _device_u8(volume)
    dz, dy, dx = vol.shape
    n = 1 << (3 * d)
    mins = torch.empty(n, dtype=torch.uint8, device=vol.device)
    maxs = torch.empty(n, dtype=torch.uint8, device=vol.device)
    N.check(N.lib().ro_node_minmax(ctx or _ctx(), vol.data_ptr(), dx, dy, dz, d, pad,
                                   mins.data_ptr(), maxs.data_ptr(), N.stream_ptr()))
    return mins, maxs


class MetadataPyramid:
    """Min / max of every node at depths 0..depth for one channel's level-0
    volume, in node-index order (level_offset(d) + local), resident in HBM,
    with a host mirror for request lookups."""

    def __init__(self, volume, depth: int, pad: int):
        vol = _device_u8(volume)
        self.depth, self.pad = depth, pad
        n_nodes = ((1 << (3 * (depth + 1))) - 1) // 7
        self.mins = torch.empty(n_nodes, dtype=torch.uint8, device=vol.device)
        self.maxs = torch.empty(n_nodes, dtype=torch.uint8, device=vol.device)
        for d in range(depth + 1):
            base = ((1 << (3 * d)) - 1) // 7
            mn, mx = node_minmax(vol, d, pad)
            self.mins[base:base + mn.numel()] = mn
            self.maxs[base:base + mx.numel()] = mx
        self._host = (self.mins.cpu().numpy(), self.maxs.cpu().numpy())

    def lookup(self, node_indices):
        """(mins, maxs) int arrays for node indices (session metadata requests)."""
        idx = np.asarray(node_indices, dtype=np.int64)
        return self._host[0][idx].astype(np.int64), self._host[1][idx].astype(np.int64)


def fill_metadata(engine, slot: int, volume):
    """engine.py:138-152 for one slot, on the device (ro_fill_metadata)."""
    vol = _device_u8(volume, engine.paging.device)
    dz, dy, dx = vol.shape
    st = engine.paging.state(with_words=True)
    N.check(N.lib().ro_fill_metadata(engine.paging.ctx, C.byref(st), slot, vol.data_ptr(),
                                     dx, dy, dz, engine.metadata_pad, N.stream_ptr()))
