"""Benchmark / test scenarios built on the GPU with plain torch ops.

Config 2 of BASELINE.json ("CyCIF-like 4-of-16 channels, 2048x2048x128
uint16 per channel, 32^3 bricks, 1920x1080, partial residency with coarser-
LOD fallback"), following SURVEY.md §8(d):

* per channel c: ~20k ellipsoidal cells (radii 3-8 voxels in x/y, 2-4 in
  z) shared by all channels, each expressing channel c with p = 0.3 at
  intensity U(20k, 60k) over a U(0, 2k) background (seeds 1000 / 1000+c);
* normalize_to_u8 (ingest.py:27-35), 2x box pyramid with round-half-up
  (ingest.py:38-59), k = 7 levels, 32^3 bricks with edge replication
  (ingest.py:71-89);
* visible channels {0, 5, 10, 15} in slots 0..3 (m = 4), octree D = 6;
* residency: every brick of levels >= 2 plus a seeded 50 % of the level-0/1
  bricks, so rays hit misses and substitute coarser levels;
* exact per-node metadata with the reference dilation
  (engine.py:109-152), semi-transparent per-channel colour ramps
  (threshold 40, max alpha 0.3) so rays stay long.

The builder returns the brick list + payloads and the metadata grids; the
product arm loads them through Engine.apply_bricks /
ResidencyOctree.write_level_metadata, the CPU-baseline arm turns them into
reference-layout arrays with numpy (``reference_state``) without touching
libresoct.so.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as Fnn

from .camera import Camera, orbit_pose
from .render import ChannelSettings, RenderConfig
from .transfer import colored_ramp_tf
from .volume import LevelDesc, VolumeManifest, metadata_pad_default, plan_levels

COLORS = [(1.0, 0.35, 0.2), (0.25, 1.0, 0.35), (0.3, 0.45, 1.0), (1.0, 0.9, 0.25)]


@dataclass
class Scenario:
    name: str
    manifest: VolumeManifest
    depth: int
    cache_slots: tuple
    channels: list
    render: RenderConfig
    camera: Camera
    brick_ids: np.ndarray                 # int64, insertion order
    payloads: torch.Tensor                # u8 [n, bz, by, bx] (device)
    meta_mins: dict = field(default_factory=dict)   # (slot, d) -> u8 [side^3]
    meta_maxs: dict = field(default_factory=dict)
    dataset_channels: tuple = ()

    @property
    def m(self) -> int:
        return len(self.dataset_channels)


def _cells(shape_zyx, n_cells, device, seed):
    nz, ny, nx = shape_zyx
    g = torch.Generator(device=device).manual_seed(seed)
    cz = torch.randint(0, nz, (n_cells,), generator=g, device=device)
    cy = torch.randint(0, ny, (n_cells,), generator=g, device=device)
    cx = torch.randint(0, nx, (n_cells,), generator=g, device=device)
    rx = 3.0 + 5.0 * torch.rand(n_cells, generator=g, device=device)
    ry = 3.0 + 5.0 * torch.rand(n_cells, generator=g, device=device)
    rz = 2.0 + 2.0 * torch.rand(n_cells, generator=g, device=device)
    return cz, cy, cx, rz, ry, rx


def cycif_channel(shape_zyx, cells, channel: int, device) -> torch.Tensor:
    """One u16-range channel (int32 tensor [z, y, x])."""
    nz, ny, nx = shape_zyx
    g = torch.Generator(device=device).manual_seed(1000 + channel)
    vol = torch.randint(0, 2001, (nz, ny, nx), generator=g, device=device,
                        dtype=torch.int32)
    cz, cy, cx, rz, ry, rx = cells
    n = cz.numel()
    express = torch.rand(n, generator=g, device=device) < 0.3
    inten = (20000 + 40000 * torch.rand(n, generator=g, device=device)).to(torch.int32)
    sel = torch.nonzero(express).flatten()
    oz, oy, ox = torch.meshgrid(torch.arange(-4, 5, device=device),
                                torch.arange(-8, 9, device=device),
                                torch.arange(-8, 9, device=device), indexing="ij")
    oz, oy, ox = oz.reshape(1, -1), oy.reshape(1, -1), ox.reshape(1, -1)
    flat = vol.view(-1)
    for chunk in torch.split(sel, 1024):
        z = cz[chunk, None] + oz
        y = cy[chunk, None] + oy
        x = cx[chunk, None] + ox
        inside = ((ox / rx[chunk, None]) ** 2 + (oy / ry[chunk, None]) ** 2 +
                  (oz / rz[chunk, None]) ** 2) <= 1.0
        inside &= (z >= 0) & (z < nz) & (y >= 0) & (y < ny) & (x >= 0) & (x < nx)
        idx = ((z * ny + y) * nx + x)[inside]
        val = inten[chunk, None].expand_as(inside)[inside]
        flat.scatter_reduce_(0, idx, val, reduce="amax")
    return vol


def normalize_to_u8(raw: torch.Tensor) -> torch.Tensor:
    """ingest.py:27-35 in fp64 on the device."""
    lo = raw.min().to(torch.float64)
    hi = raw.max().to(torch.float64)
    if hi == lo:
        return torch.zeros_like(raw, dtype=torch.uint8)
    out = torch.empty(raw.shape, dtype=torch.uint8, device=raw.device)
    scale = 255.0 / (hi - lo)
    for zs in range(0, raw.shape[0], 8):
        d = raw[zs:zs + 8].to(torch.float64)
        out[zs:zs + 8] = torch.floor((d - lo) * scale + 0.5).clamp(0, 255).to(torch.uint8)
    return out


def downsample2(level: torch.Tensor) -> torch.Tensor:
    """ingest.py:38-59 for factors (2,2,2): round-half-up of the 8-voxel mean
    (edge-replicated on odd extents)."""
    z, y, x = level.shape
    a = level
    if z % 2 or y % 2 or x % 2:
        iz = torch.arange(z + z % 2, device=a.device).clamp(max=z - 1)
        iy = torch.arange(y + y % 2, device=a.device).clamp(max=y - 1)
        ix = torch.arange(x + x % 2, device=a.device).clamp(max=x - 1)
        a = a[iz][:, iy][:, :, ix]
        z, y, x = a.shape
    s = a.to(torch.int32).reshape(z // 2, 2, y // 2, 2, x // 2, 2).sum(dim=(1, 3, 5))
    return ((s + 4) // 8).to(torch.uint8)


def bricks_of_level(level: torch.Tensor, brick) -> torch.Tensor:
    """All bricks of one level, edge-replicated: [gz, gy, gx, bz, by, bx]."""
    bx, by, bz = brick
    z, y, x = level.shape
    gz, gy, gx = -(-z // bz), -(-y // by), -(-x // bx)
    iz = torch.arange(gz * bz, device=level.device).clamp(max=z - 1)
    iy = torch.arange(gy * by, device=level.device).clamp(max=y - 1)
    ix = torch.arange(gx * bx, device=level.device).clamp(max=x - 1)
    a = level[iz][:, iy][:, :, ix]
    return a.reshape(gz, bz, gy, by, gx, bx).permute(0, 2, 4, 1, 3, 5).contiguous()


def box_minmax_levels(vol: torch.Tensor, depth: int, pad: int):
    """engine.py:138-152 on the device: for every octree depth d the min/max
    over each node's dilated level-0 box.  Separable windowed max-pooling,
    exact when every extent divides by 2^depth (else the numpy path)."""
    nz, ny, nx = vol.shape
    out = {}
    v = vol.to(torch.float32)
    for d in range(depth + 1):
        side = 1 << d
        if nz % side or ny % side or nx % side:
            raise ValueError("extent not divisible by the node grid")

        def pool(t, n, sign):
            w = n // side
            r = Fnn.max_pool1d(sign * t, kernel_size=w + 2 * pad, stride=w, padding=pad)
            return sign * r

        res = []
        for sign in (-1.0, 1.0):
            t = v.reshape(nz * ny, 1, nx)
            t = pool(t, nx, sign).reshape(nz, ny, side)
            t = t.permute(0, 2, 1).reshape(nz * side, 1, ny)
            t = pool(t, ny, sign).reshape(nz, side, side)
            t = t.permute(1, 2, 0).reshape(side * side, 1, nz)
            t = pool(t, nz, sign).reshape(side, side, side)  # [y, x, z]
            res.append(t.permute(2, 0, 1).contiguous().to(torch.uint8))
        out[d] = (res[0].reshape(-1), res[1].reshape(-1))
    return out


def cycif(device="cuda", dims=(2048, 2048, 128), n_cells=20000,
          dataset_channels=(0, 5, 10, 15), image_dims=(1920, 1080), depth=6,
          resident_fraction_fine=0.5, max_alpha=0.3, base_step=1.0 / 256.0,
          angle=0.6, budget=256) -> Scenario:
    device = torch.device(device)
    nx, ny, nz = dims
    brick = (32, 32, 32)
    k = 1
    while True:  # levels down to a single brick in x/y (grids 64^2x4 ... 1)
        lv = plan_levels(dims, brick, k, (2, 2, 2))
        if lv[-1].brick_grid_dims[0] == 1 and lv[-1].brick_grid_dims[1] == 1:
            break
        k += 1
    levels = plan_levels(dims, brick, k, (2, 2, 2))
    manifest = VolumeManifest(name="cycif", channel_count=16, brick_size=brick,
                              levels=levels)
    manifest.validate()
    pad = metadata_pad_default(k)
    cells = _cells((nz, ny, nx), n_cells, device, 1000)
    ids, pays = [], []
    mins, maxs = {}, {}
    for slot, ch in enumerate(dataset_channels):
        raw = cycif_channel((nz, ny, nx), cells, ch, device)
        lvl = normalize_to_u8(raw)
        del raw
        for d, (mn, mx) in box_minmax_levels(lvl, depth, pad).items():
            mins[(slot, d)] = mn
            maxs[(slot, d)] = mx
        pyramid = [lvl]
        for _ in range(1, k):
            pyramid.append(downsample2(pyramid[-1]))
        rng = np.random.default_rng(2024 + ch)
        for lev in range(k - 1, -1, -1):
            gx, gy, gz = levels[lev].brick_grid_dims
            b = bricks_of_level(pyramid[lev], brick).reshape(-1, *brick[::-1])
            if lev >= 2:
                keep = np.ones(gx * gy * gz, dtype=bool)
            else:
                keep = rng.random(gx * gy * gz) < resident_fraction_fine
            sel = np.flatnonzero(keep)
            zz, yy, xx = sel // (gx * gy), (sel // gx) % gy, sel % gx
            ids.append(((slot * k + lev) << 24) | (zz << 16) | (yy << 8) | xx)
            pays.append(b[torch.as_tensor(sel, device=device)])
        del pyramid, lvl
    brick_ids = np.concatenate(ids).astype(np.int64)
    payloads = torch.cat(pays)
    n = len(brick_ids)
    side = max(1, math.ceil(n ** (1 / 3)))
    while side ** 3 < n:
        side += 1
    channels = [ChannelSettings(slot=s, tf=colored_ramp_tf(40.0, COLORS[s % 4], max_alpha))
                for s in range(len(dataset_channels))]
    render = RenderConfig(image_dims=image_dims, base_step=base_step,
                          max_requests_per_frame=budget, traversal_start_level=2)
    return Scenario(name=f"cycif{nx}x{ny}x{nz}", manifest=manifest, depth=depth,
                    cache_slots=(side, side, side), channels=channels, render=render,
                    camera=orbit_pose(angle), brick_ids=brick_ids, payloads=payloads,
                    meta_mins=mins, meta_maxs=maxs,
                    dataset_channels=tuple(dataset_channels))


def build_engine(scn: Scenario, device=None):
    """Product state: batched upload through Engine.apply_bricks (kernel 3b +
    octree pass) and per-level metadata writes."""
    from .engine import Engine, EngineConfig
    eng = Engine(scn.manifest, EngineConfig(octree_depth=scn.depth,
                                            cache_slots=scn.cache_slots,
                                            channel_slots=scn.m), device=device)
    for s, c in enumerate(scn.dataset_channels):
        eng.paging.channel_mapping[s] = c
    eng.apply_bricks(scn.brick_ids, scn.payloads)
    for (slot, d), mn in scn.meta_mins.items():
        eng.octree.write_level_metadata(slot, d, mn, scn.meta_maxs[(slot, d)])
    torch.cuda.synchronize()
    return eng


def reference_state(scn: Scenario):
    """Reference-layout arrays built with numpy only (no libresoct.so):
    slots 0..n-1 in insertion order (fresh LIFO free list), leaf masks from
    brick/leaf overlap, OR closure, metadata bits from the grids.  Returns a
    dict with the fields of oracle.raycast.OracleState."""
    man = scn.manifest
    k = len(man.levels)
    m = scn.m
    dims = np.array([l.dims for l in man.levels], dtype=np.int32)
    grids = np.array([l.brick_grid_dims for l in man.levels], dtype=np.int32)
    sizes = [int(np.prod(grids[pt % k])) for pt in range(m * k)]
    pt_off = np.zeros(m * k + 1, dtype=np.int64)
    np.cumsum(sizes, out=pt_off[1:])
    E = int(pt_off[-1])
    pt_status = np.zeros(E, dtype=np.int8)
    pt_slot = np.full(E, -1, dtype=np.int32)
    ids = scn.brick_ids
    pt = (ids >> 24) & 0xFF
    slot_of, lev_of = pt // k, pt % k
    x, y, z = ids & 0xFF, (ids >> 8) & 0xFF, (ids >> 16) & 0xFF
    e = pt_off[pt] + (z * grids[lev_of, 1] + y) * grids[lev_of, 0] + x
    pt_status[e] = 1
    pt_slot[e] = np.arange(len(ids), dtype=np.int32)
    S = int(np.prod(scn.cache_slots))
    bx, by, bz = man.brick_size
    cache = np.zeros((S, bz, by, bx), dtype=np.uint8)
    cache[:len(ids)] = scn.payloads.cpu().numpy()
    D = scn.depth
    side = 1 << D
    N = ((1 << (3 * (D + 1))) - 1) // 7
    words = np.zeros((N, m), dtype=np.uint32)
    B = man.brick_size
    for s in range(m):
        leaf = np.zeros((side, side, side), dtype=np.uint32)
        sel = np.flatnonzero(slot_of == s)
        for i in sel:
            lev = int(lev_of[i])
            c = (int(x[i]), int(y[i]), int(z[i]))
            rng_ = []
            for a in range(3):
                dim = int(dims[lev, a])
                lo = max(0, (c[a] * B[a] * side) // dim)
                hi = min(side - 1, -((-(c[a] + 1) * B[a] * side) // dim) - 1)
                rng_.append((lo, hi))
            leaf[rng_[2][0]:rng_[2][1] + 1, rng_[1][0]:rng_[1][1] + 1,
                 rng_[0][0]:rng_[0][1] + 1] |= np.uint32(1 << lev)
        cur = leaf
        for d in range(D, -1, -1):
            base = ((1 << (3 * d)) - 1) // 7
            words[base:base + (1 << d) ** 3, s] = cur.reshape(-1)
            if d > 0:
                h = (1 << d) // 2
                cur = cur.reshape(h, 2, h, 2, h, 2)
                cur = np.bitwise_or.reduce(np.bitwise_or.reduce(
                    np.bitwise_or.reduce(cur, axis=5), axis=3), axis=1)
        for d in range(D + 1):
            base = ((1 << (3 * d)) - 1) // 7
            mn = scn.meta_mins[(s, d)].cpu().numpy().astype(np.uint32)
            mx = scn.meta_maxs[(s, d)].cpu().numpy().astype(np.uint32)
            words[base:base + (1 << d) ** 3, s] |= (mn << 16) | (mx << 24)
    return dict(m=m, k=k, brick_size=tuple(man.brick_size), level_dims=dims,
                level_grids=grids, pt_offsets=pt_off, pt_status=pt_status,
                pt_slot=pt_slot, cache=cache, words=words, depth=D, eps_h=0.0)


# ---------------------------------------------------------------------------
# config 4: out-of-core procedural volume
# ---------------------------------------------------------------------------

class ProceduralStore:
    """Config 4 of BASELINE.json: 60 channels x 8192x8192x256 u8 (k = 9,
    grids 256^2x8 ... 1, 599,381 bricks per channel, ~1.18 TB of bricks)
    that never exists in full: every brick is generated on request from a
    deterministic per-(channel, level, brick) hash, the way a brick server
    would read it from disk (service.py:130-136 serves a stored brick).

    Content: per channel a seeded occupancy grid of ``cell``-voxel columns
    (cell x cell in x/y, the full z extent); an occupied column holds noise in
    [16, 255] (one of ``pool`` seeded noise bricks, picked by the brick hash),
    an empty one holds 0.  A level-l voxel takes the occupancy of the column
    under its centre.  ``fetch_metadata`` (service.py:102-115's
    region_min_max) answers from the occupancy grid: (0, 0) when the box
    touches no occupied column, else a conservative (16 or 0, 255) -- exact
    for the empty test the ray caster runs, never tighter than the data.

    Transport interface of volume.LocalTransport (manifest, fetch_brick,
    fetch_metadata), so Session streams it like any other server."""

    metadata_supported = True

    def __init__(self, dims=(8192, 8192, 256), channels=60, brick=32, cell=256,
                 occupancy=0.3, pool=64, seed=4242):
        nx, ny, nz = dims
        b = (brick, brick, brick)
        k = 1
        while True:
            lv = plan_levels(dims, b, k, (2, 2, 2))
            if lv[-1].brick_grid_dims[0] == 1 and lv[-1].brick_grid_dims[1] == 1:
                break
            k += 1
        self.manifest = VolumeManifest(name=f"procedural{nx}x{ny}x{nz}",
                                       channel_count=channels, brick_size=b,
                                       levels=plan_levels(dims, b, k, (2, 2, 2)))
        self.manifest.validate()
        self.dims = dims
        self.brick_edge = brick
        self.cell = cell
        gx, gy = -(-nx // cell), -(-ny // cell)
        self.occ = np.stack([np.random.default_rng(seed + 1 + c).random((gy, gx)) < occupancy
                             for c in range(channels)])
        rng = np.random.default_rng(seed)
        self.pool = rng.integers(16, 256, size=(pool, brick, brick, brick), dtype=np.uint8)
        self.bytes_served = 0

    @property
    def brick_count(self) -> int:
        return self.manifest.channel_count * sum(
            int(np.prod(l.brick_grid_dims)) for l in self.manifest.levels)

    def fetch_brick(self, c, l, coord):
        x, y, z = coord
        B = self.brick_edge
        i = np.arange(B)
        # column of each level-l voxel centre, in level-0 voxels
        cx = np.minimum((((x * B + i) << 1) + 1) << l >> 1, self.dims[0] - 1) // self.cell
        cy = np.minimum((((y * B + i) << 1) + 1) << l >> 1, self.dims[1] - 1) // self.cell
        mask = self.occ[c][cy[:, None], cx[None, :]]
        h = (c * 73856093) ^ (l * 19349663) ^ (x * 83492791) ^ (y * 2654435761) ^ (z * 97)
        out = self.pool[h % len(self.pool)] * mask[None, :, :]
        self.bytes_served += out.nbytes
        return out

    def fetch_metadata(self, c, l, box):
        x0, y0, _, x1, y1, _ = box
        if x1 <= x0 or y1 <= y0:
            return 0, 0
        part = self.occ[c][y0 // self.cell:(y1 - 1) // self.cell + 1,
                           x0 // self.cell:(x1 - 1) // self.cell + 1]
        if not part.any():
            return 0, 0
        return (16 if part.all() else 0), 255

    def close(self):
        pass

    # VolumeStore-style names (service.py:71-115 semantics) for in-process users
    def brick(self, c, l, coord):
        return self.fetch_brick(c, l, coord)

    def region_min_max(self, c, l, box):
        return self.fetch_metadata(c, l, box)
