"""In-memory bricked multi-resolution volumes: the input side of the render path.

Not on the hot path.  This restates just enough of the reference's data
format to build render state without the on-disk LZ4 store (which is out of
scope):

* ``normalize_to_u8`` / ``downsample_box`` / ``extract_brick`` /
  ``plan_levels`` -- ``ingest.py:27-89``, ``manifest.py:137-150``;
* ``VolumeStore.brick`` / ``region_min_max`` / ``level_array`` --
  ``service.py:71-115`` (in memory instead of files);
* ``LocalTransport`` -- ``service.py:167-187``;
* synthetic generators -- ``datasets.py:23-111``.

Large scenario builders that run on the GPU (the 2048^2 x 128 CyCIF-like
bench volume) live in :mod:`paper_2309_04393_b200.scenarios`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class VolumeError(ValueError):
    pass


class BrickNotFound(KeyError):
    """service.py:26-27 -- the requested brick does not exist."""


class TransportError(RuntimeError):
    """service.py:30-31 -- reachable dataset that failed to deliver."""


# ---------------------------------------------------------------------------
# manifest-like level description (manifest.py:29-150)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LevelDesc:
    dims: tuple            # voxels (x, y, z)
    downsample_from_prev: tuple
    brick_grid_dims: tuple


@dataclass
class VolumeManifest:
    name: str
    channel_count: int
    brick_size: tuple
    levels: list = field(default_factory=list)
    dtype_original: str = "u8"

    def validate(self):
        if self.channel_count < 1:
            raise VolumeError("channelCount must be >= 1")
        for b in self.brick_size:
            if b < 2 or (b & (b - 1)) != 0:
                raise VolumeError("brick size must be a power of two >= 2")
        if not self.levels:
            raise VolumeError("at least one level required")
        for lvl in self.levels:
            for a in range(3):
                if lvl.brick_grid_dims[a] != -(-lvl.dims[a] // self.brick_size[a]):
                    raise VolumeError("brickGridDims mismatch")
                if lvl.brick_grid_dims[a] > 256:
                    raise VolumeError("brick grid exceeds 256 per axis")

    @property
    def num_levels(self) -> int:
        return len(self.levels)


def plan_levels(dims, brick_size, num_levels, factors) -> list:
    """manifest.py:137-150."""
    if num_levels < 1:
        raise VolumeError("numLevels must be >= 1")
    levels = []
    cur = tuple(dims)
    for i in range(num_levels):
        f = (1, 1, 1) if i == 0 else tuple(factors)
        if i > 0:
            cur = tuple(-(-cur[a] // f[a]) for a in range(3))
        grid = tuple(-(-cur[a] // brick_size[a]) for a in range(3))
        levels.append(LevelDesc(dims=cur, downsample_from_prev=f,
                                brick_grid_dims=grid))
    return levels


# ---------------------------------------------------------------------------
# ingest (ingest.py:27-89)
# ---------------------------------------------------------------------------

def normalize_to_u8(raw: np.ndarray) -> np.ndarray:
    data = raw.astype(np.float64)
    lo = data.min()
    hi = data.max()
    if hi == lo:
        return np.zeros(raw.shape, dtype=np.uint8)
    scaled = (data - lo) * (255.0 / (hi - lo))
    return np.floor(scaled + 0.5).clip(0, 255).astype(np.uint8)


def downsample_box(level: np.ndarray, factors) -> np.ndarray:
    """Box filter by per-axis factors in {1,2}; arrays are [z, y, x]."""
    fx, fy, fz = factors
    arr = level.astype(np.float64)
    for axis, f in ((0, fz), (1, fy), (2, fx)):
        if f == 1:
            continue
        n = arr.shape[axis]
        if n % 2 == 1:
            pad = [(0, 0)] * 3
            pad[axis] = (0, 1)
            arr = np.pad(arr, pad, mode="edge")
        shape = list(arr.shape)
        shape[axis] //= 2
        shape.insert(axis + 1, 2)
        arr = arr.reshape(shape).mean(axis=axis + 1)
    return np.floor(arr + 0.5).clip(0, 255).astype(np.uint8)


def build_pyramid(channel_u8: np.ndarray, levels) -> list:
    pyramid = [channel_u8]
    for lvl in levels[1:]:
        pyramid.append(downsample_box(pyramid[-1], lvl.downsample_from_prev))
    return pyramid


def extract_brick(level_data: np.ndarray, coord, brick_size) -> np.ndarray:
    bx, by, bz = coord
    sx, sy, sz = brick_size
    dz, dy, dx = level_data.shape
    x0, y0, z0 = bx * sx, by * sy, bz * sz
    part = level_data[z0:min(z0 + sz, dz), y0:min(y0 + sy, dy),
                      x0:min(x0 + sx, dx)]
    pad = ((0, sz - part.shape[0]), (0, sy - part.shape[1]),
           (0, sx - part.shape[2]))
    if any(p[1] for p in pad):
        part = np.pad(part, pad, mode="edge")
    return np.ascontiguousarray(part)


# ---------------------------------------------------------------------------
# store + transport (service.py:35-187, in memory)
# ---------------------------------------------------------------------------

class VolumeStore:
    """Bricked pyramids of every channel, held in host memory."""

    def __init__(self, channels_raw: list, brick_size=(32, 32, 32),
                 num_levels: int = 4, factors=(2, 2, 2), name="volume",
                 normalize: bool = True):
        if not channels_raw:
            raise VolumeError("no channels given")
        shape = channels_raw[0].shape
        for ch in channels_raw:
            if ch.shape != shape:
                raise VolumeError("all channels must share dims")
        dims = (shape[2], shape[1], shape[0])
        levels = plan_levels(dims, brick_size, num_levels, factors)
        self.manifest = VolumeManifest(name=name, channel_count=len(channels_raw),
                                       brick_size=tuple(brick_size),
                                       levels=levels)
        self.manifest.validate()
        self.pyramids = []
        for raw in channels_raw:
            base = normalize_to_u8(raw) if normalize else np.asarray(raw, np.uint8)
            self.pyramids.append(build_pyramid(base, levels))

    def _check(self, c, l, coord=None):
        if not 0 <= c < self.manifest.channel_count:
            raise BrickNotFound(f"channel {c} out of range")
        if not 0 <= l < len(self.manifest.levels):
            raise BrickNotFound(f"level {l} out of range")
        if coord is not None:
            grid = self.manifest.levels[l].brick_grid_dims
            if not all(0 <= coord[a] < grid[a] for a in range(3)):
                raise BrickNotFound(f"brick {coord} outside grid {grid}")

    def brick(self, c, l, coord) -> np.ndarray:
        self._check(c, l, coord)
        return extract_brick(self.pyramids[c][l], coord, self.manifest.brick_size)

    def brick_bytes(self, c, l, coord) -> bytes:
        """The brick as one LZ4 frame (service.py:63-69: the stored / served
        form), compressed once with liblz4 and cached."""
        from .ingest import compress_brick
        key = (c, l, tuple(coord))
        cache = self.__dict__.setdefault("_frames", {})
        data = cache.get(key)
        if data is None:
            data = cache[key] = compress_brick(self.brick(c, l, coord))
        return data

    def level_array(self, c, l) -> np.ndarray:
        self._check(c, l)
        return self.pyramids[c][l]

    def region_min_max(self, c, l, box):
        self._check(c, l)
        nx, ny, nz = self.manifest.levels[l].dims
        x0, y0, z0, x1, y1, z1 = box
        x0, y0, z0 = max(0, x0), max(0, y0), max(0, z0)
        x1, y1, z1 = min(nx, x1), min(ny, y1), min(nz, z1)
        if x0 >= x1 or y0 >= y1 or z0 >= z1:
            return 0, 0
        part = self.pyramids[c][l][z0:z1, y0:y1, x0:x1]
        return int(part.min()), int(part.max())


class LocalTransport:
    """In-process transport over a VolumeStore (service.py:167-187)."""

    metadata_supported = True

    def __init__(self, store: VolumeStore):
        self.store = store

    @property
    def manifest(self):
        return self.store.manifest

    def fetch_brick(self, c, l, coord):
        return self.store.brick(c, l, coord)

    def metadata_pyramid(self, c, depth, pad):
        """Every node's region_min_max over its dilated box (service.py:102-115
        for all nodes at once), reduced on the GPU from the level-0 volume
        (metadata.MetadataPyramid); cached per (channel, depth, pad)."""
        from .metadata import MetadataPyramid
        cache = self.__dict__.setdefault("_pyramids", {})
        key = (c, depth, pad)
        pyr = cache.get(key)
        if pyr is None:
            pyr = cache[key] = MetadataPyramid(self.store.level_array(c, 0), depth, pad)
        return pyr

    def fetch_brick_bytes(self, c, l, coord) -> bytes:
        """The LZ4 frame the server would send (service.py:130-136)."""
        return self.store.brick_bytes(c, l, coord)

    def fetch_metadata(self, c, l, box):
        return self.store.region_min_max(c, l, box)

    def close(self):
        pass


# ---------------------------------------------------------------------------
# synthetic volumes (datasets.py:23-111)
# ---------------------------------------------------------------------------

def _coords(n):
    ax = (np.arange(n, dtype=np.float64) + 0.5) / n
    return np.meshgrid(ax, ax, ax, indexing="ij")


def constant_volume(n, value=0):
    return np.full((n, n, n), value, dtype=np.uint8)


def ramp_volume(n):
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return ((x * 3 + y * 7 + z * 11) % 256).astype(np.uint8)


def shell_volume(n, radius=0.38, thickness=0.04, value=220):
    z, y, x = _coords(n)
    r = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)
    vol = np.zeros((n, n, n), dtype=np.uint8)
    vol[np.abs(r - radius) <= thickness] = value
    return vol


def vessel_volume(n, seed=7, num_branches=12, value=230):
    rng = np.random.default_rng(seed)
    vol = np.zeros((n, n, n), dtype=np.uint8)
    zi, yi, xi = np.meshgrid(np.arange(n), np.arange(n), np.arange(n),
                             indexing="ij")
    pts = np.stack([xi, yi, zi], axis=-1).astype(np.float64) / n
    for _ in range(num_branches):
        a = rng.uniform(0.15, 0.85, size=3)
        b = rng.uniform(0.15, 0.85, size=3)
        ab = b - a
        denom = float(ab @ ab)
        if denom == 0.0:
            continue
        t = np.clip(((pts - a) @ ab) / denom, 0.0, 1.0)
        closest = a + t[..., None] * ab
        dist = np.linalg.norm(pts - closest, axis=-1)
        radius = rng.uniform(0.008, 0.02)
        vol[dist <= radius] = value
    return vol


def noise_floor(n, seed, hi=15):
    rng = np.random.default_rng(seed)
    return rng.integers(1, hi + 1, size=(n, n, n)).astype(np.uint8)


def sparse_multichannel(n, channels=4, seed=11):
    out = []
    for c in range(channels):
        if c % 2 == 0:
            fg = vessel_volume(n, seed=seed + c)
        else:
            fg = shell_volume(n, radius=0.30 + 0.05 * c)
        out.append(np.maximum(fg, noise_floor(n, seed=seed + 100 + c)))
    return out


def metadata_pad_default(k: int) -> int:
    """engine.py:59-62: 1.5 * 2^(k-1) voxels, rounded up."""
    return -(-3 * (1 << (k - 1)) // 2)


def box_minmax_grid(volume: np.ndarray, side: int, pad: int):
    """engine.py:186-219: per-node min/max over dilated boxes, [z, y, x].

    Separable: min/max over each x window, then y, then z (exactly the
    min/max over the 3-D box, computed in O(n * windows) instead of per node).
    """
    nz, ny, nx = volume.shape

    def bounds(n):
        out = []
        for i in range(side):
            v0 = (i * n) // side - pad
            v1 = -((-(i + 1) * n) // side) + pad
            out.append((max(0, v0), min(n, v1)))
        return out

    def reduce_axis(arr, axis, bnds, fn, empty):
        parts = []
        for lo, hi in bnds:
            if lo >= hi:
                shp = list(arr.shape)
                shp[axis] = 1
                parts.append(np.full(shp, empty, dtype=arr.dtype))
            else:
                sl = [slice(None)] * 3
                sl[axis] = slice(lo, hi)
                parts.append(fn(arr[tuple(sl)], axis=axis, keepdims=True))
        return np.concatenate(parts, axis=axis)

    xb, yb, zb = bounds(nx), bounds(ny), bounds(nz)
    mins = volume
    maxs = volume
    for axis, b in ((2, xb), (1, yb), (0, zb)):
        mins = reduce_axis(mins, axis, b, np.min, 255)
        maxs = reduce_axis(maxs, axis, b, np.max, 0)
    # empty windows map to (0, 0) in the reference
    empty = np.zeros((side, side, side), dtype=bool)
    ex = np.array([lo >= hi for lo, hi in xb])
    ey = np.array([lo >= hi for lo, hi in yb])
    ez = np.array([lo >= hi for lo, hi in zb])
    empty |= ex[None, None, :] | ey[None, :, None] | ez[:, None, None]
    mins = np.where(empty, 0, mins).astype(np.uint8)
    maxs = np.where(empty, 0, maxs).astype(np.uint8)
    return mins, maxs
