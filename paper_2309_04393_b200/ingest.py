"""Brick ingest on the GPU.

Device-side counterparts of the reference's ingest / wire-format helpers:

* ``decompress_bricks`` -- LZ4 frames (the wire and on-disk brick format,
  ``lz4io.py:69-110`` / ``ingest.py:114-117``) decoded by ``ro_lz4_decode``,
  one warp per frame; ``Engine.apply_bricks_lz4`` decodes straight into the
  brick cache (``ro_apply_bricks_lz4``).
* ``normalize_to_u8`` (``ingest.py:27-35``), ``downsample_box``
  (``ingest.py:38-61``), ``build_pyramid`` (``ingest.py:64-72``) and
  ``extract_bricks`` (``ingest.py:75-95``, every brick of a level) on
  device-resident volumes, bit-identical to the reference's fp64 numpy.
* ``compress`` / ``compress_brick`` -- the SERVER side of the wire format
  (``lz4io.py:59-66``), host liblz4 exactly as the reference calls it; the
  client never decompresses on the CPU.
"""

from __future__ import annotations

import ctypes as C
import ctypes.util

import numpy as np
import torch

from . import _native as N


class IngestError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# host LZ4 frame compression (server side of the wire format)
# ---------------------------------------------------------------------------

_LZ4 = None


def _liblz4():
    global _LZ4
    if _LZ4 is None:
        name = ctypes.util.find_library("lz4")
        for cand in ([name] if name else []) + ["liblz4.so.1", "liblz4.so"]:
            try:
                lib = C.CDLL(cand)
                break
            except OSError:
                continue
        else:
            raise OSError("liblz4 not found")
        lib.LZ4F_compressFrameBound.restype = C.c_size_t
        lib.LZ4F_compressFrameBound.argtypes = [C.c_size_t, C.c_void_p]
        lib.LZ4F_compressFrame.restype = C.c_size_t
        lib.LZ4F_compressFrame.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p,
                                           C.c_size_t, C.c_void_p]
        lib.LZ4F_isError.restype = C.c_uint
        lib.LZ4F_isError.argtypes = [C.c_size_t]
        _LZ4 = lib
    return _LZ4


def compress(data, prefs=None) -> bytes:
    """One LZ4 frame with liblz4's default preferences (lz4io.py:59-66).
    ``prefs`` (optional) is a ctypes LZ4F_preferences_t pointer."""
    lib = _liblz4()
    src = bytes(data)
    bound = lib.LZ4F_compressFrameBound(len(src), prefs)
    dst = C.create_string_buffer(bound)
    n = lib.LZ4F_compressFrame(dst, bound, src, len(src), prefs)
    if lib.LZ4F_isError(n):
        raise IngestError("LZ4 frame compression failed")
    return dst.raw[:n]


def compress_brick(payload) -> bytes:
    """ingest.py:110-111"""
    return compress(np.ascontiguousarray(payload, dtype=np.uint8).tobytes())


def pack_frames(frames) -> tuple:
    """list of bytes -> (uint8 concatenation, int64 offsets[n+1])."""
    offs = np.zeros(len(frames) + 1, dtype=np.int64)
    np.cumsum([len(f) for f in frames], out=offs[1:])
    buf = np.frombuffer(bytearray(b"".join(frames)), dtype=np.uint8) if frames else \
        np.zeros(0, np.uint8)
    return np.ascontiguousarray(buf), offs


# ---------------------------------------------------------------------------
# device decode
# ---------------------------------------------------------------------------

LZ4_STATUS = {0: "ok", -1: "not an LZ4 frame", -2: "bad descriptor / header checksum",
              -3: "block too large", -4: "truncated", -5: "corrupt block",
              -6: "size mismatch", -7: "checksum mismatch", -8: "trailing bytes"}


_INGEST_CTX = {}


def _ctx():
    """A context for the ingest calls that need device scratch (one per
    device; the layout is a 1-brick placeholder, only the scratch is used)."""
    dev = torch.cuda.current_device()
    h = _INGEST_CTX.get(dev)
    if h is not None:
        return h
    lay = N.Layout()
    lay.m, lay.k, lay.depth = 1, 1, 0
    lay.brick = (N._i32 * 3)(2, 2, 2)
    for a in range(3):
        lay.level_dims[0][a] = 2
        lay.level_grids[0][a] = 1
    lay.pt_offsets[0], lay.pt_offsets[1] = 0, 1
    lay.num_slots = 1
    h = C.c_void_p()
    N.check(N.lib().ro_create(C.byref(lay), C.byref(h)))
    _INGEST_CTX[dev] = h
    return h


def decompress_bricks(frames, brick_size, device=None, raise_on_error=True):
    """Decode LZ4 frames into a uint8 tensor [n, bz, by, bx] on the device.

    ``frames``: list of bytes, or (concatenated uint8, offsets) from
    ``pack_frames``.  Returns (bricks, status int32[n]); with
    ``raise_on_error`` a bad frame raises IngestError naming it."""
    N.require_cuda()
    if isinstance(frames, tuple):
        buf, offs = frames
    else:
        buf, offs = pack_frames(list(frames))
    n = len(offs) - 1
    sx, sy, sz = brick_size
    bvox = sx * sy * sz
    dev = torch.device(device) if device is not None else torch.device("cuda")
    out = torch.empty((n, sz, sy, sx), dtype=torch.uint8, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    if n == 0:
        return out, status.cpu().numpy()
    d_buf = torch.from_numpy(np.ascontiguousarray(buf)).to(dev, non_blocking=False) \
        if not isinstance(buf, torch.Tensor) else buf.to(dev)
    d_off = torch.from_numpy(np.ascontiguousarray(offs, dtype=np.int64)).to(dev)
    N.check(N.lib().ro_lz4_decode(_ctx(), d_buf.data_ptr() if d_buf.numel() else None,
                                  d_off.data_ptr(), n, out.data_ptr(), bvox, bvox,
                                  status.data_ptr(), N.stream_ptr()))
    st = status.cpu().numpy()
    if raise_on_error and (st != 0).any():
        i = int(np.flatnonzero(st)[0])
        raise IngestError(f"frame {i}: {LZ4_STATUS.get(int(st[i]), 'decode error')}")
    return out, st


# ---------------------------------------------------------------------------
# device pyramid + bricks (ingest.py:27-95)
# ---------------------------------------------------------------------------

_DTYPE_CODES = {torch.uint8: 1, torch.uint16: 2, torch.uint32: 3, torch.float32: 4}


def normalize_to_u8(raw: torch.Tensor) -> torch.Tensor:
    """ingest.py:27-35: min -> 0, max -> 255, round half up, on the device."""
    N.require_cuda()
    code = _DTYPE_CODES.get(raw.dtype)
    if code is None:
        raise IngestError(f"unsupported dtype {raw.dtype} (u8, u16, u32, f32)")
    src = raw.contiguous()
    out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    N.check(N.lib().ro_normalize_to_u8(_ctx(), src.data_ptr(), code, src.numel(),
                                       out.data_ptr(), N.stream_ptr()))
    return out


def downsample_box(level: torch.Tensor, factors) -> torch.Tensor:
    """ingest.py:38-61: per-axis factors (fx, fy, fz) in {1, 2}, level [z, y, x]."""
    fx, fy, fz = (int(f) for f in factors)
    src = level.contiguous()
    dz, dy, dx = src.shape
    out = torch.empty((-(-dz // fz), -(-dy // fy), -(-dx // fx)), dtype=torch.uint8,
                      device=src.device)
    N.check(N.lib().ro_downsample_box(src.data_ptr(), dx, dy, dz, fx, fy, fz,
                                      out.data_ptr(), N.stream_ptr()))
    return out


def build_pyramid(channel_u8: torch.Tensor, levels) -> list:
    """ingest.py:64-72: level i+1 = downsample_box(level i, its factors)."""
    pyramid = [channel_u8.contiguous()]
    for lvl in levels[1:]:
        pyramid.append(downsample_box(pyramid[-1], lvl.downsample_from_prev))
    for lvl, arr in zip(levels, pyramid):
        if tuple(arr.shape) != (lvl.dims[2], lvl.dims[1], lvl.dims[0]):
            raise IngestError(f"level shape {tuple(arr.shape)} != manifest {lvl.dims}")
    return pyramid


def extract_bricks(level: torch.Tensor, brick_size) -> torch.Tensor:
    """ingest.py:75-95 for every brick of a level: [gz*gy*gx, bz, by, bx] in
    (z, y, x) grid order, edge bricks edge-replicated."""
    sx, sy, sz = brick_size
    src = level.contiguous()
    dz, dy, dx = src.shape
    nb = (-(-dx // sx)) * (-(-dy // sy)) * (-(-dz // sz))
    out = torch.empty((nb, sz, sy, sx), dtype=torch.uint8, device=src.device)
    N.check(N.lib().ro_extract_bricks(src.data_ptr(), dx, dy, dz, sx, sy, sz,
                                      out.data_ptr(), N.stream_ptr()))
    return out
