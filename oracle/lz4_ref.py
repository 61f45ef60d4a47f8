"""LZ4 frame oracle -- TEST INFRASTRUCTURE ONLY.

The reference decodes bricks with the system liblz4 frame API
(/root/reference/pkg/src/resoctree/lz4io.py:17-110: LZ4F_decompress in a loop,
errors on corrupt / truncated input and on trailing bytes or a size
mismatch).  liblz4 1.9.4 is the third-party dependency that holds the
algorithm (not vendored in the reference); it is present in this image, so
the oracle calls it exactly the way lz4io.decompress does.  ``prefs_frame``
builds frames with non-default preferences (checksums, content size, block
sizes, linked blocks, HC levels) through LZ4F_compressFrame.
"""

from __future__ import annotations

import ctypes as C
import ctypes.util

_LIB = None


class Lz4DecodeError(ValueError):
    pass


class FrameInfo(C.Structure):
    _fields_ = [("blockSizeID", C.c_int), ("blockMode", C.c_int),
                ("contentChecksumFlag", C.c_int), ("frameType", C.c_int),
                ("contentSize", C.c_ulonglong), ("dictID", C.c_uint),
                ("blockChecksumFlag", C.c_int)]


class Preferences(C.Structure):
    _fields_ = [("frameInfo", FrameInfo), ("compressionLevel", C.c_int),
                ("autoFlush", C.c_uint), ("favorDecSpeed", C.c_uint),
                ("reserved", C.c_uint * 3)]


def lib():
    global _LIB
    if _LIB is None:
        name = ctypes.util.find_library("lz4") or "liblz4.so.1"
        L = C.CDLL(name)
        L.LZ4F_isError.restype = C.c_uint
        L.LZ4F_isError.argtypes = [C.c_size_t]
        L.LZ4F_createDecompressionContext.restype = C.c_size_t
        L.LZ4F_createDecompressionContext.argtypes = [C.POINTER(C.c_void_p), C.c_uint]
        L.LZ4F_freeDecompressionContext.restype = C.c_size_t
        L.LZ4F_freeDecompressionContext.argtypes = [C.c_void_p]
        L.LZ4F_decompress.restype = C.c_size_t
        L.LZ4F_decompress.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t),
                                      C.c_void_p, C.POINTER(C.c_size_t), C.c_void_p]
        L.LZ4F_compressFrameBound.restype = C.c_size_t
        L.LZ4F_compressFrameBound.argtypes = [C.c_size_t, C.c_void_p]
        L.LZ4F_compressFrame.restype = C.c_size_t
        L.LZ4F_compressFrame.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                         C.c_void_p]
        _LIB = L
    return _LIB


def decompress(data: bytes, expected_size: int | None = None) -> bytes:
    """lz4io.py:69-110, restated call for call."""
    L = lib()
    src = bytes(data)
    if not src:
        raise Lz4DecodeError("empty LZ4 stream")
    ctx = C.c_void_p()
    if L.LZ4F_isError(L.LZ4F_createDecompressionContext(C.byref(ctx), 100)):
        raise RuntimeError("context allocation failed")
    try:
        out = bytearray()
        chunk = C.create_string_buffer(max(expected_size or 0, 1 << 16))
        src_buf = C.create_string_buffer(src, len(src))
        consumed = 0
        while True:
            dst_size = C.c_size_t(len(chunk))
            src_size = C.c_size_t(len(src) - consumed)
            hint = L.LZ4F_decompress(ctx, chunk, C.byref(dst_size),
                                     C.byref(src_buf, consumed), C.byref(src_size), None)
            if L.LZ4F_isError(hint):
                raise Lz4DecodeError("corrupt LZ4 frame")
            out += chunk.raw[:dst_size.value]
            consumed += src_size.value
            if hint == 0:
                break
            if src_size.value == 0 and dst_size.value == 0:
                raise Lz4DecodeError("truncated LZ4 frame")
        if consumed != len(src):
            raise Lz4DecodeError("trailing bytes after LZ4 frame")
    finally:
        L.LZ4F_freeDecompressionContext(ctx)
    if expected_size is not None and len(out) != expected_size:
        raise Lz4DecodeError(f"decompressed size {len(out)} != expected {expected_size}")
    return bytes(out)


def prefs_frame(data: bytes, block_size_id=4, linked=False, content_checksum=False,
                block_checksum=False, content_size=False, level=0) -> bytes:
    """LZ4F_compressFrame with explicit preferences."""
    L = lib()
    p = Preferences()
    p.frameInfo.blockSizeID = block_size_id
    p.frameInfo.blockMode = 0 if linked else 1
    p.frameInfo.contentChecksumFlag = 1 if content_checksum else 0
    p.frameInfo.blockChecksumFlag = 1 if block_checksum else 0
    p.frameInfo.contentSize = len(data) if content_size else 0
    p.compressionLevel = level
    src = bytes(data)
    bound = L.LZ4F_compressFrameBound(len(src), C.byref(p))
    dst = C.create_string_buffer(bound)
    n = L.LZ4F_compressFrame(dst, bound, src, len(src), C.byref(p))
    if L.LZ4F_isError(n):
        raise RuntimeError("LZ4F_compressFrame failed")
    return dst.raw[:n]
