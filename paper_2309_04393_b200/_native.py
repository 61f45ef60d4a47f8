"""ctypes binding of libresoct.so (include/resoct.h).

The product path has no fallback: if the library is missing or no CUDA
device is present, every call raises instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os

import torch  # noqa: F401  (loads the CUDA runtime libresoct.so links against)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RESOCT_LIB") or os.path.join(HERE, "libresoct.so")

RO_MAX_LEVELS = 16
RO_MAX_PT = 256
RO_MAX_CH = 8
RO_MAX_TF_POINTS = 16
RO_NUM_COUNTERS = 8
RO_MODE_RESIDENCY = 0
RO_MODE_REFERENCE = 1
RO_MODE_PAGETABLE = 2
RO_MODE_CLASSIC = 3
RO_PT_UNMAPPED = -1
RO_PT_EMPTY = -2
RO_SUB_EDGE = 4          # sub-block edge of ro_state.sub_max (resoct.h)
RO_SUB_EDGE_ALLOC = int(os.environ.get("RESOCT_SUB_EDGE_ALLOC", RO_SUB_EDGE))

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_d = C.c_double


class NativeLibraryMissing(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


class Layout(C.Structure):
    _fields_ = [("m", _i32), ("k", _i32), ("depth", _i32), ("brick", _i32 * 3),
                ("level_dims", (_i32 * 3) * RO_MAX_LEVELS),
                ("level_grids", (_i32 * 3) * RO_MAX_LEVELS),
                ("pt_offsets", _i64 * (RO_MAX_PT + 1)), ("num_slots", _i64)]


class State(C.Structure):
    _fields_ = [("words", _p), ("pt", _p), ("cache", _p), ("slot_brick", _p),
                ("slot_last_used", _p), ("free_stack", _p), ("free_count", _p),
                ("sub_max", _p)]


class HostState(C.Structure):
    _fields_ = [("pt_status", _p), ("pt_slot", _p), ("words", _p), ("cache", _p),
                ("slot_brick", _p), ("slot_last_used", _p), ("free_list", _p),
                ("free_count", _i64)]


class Channel(C.Structure):
    _fields_ = [("slot", _i32), ("lo", _i32), ("hi", _i32), ("npoints", _i32),
                ("tf_x", _d * RO_MAX_TF_POINTS),
                ("tf_rgba", (_d * 4) * RO_MAX_TF_POINTS),
                ("empty_below", C.c_uint16 * 256), ("zero_upto", _i32), ("_pad", _i32),
                ("tf_seg", C.c_uint8 * 256)]


class Frame(C.Structure):
    _fields_ = [("mode", _i32), ("n_ch", _i32), ("width", _i32), ("height", _i32),
                ("cam_pos", _d * 3), ("cam_fwd", _d * 3), ("cam_right", _d * 3),
                ("cam_up", _d * 3), ("tan_half", _d), ("aspect", _d),
                ("base_step", _d), ("t0", _d), ("early_alpha", _d), ("eps_h", _d),
                ("start_level", _i32), ("check_skips", _i32),
                ("lod_threshold", _d * (RO_MAX_LEVELS + 1)),
                ("step_tab", _d * RO_MAX_LEVELS),
                ("maxlev_tab", _i32 * RO_MAX_LEVELS),
                ("dt_tab", _i32 * RO_MAX_LEVELS),
                ("n_parts", _i32), ("part", _i32), ("tile_rows", _i32),
                ("cls_depth", _i32), ("ref_pt", _p), ("ref_cache", _p),
                ("cls_min", _p), ("cls_max", _p), ("shared_outputs", _i32), ("max_samples", _i32),
                ("ch", Channel * RO_MAX_CH)]


class CameraDesc(C.Structure):
    _fields_ = [("position", _d * 3), ("target", _d * 3), ("up", _d * 3), ("fov_deg", _d)]


class RenderConfigDesc(C.Structure):
    _fields_ = [("width", _i32), ("height", _i32), ("base_step", _d),
                ("lod_reference_distance", _d), ("early_term_alpha", _d),
                ("traversal_start_level", _i32), ("_pad0", _i32)]


class ChannelDesc(C.Structure):
    _fields_ = [("slot", _i32), ("level_lo", _i32), ("level_hi", _i32), ("npoints", _i32),
                ("x", _d * RO_MAX_TF_POINTS), ("rgba", (_d * 4) * RO_MAX_TF_POINTS)]


class Outputs(C.Structure):
    _fields_ = [("image", _p), ("required", _p), ("pix_required", _p),
                ("hist", _p), ("counters", _p)]


class Feedback(C.Structure):
    _fields_ = [("brick_keys", _p), ("brick_ids", _p), ("meta_keys", _p),
                ("meta_ids", _p), ("counts", _p), ("counts_dev", _p)]


_LIB = None

_SIGS = {
    "ro_abi_version": ([], _i32),
    "ro_last_error": ([], C.c_char_p),
    "ro_create": ([C.POINTER(Layout), C.POINTER(_p)], _i32),
    "ro_destroy": ([_p], _i32),
    "ro_reserve": ([_p, _i64], _i32),
    "ro_local_rows": ([_i32, _i32, _i32, _i32], _i64),
    "ro_render": ([_p, C.POINTER(Frame), C.POINTER(State), C.POINTER(Outputs), _p], _i32),
    "ro_feedback_collect": ([_p, _i64, _i32, C.POINTER(Feedback), _p], _i32),
    "ro_note_sampled": ([_p, C.POINTER(State), _p, _i64, _p], _i32),
    "ro_feedback_merge": ([_p, _p, _p, _i32, _i64, _p], _i32),
    "ro_gather_rows": ([_p, _i32, _i64, _i32, _i32, _i32, _p, _p], _i32),
    "ro_apply_bricks": ([_p, C.POINTER(State), _p, _i64, _p, _i32, _i64, _i32, _p, _p, _p], _i32),
    "ro_evict_bricks": ([_p, C.POINTER(State), _p, _i64, _i32, _p], _i32),
    "ro_mark_empty": ([_p, C.POINTER(State), _p, _i64, _p], _i32),
    "ro_apply_metadata": ([_p, C.POINTER(State), _p, _p, _p, _p, _i64, _p], _i32),
    "ro_write_level_metadata": ([_p, C.POINTER(State), _i32, _i32, _p, _p, _p], _i32),
    "ro_swap_channel": ([_p, C.POINTER(State), _i32, _i32, _p], _i32),
    "ro_octree_update": ([_p, C.POINTER(State), _p, _i64, _p], _i32),
    "ro_rebuild_masks": ([_p, C.POINTER(State), _p], _i32),
    "ro_sync": ([_p, _p], _i32),
    "ro_set_feedback_buffers": ([_p, _p, _p], _i32),
    "ro_enable_peer_access": ([_i32], _i32),
    "ro_pack_frame": ([_i32, _i32, _i32, _i32, C.POINTER(CameraDesc),
                       C.POINTER(RenderConfigDesc), C.POINTER(ChannelDesc), _i32, _d,
                       C.POINTER(Frame)], _i32),
    "ro_tf_evaluate": ([_i32, _p, _p, _d, _p], _i32),
    "ro_tf_first_support": ([_i32, _p, _p, _d, _p], _i32),
    "ro_tf_support_intervals": ([_i32, _p, _p, _p, _p], _i32),
    "ro_tf_interval_max_opacity": ([_i32, _p, _p, _d, _d, _p], _i32),
    "ro_tf_tables": ([_i32, _p, _p, _p, _p, _p, _p], _i32),
    "ro_upload_state": ([_p, C.POINTER(HostState), C.POINTER(State), _p], _i32),
    "ro_download_state": ([_p, C.POINTER(State), _p, _p, _p, _p, _p, _p, _p, _p, _p], _i32),
    "ro_apply_bricks_lz4": ([_p, C.POINTER(State), _p, _i64, _p, _p, _i32, _i64, _i32, _p,
                             _p, _p], _i32),
    "ro_lz4_decode": ([_p, _p, _p, _i64, _p, _i64, _i64, _p, _p], _i32),
    "ro_normalize_to_u8": ([_p, _p, _i32, _i64, _p, _p], _i32),
    "ro_downsample_box": ([_p, _i32, _i32, _i32, _i32, _i32, _i32, _p, _p], _i32),
    "ro_extract_bricks": ([_p, _i32, _i32, _i32, _i32, _i32, _i32, _p, _p], _i32),
    "ro_node_minmax": ([_p, _p, _i32, _i32, _i32, _i32, _i32, _p, _p, _p], _i32),
    "ro_fill_metadata": ([_p, C.POINTER(State), _i32, _p, _i32, _i32, _i32, _i32, _p], _i32),
    "ro_bricks_box_minmax": ([_p, _p, _i64, _i32, _i32, _i32, _p, _p, _p], _i32),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libresoct.so; raises NativeLibraryMissing if it was never built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        handle = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        if handle.ro_abi_version() != 1:
            raise NativeLibraryMissing("libresoct.so ABI version mismatch")
        _LIB = handle
    return _LIB


def check(rc: int):
    if rc != 0:
        msg = lib().ro_last_error().decode(errors="replace")
        raise NativeError(f"libresoct error {rc}: {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise NativeError("the residency-octree render path needs a CUDA device "
                          "(no CPU fallback exists)")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()
