"""Helpers for the GPU parity tests."""

from __future__ import annotations

import hashlib

import numpy as np


def _h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def device_state_hashes(engine_or_paging, octree=None) -> dict:
    """Hashes of the device state in the REFERENCE layout."""
    p = getattr(engine_or_paging, "paging", engine_or_paging)
    o = octree if octree is not None else getattr(engine_or_paging, "octree", None)
    out = {"pt_status": _h(p.pt_status), "pt_slot": _h(p.pt_slot),
           "slot_brick": _h(p.slot_brick), "slot_last_used": _h(p.slot_last_used),
           "cache": _h(p.cache), "free": _h(np.array(p._free, dtype=np.int64))}
    if o is not None:
        out["words"] = _h(o.words)
    return out


def diff_hashes(got: dict, want: dict) -> list:
    return [k for k in want if k in got and got[k] != want[k]]


def oracle_state_from_device(engine):
    from oracle import raycast as orc
    p, o = engine.paging, engine.octree
    return orc.OracleState(m=p.config.m, k=p.config.k, brick_size=p.config.brick_size,
                           level_dims=p.level_dims, level_grids=p.level_grids,
                           pt_offsets=p.pt_offsets, pt_status=p.pt_status,
                           pt_slot=p.pt_slot, cache=p.cache, words=o.words,
                           depth=o.config.depth, eps_h=o.config.homogeneity_eps)


def cam_tuple(cam):
    return (cam.position, cam.target, cam.up, cam.fov_deg)
