"""Config 3 of BASELINE.json: mixed per-channel resolution bias + a mid-sequence
channel switch (4 -> 4 different channels), timing the octree bitmask update
(kernel 2) and the request/usage feedback + LRU (kernel 3) per frame.

    python tools/bench_config3.py [--image W H] [--frames N]

Scene: sparse_multichannel(256, channels=8,
seed=11), 32^3 bricks, 4 levels; m = 4 slots with level ranges
(0,3), (1,3), (2,3), (3,3); octree depth 5; budget 512; a cold Session; at
frame 10 every slot s is swapped to channel 4+s; then run on.  Prints one
JSON line with per-frame device times (CUDA events) of: render (ray cast +
feedback ordering), note_sampled, apply_bricks (LRU + page tables + cache
upload + octree pass), apply_metadata; plus the oracle's (reference-
semantics Python) update time for the same brick batches when --oracle.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _percentiles(xs) -> dict:
    """p50 / p99 / max of per-frame times, and frame 1 over the median."""
    a = np.asarray(xs, dtype=np.float64)
    p50 = float(np.percentile(a, 50))
    return {"p50": round(p50, 3), "p99": round(float(np.percentile(a, 99)), 3),
            "max": round(float(a.max()), 3), "first": round(float(a[0]), 3),
            "first_over_p50": round(float(a[0]) / p50, 2) if p50 > 0 else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--image", type=int, nargs=2, default=[1920, 1080])
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--swap-at", type=int, default=10)
    ap.add_argument("--device-metadata", action="store_true",
                    help="answer metadata requests from the GPU min/max pyramid")
    ap.add_argument("--lz4", action="store_true",
                    help="fetch LZ4 frames and decode them on the GPU into the cache")
    ap.add_argument("--oracle", action="store_true",
                    help="also time the reference-semantics Python updates")
    args = ap.parse_args()

    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       RenderConfig, Session, orbit_pose)
    from paper_2309_04393_b200 import volume as V
    from paper_2309_04393_b200.transfer import colored_ramp_tf
    from paper_2309_04393_b200.scenarios import COLORS

    t0 = time.perf_counter()
    store = V.VolumeStore(V.sparse_multichannel(256, channels=8, seed=11), (32, 32, 32), 4,
                          (2, 2, 2))
    build_s = time.perf_counter() - t0
    ranges = [(0, 3), (1, 3), (2, 3), (3, 3)]
    chans = [ChannelSettings(slot=s, tf=colored_ramp_tf(40.0, COLORS[s], 0.8),
                             level_range=ranges[s]) for s in range(4)]
    rconf = RenderConfig(image_dims=tuple(args.image), base_step=1.0 / 256.0,
                         max_requests_per_frame=512, traversal_start_level=2)
    econf = EngineConfig(octree_depth=5, cache_slots=(16, 16, 8), channel_slots=4)
    sess = Session(LocalTransport(store), econf, rconf, chans,
                   device_metadata=args.device_metadata, compressed_transfer=args.lz4)
    eng = sess.engine
    pose = orbit_pose(0.6)

    from paper_2309_04393_b200.render import render_frame
    ev = lambda: torch.cuda.Event(enable_timing=True)
    rows = []
    for i in range(args.frames):
        if i == args.swap_at:
            e0, e1 = ev(), ev()
            e0.record()
            for s in range(4):
                sess.swap_channel(s, 4 + s)
            e1.record()
            torch.cuda.synchronize()
            rows.append({"swap_ms": e0.elapsed_time(e1)})
        eng.advance_frame()
        e = [ev() for _ in range(6)]
        e[0].record()
        out = render_frame(eng.paging, eng.octree, sess.channels, pose, rconf)
        e[1].record()
        eng.note_sampled(out.required_mask_device)
        e[2].record()
        torch.cuda.synchronize()
        # fetch (host, out of scope): decoded payloads from the in-memory store
        tf0 = time.perf_counter()
        ids = list(out.brick_requests)
        pays = [sess._fetch_brick(b)[1] for b in ids]
        if args.device_metadata and out.metadata_requests:
            metas = list(zip(*sess._lookup_metadata(out.metadata_requests)))
        else:
            metas = [sess._fetch_metadata(n, s) for n, s in out.metadata_requests]
        fetch_ms = (time.perf_counter() - tf0) * 1e3
        e[3].record()
        if ids:
            if args.lz4:
                eng.apply_bricks_lz4(ids, pays)
            else:   # page-locked payloads, as Session.step_frame stacks them
                eng.apply_bricks(ids, sess._pinned.stack(pays))
        e[4].record()
        if metas:
            eng.apply_metadata_batch([m[0] for m in metas], [m[1] for m in metas],
                                     [m[2] for m in metas], [m[3] for m in metas])
        e[5].record()
        torch.cuda.synchronize()
        rows.append({"frame": eng.frame, "render_ms": e[0].elapsed_time(e[1]),
                     "note_sampled_ms": e[1].elapsed_time(e[2]),
                     "apply_bricks_ms": e[3].elapsed_time(e[4]),
                     "apply_metadata_ms": e[4].elapsed_time(e[5]),
                     "host_fetch_ms": fetch_ms, "bricks": len(ids), "metas": len(metas),
                     "samples": out.stats.samples_evaluated + out.stats.samples_skipped,
                     "resident": eng.paging.occupied_slot_count()})
    frames = [r for r in rows if "frame" in r]
    upd = [r["apply_bricks_ms"] for r in frames if r["bricks"]]
    per_brick = [r["apply_bricks_ms"] / r["bricks"] for r in frames if r["bricks"]]
    line = {"config": "config 3: sparse_multichannel(256, 8), m=4 ranges (0,3)(1,3)(2,3)(3,3), "
                      f"D=5, budget 512, {args.image[0]}x{args.image[1]}, swap at frame "
                      f"{args.swap_at}",
            "frames": len(frames), "build_s": build_s,
            "render_ms_median": float(np.median([r["render_ms"] for r in frames])),
            "apply_bricks_ms_median": float(np.median(upd)) if upd else None,
            "apply_bricks_us_per_brick_median": 1e3 * float(np.median(per_brick)) if per_brick else None,
            "apply_metadata_ms_median": float(np.median([r["apply_metadata_ms"] for r in frames])),
            "host_fetch_ms_median": float(np.median([r["host_fetch_ms"] for r in frames])),
            "device_metadata": args.device_metadata, "lz4_transfer": args.lz4,
            "swap_ms": [r["swap_ms"] for r in rows if "swap_ms" in r],
            "frame_device_ms": _percentiles([r["render_ms"] + r["note_sampled_ms"]
                                             + r["apply_bricks_ms"] + r["apply_metadata_ms"]
                                             for r in frames]),
            "render_ms": _percentiles([r["render_ms"] for r in frames]),
            "per_frame": rows}
    if args.oracle:
        # reference-semantics Python update cost on a replayed batch
        from oracle.state import OracleResidency
        man = store.manifest
        st = OracleResidency(4, 4, man.brick_size, [l.dims for l in man.levels],
                             [l.brick_grid_dims for l in man.levels], (16, 16, 8), 5,
                             with_payloads=False)
        ids = [eng.paging.encode(s, lev, (x, y, z)) for s in range(4) for lev in (0, 1)
               for z in range(2) for y in range(2) for x in range(2)][:64]
        t0 = time.perf_counter()
        for b in ids:
            st.apply_brick(b, None, 1)
        line["oracle_apply_brick_ms_per_brick"] = (time.perf_counter() - t0) * 1e3 / len(ids)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
