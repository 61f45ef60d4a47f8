"""First-frame latency of a cold Session (config 3 scene): wall time of the
first frames (render + note_sampled + fetch + apply) and their split, to find
one-time costs (allocation, module loading, pinned pools).

    python tools/first_frame.py [--frames N]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--image", type=int, nargs=2, default=[1920, 1080])
    args = ap.parse_args()
    t0 = time.perf_counter()
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    t_cuda = time.perf_counter() - t0
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       RenderConfig, Session, orbit_pose)
    from paper_2309_04393_b200 import volume as V
    from paper_2309_04393_b200.transfer import colored_ramp_tf
    from paper_2309_04393_b200.scenarios import COLORS
    store = V.VolumeStore(V.sparse_multichannel(256, channels=8, seed=11), (32, 32, 32), 4,
                          (2, 2, 2))
    ranges = [(0, 3), (1, 3), (2, 3), (3, 3)]
    chans = [ChannelSettings(slot=s, tf=colored_ramp_tf(40.0, COLORS[s], 0.8),
                             level_range=ranges[s]) for s in range(4)]
    rconf = RenderConfig(image_dims=tuple(args.image), base_step=1.0 / 256.0,
                         max_requests_per_frame=512, traversal_start_level=2)
    econf = EngineConfig(octree_depth=5, cache_slots=(16, 16, 8), channel_slots=4)
    t1 = time.perf_counter()
    sess = Session(LocalTransport(store), econf, rconf, chans)
    torch.cuda.synchronize()
    t_sess = time.perf_counter() - t1
    rows = []
    for i in range(args.frames):
        ts = time.perf_counter()
        rec = sess.step_frame(orbit_pose(0.6))
        torch.cuda.synchronize()
        rows.append({"frame": i + 1, "ms": (time.perf_counter() - ts) * 1e3,
                     "render_ms": rec.output.stats.render_ms,
                     "bricks": rec.bricks_applied, "metas": rec.metadata_applied})
    steady = sorted(r["render_ms"] for r in rows[len(rows) // 2:])
    print(json.dumps({"cuda_init_s": t_cuda, "session_init_s": t_sess,
                      "module_loading": os.environ.get("CUDA_MODULE_LOADING", "default"),
                      "first_render_ms": rows[0]["render_ms"],
                      "steady_render_ms_median": steady[len(steady) // 2], "frames": rows}))


if __name__ == "__main__":
    main()
