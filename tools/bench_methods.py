"""Three-way method comparison on the B200 path (reference bench.py:98-161):
residency octree vs classic octree vs page-table only over an orbit, one JSON
line per method with the reference's summary fields (mean cache bytes,
traversal steps, skipped samples, wall ms per frame incl. D2H) plus the
ray-cast kernel time measured with CUDA events.

    python tools/bench_methods.py [--frames 36] [--size 96]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04393_b200 import (ChannelSettings, RenderConfig,  # noqa: E402
                                   grayscale_ramp_tf, methods, orbit_path)
from paper_2309_04393_b200 import render as R  # noqa: E402
from paper_2309_04393_b200 import volume as V  # noqa: E402


def kernel_ms(mode, paging, octree, chans, cam, cfg, classic, reps=5):
    fp = R.FramePass(mode, paging, octree, chans, cam, cfg, classic=classic)
    fp.render()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fp.render()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=36)
    ap.add_argument("--size", type=int, default=96)
    ap.add_argument("--n", type=int, default=256)
    args = ap.parse_args()
    store = V.VolumeStore(V.sparse_multichannel(args.n, channels=4), (32, 32, 32), 4,
                          (2, 2, 2))
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(40.0)) for s in range(4)]
    slots = {s: s for s in range(4)}
    cfg = RenderConfig(image_dims=(args.size, args.size), base_step=1.0 / 128.0,
                       max_requests_per_frame=2048, traversal_start_level=2)
    econf = methods.full_engine_config(store, 4, depth=5)
    # warm-up orbit (first-launch / allocation costs of every method), untimed
    methods.run_orbit(store, chans, slots, cfg, econf, num_frames=2)
    rows = methods.run_orbit(store, chans, slots, cfg, econf, num_frames=args.frames)
    summary = methods.summarize(rows)
    for method in summary:
        summary[method]["median_ms"] = float(np.median([r.ms for r in rows
                                                        if r.method == method]))
    # kernel-only time per method on a few poses
    eng = methods.prepare_engine(store, slots, econf)
    eng_pt = methods.prepare_pagetable_engine(store, slots, econf)
    classic = methods.build_classic(eng, store, slots)
    cams = orbit_path(args.frames)[:: max(1, args.frames // 6)]
    for method, mode, pg, oc, cl in (
            ("residency", R.MODE_RESIDENCY, eng.paging, eng.octree, None),
            ("classic", R.MODE_CLASSIC, eng.paging, None, classic),
            ("pagetable", R.MODE_PAGETABLE, eng_pt.paging, None, None),
            ("reference", R.MODE_REFERENCE, eng.paging, None, None)):
        ks = [kernel_ms(mode, pg, oc, chans, c, cfg, cl) for c in cams]
        summary.setdefault(method, {})["kernel_ms_mean"] = sum(ks) / len(ks)
    for method, s in summary.items():
        print(json.dumps({"method": method, "image": [args.size, args.size],
                          "scene": f"sparse_multichannel({args.n}, 4) 32^3 bricks D5",
                          **s}))


if __name__ == "__main__":
    main()
