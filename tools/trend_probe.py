"""One residency-mode frame of the acceptance trend scene (reference
bench.run_orbit's sparse 4-channel 256^3 volume, fully resident, exact
metadata) at --size^2: kernel time and work counters (counters 5..7 are the
RO_STATS instrumentation's when RESOCT_LIB points at such a build)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--mode", default="residency", choices=["residency", "pagetable"])
    args = ap.parse_args()
    from paper_2309_04393_b200 import ChannelSettings, RenderConfig, grayscale_ramp_tf, methods
    from paper_2309_04393_b200 import render as R
    from paper_2309_04393_b200 import volume as V
    from paper_2309_04393_b200.camera import orbit_path
    store = V.VolumeStore(V.sparse_multichannel(256, channels=4), (32, 32, 32), 4, (2, 2, 2))
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(40.0)) for s in range(4)]
    slots = {s: s for s in range(4)}
    cfg = RenderConfig(image_dims=(args.size, args.size), base_step=1.0 / 128.0,
                       max_requests_per_frame=2048, traversal_start_level=2)
    econf = methods.full_engine_config(store, 4, depth=5)
    if args.mode == "residency":
        eng = methods.prepare_engine(store, slots, econf)
        mode, oc = R.MODE_RESIDENCY, eng.octree
    else:
        eng = methods.prepare_pagetable_engine(store, slots, econf)
        mode, oc = R.MODE_PAGETABLE, None
    cam = orbit_path(12)[0]
    fp = R.FramePass(mode, eng.paging, oc, chans, cam, cfg)
    for _ in range(3):
        fp.render()
        fp.collect()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fp.render()
    e1.record()
    torch.cuda.synchronize()
    fp.collect()
    c = fp.buf.counters.cpu().tolist()
    print(json.dumps({"mode": args.mode, "size": args.size, "kernel_ms": e0.elapsed_time(e1) / 10,
                      "steps": c[0], "evaluated": c[1], "skipped": c[2], "stat5": c[5],
                      "stat6": c[6], "stat7": c[7], "fetches": int(fp.buf.hist.sum().item())}))


if __name__ == "__main__":
    main()
