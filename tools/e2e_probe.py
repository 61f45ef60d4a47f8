"""Host-side cost of render_frame() at config 2: wall time per call vs the
device time of the same frames, and the split of the host work (frame
packing, launches, post-synchronisation numpy work)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04393_b200 import render as R, scenarios  # noqa: E402
from paper_2309_04393_b200.camera import orbit_path  # noqa: E402


def main():
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cams = orbit_path(20)
    for c in cams[:3]:
        R.render_frame(eng.paging, eng.octree, scn.channels, c, scn.render)
    torch.cuda.synchronize()
    t_pack, t_call = [], []
    for c in cams:
        t0 = time.perf_counter()
        R.FramePass(R.MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, c, scn.render)
        t_pack.append(time.perf_counter() - t0)
    dev = []
    prof = None
    if os.environ.get("E2E_CPROFILE"):
        import cProfile
        prof = cProfile.Profile()
        prof.enable()
    t0 = time.perf_counter()
    for c in cams:   # outputs dropped each frame, as a viewer loop would
        t1 = time.perf_counter()
        out = R.render_frame(eng.paging, eng.octree, scn.channels, c, scn.render)
        t_call.append(time.perf_counter() - t1)
        dev.append(out.stats.render_ms)
        del out
    total = time.perf_counter() - t0
    if prof is not None:
        prof.disable()
        import pstats
        pstats.Stats(prof).sort_stats("tottime").print_stats(25)
    print(json.dumps({"render_frame_ms_mean": 1e3 * total / len(cams),
                      "framepass_ms_mean": 1e3 * sum(t_pack) / len(t_pack),
                      "render_ms_to_sync_mean": sum(dev) / len(dev),
                      "per_call_ms": [round(1e3 * t, 3) for t in t_call]}))


if __name__ == "__main__":
    main()
