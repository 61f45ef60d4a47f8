"""Breakdown of one render_frame() call at config 2 (host pack, ray cast +
request ordering, D2H, host post-processing), wall-clock with syncs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04393_b200 import render as R, scenarios  # noqa: E402


def main():
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cfg, chans, cam = scn.render, scn.channels, scn.camera
    for _ in range(3):
        R.render_frame(eng.paging, eng.octree, chans, cam, cfg)
    torch.cuda.synchronize()
    n = 20
    t = time.perf_counter()
    for _ in range(n):
        R.render_frame(eng.paging, eng.octree, chans, cam, cfg)
    e2e = (time.perf_counter() - t) / n * 1e3
    parts = {"pack": 0.0, "render+collect": 0.0, "d2h": 0.0}
    for _ in range(n):
        t0 = time.perf_counter()
        fp = R.FramePass(R.MODE_RESIDENCY, eng.paging, eng.octree, chans, cam, cfg)
        t1 = time.perf_counter()
        fp.render()
        fp.collect()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        img = torch.empty(fp.buf.image.shape, dtype=torch.float32, pin_memory=True)
        img.copy_(fp.buf.image, non_blocking=True)
        px = torch.empty(fp.buf.pix_required.shape, dtype=torch.int32, pin_memory=True)
        px.copy_(fp.buf.pix_required, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        parts["pack"] += (t1 - t0) * 1e3 / n
        parts["render+collect"] += (t2 - t1) * 1e3 / n
        parts["d2h"] += (t3 - t2) * 1e3 / n
    gb = (fp.buf.image.numel() * 4 + fp.buf.pix_required.numel() * 4) / 1e9
    print({"e2e_ms": e2e, **parts, "d2h_GBps": gb / (parts["d2h"] / 1e3)})


if __name__ == "__main__":
    main()
