"""Per-frame cost of the sort-first exchange (distributed.PeerFrame) with two
ranks, against the same rows rendered without any exchange.

    RESOCT_DIST_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 \\
        --master-addr 127.0.0.1 tools/peer_overhead.py

On ONE GPU (the only layout gpurun offers) both ranks time-share the device
and the rendezvous tokens are host-side (gloo), so the figure is the
exchange's host/latency overhead, not NVLink behaviour: per rank, wall time
of PeerFrame.frame minus the wall time of a plain render + collect of the
same part.  Prints one JSON line on rank 0.
"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group(os.environ.get("RESOCT_DIST_BACKEND", "gloo"))
    from paper_2309_04393_b200 import scenarios
    from paper_2309_04393_b200.camera import orbit_path
    from paper_2309_04393_b200.distributed import PeerFrame
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cfg = scn.render
    cams = orbit_path(12)
    passes = [FramePass(MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, c, cfg,
                        partition=(world, rank, 8), bricks_first=True) for c in cams]
    budget, m = cfg.max_requests_per_frame, eng.paging.config.m

    def timed(fn, n):
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i in range(n):
            fn(i)
        torch.cuda.synchronize()
        el = torch.tensor([(time.perf_counter() - t) / n], dtype=torch.float64)
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        return float(el[0]) * 1e3

    def plain(i):
        fp = passes[i % len(passes)]
        fp.frame.shared_outputs = 0
        fp.render()
        fp.collect()

    for i in range(3):
        plain(i)
    plain_ms = timed(plain, 12)
    peer = PeerFrame(eng.paging, eng.octree, len(scn.channels), cfg.image_dims)
    for i in range(3):
        peer.frame(passes[i], budget, m)
    peer_ms = timed(lambda i: peer.frame(passes[i % len(passes)], budget, m), 12)
    peer.close()
    if rank == 0:
        print(json.dumps({"ranks": world, "backend": dist.get_backend(), "gpus": 1,
                          "plain_part_frame_ms": plain_ms, "peer_frame_ms": peer_ms,
                          "exchange_overhead_ms": peer_ms - plain_ms,
                          "note": "both ranks on one GPU (time-shared); gloo host tokens"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
