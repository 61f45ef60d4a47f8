"""Config 5 of BASELINE.json: 3840x2160, m = 6 channels, a 120-frame camera
orbit, sort-first image tiles on 1/2/4/8 GPUs with the NCCL exchange.

    python tools/bench_config5.py [--frames 120]                 # 1 GPU
    torchrun --nproc-per-node N tools/bench_config5.py           # N GPUs

Scene: the config-2 CyCIF-like volume builder with six visible channels
{0, 3, 6, 9, 12, 15} (m = 6), levels >= 2 resident plus half of levels 0/1.
Every frame renders its rows (sort-first, 8-row blocks round-robin), orders
the feedback, and (N > 1) runs distributed.exchange (usage all-reduce, request
all-gather + merge, image gather to rank 0).  Time per frame = max over ranks
of CUDA-event time.  Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--image", type=int, nargs=2, default=[3840, 2160])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2309_04393_b200 import orbit_path, scenarios
    from paper_2309_04393_b200.distributed import exchange
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass

    scn = scenarios.cycif(device=f"cuda:{local}", dataset_channels=(0, 3, 6, 9, 12, 15),
                          image_dims=tuple(args.image))
    eng = scenarios.build_engine(scn, device=torch.device("cuda", local))
    cfg = scn.render
    cams = orbit_path(args.frames)
    m = eng.paging.config.m
    times, samples = [], 0
    stream = torch.cuda.current_stream()
    for i, cam in enumerate(cams + cams[:3]):   # 3 warm-up frames at the end
        fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, cam, cfg,
                       partition=(world, rank, 8), bricks_first=(world == 1))
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fp.render()
        fp.collect()
        if world > 1:
            b = fp.buf
            exchange(dict(image=b.image, required=b.required, pix_required=b.pix_required,
                          hist=b.hist, counters=b.counters, fb=b.fb, counts=b.counts),
                     cfg.image_dims, 8, cfg.max_requests_per_frame, m)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        c = fp.buf.counters.clone()
        if world > 1:
            t = torch.tensor([ms], device=c.device, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t[0])
            torch.distributed.all_reduce(c)
        if i >= 3 or len(cams) < 4:
            times.append(ms)
            samples += int(c[1] + c[2])
    if rank == 0:
        times = times[:args.frames]
        tot = sum(times)
        print(json.dumps({
            "config": f"config 5: {args.image[0]}x{args.image[1]}, m=6 (CyCIF-like channels "
                      "0,3,6,9,12,15), orbit_path(%d), sort-first x%d" % (args.frames, world),
            "n_gpus": world, "frames": len(times), "frames_per_s": len(times) / (tot / 1e3),
            "ms_per_frame_mean": float(np.mean(times)), "ms_per_frame_p50": float(np.median(times)),
            "ms_per_frame_max": float(np.max(times)),
            "gsamples_per_s": samples / (tot / 1e3) / 1e9}))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
