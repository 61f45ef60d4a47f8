"""Sort-first over peer memory (distributed.PeerFrame): two ranks render
their row blocks straight into rank 0's full-frame buffers and request-key
arrays through CUDA IPC; the owner's single feedback pass must equal the
single-GPU frame exactly.  Both ranks run on one GPU here (IPC within a
device; on a B200 box the same mappings are NVLink peer memory).  No kernel
waits on another: ranks synchronise with host barriers (gloo)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from test_gpu_parity import _random_partial_engine
        from paper_2309_04393_b200 import (ChannelSettings, RenderConfig, grayscale_ramp_tf,
                                           orbit_pose, render_frame)
        from paper_2309_04393_b200.distributed import PeerFrame
        from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
        eng = _random_partial_engine(7, eps=0.0, depth=3, m=4)
        chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(20.0 + 10 * s), level_range=(0, 2))
                 for s in (1, 3, 0, 2)]
        cfg = RenderConfig(image_dims=(53, 41), base_step=1 / 64, max_requests_per_frame=60)
        pose = orbit_pose(1.3, radius=1.8)
        ref = render_frame(eng.paging, eng.octree, chans, pose, cfg) if rank == 0 else None
        peer = PeerFrame(eng.paging, eng.octree, len(chans), cfg.image_dims)
        results = []
        for _ in range(2):   # twice: the owner's key arrays must come back clean
            fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, chans, pose, cfg,
                           partition=(world, rank, 8), bricks_first=True)
            bricks, metas = peer.frame(fp, cfg.max_requests_per_frame, eng.paging.config.m)
            if rank == 0:
                b = peer.bufs
                w, h = cfg.image_dims
                ok = (np.array_equal(b["image"].cpu().numpy().reshape(h, w, 4), ref.image)
                      and bricks == ref.brick_requests and metas == ref.metadata_requests
                      and np.array_equal(b["required"].cpu().numpy(), ref.required_mask)
                      and np.array_equal(b["hist"].cpu().numpy(), ref.level_histogram)
                      and np.array_equal(b["pix_required"].cpu().numpy(), ref.pixel_required)
                      and int(b["counters"][1] + b["counters"][2]) ==
                      ref.stats.samples_evaluated + ref.stats.samples_skipped)
                results.append(bool(ok))
            else:
                results.append(isinstance(bricks, list) and isinstance(metas, list))
        peer.close()
        q.put((rank, all(results)))
    except Exception as e:  # report instead of hanging the other rank
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_gpu_peer_frame_equals_single_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert res == {0: True, 1: True}, res
