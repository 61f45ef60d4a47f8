"""Brick ingest throughput: the reference path
(liblz4 frame decode on a host core, lz4io.py:69-110, then host payload
upload) vs LZ4 frames uploaded and decoded on the GPU straight into the cache
(ro_apply_bricks_lz4).  Bricks are config-2 CyCIF bricks (32^3 u8).

    python tools/bench_ingest.py [--bricks 4096]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import lz4_ref  # noqa: E402  (CPU baseline only)
from paper_2309_04393_b200 import Engine, EngineConfig, ingest, scenarios  # noqa: E402
from paper_2309_04393_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bricks", type=int, default=4096)
    args = ap.parse_args()
    scn = scenarios.cycif(device="cuda")
    man = scn.manifest
    n = min(args.bricks, scn.payloads.shape[0])
    # a spread of bricks (level 0 and coarser)
    idx = np.linspace(0, scn.payloads.shape[0] - 1, n).astype(np.int64)
    pays = scn.payloads[torch.from_numpy(idx).cuda()].cpu().numpy()
    ids = scn.brick_ids[idx]
    frames = [ingest.compress_brick(p) for p in pays]
    raw_bytes = pays.nbytes
    comp_bytes = sum(len(f) for f in frames)
    buf, offs = ingest.pack_frames(frames)

    # reference path: host liblz4 decode, one core
    t = time.perf_counter()
    for f in frames:
        lz4_ref.decompress(f, 32 * 32 * 32)
    cpu_s = time.perf_counter() - t

    # GPU decode kernel alone (frames resident in HBM)
    d_buf = torch.from_numpy(buf).cuda()
    d_off = torch.from_numpy(offs).cuda()
    out = torch.empty((n, 32, 32, 32), dtype=torch.uint8, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    ctx = ingest._ctx()

    def dec():
        N.check(N.lib().ro_lz4_decode(ctx, d_buf.data_ptr(), d_off.data_ptr(), n,
                                      out.data_ptr(), 32768, 32768, st.data_ptr(),
                                      N.stream_ptr()))
    for _ in range(3):
        dec()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        dec()
    e1.record()
    torch.cuda.synchronize()
    k_ms = e0.elapsed_time(e1) / reps
    assert np.array_equal(out.cpu().numpy(), pays)

    # end to end: host frames -> H2D -> decode -> LRU insert (+octree) on the device
    cfg = EngineConfig(octree_depth=scn.depth, cache_slots=tuple(scn.cache_slots),
                       channel_slots=scn.m)
    del scn
    torch.cuda.empty_cache()
    Engine(man, cfg).apply_bricks_lz4(list(ids[:8]), frames[:8])  # warm-up
    Engine(man, cfg).apply_bricks(list(ids[:8]), pays[:8])
    e2 = Engine(man, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e2.advance_frame()
    e2.apply_bricks_lz4(list(ids), (buf, offs))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t
    e3 = Engine(man, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e3.advance_frame()
    e3.apply_bricks(list(ids), pays)
    torch.cuda.synchronize()
    raw_s = time.perf_counter() - t
    print(json.dumps({
        "bricks": n, "raw_MB": raw_bytes / 1e6, "lz4_MB": comp_bytes / 1e6,
        "ratio": raw_bytes / comp_bytes,
        "cpu_liblz4_1core_GBps_out": raw_bytes / cpu_s / 1e9,
        "gpu_decode_kernel_ms": k_ms, "gpu_decode_GBps_out": raw_bytes / (k_ms / 1e3) / 1e9,
        "apply_bricks_lz4_ms": e2e_s * 1e3, "apply_bricks_raw_ms": raw_s * 1e3,
        "note": "apply_* = host arrays in, LRU + octree update on device, synchronised"}))


if __name__ == "__main__":
    main()
