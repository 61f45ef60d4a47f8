"""Kernel-level breakdown of one Engine.apply_bricks batch (config-3 scene,
cold cache, pageable or page-locked payloads) with torch.profiler."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from torch.profiler import ProfilerActivity, profile
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200 import volume as V
    from paper_2309_04393_b200.paging import PinnedBrickBuffer
    store = V.VolumeStore(V.sparse_multichannel(256, channels=8, seed=11), (32, 32, 32), 4,
                          (2, 2, 2))
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    for pinned in (False, True):
        eng = Engine(store.manifest, EngineConfig(octree_depth=5, cache_slots=(16, 16, 8),
                                                  channel_slots=4))
        eng.paging.ctx
        from paper_2309_04393_b200 import _native as N
        N.check(N.lib().ro_reserve(eng.paging.ctx, 512))
        ids, pays = [], []
        for s in range(4):
            for lev in (0, 1):
                g = store.manifest.levels[lev].brick_grid_dims
                for z in range(g[2]):
                    for y in range(g[1]):
                        for x in range(g[0]):
                            ids.append(eng.paging.encode(s, lev, (x, y, z)))
                            pays.append(store.brick(s, lev, (x, y, z)))
        ids, pays = ids[:2 * n], np.stack(pays[:2 * n])
        buf = PinnedBrickBuffer((32, 32, 32))
        eng.advance_frame()
        eng.apply_bricks(ids[:n], buf.stack(list(pays[:n])) if pinned else pays[:n])  # warm
        torch.cuda.synchronize()
        eng.advance_frame()
        p = buf.stack(list(pays[n:2 * n])) if pinned else pays[n:2 * n]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            e0.record()
            eng.apply_bricks(ids[n:2 * n], p)
            e1.record()
            torch.cuda.synchronize()
        print(f"--- {n} bricks, {'page-locked' if pinned else 'pageable'} payloads: "
              f"{e0.elapsed_time(e1):.3f} ms (events)")
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))


if __name__ == "__main__":
    main()
