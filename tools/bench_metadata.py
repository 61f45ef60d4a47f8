"""Culling-metadata producer throughput: every node
of a D=6 tree over one config-2 channel (2048x2048x128 u8 level 0), GPU
(ro_fill_metadata, CUDA events) vs the reference's numpy _box_minmax_grid on
one host core (engine.py:186-219, restated in volume.box_minmax_grid, timed
on a bounded subset of depths), and a cold-start Session at 256^2 with
per-request host metadata vs the GPU pyramid."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04393_b200 import scenarios  # noqa: E402
from paper_2309_04393_b200.metadata import node_minmax  # noqa: E402
from paper_2309_04393_b200.volume import box_minmax_grid  # noqa: E402


def main():
    dims = (2048, 2048, 128)
    g = torch.Generator(device="cuda").manual_seed(5)
    vol = torch.randint(0, 256, (dims[2], dims[1], dims[0]), dtype=torch.uint8, device="cuda",
                        generator=g)
    pad = 12
    D = 6
    for _ in range(2):
        for d in range(D + 1):
            node_minmax(vol, d, pad)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for d in range(D + 1):
        node_minmax(vol, d, pad)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    host = vol.cpu().numpy()
    t = time.perf_counter()
    for d in (0, 1, 2):
        box_minmax_grid(host, 1 << d, pad)
    cpu_s_012 = time.perf_counter() - t
    mn, mx = node_minmax(vol, 2, pad)
    gm, gx = box_minmax_grid(host, 4, pad)
    assert np.array_equal(mn.cpu().numpy(), gm.ravel()) and np.array_equal(mx.cpu().numpy(),
                                                                           gx.ravel())
    vol_gb = host.nbytes / 1e9
    print(json.dumps({"volume": list(dims), "depths": D + 1, "pad": pad,
                      "gpu_all_levels_ms": gpu_ms,
                      "gpu_GBps_per_level": vol_gb * (D + 1) / (gpu_ms / 1e3),
                      "cpu_numpy_levels_0_2_s": cpu_s_012,
                      "cpu_numpy_GBps_per_level": vol_gb * 3 / cpu_s_012}))


if __name__ == "__main__":
    main()
