"""A pure C host (examples/render_c.c: include/resoct.h + libresoct.so +
cudart, no Python) builds a scene, inserts bricks, fills metadata, packs
(ro_pack_frame), renders and orders feedback; the same scene through the
Python API must give the identical image, counters and ordered requests."""

import os
import subprocess

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _voxel(x, y, z):
    dx, dy, dz = 2 * x + 1 - 64, 2 * y + 1 - 64, 2 * z + 1 - 64
    d2 = dx * dx + dy * dy + dz * dz
    return np.where((d2 > 1600) & (d2 < 2400), 200, (x * 7 + y * 13 + z * 3) % 23).astype(np.uint8)


def test_gpu_c_host_matches_python_api(native_lib, tmp_path):
    from paper_2309_04393_b200 import (Camera, ChannelSettings, Engine, EngineConfig,
                                       RenderConfig, TransferFunction, render_frame)
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    exe = tmp_path / "render_c"
    lib = os.path.join(ROOT, "paper_2309_04393_b200")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "render_c.c"),
                    "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    "-L" + lib, "-lresoct", "-L/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath," + lib, "-lm", "-o", str(exe)], check=True)
    out = tmp_path / "out"
    subprocess.run([str(exe), str(out)], check=True, timeout=120)
    c_img = np.fromfile(str(out) + ".img", dtype=np.float32).reshape(32, 40, 4)
    lines = open(str(out) + ".txt").read().split()
    c_ctr = [int(v) for v in lines[:4]]
    nb, nm = int(lines[4]), int(lines[5])
    c_bricks = [int(v) for v in lines[6:6 + nb]]

    man = VolumeManifest(name="c", channel_count=1, brick_size=(16, 16, 16),
                         levels=plan_levels((64, 64, 64), (16, 16, 16), 2, (2, 2, 2)))
    eng = Engine(man, EngineConfig(octree_depth=3, cache_slots=(5, 5, 5), channel_slots=1))
    z, y, x = np.meshgrid(np.arange(64), np.arange(64), np.arange(64), indexing="ij")
    lvl0 = _voxel(x, y, z)
    ids, pays = [], []
    for lev, g in ((0, 4), (1, 2)):
        s = 1 << lev
        for bz in range(g):
            for by in range(g):
                for bx in range(g):
                    zz, yy, xx = np.meshgrid(np.arange(16), np.arange(16), np.arange(16),
                                             indexing="ij")
                    pays.append(_voxel((bx * 16 + xx) * s, (by * 16 + yy) * s, (bz * 16 + zz) * s))
                    ids.append(eng.paging.encode(0, lev, (bx, by, bz)))
    eng.apply_bricks(ids, np.stack(pays))
    eng.fill_metadata_from_volumes({0: lvl0})
    tf = TransferFunction(points=((0.0, (0.0, 0.0, 0.0, 0.0)), (40.0, (0.0, 0.0, 0.0, 0.0)),
                                  (255.0, (1.0, 1.0, 1.0, 1.0))))
    o = render_frame(eng.paging, eng.octree, [ChannelSettings(slot=0, tf=tf)],
                     Camera(position=(2.1, 1.2, 1.4), target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0),
                            fov_deg=45.0),
                     RenderConfig(image_dims=(40, 32), base_step=1.0 / 64.0,
                                  max_requests_per_frame=64, traversal_start_level=2))
    assert np.array_equal(c_img, o.image)
    assert c_ctr == [o.stats.traversal_steps, o.stats.samples_evaluated,
                     o.stats.samples_skipped, o.stats.skip_violations]
    assert c_bricks == o.brick_requests and nm == len(o.metadata_requests)
    assert o.stats.samples_evaluated > 0 and o.image[..., 3].max() > 0
