"""CPU tests: C-ABI surface, host tables, codec / geometry known answers.

Known-answer vectors are the reference's own unit-test cases (cited).
"""

import math
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT


def test_native_library_exports_every_header_symbol(native_lib):
    header = open(os.path.join(ROOT, "include", "resoct.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(ro_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    from paper_2309_04393_b200 import _native
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(native_lib, name), name
    assert native_lib.ro_abi_version() == 1


def test_ctypes_structs_match_c_layout():
    """sizeof/offsetof of every ABI struct, compiled from the header with gcc,
    equals the ctypes mirror."""
    from paper_2309_04393_b200 import _native as N
    structs = {"ro_layout": N.Layout, "ro_state": N.State, "ro_channel": N.Channel,
               "ro_frame": N.Frame, "ro_outputs": N.Outputs, "ro_feedback": N.Feedback,
               "ro_host_state": N.HostState, "ro_camera": N.CameraDesc,
               "ro_render_config": N.RenderConfigDesc, "ro_channel_desc": N.ChannelDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "resoct.h"',
             'int main(void) {']
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        got = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    for line in got.strip().splitlines():
        name, val = line.rsplit(" ", 1)
        if name.endswith(" size"):
            cname = name.split()[0]
            assert C_sizeof(structs[cname]) == int(val), cname
        else:
            cname, fname = name.split(".")
            assert getattr(structs[cname], fname).offset == int(val), name


def C_sizeof(t):
    import ctypes
    return ctypes.sizeof(t)


def test_local_rows_partition_covers_image(native_lib):
    from paper_2309_04393_b200.distributed import part_rows
    for h in (1, 7, 8, 9, 64, 1080, 2160):
        for n in (1, 2, 3, 4, 8):
            rows = []
            for p in range(n):
                pr = part_rows(h, n, p, 8)
                assert native_lib.ro_local_rows(h, n, p, 8) == len(pr)
                rows += pr
            assert sorted(rows) == list(range(h))


def test_brick_id_codec_known_answers():
    """test_paging.py:24-26 and test_acceptance.py:258-265."""
    from paper_2309_04393_b200.paging import decode_brick_id, encode_brick_id
    assert encode_brick_id(1, 2, (3, 2, 1), 4, 2) == 0x06010203
    rng = np.random.default_rng(1234)
    for _ in range(2000):
        k, m = 8, 8
        s, lev = int(rng.integers(m)), int(rng.integers(k))
        c = tuple(int(v) for v in rng.integers(0, 256, 3))
        assert decode_brick_id(encode_brick_id(s, lev, c, k, m), k) == (s, lev, c)


def test_octree_offsets_and_index_known_answers():
    """test_octree.py:44-54."""
    from paper_2309_04393_b200.octree import NodeAddress, level_offset, node_from_index
    assert [level_offset(d) for d in range(5)] == [0, 1, 9, 73, 585]
    for d in range(5):
        side = 1 << d
        for idx in range(level_offset(d), level_offset(d) + min(side ** 3, 300)):
            a = node_from_index(idx)
            assert a.d == d and a.index == idx
    assert NodeAddress(2, 3, 1, 0).index == 9 + 3 + 4


def test_lod_and_depth_known_answers():
    """test_render_units.py:54-93."""
    from paper_2309_04393_b200.render import choose_resolution_level as lod
    from paper_2309_04393_b200.render import choose_traversal_depth as td
    assert lod(0.5, 1.0) == 0 and lod(1.0, 1.0) == 0 and lod(1.9, 1.0) == 0
    assert lod(2.0, 1.0) == 1 and lod(3.9, 1.0) == 1 and lod(4.0, 1.0) == 2
    assert lod(100.0, 1.0, 0, 3) == 3 and lod(8.0, 1.0, 2, 15) == 3
    assert lod(0.1, 1.0, 2, 15) == 2 and lod(1.0, 0.25) == 2
    assert td(1 / 8, 5) == 3 and td(1 / 256, 3) == 3 and td(0.3, 5) == 1
    assert td(2.0, 5) == 0 and td(1 / 64, 6) == 6


def test_lod_thresholds_reproduce_libm_floor_log2():
    """The kernel's LOD rule (ilogb + libm-derived thresholds) equals
    floor(log2(ratio)) for ratios straddling every power of two."""
    from paper_2309_04393_b200.render import lod_thresholds
    T = lod_thresholds()

    def kernel_rule(ratio):
        if ratio < 1.0:
            return 0
        e = math.frexp(ratio)[1] - 1
        if e >= 15:
            return 15
        lev = e
        if ratio >= T[lev + 1]:
            lev += 1
        elif lev >= 1 and ratio < T[lev]:
            lev -= 1
        return lev

    rng = np.random.default_rng(3)
    vals = list(rng.uniform(1.0, 70000.0, 20000))
    for L in range(1, 16):
        x = float(2 ** L)
        y = x
        for _ in range(6):
            vals.append(y)
            y = math.nextafter(y, 0.0)
        y = x
        for _ in range(6):
            vals.append(y)
            y = math.nextafter(y, math.inf)
    for r in vals:
        want = min(int(math.floor(math.log2(r))), 15)
        assert kernel_rule(r) == want, r


def test_empty_below_equals_interval_is_empty():
    """kernels._is_empty_meta / TransferFunction.interval_is_empty
    (test_kernels.py:53-61) as the kernel's one-compare threshold."""
    from paper_2309_04393_b200.transfer import TransferFunction, grayscale_ramp_tf
    tfs = [grayscale_ramp_tf(40.0), grayscale_ramp_tf(0.0, 0.5),
           TransferFunction(points=((10.0, (1, 0, 0, 0)), (20.0, (0, 1, 0, 0.7)),
                                    (30.0, (0, 0, 1, 0.2)))),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (100.0, (1, 1, 0, 0.9)),
                                    (101.0, (0, 0, 0, 0)), (255.0, (0, 0, 0, 0)))),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (255.0, (0, 0, 0, 0)))),
           TransferFunction(points=((0.0, (0, 0, 0, 0.3)), (57.5, (0, 0, 0, 0)),
                                    (200.25, (0, 0, 0, 0)), (255.0, (1, 1, 1, 1))))]
    for tf in tfs:
        eb = tf.empty_below()
        f, op = tf.support_table()
        for mn in range(0, 256, 3):
            for mx in range(0, 256, 5):
                ref = (f[mn] > mx) or (f[mn] == mx and op[mx] == 0.0)
                assert (mx < eb[mn]) == ref, (tf, mn, mx)
                if mx >= mn:
                    assert ref == tf.interval_is_empty(mn, mx)


def test_camera_ray_basis_reproduces_generate_rays():
    """The per-pixel formula the kernel uses equals camera.py:32-51."""
    from oracle.raycast import generate_rays as oracle_rays
    from paper_2309_04393_b200.camera import Camera, ray_basis
    rng = np.random.default_rng(0)
    for _ in range(30):
        cam = Camera(position=tuple(rng.uniform(-3, 3, 3)), target=tuple(rng.uniform(0, 1, 3)),
                     fov_deg=float(rng.uniform(10, 120)))
        w, h = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        b = ray_basis(cam, w, h)
        _, d = oracle_rays(cam.position, cam.target, cam.up, cam.fov_deg, w, h)
        for j in range(h):
            for i in range(w):
                u = (((i + 0.5) / w * 2.0 - 1.0) * b.tan_half) * b.aspect
                v = (1.0 - (j + 0.5) / h * 2.0) * b.tan_half
                dd = [(b.fwd[a] + u * b.right[a]) + v * b.up[a] for a in range(3)]
                n = math.sqrt((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2])
                assert [x / n for x in dd] == list(d[j * w + i])


def test_octree_geometry_integer_form_matches_fractions():
    """Integer leaf/brick overlap ranges == the reference's Fraction form
    (octree.py:126-189), incl. non-divisible dims."""
    from fractions import Fraction

    def ceil_open(v):
        return math.floor(v)

    def floor_open(v):
        return math.ceil(v) - 1

    for dims, B, D in (((100, 64, 33), 16, 3), ((48, 48, 48), 16, 4), ((2048, 2048, 128), 32, 6)):
        side = 1 << D
        for a, dim in enumerate(dims):
            grid = -(-dim // B)
            for c in range(grid):
                lo_f = Fraction(c * B, dim) * side
                hi_f = Fraction((c + 1) * B, dim) * side
                want = (max(0, ceil_open(lo_f)), min(side - 1, floor_open(hi_f)))
                got = (max(0, (c * B * side) // dim),
                       min(side - 1, -((-(c + 1) * B * side) // dim) - 1))
                assert got == want
            for d in range(D + 1):
                sd = 1 << d
                for x in range(sd):
                    lo = Fraction(x * dim, sd * B)
                    hi = Fraction((x + 1) * dim, sd * B)
                    want = (max(0, ceil_open(lo)), min(grid - 1, floor_open(hi)))
                    got = (max(0, (x * dim) // (sd * B)),
                           min(grid - 1, -((-(x + 1) * dim) // (sd * B)) - 1))
                    assert got == want


def test_feedback_merge_rule():
    """Keyed keep-first merge of per-part lists reproduces the global
    first-seen order and the bricks-first budget (render.py:210-215)."""
    from paper_2309_04393_b200.distributed import merge_feedback
    rng = np.random.default_rng(9)
    for _ in range(200):
        events = []  # (key, kind, id)
        for key in sorted(rng.choice(10 ** 6, size=int(rng.integers(0, 60)), replace=False)):
            kind = int(rng.integers(2))
            events.append((int(key), kind, int(rng.integers(0, 25))))
        budget = int(rng.integers(1, 30))
        seen = {0: [], 1: []}
        for key, kind, v in events:
            if v not in seen[kind]:
                seen[kind].append(v)
        want_b = seen[0][:budget]
        want_m = [(v // 3, v % 3) for v in seen[1][:budget - len(want_b)]]
        n_parts = int(rng.integers(1, 4))
        parts = []
        for p in range(n_parts):
            mine = [e for i, e in enumerate(events) if i % n_parts == p]
            lists = []
            for kind in (0, 1):
                first = {}
                for key, kd, v in mine:
                    if kd == kind and v not in first:
                        first[v] = key
                items = sorted((k, v) for v, k in first.items())[:budget]
                lists.append(np.array([k for k, _ in items], dtype=np.int64))
                lists.append(np.array([v for _, v in items], dtype=np.int64))
            parts.append(tuple(lists))
        bricks, metas = merge_feedback(parts, budget, 3)
        assert bricks == want_b and metas == want_m



def test_c_pack_frame_matches_python_packing(native_lib):
    """ro_pack_frame (C / C++ hosts) fills ro_frame byte for byte like the
    Python mirror (render._pack_frame: camera basis, LOD thresholds, step /
    depth tables, channel clamps, TF emptiness tables), no GPU needed."""
    import ctypes as C
    import numpy as np
    from paper_2309_04393_b200 import _native as N
    from paper_2309_04393_b200 import Camera, ChannelSettings, RenderConfig, TransferFunction
    from paper_2309_04393_b200.render import _pack_frame, _pack_frame_py

    class _P:  # the layout facts _pack_frame reads
        def __init__(self, k, m):
            self.config = type("cfg", (), {"k": k, "m": m})()

    rng = np.random.default_rng(3)
    for trial in range(40):
        k, m = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        depth = int(rng.integers(0, 8))
        n_ch = int(rng.integers(1, min(m, 4) + 1))
        chans = []
        for s in rng.permutation(m)[:n_ch]:
            n = int(rng.integers(2, 8))
            xs = np.sort(rng.choice(np.arange(0, 256), size=n, replace=False)).astype(float)
            pts = tuple((float(x), tuple(float(v) for v in rng.random(4)) if rng.random() < 0.6
                         else (0.1, 0.2, 0.3, 0.0)) for x in xs)
            lo = int(rng.integers(0, 12))
            chans.append(ChannelSettings(slot=int(s), tf=TransferFunction(points=pts),
                                         level_range=(lo, lo + int(rng.integers(0, 6)))))
        cam = Camera(position=tuple(float(v) for v in rng.uniform(-3, 3, 3)),
                     target=tuple(float(v) for v in rng.uniform(0, 1, 3)),
                     up=(0.0, 1.0, 0.0), fov_deg=float(rng.uniform(20, 90)))
        cfg = RenderConfig(image_dims=(int(rng.integers(1, 4000)), int(rng.integers(1, 3000))),
                           base_step=float(rng.choice([1 / 64, 1 / 256, 1 / 1000, 0.3])),
                           lod_reference_distance=float(rng.uniform(0.2, 3.0)),
                           early_term_alpha=0.99, traversal_start_level=int(rng.integers(0, 4)))
        eps = float(rng.choice([0.0, 2.5]))
        py = _pack_frame_py(0, _P(k, m), chans, cam, cfg, depth, eps)
        cd = N.CameraDesc((C.c_double * 3)(*cam.position), (C.c_double * 3)(*cam.target),
                          (C.c_double * 3)(*cam.up), cam.fov_deg)
        rc = N.RenderConfigDesc(cfg.image_dims[0], cfg.image_dims[1], cfg.base_step,
                                cfg.lod_reference_distance, cfg.early_term_alpha,
                                cfg.traversal_start_level, 0)
        descs = (N.ChannelDesc * n_ch)()
        for i, c in enumerate(chans):
            descs[i].slot, descs[i].level_lo, descs[i].level_hi = c.slot, *c.level_range
            descs[i].npoints = len(c.tf.points)
            for j, (x, rgba) in enumerate(c.tf.points):
                descs[i].x[j] = x
                for q in range(4):
                    descs[i].rgba[j][q] = rgba[q]
        out = N.Frame()
        N.check(native_lib.ro_pack_frame(k, m, depth, 0, C.byref(cd), C.byref(rc), descs, n_ch,
                                         eps, C.byref(out)))
        assert bytes(out) == bytes(py), trial
        assert bytes(_pack_frame(0, _P(k, m), chans, cam, cfg, depth, eps)) == bytes(py), trial


def test_host_result_pool_recycles_only_dropped_buffers():
    """render._ResultPool: a frame's page-locked result set is reused only
    after every array handed out from it -- and every view derived from
    those -- is gone; with all sets held, frames land in the private staging
    set (copied out) instead of allocating more page-locked memory."""
    import gc

    import torch
    from paper_2309_04393_b200 import render as R
    pool = R._ResultPool(depth=2, pin=False)
    shapes = (((8, 4), torch.float32),)

    def frame():
        (t,), owned = pool.acquire(shapes)
        if not owned:
            return None, t.data_ptr(), False
        (arr,) = pool.handout(shapes, (t,), (t,))
        return arr.reshape(32)[3:], t.data_ptr(), True   # the caller keeps a slice only

    o1, p1, _ = frame()
    o2, p2, _ = frame()
    assert p1 != p2                      # o1 still alive: a second set
    _, p3, owned3 = frame()
    assert not owned3 and p3 not in (p1, p2)   # depth reached: staging, not a third set
    held = torch.from_numpy(o2)          # a torch view of a numpy view keeps it alive too
    del o1
    gc.collect()
    o4, p4, owned4 = frame()
    assert owned4 and p4 == p1           # recycled once every view of it was gone
    del o2
    gc.collect()
    _, p5, owned5 = frame()
    assert not owned5                    # `held` still references set 2
    del held
    gc.collect()
    o6, p6, owned6 = frame()
    assert owned6 and p6 == p2
    del o4, o6


def test_procedural_store_metadata_is_conservative():
    """Config-4 procedural store: the occupancy-grid metadata answer bounds
    the real level-0 voxels of every queried box ((0, 0) only where every
    voxel is 0), and bricks are deterministic per (channel, level, brick)."""
    from paper_2309_04393_b200.scenarios import ProceduralStore
    st = ProceduralStore(dims=(256, 256, 32), channels=3, brick=16, cell=32,
                         occupancy=0.3, pool=4, seed=5)
    man = st.manifest
    gx, gy, gz = man.levels[0].brick_grid_dims
    rng = np.random.default_rng(0)
    for c in range(3):
        vol = np.zeros((32, 256, 256), dtype=np.uint8)
        for z in range(gz):
            for y in range(gy):
                for x in range(gx):
                    vol[z * 16:(z + 1) * 16, y * 16:(y + 1) * 16,
                        x * 16:(x + 1) * 16] = st.fetch_brick(c, 0, (x, y, z))
        for _ in range(200):
            lo = rng.integers(0, [256, 256, 32])
            hi = lo + rng.integers(1, [120, 120, 32])
            box = (*lo.tolist(), *np.minimum(hi, [256, 256, 32]).tolist())
            part = vol[box[2]:box[5], box[1]:box[4], box[0]:box[3]]
            mn, mx = st.region_min_max(c, 0, box)
            if (mn, mx) == (0, 0):
                assert part.max() == 0
            else:
                assert mn <= part.min() and mx >= part.max()
        assert np.array_equal(st.fetch_brick(c, 2, (1, 0, 0)), st.fetch_brick(c, 2, (1, 0, 0)))
