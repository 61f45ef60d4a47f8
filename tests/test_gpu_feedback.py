"""The request-ordering kernel (csrc/feedback.cu k_feedback) against a numpy
sort: random first-seen key sets written straight into caller-owned key
arrays (ro_set_feedback_buffers), then ro_feedback_collect.  Covers every
shape of the selection: everything survives, radix-selected budgets, budgets
above one shared-memory sort chunk (rank chunks), keys needing more than 32
packed bits (large pixel and event indices: the 4K / many-event case),
bricks-first and per-list budgets, the asynchronous (device-counts) form,
and that every key array is reset for the next frame.

The bricks-first rule is render.py:210-215; the first-seen order it cuts is
kernels.py:457-517 (ordered by (pixel, event) key, see raycast.cu)."""

import ctypes as C

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def eng(native_lib):
    import torch
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    torch.cuda.set_device(0)
    # 4 slots x (8192 + 1024 + 256 + 64) page-table entries, 4 x 4681 metadata entries
    levels = plan_levels((2048, 2048, 64), (32, 32, 32), 4, (2, 2, 2))
    man = VolumeManifest("fb", 4, (32, 32, 32), levels)
    e = Engine(man, EngineConfig(octree_depth=4, cache_slots=(2, 2, 2), channel_slots=4))
    return e


def _entry_to_id(p, e):
    pt = int(np.searchsorted(p.pt_offsets, e, side="right") - 1)
    lev = pt % p.config.k
    gx, gy, _ = (int(v) for v in p.level_grids[lev])
    local = e - int(p.pt_offsets[pt])
    x, y, z = local % gx, (local // gx) % gy, local // (gx * gy)
    return (pt << 24) | (z << 16) | (y << 8) | x


def _random_keys(rng, n_entries, n_touch, pix_bits, ev_bits, used):
    ent = rng.choice(n_entries, size=n_touch, replace=False)
    keys = set()
    out = []
    while len(out) < n_touch:
        k = (int(rng.integers(0, 1 << pix_bits)) << 32) | int(rng.integers(0, 1 << ev_bits))
        if k not in used and k not in keys:
            keys.add(k)
            out.append(k)
    used.update(keys)
    return ent, np.array(out, dtype=np.uint64)


CASES = [  # (bricks touched, metas touched, pixel bits, event bits, budget, bricks_first)
    (0, 0, 21, 10, 256, 1),
    (37, 5, 21, 10, 256, 1),          # everything survives
    (3000, 400, 21, 10, 256, 1),      # radix select, bricks fill the budget
    (200, 3000, 21, 10, 256, 1),      # metas get budget - bricks
    (3000, 3000, 21, 10, 512, 0),     # per-list budgets (sort-first parts)
    (20000, 9000, 23, 20, 20000, 1),  # > one sort chunk; 43-bit packed keys
    (30000, 9000, 23, 31, 12000, 0),  # 54-bit packed keys, chunked metas
    (5000, 100, 13, 0, 4096, 1),      # no event bits
    (9000, 0, 23, 31, 8192, 1),       # exactly one chunk, one left over
]


@pytest.mark.parametrize("nb,nm,pb,eb,budget,bf", CASES)
def test_gpu_feedback_orders_and_cuts_like_a_sort(eng, nb, nm, pb, eb, budget, bf):
    import torch
    from paper_2309_04393_b200 import _native as N
    p = eng.paging
    ctx = p.ctx
    E = p.total_entries
    n_nodes = ((1 << (3 * (eng.octree.config.depth + 1))) - 1) // 7
    n_meta = n_nodes * p.config.m
    rng = np.random.default_rng(nb * 7 + nm + budget)
    used = set()
    be, bk = _random_keys(rng, E, nb, pb, eb, used)
    me, mk = _random_keys(rng, n_meta, nm, pb, eb, used)
    dev = p.device
    bkeys = torch.full((E,), -1, dtype=torch.int64, device=dev)
    mkeys = torch.full((n_meta,), -1, dtype=torch.int64, device=dev)
    bkeys[torch.as_tensor(be, device=dev)] = torch.as_tensor(bk.view(np.int64), device=dev)
    mkeys[torch.as_tensor(me, device=dev)] = torch.as_tensor(mk.view(np.int64), device=dev)
    N.check(N.lib().ro_set_feedback_buffers(ctx, bkeys.data_ptr(), mkeys.data_ptr()))
    try:
        out = torch.zeros((4, max(budget, 1)), dtype=torch.int64, device=dev)
        counts = np.zeros(4, dtype=np.int64)
        cdev = torch.zeros(4, dtype=torch.int64, device=dev)
        fb = N.Feedback(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
                        out[3].data_ptr(), counts.ctypes.data, cdev.data_ptr())
        N.check(N.lib().ro_feedback_collect(ctx, budget, bf, C.byref(fb), N.stream_ptr()))
        got = out.cpu().numpy()
        # every key array is reset for the next frame
        assert bool((bkeys == -1).all()) and bool((mkeys == -1).all())
    finally:
        N.check(N.lib().ro_set_feedback_buffers(ctx, None, None))
    kb = min(nb, budget)
    km = min(nm, budget - kb if bf else budget)
    assert counts.tolist() == [nb, nm, kb, km]
    assert cdev.cpu().numpy().tolist() == [nb, nm, kb, km]
    ob = np.argsort(bk, kind="stable")[:kb]
    om = np.argsort(mk, kind="stable")[:km]
    assert got[0, :kb].view(np.uint64).tolist() == bk[ob].tolist()
    assert got[1, :kb].tolist() == [_entry_to_id(p, int(e)) for e in be[ob]]
    assert got[2, :km].view(np.uint64).tolist() == mk[om].tolist()
    assert got[3, :km].tolist() == me[om].tolist()


def test_gpu_feedback_async_form_needs_no_host_counts(eng):
    """counts == NULL: nothing waits; the device counts arrive on the stream."""
    import torch
    from paper_2309_04393_b200 import _native as N
    p = eng.paging
    dev = p.device
    E = p.total_entries
    bkeys = torch.full((E,), -1, dtype=torch.int64, device=dev)
    n_meta = (((1 << (3 * (eng.octree.config.depth + 1))) - 1) // 7) * p.config.m
    mkeys = torch.full((n_meta,), -1, dtype=torch.int64, device=dev)
    bkeys[5] = (3 << 32) | 1
    bkeys[9] = (2 << 32) | 7
    mkeys[4] = (2 << 32) | 3
    N.check(N.lib().ro_set_feedback_buffers(p.ctx, bkeys.data_ptr(), mkeys.data_ptr()))
    try:
        out = torch.zeros((4, 8), dtype=torch.int64, device=dev)
        cdev = torch.zeros(4, dtype=torch.int64, device=dev)
        fb = N.Feedback(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
                        out[3].data_ptr(), None, cdev.data_ptr())
        N.check(N.lib().ro_feedback_collect(p.ctx, 8, 1, C.byref(fb), N.stream_ptr()))
        torch.cuda.synchronize()
    finally:
        N.check(N.lib().ro_set_feedback_buffers(p.ctx, None, None))
    assert cdev.cpu().tolist() == [2, 1, 2, 1]
    o = out.cpu().numpy()
    assert o[0, :2].tolist() == [(2 << 32) | 7, (3 << 32) | 1]
    assert o[1, :2].tolist() == [_entry_to_id(p, 9), _entry_to_id(p, 5)]
    assert o[2, 0] == (2 << 32) | 3 and o[3, 0] == 4
