"""Residency-state API semantics restated from the reference's own unit tests
(pkg/tests/test_paging.py, test_octree.py, test_engine.py), run against the
mirror package whose state lives on the GPU.  Each test names the reference
test whose behaviour it pins."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def _paging(m=2, k=3, cache=(3, 3, 3)):
    from paper_2309_04393_b200 import MultiChannelPaging, PagingConfig
    cfg = PagingConfig(brick_size=(16, 16, 16), cache_slots=cache, m=m, k=k)
    dims = [(64, 64, 64), (32, 32, 32), (16, 16, 16)][:k]
    grids = [(4, 4, 4), (2, 2, 2), (1, 1, 1)][:k]
    return MultiChannelPaging(cfg, dims, grids)


def _octree(depth=3, m=2, k=3, cache=(3, 3, 3)):
    from paper_2309_04393_b200 import OctreeConfig, ResidencyOctree
    p = _paging(m, k, cache)
    return ResidencyOctree(OctreeConfig(depth=depth, channel_slots=m), p), p


def _brick(v=0):
    return np.full((16, 16, 16), v, dtype=np.uint8)


def _engine(depth=3, cache=(3, 3, 3), m=2):
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    man = VolumeManifest(name="t", channel_count=3, brick_size=(16, 16, 16),
                         levels=plan_levels((64, 64, 64), (16, 16, 16), 3, (2, 2, 2)))
    return Engine(man, EngineConfig(octree_depth=depth, cache_slots=cache, channel_slots=m))


# -- paging (test_paging.py) ---------------------------------------------------

def test_translate_unmapped_then_mapped():
    """test_paging.py:66-78"""
    from paper_2309_04393_b200 import MAPPED, UNMAPPED
    from paper_2309_04393_b200.paging import VirtualAddress
    p = _paging()
    a = VirtualAddress(level=0, channel_slot=0, position=(0.3, 0.6, 0.9))
    assert p.translate(a).status == UNMAPPED
    p.insert_brick(p.encode(0, 0, (1, 2, 3)), _brick(9), frame=1)
    t = p.translate(a)
    assert t.status == MAPPED
    for got, want in zip(t.local_coord, (0.3 * 64 - 16, 0.6 * 64 - 32, 0.9 * 64 - 48)):
        assert got == pytest.approx(want)


def test_brick_coord_of_partial_grid():
    """test_paging.py:81-87: a 48-voxel level in 32-voxel bricks."""
    from paper_2309_04393_b200 import MultiChannelPaging, PagingConfig
    p = MultiChannelPaging(PagingConfig(brick_size=(32, 32, 32), cache_slots=(2, 2, 2),
                                        m=1, k=1), [(48, 48, 48)], [(2, 2, 2)])
    assert p.brick_coord_of(0, (32 / 48, 0.0, 0.0)) == (1, 0, 0)
    assert p.brick_coord_of(0, (0.66, 0.0, 0.99)) == (0, 0, 1)


def test_sample_matches_weighted_taps():
    """test_paging.py:90-118: paging.sample == the 8-tap weighted sum, and a
    constant brick samples exactly."""
    p = _paging()
    rng = np.random.default_rng(4)
    data = rng.integers(0, 256, size=(16, 16, 16), dtype=np.uint8)
    slot, _ = p.insert_brick(p.encode(0, 0, (0, 0, 0)), data, frame=1)
    for _ in range(30):
        loc = tuple(float(v) for v in rng.uniform(0.5, 15.5, 3))
        f = [c - 0.5 for c in loc]
        i = [int(v) for v in f]
        t = [f[a] - i[a] for a in range(3)]
        want = sum(((t[0] if dx else 1 - t[0]) * (t[1] if dy else 1 - t[1]) *
                    (t[2] if dz else 1 - t[2])) *
                   float(data[min(i[2] + dz, 15), min(i[1] + dy, 15), min(i[0] + dx, 15)])
                   for dz in (0, 1) for dy in (0, 1) for dx in (0, 1))
        assert p.sample(slot, loc) == pytest.approx(want, abs=1e-9)
    s2, _ = p.insert_brick(p.encode(0, 0, (1, 0, 0)), _brick(137), frame=1)
    assert p.sample(s2, (0.1, 8.0, 15.9)) == 137.0


def test_reinsert_is_noop_and_mark_used_monotone():
    """test_paging.py:147-163"""
    from paper_2309_04393_b200 import PagingError
    p = _paging()
    b = p.encode(0, 0, (0, 0, 0))
    s1, ev1 = p.insert_brick(b, _brick(1), frame=1)
    s2, ev2 = p.insert_brick(b, _brick(2), frame=2)
    assert s1 == s2 and ev1 is None and ev2 is None
    assert p.occupied_slot_count() == 1
    p.mark_used(s1, 5)
    with pytest.raises(PagingError):
        p.mark_used(s1, 4)


def test_mark_empty_frees_slot_and_swap_frees_only_that_slot():
    """test_paging.py:166-190"""
    from paper_2309_04393_b200 import EMPTY
    from paper_2309_04393_b200.paging import VirtualAddress
    p = _paging()
    a, b = p.encode(0, 0, (0, 0, 0)), p.encode(1, 0, (0, 0, 0))
    p.insert_brick(a, _brick(1), frame=1)
    p.insert_brick(b, _brick(2), frame=1)
    p.mark_empty(a)
    assert p.resident_slot(a) is None and p.occupied_slot_count() == 1
    assert p.translate(VirtualAddress(level=0, channel_slot=0,
                                      position=(0.01, 0.01, 0.01))).status == EMPTY
    c = p.encode(0, 1, (0, 0, 0))
    p.insert_brick(c, _brick(3), frame=2)
    p.set_channel_mapping(0, 2)
    assert p.resident_slot(c) is None and p.resident_slot(b) is not None
    p.check_bijection()


def test_lru_victim_is_least_recent_then_lowest_slot():
    """test_paging.py:121-144 (LRU model): with the cache full, the victim is
    the occupied slot with the smallest (last_used, slot)."""
    p = _paging(cache=(2, 1, 1))
    a, b, c = (p.encode(0, 0, (x, 0, 0)) for x in range(3))
    p.insert_brick(a, _brick(), frame=1)
    p.insert_brick(b, _brick(), frame=2)
    _, ev = p.insert_brick(c, _brick(), frame=3)
    assert ev == a
    d = p.encode(0, 0, (3, 0, 0))
    p.mark_used(p.slot_triple(p.resident_slot(b)), 4)
    _, ev = p.insert_brick(d, _brick(), frame=4)
    assert ev == c


# -- octree (test_octree.py) ------------------------------------------------------

def test_insert_sets_bits_and_propagates():
    """test_octree.py:145-160: a level-1 brick marks exactly the low octant."""
    from paper_2309_04393_b200 import NodeAddress
    o, p = _octree()
    b = p.encode(0, 1, (0, 0, 0))
    p.insert_brick(b, _brick(), frame=1)
    o.on_brick_inserted(b)
    assert o.residency_mask(NodeAddress(0, 0, 0, 0), 0) == 0b10
    assert o.residency_mask(NodeAddress(0, 0, 0, 0), 1) == 0
    w = o.words
    for z in range(8):
        for y in range(8):
            for x in range(8):
                idx = NodeAddress(3, x, y, z).index
                assert (int(w[idx, 0]) & 0xFFFF) == (0b10 if max(x, y, z) < 4 else 0)
    o.check_mask_consistency()
    o.check_leaf_ground_truth()


def test_evict_clears_only_unbacked_leaves_and_keeps_other_levels():
    """test_octree.py:163-196"""
    from paper_2309_04393_b200 import NodeAddress
    o, p = _octree()
    a, b = p.encode(0, 0, (0, 0, 0)), p.encode(0, 0, (1, 0, 0))
    for bid in (a, b):
        p.insert_brick(bid, _brick(), frame=1)
        o.on_brick_inserted(bid)
    p.evict_bricks([a])
    o.on_brick_evicted(a)
    assert o.residency_mask(NodeAddress(3, 0, 0, 0), 0) == 0
    assert o.residency_mask(NodeAddress(3, 2, 0, 0), 0) == 0b01
    o2, p2 = _octree()
    lv1, lv0 = p2.encode(0, 1, (0, 0, 0)), p2.encode(0, 0, (0, 0, 0))
    for bid in (lv1, lv0):
        p2.insert_brick(bid, _brick(), frame=1)
        o2.on_brick_inserted(bid)
    leaf = NodeAddress(3, 1, 1, 1)
    assert o2.residency_mask(leaf, 0) == 0b11
    p2.evict_bricks([lv0])
    o2.on_brick_evicted(lv0)
    assert o2.residency_mask(leaf, 0) == 0b10
    o2.check_leaf_ground_truth()


def test_random_insert_evict_matches_full_scan():
    """test_octree.py:199-222"""
    o, p = _octree(depth=2, m=2, k=3, cache=(2, 2, 2))
    rng = np.random.default_rng(99)
    for step in range(300):
        slot, level = int(rng.integers(2)), int(rng.integers(3))
        grid = [int(v) for v in p.level_grids[level]]
        bid = p.encode(slot, level, tuple(int(rng.integers(g)) for g in grid))
        if rng.random() < 0.7:
            _, ev = p.insert_brick(bid, _brick(), frame=step)
            if ev is not None:
                o.on_brick_evicted(ev)
            o.on_brick_inserted(bid)
        elif p.resident_slot(bid) is not None:
            p.evict_bricks([bid])
            o.on_brick_evicted(bid)
        if step % 75 == 0:
            o.check_mask_consistency()
            o.check_leaf_ground_truth()
    o.check_mask_consistency()
    o.check_leaf_ground_truth()
    p.check_bijection()


def test_metadata_word_layout():
    """test_octree.py:225-240"""
    from paper_2309_04393_b200 import INVALID_WORD, NodeAddress, OctreeError
    o, _ = _octree()
    a = NodeAddress(2, 1, 2, 3)
    assert o.metadata(a, 0) is None
    assert int(o.words[a.index, 0]) == int(INVALID_WORD)
    o.set_node_metadata(a, 0, 17, 200)
    assert o.metadata(a, 0) == (17, 200)
    w = int(o.words[a.index, 0])
    assert (w >> 16) & 0xFF == 17 and (w >> 24) & 0xFF == 200
    o.words_dev[a.index, 0] |= 0b101        # residency bits and metadata are disjoint
    o.set_node_metadata(a, 0, 3, 9)
    assert o.residency_mask(a, 0) == 0b101
    with pytest.raises(OctreeError):
        o.set_node_metadata(a, 0, 10, 9)


# -- engine (test_engine.py) ---------------------------------------------------

def test_lru_eviction_updates_octree_and_note_sampled_protects():
    """test_engine.py:34-65"""
    eng = _engine(cache=(2, 1, 1))
    a, b, c = (eng.paging.encode(0, 0, (x, 0, 0)) for x in range(3))
    eng.apply_brick(a, _brick())
    eng.advance_frame()
    eng.apply_brick(b, _brick())
    eng.advance_frame()
    eng.apply_brick(c, _brick())          # a is least recently used
    assert eng.paging.resident_slot(a) is None
    eng.octree.check_mask_consistency()
    eng.octree.check_leaf_ground_truth()
    eng2 = _engine(cache=(2, 1, 1))
    eng2.apply_brick(a, _brick())
    eng2.advance_frame()
    eng2.apply_brick(b, _brick())
    mask = np.zeros(eng2.paging.total_entries, dtype=np.uint8)
    s, lev, coord = eng2.paging.decode(a)
    mask[eng2.paging._entry_index(s, lev, coord)] = 1
    eng2.advance_frame()
    eng2.note_sampled(mask)               # touching a makes b the victim
    eng2.apply_brick(c, _brick())
    assert eng2.paging.resident_slot(a) is not None
    assert eng2.paging.resident_slot(b) is None


def test_apply_metadata_swap_and_fill_preserve_residency_bits():
    """test_engine.py:68-95, 134-141"""
    import torch
    from paper_2309_04393_b200 import INVALID_WORD, NodeAddress
    eng = _engine(depth=2)
    addr = NodeAddress(2, 3, 1, 0)
    eng.apply_metadata(addr.index, 1, 4, 77)
    assert eng.octree.metadata(addr, 1) == (4, 77)
    b = eng.paging.encode(1, 0, (0, 0, 0))
    eng.apply_brick(b, _brick(5))
    root = NodeAddress(0, 0, 0, 0)
    assert eng.octree.residency_mask(root, 1) == 0b001
    eng.fill_metadata_from_volumes({1: torch.zeros((64, 64, 64), dtype=torch.uint8)})
    assert eng.octree.residency_mask(root, 1) == 0b001
    assert eng.octree.metadata(root, 1) == (0, 0)
    eng.swap_channel(1, 2)
    assert eng.paging.resident_slot(b) is None
    assert (eng.octree.words[:, 1] == INVALID_WORD).all()
    assert eng.paging.channel_mapping[1] == 2


def test_metadata_box_dilation_and_prefill_overflow():
    """test_engine.py:96-116, 144-160"""
    from paper_2309_04393_b200 import EngineError, NodeAddress
    eng = _engine(depth=2)
    pad = eng.metadata_pad
    assert pad == 6          # ceil(1.5 * 2^(k-1)) with k = 3
    lo, hi = eng.metadata_box(NodeAddress(2, 1, 0, 3))
    assert lo == (16 - pad, 0, 48 - pad) and hi == (32 + pad, 16 + pad, 64)
    small = _engine(cache=(2, 2, 2))
    with pytest.raises(EngineError):
        small.prefill(lambda s, lev, c: _brick(), slots=[0])


# -- engine metadata fill / prefill (test_engine.py:118-194) -------------------

def test_fill_metadata_equals_per_node_scan_and_keeps_masks():
    """test_engine.py:118-141: every node's (min, max) after the device fill
    equals the per-node local scan, other slots stay INVALID, and the fill
    leaves residency bits alone."""
    from paper_2309_04393_b200.octree import NodeAddress
    from paper_2309_04393_b200.volume import shell_volume
    eng = _engine(depth=2, cache=(5, 5, 5))
    bid = eng.paging.encode(0, 0, (0, 0, 0))
    eng.apply_brick(bid, _brick(3))
    mask = eng.octree.residency_mask(NodeAddress(2, 0, 0, 0), 0)
    assert mask != 0
    vol = shell_volume(64)
    eng.fill_metadata_from_volumes({0: vol})
    for d in range(3):
        s = 1 << d
        for z in range(s):
            for y in range(s):
                for x in range(s):
                    a = NodeAddress(d, x, y, z)
                    assert eng.octree.metadata(a, 0) == eng.compute_metadata_local(a, 0, vol)
    assert eng.octree.metadata(NodeAddress(0, 0, 0, 0), 1) is None
    assert eng.octree.residency_mask(NodeAddress(2, 0, 0, 0), 0) == mask


def test_prefill_all_levels_and_overflow():
    """test_engine.py:144-160: prefill makes 4^3 + 2^3 + 1 bricks resident;
    a cache too small for that raises."""
    from paper_2309_04393_b200 import EngineError
    eng = _engine(depth=2, cache=(5, 5, 5), m=1)
    eng.prefill(lambda slot, level, coord: _brick(level), slots=[0])
    assert eng.paging.occupied_slot_count() == 73
    for lev, g in [(0, 4), (1, 2), (2, 1)]:
        for z in range(g):
            assert eng.paging.resident_slot(eng.paging.encode(0, lev, (z, 0, 0))) is not None
    with pytest.raises(EngineError):
        _engine(depth=2, cache=(2, 2, 2), m=1).prefill(
            lambda slot, level, coord: _brick(level), slots=[0])


def test_metadata_bounds_samples_of_every_level():
    """test_engine.py:163-194: the dilated node (min, max) bounds the
    trilinear sample of every level's brick at random points."""
    from paper_2309_04393_b200.octree import NodeAddress
    from paper_2309_04393_b200.volume import build_pyramid, shell_volume
    eng = _engine(depth=2, cache=(6, 6, 6), m=1)
    vol = shell_volume(64)
    pyr = build_pyramid(vol, eng.manifest.levels)

    def fetch(slot, level, coord):
        x, y, z = coord
        out = np.zeros((16, 16, 16), np.uint8)
        part = pyr[level][z * 16:(z + 1) * 16, y * 16:(y + 1) * 16, x * 16:(x + 1) * 16]
        out[:part.shape[0], :part.shape[1], :part.shape[2]] = part
        return out

    eng.prefill(fetch, slots=[0])
    eng.fill_metadata_from_volumes({0: vol})
    rng = np.random.default_rng(7)
    for _ in range(200):
        p = rng.uniform(0.0, 1.0, 3)
        mn, mx = eng.octree.metadata(NodeAddress(2, *(min(int(v * 4), 3) for v in p)), 0)
        for lev in range(3):
            coord = eng.paging.brick_coord_of(lev, tuple(p))
            lin = eng.paging.resident_slot(eng.paging.encode(0, lev, coord))
            dims = eng.paging.level_dims[lev]
            local = tuple(float(p[a] * dims[a] - coord[a] * 16) for a in range(3))
            v = eng.paging.sample(eng.paging.slot_triple(lin), local)
            assert mn - 1e-9 <= v <= mx + 1e-9, (p, lev, v, mn, mx)


def test_pinned_payloads_upload_like_pageable():
    """ro_apply_bricks with payloads in page-locked memory (direct DMA from
    the caller's buffer) leaves the same cache / page table / LRU / octree
    as the pageable staging path, batch after batch with evictions, and the
    recycled PinnedBrickBuffer can be refilled right after each call."""
    import torch
    from paper_2309_04393_b200.paging import PinnedBrickBuffer
    a, b = _engine(cache=(2, 2, 2)), _engine(cache=(2, 2, 2))
    pinned = PinnedBrickBuffer((16, 16, 16))
    rng = np.random.default_rng(3)
    for frame in range(1, 7):
        a.advance_frame(), b.advance_frame()
        ids, seen = [], set()
        while len(ids) < 5:
            slot, level = int(rng.integers(2)), int(rng.integers(3))
            grid = [int(v) for v in a.paging.level_grids[level]]
            bid = a.paging.encode(slot, level, tuple(int(rng.integers(g)) for g in grid))
            if bid not in seen:
                seen.add(bid)
                ids.append(bid)
        pays = [rng.integers(0, 256, (16, 16, 16), dtype=np.uint8) for _ in ids]
        a.apply_bricks(ids, np.stack(pays))
        view = pinned.stack(pays)
        assert isinstance(view, torch.Tensor) and view.is_pinned()
        b.apply_bricks(ids, view)
        torch.cuda.synchronize()
        for name in ("pt_status", "pt_slot", "slot_brick", "slot_last_used", "cache"):
            assert np.array_equal(getattr(a.paging, name), getattr(b.paging, name)), name
        assert np.array_equal(a.octree.words, b.octree.words)


@pytest.mark.gpu
def test_gpu_chunked_upload_paths_agree():
    """apply_bricks batches larger than one upload chunk (256 bricks): the
    page-locked and pageable host paths DMA in chunks and copy each chunk
    into the cache (fused with its sub-block maxima) as it lands, with the
    octree update under the transfer; the device-payload path does it in one
    pass.  All three end in the same page table, LRU arrays, cache, octree
    words and sub-block maxima, every resident brick holds its payload, and
    a frame rendered from each is identical."""
    import torch
    from paper_2309_04393_b200 import (ChannelSettings, Engine, EngineConfig, RenderConfig,
                                       grayscale_ramp_tf, orbit_pose, render_frame)
    from paper_2309_04393_b200.paging import PinnedBrickBuffer
    from gpu_helpers import device_state_hashes, diff_hashes
    import scenes
    st = scenes.store("sparse256x4")
    rng = np.random.default_rng(5)
    ids, pays = [], []
    probe = Engine(st.manifest, EngineConfig(octree_depth=4, cache_slots=(12, 12, 12),
                                             channel_slots=4))
    for s in range(4):
        for lev in range(len(st.manifest.levels)):
            gx, gy, gz = st.manifest.levels[lev].brick_grid_dims
            for z in range(gz):
                for y in range(gy):
                    for x in range(gx):
                        ids.append(probe.paging.encode(s, lev, (x, y, z)))
                        pays.append((s, lev, (x, y, z)))
    order = rng.permutation(len(ids))
    ids = [ids[i] for i in order]
    payload = np.stack([st.brick(s, lev, c) for s, lev, c in (pays[i] for i in order)])
    batches = [(0, 1500), (1500, 2300)]   # the second batch evicts
    engines = []
    for kind in ("pinned", "pageable", "device"):
        eng = Engine(st.manifest, EngineConfig(octree_depth=4, cache_slots=(12, 12, 12),
                                               channel_slots=4))
        eng.fill_metadata_from_volumes({s: st.level_array(s, 0) for s in range(4)})
        buf = PinnedBrickBuffer((32, 32, 32))
        for a, b in batches:
            eng.advance_frame()
            chunk = payload[a:b]
            if kind == "pinned":
                arg = buf.stack(list(chunk))
            elif kind == "pageable":
                arg = chunk
            else:
                arg = torch.from_numpy(chunk).cuda()
            slots, _ = eng.apply_bricks(ids[a:b], arg, return_slots=True)
        torch.cuda.synchronize()
        engines.append((kind, eng, slots))
    ref = device_state_hashes(engines[2][1])
    ref_sub = engines[2][1].paging.sub_max.cpu().numpy()
    for kind, eng, _ in engines[:2]:
        assert not diff_hashes(device_state_hashes(eng), ref), kind
        assert np.array_equal(eng.paging.sub_max.cpu().numpy(), ref_sub), kind
    kind, eng, slots = engines[0]
    cache = eng.paging.cache_dev.reshape(eng.paging.num_slots, 32, 32, 32)
    a, b = batches[-1]
    for j in rng.choice(b - a, 40, replace=False):
        assert np.array_equal(cache[int(slots[j])].cpu().numpy(), payload[a + j])
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(40.0)) for s in range(4)]
    cfg = RenderConfig(image_dims=(64, 48), base_step=1 / 128, max_requests_per_frame=256)
    imgs = [render_frame(e.paging, e.octree, chans, orbit_pose(0.7), cfg).image
            for _, e, _ in engines]
    assert np.array_equal(imgs[0], imgs[2]) and np.array_equal(imgs[1], imgs[2])
