"""CUDA path vs the reference's golden outputs and the CPU oracle.

Bar: request lists (ordered), usage mask, octree words,
page tables, slot arrays, counters and histograms bit-exact; images
bit-exact too (the kernel replays the reference's fp64 operation order,
-fmad=false).  IMAGE_ATOL is the north-star bound (1/255) used only by the
full-size property tests where the oracle is not run on every pixel.
"""

import math

import numpy as np
import pytest

from conftest import cuda_ok, load_golden
import scenes
from gpu_helpers import (cam_tuple, device_state_hashes, diff_hashes,
                         oracle_state_from_device)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

IMAGE_ATOL = 1.0 / 255.0


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib, oracle_lib):
    return native_lib


def _check(rec, prefix, out):
    return scenes.check_frame(rec, prefix, out.image, out.brick_requests,
                              out.metadata_requests, out.required_mask,
                              out.level_histogram, out.pixel_required,
                              [out.stats.traversal_steps, out.stats.samples_evaluated,
                               out.stats.samples_skipped, out.stats.skip_violations])


def test_gpu_session_mc64_matches_reference():
    from paper_2309_04393_b200 import EngineConfig, LocalTransport, Session
    meta, rec = load_golden("session_mc64")
    e = meta["engine"]
    sess = Session(LocalTransport(scenes.store("mc64")),
                   EngineConfig(octree_depth=e["depth"], cache_slots=tuple(e["cache_slots"]),
                                channel_slots=e["m"]),
                   scenes.render_config(meta["render"]),
                   scenes.product_channels(meta["channels"]))
    from paper_2309_04393_b200 import Camera
    for item in meta["script"]:
        if "swap" in item:
            for slot, ch in item["swap"]:
                sess.swap_channel(slot, ch)
            assert not diff_hashes(device_state_hashes(sess.engine), item["after_swap"])
            continue
        i = item["frame"]
        pos, tgt, up, fov = item["pose"]
        r = sess.step_frame(Camera(position=tuple(pos), target=tuple(tgt), up=tuple(up),
                                   fov_deg=fov))
        bad = _check(rec, f"f{i}_", r.output)
        assert not bad, (i, bad)
        assert r.bricks_applied == item["bricks_applied"]
        assert r.metadata_applied == item["metadata_applied"]
        d = diff_hashes(device_state_hashes(sess.engine), item["after"])
        assert not d, (i, d)
    sess.close()


def _prepared_engine(kind, m=1, depth=5, slots_to_channels=None):
    from paper_2309_04393_b200 import Engine, EngineConfig
    st = scenes.store(kind)
    slots_to_channels = slots_to_channels or {0: 0}
    eng = Engine(st.manifest, EngineConfig(octree_depth=depth,
                                           cache_slots=scenes.full_cache_slots(st, m),
                                           channel_slots=m))
    for s, c in slots_to_channels.items():
        eng.paging.channel_mapping[s] = c
    eng.prefill(lambda s, lev, c: st.brick(slots_to_channels[s], lev, c),
                slots=sorted(slots_to_channels))
    eng.fill_metadata_from_volumes({s: st.level_array(c, 0)
                                    for s, c in slots_to_channels.items()})
    return eng


def test_gpu_vessel256_matches_reference():
    """Config 1 (test_acceptance.py:44-123): fully resident vessel 256^3,
    residency == reference mode == reference outputs, five poses."""
    from paper_2309_04393_b200 import orbit_pose, render_frame, render_reference
    meta, rec = load_golden("vessel256_full")
    eng = _prepared_engine("vessel256", depth=meta["engine"]["depth"])
    assert not diff_hashes(device_state_hashes(eng), meta["state"])
    chans = scenes.product_channels(meta["channels"])
    cfg = scenes.render_config(meta["render"])
    for i, a in enumerate(meta["angles"]):
        pose = orbit_pose(a)
        out = render_frame(eng.paging, eng.octree, chans, pose, cfg)
        assert not _check(rec, f"res{i}_", out), i
        ref = render_reference(eng.paging, chans, pose, cfg)
        assert not _check(rec, f"ref{i}_", ref), i
        assert np.array_equal(out.image, ref.image)


def test_gpu_skip_audit_matches_reference():
    from paper_2309_04393_b200 import (EngineConfig, LocalTransport, Session,
                                       orbit_pose, render_frame)
    meta, rec = load_golden("skip_audit_shell64")
    e = meta["engine"]
    ref_eng = _prepared_engine("shell64", depth=e["depth"])
    assert not diff_hashes(device_state_hashes(ref_eng), meta["ref_state"])
    cfg = scenes.render_config(meta["render"])
    poses = [orbit_pose(a) for a in meta["poses"]]
    for r, run in enumerate(meta["runs"]):
        chans = scenes.product_channels([{"slot": 0, "tf": run["tf"], "level_range": [0, 15]}])
        sess = Session(LocalTransport(scenes.store("shell64")),
                       EngineConfig(octree_depth=e["depth"],
                                    cache_slots=tuple(e["cache_slots"]), channel_slots=1),
                       cfg, chans)
        recs = sess.run_until_converged(poses[0], max_frames=50)
        assert sess.converged and len(recs) == run["frames"]
        assert not diff_hashes(device_state_hashes(sess.engine), run["state"])
        for j, pose in enumerate(poses):
            out = render_frame(sess.engine.paging, sess.engine.octree, chans, pose, cfg,
                               reference_paging=ref_eng.paging)
            assert not _check(rec, f"r{r}p{j}_", out), (r, j)
            assert out.stats.skip_violations == 0
        sess.close()


def test_gpu_lru_replay_matches_reference():
    """Op-by-op replay of the reference's randomised residency workload."""
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    meta, _ = load_golden("lru_replay")
    levels = plan_levels(tuple(meta["dims"]), tuple(meta["brick"]), meta["levels"], (2, 2, 2))
    man = VolumeManifest(name="t", channel_count=3, brick_size=tuple(meta["brick"]),
                         levels=levels)
    eng = Engine(man, EngineConfig(octree_depth=meta["depth"],
                                   cache_slots=tuple(meta["cache_slots"]),
                                   channel_slots=meta["m"]))
    sx, sy, sz = meta["brick"]
    E = eng.paging.total_entries
    for op in meta["ops"]:
        kind = op[0]
        if kind == "insert":
            payload = np.full((1, sz, sy, sx), op[2], dtype=np.uint8)
            _, ev = eng.apply_bricks([op[1]], payload, return_slots=True)
            assert int(ev[0]) == op[3]
        elif kind == "evict":
            eng.evict_bricks([op[1]])
        elif kind == "advance_note":
            eng.advance_frame()
            mask = np.zeros(E, dtype=np.uint8)
            mask[op[1]] = 1
            eng.note_sampled(mask)
        elif kind == "meta":
            eng.apply_metadata(op[1], op[2], op[3], op[4])
        elif kind == "swap":
            eng.swap_channel(op[1], op[2])
        elif kind == "check":
            d = diff_hashes(device_state_hashes(eng), op[1])
            assert not d, d
    eng.paging.check_bijection()
    eng.octree.check_mask_consistency()
    eng.octree.check_leaf_ground_truth()


@pytest.mark.parametrize("seed", list(range(int(__import__("os").environ.get("RESOCT_LRU_N",
                                                                             "3")))))
def test_gpu_batched_lru_equals_sequential(seed):
    """Whole-frame batches (free-list pops, stale victims in (last_used, slot)
    order, slot-0 thrash once every slot is stamped this frame) equal the
    reference's one-by-one insert_brick + octree updates."""
    from oracle.session import state_hashes
    from oracle.state import OracleResidency
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    rng = np.random.default_rng(seed)
    levels = plan_levels((64, 40, 48), (8, 8, 8), 3, (2, 2, 2))
    man = VolumeManifest(name="t", channel_count=2, brick_size=(8, 8, 8), levels=levels)
    cache = (5, 3, 2)
    eng = Engine(man, EngineConfig(octree_depth=4, cache_slots=cache, channel_slots=2))
    ora = OracleResidency(2, 3, (8, 8, 8), [l.dims for l in levels],
                          [l.brick_grid_dims for l in levels], cache, 4)
    E = eng.paging.total_entries
    for step in range(40):
        eng.advance_frame()
        mask = (rng.random(E) < 0.3).astype(np.uint8)
        eng.note_sampled(mask)
        ora.note_sampled(mask, eng.frame)
        # a batch of unique, currently unmapped bricks (size up to 2x cache)
        unm = np.flatnonzero(ora.pt_status == 0)
        nb = int(rng.integers(1, min(len(unm), 60) + 1))
        entries = rng.choice(unm, size=nb, replace=False)
        ids = []
        for e in entries:
            pt = int(np.searchsorted(ora.pt_offsets, e, side="right") - 1)
            slot, lev = pt // 3, pt % 3
            g = ora.level_grids[lev]
            loc = int(e - ora.pt_offsets[pt])
            x, y, z = loc % g[0], (loc // g[0]) % g[1], loc // (g[0] * g[1])
            ids.append(((slot * 3 + lev) << 24) | (int(z) << 16) | (int(y) << 8) | int(x))
        pay = rng.integers(0, 256, size=(nb, 8, 8, 8), dtype=np.uint8)
        slots, evicted = eng.apply_bricks(ids, pay, return_slots=True)
        for i, b in enumerate(ids):
            lin, ev = ora.apply_brick(b, pay[i], eng.frame)
            assert int(slots[i]) == lin and int(evicted[i]) == (-1 if ev is None else ev)
        if step % 7 == 3:
            s = int(rng.integers(2))
            eng.swap_channel(s, int(rng.integers(2)))
            ora.swap_channel(s)
        d = diff_hashes(device_state_hashes(eng), state_hashes(ora))
        assert not d, (step, d)


def _random_partial_engine(seed, eps=0.0, depth=3, m=4, cache=(6, 6, 6)):
    """mc64 channels with a random resident subset and random INVALID /
    valid metadata: exercises MISSU, MISSP, substitution, meta requests."""
    from paper_2309_04393_b200 import Engine, EngineConfig
    st = scenes.store("mc64")
    rng = np.random.default_rng(seed)
    eng = Engine(st.manifest, EngineConfig(octree_depth=depth, cache_slots=cache,
                                           channel_slots=m, homogeneity_eps=eps))
    k = len(st.manifest.levels)
    ids, pays = [], []
    for s in range(m):
        for lev in range(k):
            gx, gy, gz = st.manifest.levels[lev].brick_grid_dims
            for z in range(gz):
                for y in range(gy):
                    for x in range(gx):
                        if rng.random() < 0.45:
                            ids.append(eng.paging.encode(s, lev, (x, y, z)))
                            pays.append(st.brick(s % 4, lev, (x, y, z)))
    order = rng.permutation(len(ids))
    ids = [ids[i] for i in order][:eng.paging.num_slots]
    pays = np.stack([pays[i] for i in order][:eng.paging.num_slots])
    eng.apply_bricks(ids, pays)
    eng.fill_metadata_from_volumes({s: st.level_array(s % 4, 0) for s in range(m)})
    # knock out metadata at random nodes -> INVALID words
    words = eng.octree.words.copy()
    kill = rng.random(words.shape) < 0.25
    words[kill] = (words[kill] & np.uint32(0xFFFF)) | np.uint32(0x00FF0000)
    eng.octree.upload_words(words)
    return eng


@pytest.mark.parametrize("seed,eps,ranges", [
    (0, 0.0, [(0, 2), (0, 2), (0, 2), (0, 2)]),
    (1, 0.0, [(0, 0), (1, 2), (2, 2), (0, 1)]),
    (2, 12.0, [(0, 2), (1, 1), (0, 2), (2, 2)]),
    (3, 3.0, [(1, 2), (0, 2), (0, 0), (0, 2)]),
])
def test_gpu_partial_residency_matches_oracle(seed, eps, ranges):
    from oracle import raycast as orc
    from paper_2309_04393_b200 import (ChannelSettings, RenderConfig, TransferFunction,
                                       grayscale_ramp_tf, orbit_pose, render_frame,
                                       render_reference)
    eng = _random_partial_engine(seed, eps=eps)
    tfs = [grayscale_ramp_tf(40.0),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (20.0, (0.1, 0.9, 0.2, 0.0)),
                                    (90.0, (1.0, 0.2, 0.1, 0.5)), (255.0, (0.2, 0.4, 1.0, 0.8)))),
           grayscale_ramp_tf(10.0, max_alpha=0.4),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (100.0, (1, 1, 0, 0.9)),
                                    (101.0, (0, 0, 0, 0)), (255.0, (0, 0, 0, 0))))]
    order = [2, 0, 3, 1] if seed % 2 else [0, 1, 2, 3]
    chans = [ChannelSettings(slot=s, tf=tfs[s], level_range=ranges[s]) for s in order]
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    for angle, dims, step, budget in ((0.4, (61, 37), 1 / 64, 40), (2.9, (32, 48), 1 / 100, 7),
                                      (4.6, (50, 50), 1 / 40, 300)):
        cfg = RenderConfig(image_dims=dims, base_step=step, max_requests_per_frame=budget)
        pose = orbit_pose(angle, radius=1.7)
        out = render_frame(eng.paging, eng.octree, chans, pose, cfg)
        want = orc.render(ost, och, cam_tuple(pose), dims, step, budget=budget)
        assert np.array_equal(out.image, want.image), (
            int((out.image != want.image).sum()), float(np.abs(out.image - want.image).max()))
        assert out.brick_requests == want.brick_requests
        assert out.metadata_requests == want.metadata_requests
        assert np.array_equal(out.required_mask, want.required_mask)
        assert np.array_equal(out.level_histogram, want.level_histogram)
        assert np.array_equal(out.pixel_required, want.pixel_required)
        assert [out.stats.traversal_steps, out.stats.samples_evaluated,
                out.stats.samples_skipped] == list(want.counters[:3])
        ref = render_reference(eng.paging, chans, pose, cfg)
        wr = orc.render(ost, och, cam_tuple(pose), dims, step, budget=budget,
                        mode=orc.MODE_REFERENCE)
        assert np.array_equal(ref.image, wr.image)
        assert np.array_equal(ref.required_mask, wr.required_mask)
        assert np.array_equal(ref.level_histogram, wr.level_histogram)


@pytest.mark.parametrize("depth,m", [(7, 4), (8, 1), (5, 6), (4, 8)])
def test_gpu_path_class_layouts_match_oracle(depth, m):
    """The residency walk's per-frame node classes in every layout the ray
    caster switches between: D <= 7 with <= 4 channels (plain + ZERO bits
    per path), D <= 7 with 5..8 channels (plain bits only), D = 8 (no path
    classes: fast flag + channel-0 parallel descent).  Random residency and
    INVALID metadata; image, requests, usage, histogram and counters equal
    the oracle's."""
    from oracle import raycast as orc
    from paper_2309_04393_b200 import (ChannelSettings, RenderConfig, TransferFunction,
                                       grayscale_ramp_tf, orbit_pose, render_frame)
    eng = _random_partial_engine(20 + depth, depth=depth, m=m)
    tfs = [grayscale_ramp_tf(40.0),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (20.0, (0.1, 0.9, 0.2, 0.0)),
                                    (90.0, (1.0, 0.2, 0.1, 0.5)), (255.0, (0.2, 0.4, 1.0, 0.8)))),
           grayscale_ramp_tf(10.0, max_alpha=0.4),
           TransferFunction(points=((0.0, (0, 0, 0, 0)), (100.0, (1, 1, 0, 0.9)),
                                    (101.0, (0, 0, 0, 0)), (255.0, (0, 0, 0, 0))))]
    chans = [ChannelSettings(slot=s, tf=tfs[s % 4], level_range=(s % 2, 2)) for s in range(m)]
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    for angle, dims, step, budget in ((0.4, (48, 40), 1 / 80, 60), (3.3, (40, 32), 1 / 200, 500)):
        cfg = RenderConfig(image_dims=dims, base_step=step, max_requests_per_frame=budget,
                           traversal_start_level=min(depth, 2))
        pose = orbit_pose(angle, radius=1.7)
        out = render_frame(eng.paging, eng.octree, chans, pose, cfg)
        want = orc.render(ost, och, cam_tuple(pose), dims, step, budget=budget,
                          start_level=cfg.traversal_start_level)
        assert np.array_equal(out.image, want.image), int((out.image != want.image).sum())
        assert out.brick_requests == want.brick_requests
        assert out.metadata_requests == want.metadata_requests
        assert np.array_equal(out.required_mask, want.required_mask)
        assert np.array_equal(out.level_histogram, want.level_histogram)
        assert [out.stats.traversal_steps, out.stats.samples_evaluated,
                out.stats.samples_skipped] == list(want.counters[:3])


def test_gpu_wide_request_keys_match_oracle():
    """Request keys wider than 32 bits end to end: a 4096x2048 frame (pixel
    index >= 2^22) whose rows 1024..1031 are rendered (sort-first part 128
    of 256), every node's metadata INVALID so every node visit is a request
    event (> 2^9 events per pixel with a 1/1024 step) -- packed keys of
    > 32 bits through the ray caster's RED.MIN and the feedback kernel's
    select / sort.  Ordered lists, usage, histogram and image equal the
    oracle's for the same rows."""
    import os
    from oracle import raycast as orc
    from paper_2309_04393_b200 import ChannelSettings, RenderConfig, grayscale_ramp_tf, orbit_pose
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
    eng = _random_partial_engine(11, depth=4)
    words = eng.octree.words.copy()
    words[:] = (words & np.uint32(0xFFFF)) | np.uint32(0x00FF0000)   # all INVALID
    eng.octree.upload_words(words)
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(180.0, max_alpha=0.05),
                             level_range=(0, 2)) for s in (0, 1, 2, 3)]
    w, h = 4096, 2048
    budget = 40000
    cfg = RenderConfig(image_dims=(w, h), base_step=1 / 1024, max_requests_per_frame=budget)
    pose = orbit_pose(0.8, radius=1.7)
    fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, chans, pose, cfg,
                   partition=(h // 8, 128, 8), bricks_first=True)
    fp.render()
    fp.collect()
    b = fp.buf
    nb, nm = b.n_bricks, b.n_metas
    fb = b.fb.cpu().numpy()
    m = eng.paging.config.m
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    want = orc.render(ost, och, cam_tuple(pose), (w, h), cfg.base_step, budget=budget,
                      rows=(1024, 1032), threads=os.cpu_count() or 1)
    assert [divmod(int(v), m) for v in fb[3][:nm]] == want.metadata_requests
    assert fb[1][:nb].tolist() == want.brick_requests
    assert np.array_equal(b.image.cpu().numpy().reshape(8, w, 4), want.image[1024:1032])
    assert np.array_equal(b.required.cpu().numpy(), want.required_mask)
    assert np.array_equal(b.hist.cpu().numpy(), want.level_histogram)
    # the keys really were wide: pixel >= 2^22 and events >= 2^9 in one key set
    keys = fb[2][:nm].astype(np.uint64)
    assert nm > 100
    assert int((keys >> np.uint64(32)).max()) >= (1 << 22)
    assert int((keys & np.uint64(0xFFFFFFFF)).max()) >= (1 << 9)


@pytest.mark.parametrize("n_parts", [2, 3, 5])
def test_gpu_sort_first_parts_merge_to_full_frame(n_parts):
    """Sort-first partition (row blocks round-robin over parts): per-part
    images, usage masks, counters and (key, id) request lists merge into the
    single-GPU frame exactly -- the multi-GPU parity mode of SURVEY §8(e)."""
    import torch
    from paper_2309_04393_b200 import (ChannelSettings, RenderConfig, grayscale_ramp_tf,
                                       orbit_pose, render_frame)
    from paper_2309_04393_b200.distributed import merge_parts, part_rows
    from paper_2309_04393_b200.render import MODE_RESIDENCY, render_frame_device
    eng = _random_partial_engine(7)
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(30.0)) for s in range(4)]
    cfg = RenderConfig(image_dims=(45, 70), base_step=1 / 64, max_requests_per_frame=50)
    pose = orbit_pose(1.3, radius=1.8)
    full = render_frame(eng.paging, eng.octree, chans, pose, cfg)
    parts = []
    for p in range(n_parts):
        buf = render_frame_device(MODE_RESIDENCY, eng.paging, eng.octree, chans, pose, cfg,
                                  partition=(n_parts, p, 8), bricks_first=False)
        parts.append({k: v.clone() if isinstance(v, torch.Tensor) else v
                      for k, v in dict(image=buf.image, required=buf.required,
                                       pix_required=buf.pix_required, hist=buf.hist,
                                       counters=buf.counters, fb=buf.fb,
                                       counts=buf.counts.copy()).items()})
    merged = merge_parts(parts, cfg.image_dims, n_parts, 8, cfg.max_requests_per_frame,
                         eng.paging.config.m)
    assert np.array_equal(merged["image"], full.image)
    assert merged["bricks"] == full.brick_requests
    assert merged["metas"] == full.metadata_requests
    assert np.array_equal(merged["required"], full.required_mask)
    assert np.array_equal(merged["hist"], full.level_histogram)
    assert np.array_equal(merged["pix_required"], full.pixel_required)
    assert merged["counters"][0] == full.stats.traversal_steps
    rows = sum(len(part_rows(cfg.image_dims[1], n_parts, p, 8)) for p in range(n_parts))
    assert rows == cfg.image_dims[1]
    # the device form of the same merge (distributed.exchange with a GPU
    # replica): ro_feedback_merge + ro_feedback_collect, ro_gather_rows
    import ctypes as C
    from paper_2309_04393_b200 import _native as N
    budget = cfg.max_requests_per_frame
    blocks = torch.stack([p["fb"] for p in parts]).contiguous()
    counts = torch.as_tensor(np.stack([p["counts"] for p in parts]), device=blocks.device)
    out = torch.zeros((4, budget), dtype=torch.int64, device=blocks.device)
    cdev = torch.zeros(4, dtype=torch.int64, device=blocks.device)
    N.check(N.lib().ro_feedback_merge(eng.paging.ctx, blocks.data_ptr(), counts.data_ptr(),
                                      n_parts, budget, N.stream_ptr()))
    fb = N.Feedback(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), out[3].data_ptr(),
                    None, cdev.data_ptr())
    N.check(N.lib().ro_feedback_collect(eng.paging.ctx, budget, 1, C.byref(fb), N.stream_ptr()))
    c = cdev.cpu().numpy()
    o = out.cpu().numpy()
    m = eng.paging.config.m
    assert o[1][:c[2]].tolist() == full.brick_requests
    assert [divmod(int(v), m) for v in o[3][:c[3]]] == full.metadata_requests
    w, h = cfg.image_dims
    max_rows = max(len(part_rows(h, n_parts, p, 8)) for p in range(n_parts))
    stacked = torch.zeros((n_parts, max_rows * w, 4), dtype=torch.float32, device=blocks.device)
    for i, p in enumerate(parts):
        stacked[i, :p["image"].shape[0]] = p["image"]
    img = torch.empty((h, w, 4), dtype=torch.float32, device=blocks.device)
    N.check(N.lib().ro_gather_rows(stacked.data_ptr(), n_parts, max_rows * w * 4, h, w, 8,
                                   img.data_ptr(), N.stream_ptr()))
    assert np.array_equal(img.cpu().numpy(), full.image)


def test_gpu_edge_cases():
    """1x1 image, a camera looking away from the volume (every ray misses),
    single channel k=1 depth 0, budget 1, eight channel slots."""
    from oracle import raycast as orc
    from paper_2309_04393_b200 import (Camera, ChannelSettings, Engine, EngineConfig,
                                       RenderConfig, grayscale_ramp_tf, orbit_pose,
                                       render_frame)
    from paper_2309_04393_b200 import volume as V
    st = V.VolumeStore([V.ramp_volume(32)] * 8, (16, 16, 16), 1, (2, 2, 2), normalize=False)
    eng = Engine(st.manifest, EngineConfig(octree_depth=0, cache_slots=(4, 4, 4),
                                           channel_slots=8))
    eng.prefill(lambda s, lev, c: st.brick(s, lev, c))
    eng.fill_metadata_from_volumes({s: st.level_array(s, 0) for s in range(8)})
    chans = [ChannelSettings(slot=s, tf=grayscale_ramp_tf(20.0 * s, max_alpha=0.1))
             for s in range(8)]
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    for cam, dims, budget in ((orbit_pose(0.3), (1, 1), 1),
                              (Camera(position=(3.0, 3.0, 3.0), target=(6.0, 6.0, 6.0)),
                               (9, 7), 1),
                              (orbit_pose(2.2, radius=1.3), (23, 19), 1)):
        cfg = RenderConfig(image_dims=dims, base_step=1 / 50, max_requests_per_frame=budget)
        out = render_frame(eng.paging, eng.octree, chans, cam, cfg)
        want = orc.render(ost, och, cam_tuple(cam), dims, 1 / 50, budget=budget)
        assert np.array_equal(out.image, want.image)
        assert out.brick_requests == want.brick_requests
        assert out.metadata_requests == want.metadata_requests
        assert np.array_equal(out.level_histogram, want.level_histogram)


def test_gpu_octree_incremental_equals_rebuild():
    """Incremental octree pass after many batches == masks recomputed from
    the resident set (leaf ground truth + OR closure)."""
    eng = _random_partial_engine(11, depth=4, cache=(4, 4, 4))
    before = eng.octree.words.copy()
    eng.octree.rebuild_masks()
    assert np.array_equal(before, eng.octree.words)
    eng.octree.check_mask_consistency()
    eng.octree.check_leaf_ground_truth()


def test_gpu_cycif_small_scenario_matches_oracle():
    """The bench scenario builder at reduced size: engine state built through
    apply_bricks / write_level_metadata equals the numpy reference-layout
    state, and a partial-residency multi-channel frame equals the oracle."""
    import torch
    from oracle import raycast as orc
    from paper_2309_04393_b200 import render_frame, scenarios
    scn = scenarios.cycif(device="cuda", dims=(256, 256, 32), n_cells=400,
                          image_dims=(96, 54), depth=4)
    eng = scenarios.build_engine(scn)
    ref = orc.OracleState(**scenarios.reference_state(scn))
    assert np.array_equal(eng.octree.words, ref.words)
    assert np.array_equal(eng.paging.pt_status, ref.pt_status)
    assert np.array_equal(eng.paging.pt_slot, ref.pt_slot)
    out = render_frame(eng.paging, eng.octree, scn.channels, scn.camera, scn.render)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in scn.channels]
    want = orc.render(ref, och, cam_tuple(scn.camera), scn.render.image_dims,
                      scn.render.base_step, budget=scn.render.max_requests_per_frame)
    assert np.array_equal(out.image, want.image)
    assert out.brick_requests == want.brick_requests
    assert out.metadata_requests == want.metadata_requests
    assert np.array_equal(out.required_mask, want.required_mask)
    assert np.array_equal(out.level_histogram, want.level_histogram)
    torch.cuda.synchronize()


def test_gpu_config3_mixed_bias_swap_session_matches_oracle():
    """Config 3 (scaled): 8-channel sparse volume, m = 4 slots with mixed
    level ranges, cold session with budget pressure, a mid-sequence swap of
    all four slots to the other four channels, run on; every frame's image,
    ordered requests, usage mask and the full state equal the oracle."""
    from oracle.session import OracleSession, state_hashes
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       RenderConfig, Session, grayscale_ramp_tf, orbit_pose)
    from paper_2309_04393_b200 import volume as V
    from oracle import raycast as orc
    store = V.VolumeStore(V.sparse_multichannel(64, channels=8), (16, 16, 16), 3, (2, 2, 2))
    ranges = [(0, 2), (1, 2), (2, 2), (0, 1)]
    tfs = [grayscale_ramp_tf(40.0), grayscale_ramp_tf(30.0, 0.6),
           grayscale_ramp_tf(50.0), grayscale_ramp_tf(20.0, 0.8)]
    chans = [ChannelSettings(slot=s, tf=tfs[s], level_range=ranges[s]) for s in range(4)]
    rconf = RenderConfig(image_dims=(56, 48), base_step=1 / 64, max_requests_per_frame=40)
    econf = EngineConfig(octree_depth=3, cache_slots=(5, 5, 4), channel_slots=4)
    sess = Session(LocalTransport(store), econf, rconf, chans)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    ora = OracleSession(store, 4, 3, (5, 5, 4), och,
                        dict(image_dims=(56, 48), base_step=1 / 64, budget=40),
                        sess.engine.metadata_pad)
    pose = orbit_pose(2.6, radius=2.0)
    cam = cam_tuple(pose)
    for i in range(16):
        if i == 8:
            for s in range(4):
                sess.swap_channel(s, 4 + s)
                ora.swap_channel(s, 4 + s)
        r = sess.step_frame(pose)
        o = ora.step_frame(cam)
        assert np.array_equal(r.output.image, o.image), i
        assert r.output.brick_requests == o.brick_requests, i
        assert r.output.metadata_requests == o.metadata_requests, i
        assert np.array_equal(r.output.required_mask, o.required_mask), i
        d = diff_hashes(device_state_hashes(sess.engine), state_hashes(ora.st))
        assert not d, (i, d)
    sess.close()


def _baseline_engines(kind, m, meta):
    """Product-side states of a baselines fixture (methods.py), each pinned to
    the reference's state hashes."""
    from paper_2309_04393_b200 import methods
    st = scenes.store(kind)
    slots = {s: s for s in range(m)}
    econf = methods.full_engine_config(st, m, depth=meta["engine"]["depth"])
    assert list(econf.cache_slots) == meta["engine"]["cache_slots"]
    k = len(st.manifest.levels)
    keep = lambda s, l, x, y, z: scenes.keep_partial(s, l, x, y, z, k)  # noqa: E731
    eng = methods.prepare_engine(st, slots, econf)
    if "state" in meta:
        assert not diff_hashes(device_state_hashes(eng), meta["state"])
    pt = methods.prepare_pagetable_engine(st, slots, econf)
    assert not diff_hashes(device_state_hashes(pt.paging), meta["pagetable_state"])
    part = methods.prepare_partial_engine(st, slots, econf, keep)
    assert not diff_hashes(device_state_hashes(part.paging), meta["partial_state"])
    ppt = methods.prepare_pagetable_engine(st, slots, econf, keep=keep)
    assert not diff_hashes(device_state_hashes(ppt.paging),
                           meta["partial_pagetable_state"])
    classic = methods.build_classic(eng, st, slots)
    return eng, pt, part, ppt, classic


def test_gpu_baselines_sparse256x4_match_reference():
    """The paper's three-way comparison (bench.py:98-145): residency,
    classic-octree and page-table-only modes of the CUDA kernel, fully and
    partially resident, bit-identical to the reference's outputs."""
    from paper_2309_04393_b200 import (orbit_path, render_classic_octree, render_frame,
                                       render_pagetable_only)
    meta, rec = load_golden("baselines_sparse256x4")
    eng, pt, part, ppt, classic = _baseline_engines("sparse256x4", 4, meta)
    assert np.array_equal(classic.min_arr.cpu().numpy(), rec["classic_min"])
    assert np.array_equal(classic.max_arr.cpu().numpy(), rec["classic_max"])
    chans = scenes.product_channels(meta["channels"])
    cfg = scenes.render_config(meta["render"])
    cams = orbit_path(meta["orbit"]["num_frames"])
    for i in meta["orbit"]["frames"]:
        cam = cams[i]
        outs = {"res": render_frame(eng.paging, eng.octree, chans, cam, cfg),
                "cls": render_classic_octree(eng.paging, classic, chans, cam, cfg),
                "pt": render_pagetable_only(pt.paging, chans, cam, cfg),
                "pcls": render_classic_octree(part.paging, classic, chans, cam, cfg),
                "ppt": render_pagetable_only(ppt.paging, chans, cam, cfg)}
        for pre, out in outs.items():
            bad = _check(rec, f"{pre}{i}_", out)
            assert not bad, (i, pre, bad)


def test_gpu_baselines_vessel256_match_reference():
    """Baselines with all-zero bricks: EMPTY entries (brick-exit skips) and
    empty classic nodes (node-exit skips), fully and partially resident."""
    from paper_2309_04393_b200 import (orbit_pose, render_classic_octree,
                                       render_pagetable_only)
    meta, rec = load_golden("baselines_vessel256")
    eng, pt, part, ppt, classic = _baseline_engines("vessel256", 1, meta)
    chans = scenes.product_channels(meta["channels"])
    cfg = scenes.render_config(meta["render"])
    for i, a in enumerate(meta["angles"]):
        cam = orbit_pose(a)
        outs = {"cls": render_classic_octree(eng.paging, classic, chans, cam, cfg),
                "pt": render_pagetable_only(pt.paging, chans, cam, cfg),
                "pcls": render_classic_octree(part.paging, classic, chans, cam, cfg),
                "ppt": render_pagetable_only(ppt.paging, chans, cam, cfg)}
        for pre, out in outs.items():
            bad = _check(rec, f"{pre}{i}_", out)
            assert not bad, (i, pre, bad)


def test_gpu_baselines_errors():
    """ClassicMetadata / render_classic_octree validation (render.py:282-295)."""
    from paper_2309_04393_b200 import (ClassicMetadata, Engine, EngineConfig,
                                       RenderError)
    from paper_2309_04393_b200.volume import VolumeManifest, plan_levels
    man = VolumeManifest(name="t", channel_count=1, dtype_original="u8",
                         brick_size=(16, 16, 16),
                         levels=plan_levels((64, 48, 40), (16, 16, 16), 3, (2, 2, 2)))
    eng = Engine(man, EngineConfig(octree_depth=3, cache_slots=(2, 2, 2), channel_slots=1))
    with pytest.raises(RenderError):
        ClassicMetadata(eng.paging)


def test_gpu_sub_block_maxima_and_skip_is_exact():
    """ro_state.sub_max == max over each 4^3 sub-block dilated by one voxel
    (clipped) for every occupied slot, kept across LRU replacement; rendering
    with the table and without it (NULL) gives identical outputs."""
    import torch
    import torch.nn.functional as Fn
    from paper_2309_04393_b200 import render as R
    from paper_2309_04393_b200 import _native as N
    eng = _prepared_engine("shell64", depth=3)
    p = eng.paging
    e = N.RO_SUB_EDGE
    occ = torch.nonzero(p.slot_brick_dev >= 0).flatten()
    cache = p.cache_dev[occ].float()
    ref = Fn.max_pool3d(cache.unsqueeze(1), kernel_size=e + 2, stride=e, padding=1)
    bz, by, bx = p.cache_dev.shape[1:]
    nsb = (bx // e) * (by // e) * (bz // e)
    got = p.sub_max.view(-1, nsb)[occ].float()
    assert torch.equal(got, ref.reshape(len(occ), -1))
    # LRU replacement rewrites the table of the reused slots
    st = scenes.store("shell64")
    g = st.manifest.levels[0].brick_grid_dims
    ids = [eng.paging.encode(0, 0, (x, y, z)) for z in range(g[2]) for y in range(g[1])
           for x in range(g[0])][:3]
    eng.evict_bricks(ids)
    eng.advance_frame()
    eng.apply_bricks(ids, np.stack([np.full((bz, by, bx), 7, np.uint8)] * 3))
    for b in ids:
        s = int(p.pt[eng.paging._entry_index(*eng.paging.decode(b))])
        assert int(p.sub_max.view(-1, nsb)[s].max()) == 7
    # identical render with the table switched off
    chans = [R.ChannelSettings(slot=0, tf=__import__(
        "paper_2309_04393_b200").grayscale_ramp_tf(40.0))]
    from paper_2309_04393_b200 import RenderConfig, orbit_pose
    cfg = RenderConfig(image_dims=(96, 80), base_step=1.0 / 64.0, max_requests_per_frame=256)
    a = R.render_frame(p, eng.octree, chans, orbit_pose(0.9), cfg)
    keep = p.sub_max
    p.sub_max = None
    try:
        b = R.render_frame(p, eng.octree, chans, orbit_pose(0.9), cfg)
    finally:
        p.sub_max = keep
    assert np.array_equal(a.image, b.image)
    assert a.brick_requests == b.brick_requests
    assert np.array_equal(a.required_mask, b.required_mask)
    assert np.array_equal(a.level_histogram, b.level_histogram)


def test_gpu_config2_full_size_properties():
    """BASELINE config 2 at full size (2048x2048x128 x4 channels, 1080p):
    sampled row bands bit-exact against the oracle (usage mask and
    histogram of the bands contained in the frame's), and the frame split
    sort-first into 3 parts and merged equals the single-pass frame
    (image, ordered requests, usage, histogram, counters)."""
    import os
    import torch
    from oracle import raycast as orc
    from paper_2309_04393_b200 import render_frame, scenarios
    from paper_2309_04393_b200.distributed import merge_parts
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cfg = scn.render
    w, h = cfg.image_dims
    out = render_frame(eng.paging, eng.octree, scn.channels, scn.camera, cfg)
    ref = orc.OracleState(**scenarios.reference_state(scn))
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in scn.channels]
    for a in (0, 300, 536, 760, 1076):
        o = orc.render(ref, och, cam_tuple(scn.camera), cfg.image_dims, cfg.base_step,
                       budget=cfg.max_requests_per_frame, rows=(a, a + 4),
                       threads=os.cpu_count() or 1)
        assert np.array_equal(out.image[a:a + 4], o.image[a:a + 4]), a
        assert not (o.required_mask & ~out.required_mask).any(), a
        assert (o.level_histogram <= out.level_histogram).all(), a
    parts = []
    for p in range(3):
        fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, scn.camera, cfg,
                       partition=(3, p, 8), bricks_first=False)
        fp.render()
        fp.collect()
        b = fp.buf
        parts.append({k: (v.clone() if isinstance(v, torch.Tensor) else v.copy())
                      for k, v in dict(image=b.image, required=b.required,
                                       pix_required=b.pix_required, hist=b.hist,
                                       counters=b.counters, fb=b.fb, counts=b.counts).items()})
    merged = merge_parts(parts, cfg.image_dims, 3, 8, cfg.max_requests_per_frame,
                         eng.paging.config.m)
    assert np.array_equal(merged["image"], out.image)
    assert merged["bricks"] == out.brick_requests
    assert merged["metas"] == out.metadata_requests
    assert np.array_equal(merged["required"], out.required_mask)
    assert np.array_equal(merged["hist"], out.level_histogram)
    assert np.array_equal(merged["pix_required"], out.pixel_required)
    assert int(merged["counters"][1] + merged["counters"][2]) == \
        out.stats.samples_evaluated + out.stats.samples_skipped


@pytest.mark.parametrize("budget", [256, 65536])
def test_gpu_config2_full_frame_matches_oracle(budget):
    """BASELINE config 2 at full size, the WHOLE 1920x1080 frame against the
    C oracle (the reference's algorithm, pinned to reference-generated
    fixtures at this k = 7 / D = 6 scale by tests/test_oracle_golden.py):
    image, ordered brick and metadata request lists, usage mask, level
    histogram, per-pixel brick switches and work counters bit-exact.  With
    budget 65536 every touched entry is emitted, so the complete first-seen
    order is compared (and the feedback kernel sorts in several chunks)."""
    import dataclasses
    import os
    from oracle import raycast as orc
    from paper_2309_04393_b200 import render_frame, scenarios
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cfg = dataclasses.replace(scn.render, max_requests_per_frame=budget)
    out = render_frame(eng.paging, eng.octree, scn.channels, scn.camera, cfg)
    ref = orc.OracleState(**scenarios.reference_state(scn))
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in scn.channels]
    o = orc.render(ref, och, cam_tuple(scn.camera), cfg.image_dims, cfg.base_step,
                   budget=budget, threads=os.cpu_count() or 1)
    assert np.array_equal(out.image, o.image)
    assert out.brick_requests == o.brick_requests
    assert out.metadata_requests == o.metadata_requests
    assert np.array_equal(out.required_mask, o.required_mask)
    assert np.array_equal(out.level_histogram, o.level_histogram)
    assert np.array_equal(out.pixel_required.reshape(-1), o.pixel_required.reshape(-1))
    assert [out.stats.traversal_steps, out.stats.samples_evaluated,
            out.stats.samples_skipped, out.stats.livelocked_rays] == \
        [int(o.counters[0]), int(o.counters[1]), int(o.counters[2]), int(o.counters[4])]
    if budget > 256:
        assert len(out.brick_requests) > 256  # the complete order, not just a prefix


@pytest.mark.parametrize("part", [40, 135, 230])
def test_gpu_config5_row_bands_match_oracle(part):
    """BASELINE config 5 (3840x2160, m = 6 visible channels, the config-2
    volume builder): one sort-first part of 8 rows rendered by the product
    path (FramePass with partition (270, part, 8), bricks-first feedback)
    equals the C oracle over the same rows -- image, ordered brick / metadata
    request lists, usage mask, level histogram and work counters.  4K pixel
    indices take 23 bits, so request keys are wider than 32 bits whenever a
    pixel passes 2^9 request events."""
    import os
    from oracle import raycast as orc
    from paper_2309_04393_b200 import orbit_path, scenarios
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
    scn = _config5_scene()
    eng = scenarios.build_engine(scn)
    cfg = scn.render
    w, h = cfg.image_dims
    cam = orbit_path(120)[part % 120]
    fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, cam, cfg,
                   partition=(h // 8, part, 8), bricks_first=True)
    fp.render()
    fp.collect()
    b = fp.buf
    m = eng.paging.config.m
    nb, nm = b.n_bricks, b.n_metas
    fb = b.fb.cpu().numpy()
    ref = orc.OracleState(**scenarios.reference_state(scn))
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in scn.channels]
    r0 = 8 * part
    want = orc.render(ref, och, cam_tuple(cam), (w, h), cfg.base_step,
                      budget=cfg.max_requests_per_frame, rows=(r0, r0 + 8),
                      threads=os.cpu_count() or 1)
    assert np.array_equal(b.image.cpu().numpy().reshape(8, w, 4), want.image[r0:r0 + 8])
    assert fb[1][:nb].tolist() == want.brick_requests
    assert [divmod(int(v), m) for v in fb[3][:nm]] == want.metadata_requests
    assert np.array_equal(b.required.cpu().numpy(), want.required_mask)
    assert np.array_equal(b.hist.cpu().numpy(), want.level_histogram)
    c = b.counters.cpu().numpy()
    assert [int(c[0]), int(c[1]), int(c[2])] == [int(v) for v in want.counters[:3]]


_C5 = {}


def _config5_scene():
    from paper_2309_04393_b200 import scenarios
    if "scn" not in _C5:
        _C5["scn"] = scenarios.cycif(device="cuda", dataset_channels=(0, 3, 6, 9, 12, 15),
                                     image_dims=(3840, 2160))
    return _C5["scn"]


def test_gpu_capacity_mode_parts_converge_to_single_gpu_image():
    """Sort-first capacity mode: two part sessions, each
    with its own cache / LRU / octree fed only by its own rows' requests,
    converge independently; their stitched rows equal the single-session
    converged image and the full-residency reference render (parity at image
    level once every desired brick is resident)."""
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       RenderConfig, Session, grayscale_ramp_tf, orbit_pose,
                                       render_reference)
    from paper_2309_04393_b200.distributed import part_rows
    st = scenes.store("vessel256")
    econf = EngineConfig(octree_depth=5, cache_slots=(9, 9, 9), channel_slots=1)
    cfg = RenderConfig(image_dims=(160, 120), base_step=1.0 / 128.0,
                       max_requests_per_frame=512, traversal_start_level=2)
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0))]
    pose = orbit_pose(0.8)
    single = Session(LocalTransport(st), econf, cfg, chans)
    single.run_until_converged(pose, max_frames=50)
    assert single.converged
    ref_img = single.history[-1].output.image
    w, h = cfg.image_dims
    stitched = np.zeros_like(ref_img)
    resident = []
    for p in range(2):
        sess = Session(LocalTransport(st), econf, cfg, chans, partition=(2, p, 8))
        recs = sess.run_until_converged(pose, max_frames=50)
        assert sess.converged, p
        rows = part_rows(h, 2, p, 8)
        assert recs[-1].output.image.shape == (len(rows), w, 4)
        stitched[rows] = recs[-1].output.image
        resident.append(sess.engine.paging.occupied_slot_count())
        sess.close()
    assert np.array_equal(stitched, ref_img)
    full = _prepared_engine("vessel256", depth=5)
    assert np.array_equal(render_reference(full.paging, chans, pose, cfg).image, ref_img)
    # each part caches only what its own rows need
    assert max(resident) < single.engine.paging.occupied_slot_count() <= sum(resident)
    single.close()


def test_gpu_upload_reference_state_through_c_abi():
    """INTEGRATION.md path B: a reference-layout state (pt_status + pt_slot,
    words, cache, LRU arrays, free list) adopted through ro_upload_state
    renders the reference's golden frames; ro_download_state returns it."""
    import ctypes as C
    from oracle.session import prepare_full
    from paper_2309_04393_b200 import Engine, EngineConfig, orbit_pose, render_frame
    from paper_2309_04393_b200 import _native as N
    from paper_2309_04393_b200.volume import box_minmax_grid
    meta, rec = load_golden("vessel256_full")
    e = meta["engine"]
    st = scenes.store("vessel256")
    ref = prepare_full(st, {0: 0}, 1, e["depth"], e["cache_slots"], e["pad"], box_minmax_grid)
    eng = Engine(st.manifest, EngineConfig(octree_depth=e["depth"],
                                           cache_slots=tuple(e["cache_slots"]), channel_slots=1))
    eng.paging.load_reference_state(ref.pt_status, ref.pt_slot, ref.cache, ref.slot_brick,
                                    ref.slot_last_used, ref.free, words=ref.words)
    assert not diff_hashes(device_state_hashes(eng), meta["state"])
    chans = scenes.product_channels(meta["channels"])
    cfg = scenes.render_config(meta["render"])
    for i, a in enumerate(meta["angles"][:2]):
        out = render_frame(eng.paging, eng.octree, chans, orbit_pose(a), cfg)
        assert not _check(rec, f"res{i}_", out), i
    p = eng.paging
    E, S = p.total_entries, p.num_slots
    ps, sl = np.zeros(E, np.int8), np.zeros(E, np.int32)
    sb, lu = np.zeros(S, np.int64), np.zeros(S, np.int64)
    fl, fc = np.zeros(S, np.int32), C.c_int64(0)
    N.check(N.lib().ro_download_state(p.ctx, C.byref(p.state()), ps.ctypes.data, sl.ctypes.data,
                                      None, None, sb.ctypes.data, lu.ctypes.data, fl.ctypes.data,
                                      C.byref(fc), N.stream_ptr()))
    assert np.array_equal(ps, ref.pt_status) and np.array_equal(sl, ref.pt_slot)
    assert np.array_equal(sb, ref.slot_brick) and np.array_equal(lu, ref.slot_last_used)
    assert list(fl[:fc.value]) == list(ref.free)


def _random_tf(rng):
    from paper_2309_04393_b200 import TransferFunction
    n = int(rng.integers(2, 7))
    xs = np.sort(rng.choice(np.arange(0, 256), size=n, replace=False)).astype(float)
    pts = []
    for x in xs:
        a = 0.0 if rng.random() < 0.35 else float(rng.uniform(0.01, 1.0))
        pts.append((float(x), (float(rng.random()), float(rng.random()),
                               float(rng.random()), a)))
    return TransferFunction(points=tuple(pts))


@pytest.mark.parametrize("seed", list(range(int(__import__("os").environ.get("RESOCT_FUZZ_N",
                                                                             "24")))))
def test_gpu_randomized_frames_match_oracle(seed):
    """Randomised sweep beyond the golden scenes: random residency and INVALID
    metadata, random TFs / level ranges / channel order / eps, odd image sizes
    with exactly axis-aligned centre rays (the |d| < 1e-12 box branches),
    cameras inside the volume, random t0 / start level / early termination /
    budget.  Everything bit-exact against the C oracle."""
    from oracle import raycast as orc
    from paper_2309_04393_b200 import Camera, ChannelSettings, RenderConfig, render_frame
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(1, 9))      # m = 4 takes the vector word load, others the scalar one
    depth = int(rng.integers(2, 5))
    eps = float(rng.choice([0.0, 3.0, 12.0]))
    eng = _random_partial_engine(seed, eps=eps, depth=depth, m=m,
                                 cache=(6, 6, 6) if m <= 4 else (8, 8, 8))
    k = eng.paging.config.k
    chans = []
    for s in rng.permutation(m):
        lo = int(rng.integers(0, k))
        hi = int(rng.integers(lo, k))
        chans.append(ChannelSettings(slot=int(s), tf=_random_tf(rng), level_range=(lo, hi)))
    kind = seed % 3
    if kind == 0:      # axis-aligned view, odd size: the centre ray has dx = dy = 0
        cam = Camera(position=(0.5, 0.5, -1.2), target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0),
                     fov_deg=40.0)
        dims = (int(rng.integers(8, 20)) * 2 + 1, int(rng.integers(6, 16)) * 2 + 1)
    elif kind == 1:    # camera inside the volume
        pos = tuple(float(v) for v in rng.uniform(0.2, 0.8, 3))
        cam = Camera(position=pos, target=(0.5, 0.5, 0.5 + 1e-3 if pos == (0.5,) * 3 else 0.5),
                     up=(0.0, 0.0, 1.0), fov_deg=float(rng.uniform(30, 90)))
        dims = (int(rng.integers(16, 40)), int(rng.integers(12, 30)))
    else:              # random outside orbit
        a = float(rng.uniform(0, 6.28))
        r = float(rng.uniform(1.2, 2.6))
        cam = Camera(position=(0.5 + r * np.cos(a), 0.5 + float(rng.uniform(-0.8, 0.8)),
                               0.5 + r * np.sin(a)), target=(0.5, 0.5, 0.5), fov_deg=45.0)
        dims = (int(rng.integers(16, 48)), int(rng.integers(12, 36)))
    cfg = RenderConfig(image_dims=dims, base_step=float(rng.choice([1 / 32, 1 / 50, 1 / 64, 1 / 100])),
                       lod_reference_distance=float(rng.choice([0.5, 1.0, 1.7])),
                       early_term_alpha=float(rng.choice([0.5, 0.99, 1.0])),
                       max_requests_per_frame=int(rng.integers(1, 400)),
                       traversal_start_level=int(rng.integers(0, 4)))
    out = render_frame(eng.paging, eng.octree, chans, cam, cfg)
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    want = orc.render(ost, och, cam_tuple(cam), dims, cfg.base_step,
                      t0=cfg.lod_reference_distance, early_alpha=cfg.early_term_alpha,
                      budget=cfg.max_requests_per_frame,
                      start_level=cfg.traversal_start_level)
    assert np.array_equal(out.image, want.image), (
        int((out.image != want.image).sum()), float(np.abs(out.image - want.image).max()))
    assert out.brick_requests == want.brick_requests
    assert out.metadata_requests == want.metadata_requests
    assert np.array_equal(out.required_mask, want.required_mask)
    assert np.array_equal(out.level_histogram, want.level_histogram)
    assert np.array_equal(out.pixel_required, want.pixel_required)
    assert [out.stats.traversal_steps, out.stats.samples_evaluated,
            out.stats.samples_skipped] == list(want.counters[:3])


@pytest.mark.parametrize("depth", [7, 8])
def test_gpu_deep_octree_matches_oracle(depth):
    """Deep trees as config 4 uses (D = 7: 2.4 M nodes, D = 8: 19.2 M): the
    vessel 256^3 volume with a random third of its bricks evicted and
    random INVALID metadata; incremental masks == a from-scratch rebuild,
    and residency frames (long parallel descents, deep skips) equal the
    oracle bit for bit."""
    from oracle import raycast as orc
    from paper_2309_04393_b200 import (ChannelSettings, RenderConfig, grayscale_ramp_tf,
                                       orbit_pose, render_frame)
    eng = _prepared_engine("vessel256", depth=depth)
    rng = np.random.default_rng(depth)
    ids = eng.paging.resident_brick_ids()
    eng.evict_bricks([int(b) for b in rng.choice(ids, size=len(ids) // 3, replace=False)])
    words = eng.octree.words.copy()
    kill = rng.random(words.shape) < 0.1
    words[kill] = (words[kill] & np.uint32(0xFFFF)) | np.uint32(0x00FF0000)
    eng.octree.upload_words(words)
    before = eng.octree.words.copy()
    eng.octree.rebuild_masks()
    assert np.array_equal(before, eng.octree.words)
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0))]
    ost = oracle_state_from_device(eng)
    och = [orc.OracleChannel(slot=0, points=chans[0].tf.points, level_range=(0, 15))]
    for angle, step in ((0.7, 1 / 256), (3.3, 1 / 1000)):
        cfg = RenderConfig(image_dims=(48, 36), base_step=step, max_requests_per_frame=300,
                           traversal_start_level=2)
        pose = orbit_pose(angle)
        out = render_frame(eng.paging, eng.octree, chans, pose, cfg)
        want = orc.render(ost, och, cam_tuple(pose), cfg.image_dims, step, budget=300,
                          threads=8)
        assert np.array_equal(out.image, want.image)
        assert out.brick_requests == want.brick_requests
        assert out.metadata_requests == want.metadata_requests
        assert np.array_equal(out.required_mask, want.required_mask)
        assert [out.stats.traversal_steps, out.stats.samples_evaluated,
                out.stats.samples_skipped] == list(want.counters[:3])


def test_gpu_out_of_core_procedural_session_matches_oracle():
    """Config 4 (scaled): the procedural out-of-core store streamed through a
    Session whose cache holds a fraction of the working set (LRU evictions
    every frame) along a moving orbit, with a mid-sequence channel swap;
    every frame's image, ordered requests, usage mask and the full state
    equal the oracle session fed by the same store."""
    from oracle.session import OracleSession, state_hashes
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, RenderConfig, Session,
                                       orbit_path)
    from paper_2309_04393_b200.scenarios import COLORS, ProceduralStore
    from paper_2309_04393_b200.transfer import colored_ramp_tf
    from oracle import raycast as orc
    store = ProceduralStore(dims=(512, 512, 64), channels=12, brick=16, cell=64,
                            occupancy=0.3, pool=8, seed=99)
    chans = [ChannelSettings(slot=s, tf=colored_ramp_tf(40.0, COLORS[s], 0.3))
             for s in range(4)]
    rconf = RenderConfig(image_dims=(64, 48), base_step=1 / 128, max_requests_per_frame=48)
    econf = EngineConfig(octree_depth=4, cache_slots=(6, 6, 5), channel_slots=4)
    sess = Session(store, econf, rconf, chans)
    och = [orc.OracleChannel(slot=c.slot, points=c.tf.points, level_range=c.level_range)
           for c in chans]
    ora = OracleSession(store, 4, 4, (6, 6, 5), och,
                        dict(image_dims=(64, 48), base_step=1 / 128, budget=48),
                        sess.engine.metadata_pad)
    for s, c in enumerate((0, 3, 6, 9)):
        sess.swap_channel(s, c)
        ora.swap_channel(s, c)
    evicting = False
    for i, pose in enumerate(orbit_path(14)):
        if i == 7:
            for s in range(4):
                sess.swap_channel(s, 1 + 3 * s)
                ora.swap_channel(s, 1 + 3 * s)
        r = sess.step_frame(pose)
        o = ora.step_frame(cam_tuple(pose))
        assert np.array_equal(r.output.image, o.image), i
        assert r.output.brick_requests == o.brick_requests, i
        assert r.output.metadata_requests == o.metadata_requests, i
        assert np.array_equal(r.output.required_mask, o.required_mask), i
        d = diff_hashes(device_state_hashes(sess.engine), state_hashes(ora.st))
        assert not d, (i, d)
        evicting |= len(ora.st.free) == 0
    assert evicting
    sess.close()
