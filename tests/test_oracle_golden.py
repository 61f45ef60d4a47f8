"""Pin the CPU oracle to the reference's own outputs (tests/golden/).

The fixtures were produced by running the reference (tests/golden/
make_golden.py); these tests need no GPU and no /root/reference.
"""

import numpy as np
import pytest

from conftest import load_golden
import scenes


def test_restated_ingest_matches_reference_pyramids():
    for name, kind, chans in (("session_mc64", "mc64", range(4)),
                              ("skip_audit_shell64", "shell64", [0]),
                              ("vessel256_full", "vessel256", [0])):
        meta, _ = load_golden(name)
        assert scenes.pyramid_sha(scenes.store(kind), chans) == meta["pyramid_sha"], name


def test_oracle_session_mc64_matches_reference(oracle_lib):
    """Cold 4-channel session with LRU pressure, mixed level ranges and a
    mid-stream double channel swap: every frame's image, ordered requests,
    usage mask, histogram, counters and the full state after each step."""
    from oracle.session import OracleSession, state_hashes
    meta, rec = load_golden("session_mc64")
    e = meta["engine"]
    sess = OracleSession(scenes.store("mc64"), e["m"], e["depth"], e["cache_slots"],
                         scenes.oracle_channels(meta["channels"]),
                         scenes.render_kw(meta["render"]), e["pad"])
    for item in meta["script"]:
        if "swap" in item:
            for slot, ch in item["swap"]:
                sess.swap_channel(slot, ch)
            assert state_hashes(sess.st) == item["after_swap"]
            continue
        i = item["frame"]
        out = sess.step_frame(tuple(item["pose"]))
        bad = scenes.check_frame(rec, f"f{i}_", out.image, out.brick_requests,
                                 out.metadata_requests, out.required_mask,
                                 out.level_histogram, out.pixel_required, out.counters)
        assert not bad, (i, bad)
        assert state_hashes(sess.st) == item["after"], i


def test_oracle_vessel256_matches_reference(oracle_lib):
    """Config 1: fully resident vessel 256^3, residency and reference modes,
    five orbit poses, bit-identical to the reference (test_acceptance.py:104-123)."""
    from oracle import raycast as orc
    from oracle.session import prepare_full, state_hashes
    from paper_2309_04393_b200.camera import orbit_pose
    from paper_2309_04393_b200.volume import box_minmax_grid
    meta, rec = load_golden("vessel256_full")
    e = meta["engine"]
    st = prepare_full(scenes.store("vessel256"), {0: 0}, 1, e["depth"],
                      e["cache_slots"], e["pad"], box_minmax_grid)
    assert state_hashes(st) == meta["state"]
    ostate = orc.OracleState(m=1, k=st.k, brick_size=st.brick_size,
                             level_dims=st.level_dims, level_grids=st.level_grids,
                             pt_offsets=st.pt_offsets, pt_status=st.pt_status,
                             pt_slot=st.pt_slot, cache=st.cache, words=st.words,
                             depth=st.depth)
    chans = scenes.oracle_channels(meta["channels"])
    kw = scenes.render_kw(meta["render"])
    for i, a in enumerate(meta["angles"]):
        p = orbit_pose(a)
        cam = (p.position, p.target, p.up, p.fov_deg)
        for mode, pre in ((orc.MODE_RESIDENCY, "res"), (orc.MODE_REFERENCE, "ref")):
            out = orc.render(ostate, chans, cam, mode=mode, threads=4, **kw)
            bad = scenes.check_frame(rec, f"{pre}{i}_", out.image, out.brick_requests,
                                     out.metadata_requests, out.required_mask,
                                     out.level_histogram, out.pixel_required,
                                     out.counters)
            assert not bad, (i, pre, bad)


def test_oracle_skip_audit_matches_reference(oracle_lib):
    """Skip soundness audit (test_acceptance.py:138-160): converged sessions
    under random TFs, audited against a fully resident reference paging."""
    from oracle import raycast as orc
    from oracle.session import OracleSession, prepare_full, state_hashes
    from paper_2309_04393_b200.camera import orbit_pose
    from paper_2309_04393_b200.volume import box_minmax_grid
    meta, rec = load_golden("skip_audit_shell64")
    e = meta["engine"]
    store = scenes.store("shell64")
    ref = prepare_full(store, {0: 0}, 1, e["depth"], scenes.full_cache_slots(store, 1),
                       e["pad"], box_minmax_grid)
    assert state_hashes(ref) == meta["ref_state"]
    ref_state = orc.OracleState(m=1, k=ref.k, brick_size=ref.brick_size,
                                level_dims=ref.level_dims, level_grids=ref.level_grids,
                                pt_offsets=ref.pt_offsets, pt_status=ref.pt_status,
                                pt_slot=ref.pt_slot, cache=ref.cache)
    poses = [orbit_pose(a) for a in meta["poses"]]
    cams = [(p.position, p.target, p.up, p.fov_deg) for p in poses]
    for r, run in enumerate(meta["runs"]):
        chans = scenes.oracle_channels([{"slot": 0, "tf": run["tf"],
                                         "level_range": [0, 15]}])
        sess = OracleSession(store, 1, e["depth"], e["cache_slots"], chans,
                             scenes.render_kw(meta["render"]), e["pad"])
        streak, last, frames = 0, None, 0
        for _ in range(50):
            out = sess.step_frame(cams[0])
            frames += 1
            dig = out.image.tobytes()
            nreq = len(out.brick_requests) + len(out.metadata_requests)
            streak = streak + 1 if (nreq == 0 and dig == last) else (1 if nreq == 0 else 0)
            last = dig
            if streak >= 2:
                break
        assert frames == run["frames"]
        assert state_hashes(sess.st) == run["state"]
        for j, cam in enumerate(cams):
            out = sess.render(cam, reference_state=ref_state)
            bad = scenes.check_frame(rec, f"r{r}p{j}_", out.image, out.brick_requests,
                                     out.metadata_requests, out.required_mask,
                                     out.level_histogram, out.pixel_required,
                                     out.counters)
            assert not bad, (r, j, bad)
            assert out.counters[3] == 0


def test_oracle_lru_replay_matches_reference():
    """Randomised insert / explicit evict / LRU touch / metadata / swap
    sequence (verify.py:88-136 + frame advances): state hashes at every
    checkpoint and every evicted id."""
    from oracle.session import state_hashes
    from oracle.state import OracleResidency
    meta, _ = load_golden("lru_replay")
    from paper_2309_04393_b200.volume import plan_levels
    levels = plan_levels(tuple(meta["dims"]), tuple(meta["brick"]), meta["levels"], (2, 2, 2))
    st = OracleResidency(meta["m"], meta["levels"], tuple(meta["brick"]),
                         [l.dims for l in levels], [l.brick_grid_dims for l in levels],
                         tuple(meta["cache_slots"]), meta["depth"])
    frame = 0
    sx, sy, sz = meta["brick"]
    for op in meta["ops"]:
        kind = op[0]
        if kind == "insert":
            payload = np.full((sz, sy, sx), op[2], dtype=np.uint8)
            _, ev = st.apply_brick(op[1], payload, frame)
            assert (-1 if ev is None else ev) == op[3]
        elif kind == "evict":
            slot, lev, coord = __import__("oracle.state", fromlist=["decode"]).decode(op[1], st.k)
            e = st.entry(slot, lev, coord)
            lin = int(st.pt_slot[e])
            st.pt_status[e] = 0
            st.pt_slot[e] = -1
            st.release_slot(lin)
            st.on_brick_evicted(op[1])
        elif kind == "advance_note":
            frame += 1
            mask = np.zeros(int(st.pt_offsets[-1]), dtype=np.uint8)
            mask[op[1]] = 1
            st.note_sampled(mask, frame)
        elif kind == "meta":
            st.set_node_metadata(op[1], op[2], op[3], op[4])
        elif kind == "swap":
            st.swap_channel(op[1])
        elif kind == "check":
            assert state_hashes(st) == op[1]


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_row_bands_merge_to_full_frame(oracle_lib, threads):
    """Row-band rendering + scanline-order merge equals one full pass (the
    CPU-baseline and sort-first merge rule)."""
    from oracle import raycast as orc
    from oracle.session import OracleSession
    meta, _ = load_golden("session_mc64")
    e = meta["engine"]
    sess = OracleSession(scenes.store("mc64"), e["m"], e["depth"], e["cache_slots"],
                         scenes.oracle_channels(meta["channels"]),
                         scenes.render_kw(meta["render"]), e["pad"])
    cam = tuple(meta["script"][0]["pose"])
    for _ in range(3):
        sess.step_frame(cam)
    full = sess.render(cam)
    par = sess.render(cam, threads=threads)
    assert np.array_equal(full.image, par.image)
    assert full.all_brick_requests == par.all_brick_requests
    assert full.all_metadata_requests == par.all_metadata_requests
    assert np.array_equal(full.required_mask, par.required_mask)
    assert np.array_equal(full.counters, par.counters)


def _baseline_states(store, m, meta):
    """Full, page-table-only and partial states of a baselines fixture, each
    pinned to the reference's own state hashes."""
    from oracle.session import prepare_full, prepare_paging, state_hashes
    from paper_2309_04393_b200.volume import box_minmax_grid
    e = meta["engine"]
    slots = {s: s for s in range(m)}
    k = len(store.manifest.levels)
    keep = lambda s, l, x, y, z: scenes.keep_partial(s, l, x, y, z, k)  # noqa: E731
    out = {}
    if "state" in meta:
        full = prepare_full(store, slots, m, e["depth"], e["cache_slots"], e["pad"],
                            box_minmax_grid)
        assert state_hashes(full) == meta["state"]
        out["full"] = full
    pt = prepare_paging(store, slots, m, e["depth"], e["cache_slots"], zero_as_empty=True)
    assert scenes.paging_hashes(pt) == meta["pagetable_state"]
    part = prepare_paging(store, slots, m, e["depth"], e["cache_slots"], keep=keep)
    assert scenes.paging_hashes(part) == meta["partial_state"]
    ppt = prepare_paging(store, slots, m, e["depth"], e["cache_slots"], keep=keep,
                         zero_as_empty=True)
    assert scenes.paging_hashes(ppt) == meta["partial_pagetable_state"]
    out.update(pt=pt, part=part, ppt=ppt)
    return out


def test_oracle_baselines_sparse256x4_match_reference(oracle_lib):
    """The paper's three-way comparison (bench.py:98-145): residency,
    classic-octree (kernels.py:359-429) and page-table-only (316-357) renders
    of the trend scene, fully and partially resident, bit-identical to the
    reference; the classic metadata pyramid equals ClassicMetadata's."""
    from oracle import raycast as orc
    from oracle.session import classic_metadata
    from paper_2309_04393_b200.camera import orbit_path
    meta, rec = load_golden("baselines_sparse256x4")
    store = scenes.store("sparse256x4")
    assert scenes.pyramid_sha(store, range(4)) == meta["pyramid_sha"]
    sts = _baseline_states(store, 4, meta)
    k = len(store.manifest.levels)
    cls = classic_metadata({s: store.level_array(s, 0) for s in range(4)}, 4, k)
    assert np.array_equal(cls[0], rec["classic_min"])
    assert np.array_equal(cls[1], rec["classic_max"])
    chans = scenes.oracle_channels(meta["channels"])
    kw = scenes.render_kw(meta["render"])
    cams = orbit_path(meta["orbit"]["num_frames"])
    runs = (("res", "full", orc.MODE_RESIDENCY), ("cls", "full", orc.MODE_CLASSIC),
            ("pt", "pt", orc.MODE_PAGETABLE), ("pcls", "part", orc.MODE_CLASSIC),
            ("ppt", "ppt", orc.MODE_PAGETABLE))
    for i in meta["orbit"]["frames"]:
        c = cams[i]
        cam = (c.position, c.target, c.up, c.fov_deg)
        for pre, which, mode in runs:
            st = scenes.oracle_render_state(sts[which], with_words=(mode == orc.MODE_RESIDENCY))
            out = orc.render(st, chans, cam, mode=mode, threads=4, classic=cls, **kw)
            bad = scenes.check_frame(rec, f"{pre}{i}_", out.image, out.brick_requests,
                                     out.metadata_requests, out.required_mask,
                                     out.level_histogram, out.pixel_required, out.counters)
            assert not bad, (i, pre, bad)


def test_oracle_baselines_vessel256_match_reference(oracle_lib):
    """Baselines on a volume with all-zero bricks: EMPTY page-table entries
    skip to their brick exit, empty classic nodes skip to their node exit."""
    from oracle import raycast as orc
    from oracle.session import classic_metadata, prepare_paging
    from paper_2309_04393_b200.camera import orbit_pose
    meta, rec = load_golden("baselines_vessel256")
    store = scenes.store("vessel256")
    sts = _baseline_states(store, 1, meta)
    assert int((sts["pt"].pt_status == 2).sum()) == meta["empty_entries"] > 0
    k = len(store.manifest.levels)
    cls = classic_metadata({0: store.level_array(0, 0)}, 1, k)
    e = meta["engine"]  # classic renders use a fully resident paging
    full = prepare_paging(store, {0: 0}, 1, e["depth"], e["cache_slots"])
    chans = scenes.oracle_channels(meta["channels"])
    kw = scenes.render_kw(meta["render"])
    runs = (("cls", full, orc.MODE_CLASSIC), ("pt", sts["pt"], orc.MODE_PAGETABLE),
            ("pcls", sts["part"], orc.MODE_CLASSIC), ("ppt", sts["ppt"], orc.MODE_PAGETABLE))
    skipped = 0
    for i, a in enumerate(meta["angles"]):
        p = orbit_pose(a)
        cam = (p.position, p.target, p.up, p.fov_deg)
        for pre, st, mode in runs:
            out = orc.render(scenes.oracle_render_state(st), chans, cam, mode=mode,
                             threads=4, classic=cls, **kw)
            bad = scenes.check_frame(rec, f"{pre}{i}_", out.image, out.brick_requests,
                                     out.metadata_requests, out.required_mask,
                                     out.level_histogram, out.pixel_required, out.counters)
            assert not bad, (i, pre, bad)
            if mode == orc.MODE_PAGETABLE:
                skipped += int(out.counters[2])
    assert skipped > 0  # the EMPTY brick-exit skip was exercised


def test_oracle_config2_bands_match_reference(oracle_lib):
    """BASELINE config 2 at its benchmarked scale (k = 7, D = 6, 4 of 16
    CyCIF-like 2048x2048x128 channels, partial residency with coarser-LOD
    substitution, 1080p): row bands rendered by the reference's own kernel
    (tests/golden/make_golden.py config2_bands) -- image rows, complete
    ordered brick / metadata request lists, usage mask, histogram, per-pixel
    brick switches and counters -- equal the C oracle's, which the GPU test
    test_gpu_config2_full_frame_matches_oracle holds the CUDA kernel to over
    the whole frame."""
    import os
    from oracle import raycast as orc
    meta, rec = load_golden("config2_bands")
    st = orc.OracleState(m=meta["m"], k=meta["k"], brick_size=tuple(meta["brick_size"]),
                         level_dims=rec["level_dims"], level_grids=rec["level_grids"],
                         pt_offsets=rec["pt_offsets"], pt_status=rec["pt_status"],
                         pt_slot=rec["pt_slot"], cache=rec["cache"], words=rec["words"],
                         depth=meta["depth"], eps_h=meta["eps_h"])
    chans = [orc.OracleChannel(slot=c["slot"],
                               points=tuple((x, tuple(v)) for x, v in c["tf"]),
                               level_range=tuple(c["level_range"])) for c in meta["channels"]]
    cam = meta["camera"]
    r = meta["render"]
    w, hh = meta["image"]
    m = meta["m"]
    for i, (a, b) in enumerate(meta["bands"]):
        o = orc.render(st, chans, (tuple(cam["position"]), tuple(cam["target"]),
                                   tuple(cam["up"]), cam["fov_deg"]), (w, hh), r["base_step"],
                       t0=r["t0"], early_alpha=r["early_alpha"], budget=1 << 16,
                       start_level=r["start_level"], rows=(a, b), threads=os.cpu_count() or 1)
        assert np.array_equal(o.image[a:b], rec[f"b{i}_image"]), a
        assert o.brick_requests == rec[f"b{i}_bricks"].tolist(), a
        assert o.metadata_requests == [divmod(int(v), m) for v in rec[f"b{i}_metas"]], a
        assert np.array_equal(np.flatnonzero(o.required_mask), rec[f"b{i}_required"]), a
        assert np.array_equal(o.level_histogram, rec[f"b{i}_hist"]), a
        assert np.array_equal(o.pixel_required.reshape(-1)[a * w:b * w], rec[f"b{i}_pix_required"])
        assert np.array_equal(o.counters[:4], rec[f"b{i}_counters"]), a
        assert len(rec[f"b{i}_bricks"]) > 0 or len(rec[f"b{i}_metas"]) > 0
