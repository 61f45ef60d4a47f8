"""The reference's end-to-end acceptance criteria on the CUDA path.

Restates /root/reference/pkg/tests/test_acceptance.py for every criterion
that exercises the hot path (1-7 and 9; 8 = codec/LZ4/manifest round trips
lives in tests/test_ingest_golden.py and tests/test_gpu_ingest.py).  The reference's own run printed exact verdict numbers
(pkg/test_output.txt:180-188, reproduced in this container by SURVEY.md §8's
acceptance re-run); the CUDA path is bit-exact, so these tests assert the
SAME numbers, not just the same inequalities.
"""

import numpy as np
import pytest

from conftest import cuda_ok
import scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def _cfgs():
    from paper_2309_04393_b200 import EngineConfig, RenderConfig
    return dict(
        RENDER_64=RenderConfig(image_dims=(128, 128), base_step=1.0 / 64.0,
                               max_requests_per_frame=512, traversal_start_level=2),
        ENGINE_64=EngineConfig(octree_depth=3, cache_slots=(9, 9, 9), channel_slots=1),
        RENDER_256=RenderConfig(image_dims=(256, 256), base_step=1.0 / 128.0,
                                max_requests_per_frame=2048, traversal_start_level=2),
        ENGINE_256=EngineConfig(octree_depth=5, cache_slots=(9, 9, 9), channel_slots=1),
        TREND_RENDER=RenderConfig(image_dims=(96, 96), base_step=1.0 / 128.0,
                                  max_requests_per_frame=2048, traversal_start_level=2))


def _tf40():
    from paper_2309_04393_b200 import grayscale_ramp_tf
    return grayscale_ramp_tf(threshold=40.0)


def _poses():
    from paper_2309_04393_b200 import orbit_pose
    return [orbit_pose(a) for a in (0.0, 1.1, 2.4, 3.7, 5.2)]


def _converged(store, econf, rconf, pose, channels):
    from paper_2309_04393_b200 import LocalTransport, Session
    sess = Session(LocalTransport(store), econf, rconf, channels)
    sess.run_until_converged(pose, max_frames=50)
    assert sess.converged
    return sess


def test_acceptance_1_oracle_equivalence():
    """test_acceptance.py:104-123: converged sessions (LRU pressure: 729
    slots), render_frame == render_reference bit-identical, 5 poses x 2
    datasets."""
    from paper_2309_04393_b200 import ChannelSettings, render_frame, render_reference
    c = _cfgs()
    chans = [ChannelSettings(slot=0, tf=_tf40())]
    for kind, econf, rconf in (("shell64", c["ENGINE_64"], c["RENDER_64"]),
                               ("vessel256", c["ENGINE_256"], c["RENDER_256"])):
        for pose in _poses():
            sess = _converged(scenes.store(kind), econf, rconf, pose, chans)
            ours = render_frame(sess.engine.paging, sess.engine.octree, chans, pose, rconf)
            ref = render_reference(sess.engine.paging, chans, pose, rconf)
            assert np.array_equal(ours.image, ref.image), (kind, pose)
            sess.close()


def test_acceptance_2_skipping_soundness():
    """test_acceptance.py:126-160: 10 random TFs x 3 poses, every skipped or
    zero sample audited against a fully resident paging: 0 violations and
    943,162 skipped samples (test_output.txt:181)."""
    from paper_2309_04393_b200 import (ChannelSettings, TransferFunction, orbit_pose,
                                       render_frame)
    from paper_2309_04393_b200 import methods
    c = _cfgs()
    st = scenes.store("shell64")
    ref_engine = methods.prepare_engine(st, {0: 0}, methods.full_engine_config(st, 1, 3))
    rng = np.random.default_rng(42)
    poses = [orbit_pose(a) for a in (0.3, 2.0, 4.4)]
    total = 0
    for _ in range(10):
        xs = np.sort(rng.choice(np.arange(1.0, 255.0), size=5, replace=False))
        pts = [(0.0, (0.0, 0.0, 0.0, 0.0))]
        for x in xs:
            alpha = 0.0 if rng.random() < 0.5 else float(rng.uniform(0.05, 1.0))
            pts.append((float(x), (float(rng.random()), float(rng.random()),
                                   float(rng.random()), alpha)))
        chans = [ChannelSettings(slot=0, tf=TransferFunction(points=tuple(pts)))]
        sess = _converged(st, c["ENGINE_64"], c["RENDER_64"], poses[0], chans)
        for pose in poses:
            out = render_frame(sess.engine.paging, sess.engine.octree, chans, pose,
                               c["RENDER_64"], reference_paging=ref_engine.paging)
            assert out.stats.skip_violations == 0
            total += out.stats.samples_skipped
        sess.close()
    assert total == 943162


@pytest.fixture(scope="module")
def trend_rows():
    """test_acceptance.py:84-91: 36-frame orbit, three methods."""
    from paper_2309_04393_b200 import ChannelSettings, methods
    st = scenes.store("sparse256x4")
    chans = [ChannelSettings(slot=s, tf=_tf40()) for s in range(4)]
    econf = methods.full_engine_config(st, 4, depth=5)
    return methods.run_orbit(st, chans, {s: s for s in range(4)}, _cfgs()["TREND_RENDER"],
                             econf, num_frames=36)


def test_acceptance_4_working_set_trend(trend_rows):
    """test_acceptance.py:177-190 / test_output.txt:183: mean cache bytes
    ours 8.64 MB <= classic 9.17 MB <= page table 20.80 MB, 58% reduction."""
    from paper_2309_04393_b200 import methods
    s = methods.summarize(trend_rows)
    ours = s["residency"]["mean_cache_bytes"]
    classic = s["classic"]["mean_cache_bytes"]
    pagetable = s["pagetable"]["mean_cache_bytes"]
    assert ours <= classic <= pagetable * 1.05
    assert 1.0 - ours / pagetable >= 0.20
    assert (round(ours / 1e6, 2), round(classic / 1e6, 2), round(pagetable / 1e6, 2)) == \
        (8.64, 9.17, 20.80)
    assert round(100 * (1.0 - ours / pagetable)) == 58


def test_acceptance_5_traversal_efficiency(trend_rows):
    """test_acceptance.py:193-198 / test_output.txt:184: mean traversal steps
    ours 490,431 < classic 1,098,886."""
    from paper_2309_04393_b200 import methods
    s = methods.summarize(trend_rows)
    ours = s["residency"]["mean_steps"]
    classic = s["classic"]["mean_steps"]
    assert ours < classic
    assert (round(ours), round(classic)) == (490431, 1098886)


def test_acceptance_6_mixed_resolution_memory():
    """test_acceptance.py:201-233 / test_output.txt:185: pinning one channel to
    the coarsest level saves 53% cache bytes; the other channels' sampled
    levels are unchanged."""
    from paper_2309_04393_b200 import ChannelSettings, methods, orbit_pose, render_frame
    st = scenes.store("sparse256x4")
    k = len(st.manifest.levels)
    eng = methods.prepare_engine(st, {s: s for s in range(4)},
                                 methods.full_engine_config(st, 4, depth=5))
    tf = _tf40()
    finest = [ChannelSettings(slot=s, tf=tf, level_range=(0, 0)) for s in range(4)]
    pinned = [ChannelSettings(slot=s, tf=tf, level_range=(k - 1, k - 1) if s == 3 else (0, 0))
              for s in range(4)]
    cfg = _cfgs()["TREND_RENDER"]
    bytes_f = bytes_p = 0
    hist_f = hist_p = None
    for a in np.linspace(0, 2 * np.pi, 12, endpoint=False):
        pose = orbit_pose(a)
        of = render_frame(eng.paging, eng.octree, finest, pose, cfg)
        op = render_frame(eng.paging, eng.octree, pinned, pose, cfg)
        bytes_f += of.stats.required_bytes
        bytes_p += op.stats.required_bytes
        hist_f = of.level_histogram if hist_f is None else hist_f + of.level_histogram
        hist_p = op.level_histogram if hist_p is None else hist_p + op.level_histogram
    assert bytes_p < bytes_f
    for c in range(3):
        assert set(np.flatnonzero(hist_f[c])) == set(np.flatnonzero(hist_p[c]))
    assert set(np.flatnonzero(hist_p[3])) == {k - 1}
    assert round(100 * (1.0 - bytes_p / bytes_f)) == 53


def test_acceptance_7_convergence():
    """test_acceptance.py:238-250 / test_output.txt:186: a cold session
    reaches a zero-request fixed point in 14 frames (LocalTransport; the HTTP
    transport is off the path)."""
    from paper_2309_04393_b200 import ChannelSettings, LocalTransport, Session, orbit_pose
    c = _cfgs()
    sess = Session(LocalTransport(scenes.store("vessel256")), c["ENGINE_256"],
                   c["RENDER_256"], [ChannelSettings(slot=0, tf=_tf40())])
    recs = sess.run_until_converged(orbit_pose(0.8), max_frames=50)
    assert sess.converged
    assert recs[-1].output.stats.requests_issued == 0
    assert recs[-1].image_digest == recs[-2].image_digest
    assert len(recs) == 14
    sess.close()


def test_acceptance_9_channel_swap():
    """test_acceptance.py:285-302: a mid-stream swap converges to exactly the
    image of a fresh session started on the new channel."""
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       Session, orbit_pose)
    c = _cfgs()
    st = scenes.store("mc64")
    econf = EngineConfig(octree_depth=3, cache_slots=(9, 9, 9), channel_slots=2)
    chans = [ChannelSettings(slot=0, tf=_tf40())]
    pose = orbit_pose(1.9)
    sess = Session(LocalTransport(st), econf, c["RENDER_64"], chans)
    sess.run_until_converged(pose, max_frames=50)
    sess.swap_channel(0, 2)
    recs = sess.run_until_converged(pose, max_frames=50)
    fresh = Session(LocalTransport(st), econf, c["RENDER_64"], chans)
    fresh.swap_channel(0, 2)
    fresh.run_until_converged(pose, max_frames=50)
    assert sess.converged and fresh.converged
    assert np.array_equal(recs[-1].output.image, fresh.history[-1].output.image)
    sess.close()
    fresh.close()


def test_acceptance_3_structural_invariants():
    """test_acceptance.py:165-172 / verify.py:88-140: 10,000 randomised
    insert / evict / swap operations on the shell 64^3 dataset with a full
    scan (page-table <-> slot bijection, mask OR-closure, leaf ground truth)
    every 100 operations, within the reference's 30 s criterion."""
    import time
    from paper_2309_04393_b200 import Engine, EngineConfig
    st = scenes.store("shell64")
    man = st.manifest
    eng = Engine(man, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4), channel_slots=1))
    rng = np.random.default_rng(0)
    k = len(man.levels)
    t0 = time.perf_counter()
    for i in range(10_000):
        op = rng.random()
        slot = int(rng.integers(1))
        lev = int(rng.integers(k))
        grid = man.levels[lev].brick_grid_dims
        coord = tuple(int(rng.integers(grid[a])) for a in range(3))
        bid = eng.paging.encode(slot, lev, coord)
        if op < 0.75:
            eng.apply_brick(bid, st.brick(eng.paging.channel_mapping[slot], lev, coord))
        elif op < 0.9:
            resident = eng.paging.resident_brick_ids()
            if resident:
                eng.evict_bricks([int(resident[int(rng.integers(len(resident)))])])
        else:
            eng.swap_channel(slot, int(rng.integers(man.channel_count)))
        if (i + 1) % 100 == 0:
            eng.paging.check_bijection()
            eng.octree.check_mask_consistency()
            eng.octree.check_leaf_ground_truth()
    elapsed = time.perf_counter() - t0
    assert elapsed < 30.0, elapsed
