"""The reference's hand-traced render units on the CUDA ray caster.

Restates /root/reference/pkg/tests/test_render_units.py -- compositing
closed forms (98-138), alternative-brick selection (143-176) and the
multi-channel traversal traces (194-269) -- through 1-pixel launches:
``probe_sample`` resolves exactly one sample at a chosen position, desired
level, traversal depth and cursor start depth with the product kernel
(ro_frame.max_samples = 1), and the traces are checked on what that sample
leaves behind: node visits, first-seen brick / metadata requests, the level
sampled (level histogram), the brick used (usage mask), the composited RGBA
and whether the sample was skippable (skip-loop samples).
"""

import math

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def make_octree(depth=3, m=2, k=3, cache=(3, 3, 3), eps=0.0):
    """test_render_units.py:17-23"""
    from paper_2309_04393_b200 import (MultiChannelPaging, OctreeConfig, PagingConfig,
                                       ResidencyOctree)
    cfg = PagingConfig(brick_size=(16, 16, 16), cache_slots=cache, m=m, k=k)
    dims = [(64, 64, 64), (32, 32, 32), (16, 16, 16)][:k]
    grids = [(4, 4, 4), (2, 2, 2), (1, 1, 1)][:k]
    paging = MultiChannelPaging(cfg, dims, grids)
    octree = ResidencyOctree(OctreeConfig(depth=depth, channel_slots=m, homogeneity_eps=eps),
                             paging)
    return octree, paging


def insert(octree, paging, slot, level, coord, value=0, frame=1):
    """test_render_units.py:30-37"""
    bid = paging.encode(slot, level, coord)
    _, evicted = paging.insert_brick(bid, np.full((16, 16, 16), value, np.uint8), frame)
    if evicted is not None:
        octree.on_brick_evicted(evicted)
    octree.on_brick_inserted(bid)
    return bid


def set_meta_all(octree, slot, mn, mx, depth=3):
    """test_render_units.py:183-191 (one batched upload)"""
    from paper_2309_04393_b200.octree import total_nodes
    n = total_nodes(depth)
    octree.set_metadata_batch(np.arange(n), np.full(n, slot), np.full(n, mn), np.full(n, mx))


def node_index(d, x, y, z):
    from paper_2309_04393_b200.octree import NodeAddress
    return NodeAddress(d, x, y, z).index


def _tf40():
    from paper_2309_04393_b200 import grayscale_ramp_tf
    return grayscale_ramp_tf(threshold=40.0)


def _flat_tf(rgba):
    from paper_2309_04393_b200 import TransferFunction
    return TransferFunction(points=((0.0, tuple(rgba)), (255.0, tuple(rgba))))


def _used(out, paging, slot, level, coord) -> bool:
    return bool(out.required_mask[paging._entry_index(slot, level, coord)])


# -- compositing (test_render_units.py:98-138) ---------------------------------

def _composite_scene(m, rgba, level):
    """m channels, constant TF, every node (0, 255), the bricks under
    (0.4, 0.4, 0.4) resident at ``level`` for every slot."""
    from paper_2309_04393_b200 import ChannelSettings
    octree, paging = make_octree(m=m)
    for s in range(m):
        set_meta_all(octree, s, 0, 255)
        insert(octree, paging, s, level, paging.brick_coord_of(level, (0.4, 0.4, 0.4)), 77)
    chans = [ChannelSettings(slot=s, tf=_flat_tf(rgba)) for s in range(m)]
    return octree, paging, chans


def test_composite_single_channel_closed_form():
    """test_render_units.py:98-105: one sample over nothing = (r a, g a, b a, a)."""
    from paper_2309_04393_b200 import probe_sample
    octree, paging, chans = _composite_scene(1, (1.0, 0.5, 0.25, 0.4), 0)
    r = probe_sample(paging, octree, chans, (0.4, 0.4, 0.4), [0], 3, start_depth=0)
    assert r.sampled_levels == [0] and not r.skippable
    assert r.rgba == pytest.approx((0.4, 0.2, 0.1, 0.4), rel=1e-6)


def test_composite_opacity_correction():
    """test_render_units.py:108-117: a step twice the base step (desired
    level 1) doubles optical depth, a = 1 - (1 - a0)^2, colour scaled alike."""
    from paper_2309_04393_b200 import probe_sample
    octree, paging, chans = _composite_scene(1, (1.0, 1.0, 1.0, 0.3), 1)
    r = probe_sample(paging, octree, chans, (0.4, 0.4, 0.4), [1], 3, start_depth=0)
    assert r.sampled_levels == [1]
    want = 1.0 - 0.7 ** 2
    assert r.rgba[3] == pytest.approx(want, rel=1e-6)
    assert r.rgba[0] == pytest.approx(want, rel=1e-6)


@pytest.mark.parametrize("m,a,level", [(1, 0.3, 0), (2, 0.25, 0), (2, 0.6, 1), (4, 0.1, 0),
                                       (4, 0.45, 2)])
def test_composite_channel_count_alpha(m, a, level):
    """test_render_units.py:120-126: m channels of equal opacity blend to
    1 - ((1 - a)^m)^ratio, ratio = 2^level."""
    from paper_2309_04393_b200 import probe_sample
    octree, paging, chans = _composite_scene(m, (0.5, 0.5, 0.5, a), level)
    r = probe_sample(paging, octree, chans, (0.4, 0.4, 0.4), [level] * m, 3, start_depth=0)
    assert r.sampled_levels == [level] * m
    want = 1.0 - ((1.0 - a) ** m) ** (2 ** level)
    assert r.rgba[3] == pytest.approx(want, abs=1e-6)   # f32 image of an fp64 composite


def test_composite_zero_alpha_noop():
    """test_render_units.py:129-131: zero-opacity channels composite nothing
    (and the sample is skippable: its channels resolve ZERO)."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging, _ = _composite_scene(2, (1.0, 1.0, 1.0, 0.0), 0)
    chans = [ChannelSettings(slot=0, tf=_flat_tf((1.0, 1.0, 1.0, 0.0))),
             ChannelSettings(slot=1, tf=_flat_tf((0.5, 0.0, 0.0, 0.0)))]
    r = probe_sample(paging, octree, chans, (0.4, 0.4, 0.4), [0, 0], 3, start_depth=0)
    assert r.rgba == (0.0, 0.0, 0.0, 0.0)
    assert r.skippable and r.sampled_levels == [None, None]


# -- alternative brick selection (test_render_units.py:143-176) ----------------

def test_alternative_prefers_nearest_then_coarser():
    """test_render_units.py:143-161: with the desired level missing the
    sample falls to the nearest resident level of the node, the coarser one
    on a tie; the desired brick is requested."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree(k=3)
    set_meta_all(octree, 0, 0, 255)
    chans = [ChannelSettings(slot=0, tf=_tf40())]
    pos = (0.1, 0.1, 0.1)
    r = probe_sample(paging, octree, chans, pos, [1], 3)
    assert r.sampled_levels == [None]                       # nothing resident
    assert r.brick_requests == [paging.encode(0, 1, (0, 0, 0))]
    insert(octree, paging, 0, 0, (0, 0, 0), 90)
    r = probe_sample(paging, octree, chans, pos, [1], 3)
    assert r.sampled_levels == [0] and _used(r.output, paging, 0, 0, (0, 0, 0))
    assert r.brick_requests == [paging.encode(0, 1, (0, 0, 0))]
    insert(octree, paging, 0, 2, (0, 0, 0), 90)
    r = probe_sample(paging, octree, chans, pos, [1], 3)
    assert r.sampled_levels == [2] and _used(r.output, paging, 0, 2, (0, 0, 0))
    insert(octree, paging, 0, 1, (0, 0, 0), 90)
    r = probe_sample(paging, octree, chans, pos, [1], 3)     # desired now resident
    assert r.sampled_levels == [1] and r.brick_requests == []
    paging.evict_bricks([paging.encode(0, 0, (0, 0, 0))], update_octree=True)
    r = probe_sample(paging, octree, chans, pos, [0], 3)     # desired 0 gone: nearest is 1
    assert r.sampled_levels == [1]
    assert r.brick_requests == [paging.encode(0, 0, (0, 0, 0))]


def test_alternative_respects_position_and_slot():
    """test_render_units.py:164-176: substitution looks at the sample's own
    bricks and the channel's own slot."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree(k=3)
    for s in range(2):
        set_meta_all(octree, s, 0, 255)
    insert(octree, paging, 1, 0, (3, 3, 3), 90)
    tf = _tf40()
    r = probe_sample(paging, octree, [ChannelSettings(slot=1, tf=tf)], (0.95, 0.95, 0.95),
                     [1], 3)
    assert r.sampled_levels == [0] and _used(r.output, paging, 1, 0, (3, 3, 3))
    r = probe_sample(paging, octree, [ChannelSettings(slot=0, tf=tf)], (0.95, 0.95, 0.95),
                     [1], 3)
    assert r.sampled_levels == [None]                         # other slot sees nothing
    r = probe_sample(paging, octree, [ChannelSettings(slot=1, tf=tf)], (0.99, 0.99, 0.99),
                     [1], 3)
    assert r.sampled_levels == [0] and _used(r.output, paging, 1, 0, (3, 3, 3))


# -- multi-channel traversal (test_render_units.py:194-269) --------------------

def test_traverse_empty_channel_resolves_at_start_depth():
    """test_render_units.py:194-203: ZERO at the start depth, one visit, no
    requests, skippable over node (1, 0, 0, 0): from x = 0.3 along +x the
    skip region ends at x = 0.5, i.e. 2 skipped samples of step 1/8 (the
    root would give 6)."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree()
    set_meta_all(octree, 0, 0, 10)
    r = probe_sample(paging, octree, [ChannelSettings(0, _tf40())], (0.3, 0.3, 0.3), [0], 3,
                     start_depth=1)
    assert r.steps == 1
    assert r.brick_requests == [] and r.metadata_requests == []
    assert r.skippable and r.sampled_levels == [None]
    assert r.output.stats.samples_skipped == 2 and r.output.stats.samples_evaluated == 0


def test_traverse_homogeneous_is_const():
    """test_render_units.py:206-214: a homogeneous node resolves CONST with
    value = node min (100), composited over the whole skip region (6 samples
    of step 1/8 from x = 0.3 to the root's exit)."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree(eps=2.0)
    set_meta_all(octree, 0, 100, 101)
    tf = _tf40()
    r = probe_sample(paging, octree, [ChannelSettings(0, tf)], (0.3, 0.3, 0.3), [0], 3,
                     start_depth=0)
    assert r.steps == 1 and r.skippable and r.sampled_levels == [None]
    a = tf.evaluate(100.0)[3]
    assert a > 0.0
    assert r.output.stats.samples_evaluated == 6
    assert r.rgba[3] == pytest.approx(1.0 - (1.0 - a) ** 6, rel=1e-6)


def test_traverse_invalid_metadata_requests_and_descends():
    """test_render_units.py:217-227: INVALID everywhere and nothing resident:
    metadata requested for the node visited, then the empty mask makes it an
    unmapped miss -- the desired brick is requested, the sample skippable."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree()
    r = probe_sample(paging, octree, [ChannelSettings(0, _tf40())], (0.9, 0.9, 0.9), [0], 3,
                     start_depth=2)
    assert r.metadata_requests == [(node_index(2, 3, 3, 3), 0)]
    assert r.brick_requests == [paging.encode(0, 0, (3, 3, 3))]
    assert r.sampled_levels == [None] and r.skippable


def test_traverse_descends_to_depth_limit_and_samples():
    """test_render_units.py:230-241: visits depths 1, 2, 3 and samples level
    0 brick (1, 1, 1); not skippable."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree()
    set_meta_all(octree, 0, 0, 255)
    insert(octree, paging, 0, 0, (1, 1, 1), value=50)
    r = probe_sample(paging, octree, [ChannelSettings(0, _tf40())], (0.4, 0.4, 0.4), [0], 3,
                     start_depth=1)
    assert r.steps == 3
    assert r.sampled_levels == [0] and _used(r.output, paging, 0, 0, (1, 1, 1))
    assert not r.skippable and r.brick_requests == []
    assert r.output.stats.samples_evaluated == 1 and r.output.stats.samples_skipped == 0


def test_traverse_shares_descent_across_channels():
    """test_render_units.py:244-256: channel 0 descends 1 -> 3 (3 visits);
    the empty channel 1 resolves at depth 3 in one more visit because the
    cursor never re-ascends: 4 visits, not skippable."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree(m=2)
    set_meta_all(octree, 0, 0, 255)
    set_meta_all(octree, 1, 0, 10)
    insert(octree, paging, 0, 0, (1, 1, 1), value=50)
    tf = _tf40()
    r = probe_sample(paging, octree, [ChannelSettings(0, tf), ChannelSettings(1, tf)],
                     (0.4, 0.4, 0.4), [0, 0], 3, start_depth=1)
    assert r.steps == 4
    assert r.sampled_levels == [0, None]
    assert not r.skippable


def test_traverse_miss_with_substitute_not_skippable():
    """test_render_units.py:259-269: desired level 0 missing -> requested,
    the level-1 substitute rendered; not skippable."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree()
    set_meta_all(octree, 0, 0, 255)
    insert(octree, paging, 0, 1, (0, 0, 0), value=80)
    r = probe_sample(paging, octree, [ChannelSettings(0, _tf40())], (0.3, 0.3, 0.3), [0], 3,
                     start_depth=0)
    assert r.brick_requests == [paging.encode(0, 0, (1, 1, 1))]
    assert r.sampled_levels == [1] and _used(r.output, paging, 0, 1, (0, 0, 0))
    assert not r.skippable


def test_probe_matches_oracle_first_sample():
    """The probe is the product ray caster, not a separate code path: a
    1-pixel full ray whose first sample is opaque (early termination after
    it) gives the same image / requests / counters as the probe."""
    from paper_2309_04393_b200 import (Camera, ChannelSettings, RenderConfig, probe_sample,
                                       render_frame)
    octree, paging, chans = _composite_scene(1, (0.2, 0.9, 0.4, 1.0), 0)
    pos = (0.4, 0.4, 0.4)
    r = probe_sample(paging, octree, chans, pos, [0], 3, start_depth=0)
    cfg = RenderConfig(image_dims=(1, 1), base_step=1.0 / 8.0, traversal_start_level=1)
    cam = Camera(position=pos, target=(1.4, 0.4, 0.4))
    chans0 = [ChannelSettings(slot=0, tf=chans[0].tf, level_range=(0, 0))]
    full = render_frame(paging, octree, chans0, cam, cfg)
    assert np.array_equal(full.image, r.output.image)
    assert full.stats.traversal_steps == r.steps
    assert full.brick_requests == r.brick_requests
    assert math.isclose(r.rgba[3], 1.0)


# -- sampling helpers (test_kernels.py:11-38, 122-145) -------------------------

def _value_scene(payload, coord=(1, 1, 1)):
    """One level-0 brick; TF alpha 1 everywhere with red = value / 255, so a
    single composited sample returns its interpolated value in the red
    channel."""
    from paper_2309_04393_b200 import ChannelSettings, TransferFunction
    octree, paging = make_octree(m=1)
    set_meta_all(octree, 0, 0, 255)
    bid = paging.encode(0, 0, coord)
    paging.insert_brick(bid, payload, 1)
    octree.on_brick_inserted(bid)
    tf = TransferFunction(points=((0.0, (0.0, 0.0, 0.0, 1.0)), (255.0, (1.0, 1.0, 1.0, 1.0))))
    return octree, paging, [ChannelSettings(slot=0, tf=tf)]


def _trilinear(brick, l):
    """kernels.py:137-180 restated: voxel centres at +0.5, clamped to the
    brick interior, x fastest."""
    B = brick.shape[0]
    f = [min(max(c - 0.5, 0.0), B - 1.0) for c in l]
    i0 = [int(v) for v in f]
    i1 = [min(v + 1, B - 1) for v in i0]
    t = [f[a] - i0[a] for a in range(3)]

    def lerp(a, b, w):
        return a + (b - a) * w

    def at(z, y, x):
        return float(brick[z, y, x])
    c00 = lerp(at(i0[2], i0[1], i0[0]), at(i0[2], i0[1], i1[0]), t[0])
    c10 = lerp(at(i0[2], i1[1], i0[0]), at(i0[2], i1[1], i1[0]), t[0])
    c01 = lerp(at(i1[2], i0[1], i0[0]), at(i1[2], i0[1], i1[0]), t[0])
    c11 = lerp(at(i1[2], i1[1], i0[0]), at(i1[2], i1[1], i1[0]), t[0])
    return lerp(lerp(c00, c10, t[1]), lerp(c01, c11, t[1]), t[2])


def test_trilinear_constant_brick_exact():
    """test_kernels.py:26-38: a constant brick samples to its value exactly
    anywhere, the brick faces included."""
    from paper_2309_04393_b200 import probe_sample
    octree, paging, chans = _value_scene(np.full((16, 16, 16), 173, np.uint8))
    for pos in ((0.25, 0.25, 0.25), (0.3, 0.4, 0.49), (0.499, 0.251, 0.37)):
        r = probe_sample(paging, octree, chans, pos, [0], 3, start_depth=0)
        assert r.sampled_levels == [0]
        assert r.rgba[0] == float(np.float32(173.0 / 255.0)) and r.rgba[3] == 1.0


def test_trilinear_matches_python_sampler():
    """test_kernels.py:11-23: the sampled value equals a plain-Python
    trilinear sampler at random positions inside the brick (read back
    through the f32 image, hence the 1e-6 tolerance)."""
    from paper_2309_04393_b200 import probe_sample
    rng = np.random.default_rng(5)
    brick = rng.integers(0, 256, size=(16, 16, 16), dtype=np.uint8)
    octree, paging, chans = _value_scene(brick)
    for _ in range(24):
        pos = tuple(float(v) for v in rng.uniform(0.25, 0.4999, 3))
        r = probe_sample(paging, octree, chans, pos, [0], 3, start_depth=0)
        want = _trilinear(brick, [p * 64.0 - 16.0 for p in pos]) / 255.0
        assert r.rgba[0] == pytest.approx(want, rel=1e-6, abs=1e-7), pos


def test_brick_coordinates_and_entries_match_paging():
    """test_kernels.py:122-145: the brick the kernel uses for a position is
    paging.brick_coord_of (clamped to the grid) and its usage-mask entry is
    paging's entry index, for every level."""
    from paper_2309_04393_b200 import ChannelSettings, probe_sample
    octree, paging = make_octree(m=1, k=3, cache=(4, 4, 4))
    set_meta_all(octree, 0, 0, 255)
    rng = np.random.default_rng(9)
    tf = _tf40()
    for lev in range(3):
        for _ in range(6):
            pos = tuple(float(v) for v in rng.uniform(0.0, 0.9999, 3))
            coord = paging.brick_coord_of(lev, pos)
            bid = paging.encode(0, lev, coord)
            if paging.resident_slot(bid) is None:
                paging.insert_brick(bid, np.full((16, 16, 16), 120, np.uint8), 1)
                octree.on_brick_inserted(bid)
            r = probe_sample(paging, octree, [ChannelSettings(0, tf)], pos, [lev], 3)
            assert r.sampled_levels == [lev]
            used = np.flatnonzero(r.output.required_mask)
            assert list(used) == [paging._entry_index(0, lev, coord)]
