"""Octree / paging query API of the mirror against the reference's own unit
tests (pkg/tests/test_octree.py:250-320 choose_metadata_level,
compute_metadata_vs_dense_scan, culling queries) and the Session's
metadata-from-bricks fallback (session.py:147-156)."""

import numpy as np
import pytest

from conftest import cuda_ok
import scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def make_octree(depth=3, m=2, k=3, cache=(3, 3, 3), eps=0.0, min_vox=1):
    """test_octree.py:15-23"""
    from paper_2309_04393_b200 import (MultiChannelPaging, OctreeConfig, PagingConfig,
                                       ResidencyOctree)
    config = PagingConfig(brick_size=(16, 16, 16), cache_slots=cache, m=m, k=k)
    dims = [(64, 64, 64), (32, 32, 32), (16, 16, 16)][:k]
    grids = [(4, 4, 4), (2, 2, 2), (1, 1, 1)][:k]
    paging = MultiChannelPaging(config, dims, grids)
    octree = ResidencyOctree(OctreeConfig(depth=depth, channel_slots=m, homogeneity_eps=eps,
                                          min_metadata_voxels=min_vox), paging)
    return octree, paging


def test_gpu_choose_metadata_level():
    from paper_2309_04393_b200 import NodeAddress
    octree, _ = make_octree(depth=3, k=3)
    assert octree.choose_metadata_level(NodeAddress(0, 0, 0, 0)) == 2
    assert octree.choose_metadata_level(NodeAddress(3, 0, 0, 0)) == 2
    octree2, _ = make_octree(depth=3, k=3, min_vox=64)
    assert octree2.choose_metadata_level(NodeAddress(3, 0, 0, 0)) == 1


def test_gpu_compute_metadata_vs_dense_scan():
    from paper_2309_04393_b200 import NodeAddress
    from paper_2309_04393_b200.volume import build_pyramid, plan_levels, shell_volume
    octree, _ = make_octree(depth=3, k=3)
    pyr = build_pyramid(shell_volume(64), plan_levels((64,) * 3, (16,) * 3, 3, (2, 2, 2)))
    levels_meta = [(64, 64, 64), (32, 32, 32), (16, 16, 16)]

    def fetch(slot, level, coord):
        x, y, z = coord
        return pyr[level][z * 16:(z + 1) * 16, y * 16:(y + 1) * 16, x * 16:(x + 1) * 16]

    rng = np.random.default_rng(1234)
    for _ in range(30):
        d = int(rng.integers(4))
        side = 1 << d
        addr = NodeAddress(d, *(int(rng.integers(side)) for _ in range(3)))
        mn, mx = octree.compute_node_metadata_from_bricks(addr, 0, fetch)
        level = octree.choose_metadata_level(addr)
        arr = pyr[level]
        n = levels_meta[level][0]
        lo = [(c * n) // side for c in (addr.z, addr.y, addr.x)]
        hi = [-(-((c + 1) * n) // side) for c in (addr.z, addr.y, addr.x)]
        part = arr[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
        assert (mn, mx) == (int(part.min()), int(part.max())), addr


def test_gpu_culling_queries():
    """test_octree.py:309-330 (is_empty / is_homogeneous)."""
    from paper_2309_04393_b200 import NodeAddress, grayscale_ramp_tf
    octree, _ = make_octree(eps=2.0)
    tf = grayscale_ramp_tf(threshold=40.0)
    addr = NodeAddress(1, 0, 0, 0)
    assert not octree.is_empty(addr, [0], {0: tf})      # INVALID -> not empty
    assert not octree.is_homogeneous(addr, [0])
    octree.set_node_metadata(addr, 0, 5, 39)
    assert octree.is_empty(addr, [0], {0: tf})
    assert not octree.is_homogeneous(addr, [0])
    octree.set_node_metadata(addr, 0, 38, 40)
    assert octree.is_homogeneous(addr, [0])
    octree.set_node_metadata(addr, 0, 38, 41)
    assert not octree.is_empty(addr, [0], {0: tf})


def test_gpu_overlapping_leaves_and_sample():
    from fractions import Fraction
    from paper_2309_04393_b200 import NodeAddress
    octree, paging = make_octree(depth=2)
    # open box (1/4, 1/2) x (0, 1/4) x (0, 1/4): exactly leaf x = 1 (faces do not count)
    got = octree.overlapping_leaves((Fraction(1, 4), 0, 0), (Fraction(1, 2), Fraction(1, 4),
                                                             Fraction(1, 4)))
    assert got == [NodeAddress(2, 1, 0, 0)]
    assert len(octree.overlapping_leaves((0, 0, 0), (1, 1, 1))) == 64
    # paging.sample: trilinear inside a slot (paging.py:241-261)
    pay = (np.arange(16 ** 3, dtype=np.int64) % 251).astype(np.uint8).reshape(16, 16, 16)
    slot, _ = paging.insert_brick(paging.encode(0, 0, (0, 0, 0)), pay, 0)
    v = paging.sample(slot, (3.5, 4.5, 5.5))
    assert v == float(pay[5, 4, 3])
    v2 = paging.sample(slot, (3.75, 4.5, 5.5))
    assert abs(v2 - (pay[5, 4, 3] + 0.25 * (float(pay[5, 4, 4]) - pay[5, 4, 3]))) < 1e-12


def test_gpu_session_metadata_from_bricks_fallback():
    """A plain-file server (no metadata endpoint): the session computes node
    metadata from bricks on the GPU and still converges."""
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, LocalTransport,
                                       RenderConfig, Session, grayscale_ramp_tf, orbit_pose)
    from paper_2309_04393_b200.volume import TransportError

    class PlainFiles(LocalTransport):
        metadata_supported = False

        def fetch_metadata(self, c, l, box):
            raise TransportError("metadata unsupported")

    st = scenes.store("shell64")
    sess = Session(PlainFiles(st), EngineConfig(octree_depth=3, cache_slots=(9, 9, 9),
                                                channel_slots=1),
                   RenderConfig(image_dims=(64, 64), base_step=1.0 / 64.0,
                                max_requests_per_frame=512),
                   [ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0))])
    recs = sess.run_until_converged(orbit_pose(0.3), max_frames=50)
    assert sess.converged
    assert sum(r.metadata_applied for r in recs) > 0
    assert recs[-1].output.image[..., 3].max() > 0
    sess.close()
