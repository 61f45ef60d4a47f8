"""Session semantics restated from the reference's pkg/tests/test_session.py
(convergence, plain-file metadata fallback, transport retries and drops,
channel swaps and TF changes, PNG frames), on the GPU-resident engine."""

import struct
import zlib

import numpy as np
import pytest

from conftest import cuda_ok
import scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def _cfg():
    from paper_2309_04393_b200 import (ChannelSettings, EngineConfig, RenderConfig,
                                       grayscale_ramp_tf, orbit_pose)
    return (EngineConfig(octree_depth=3, cache_slots=(8, 8, 8), channel_slots=2),
            RenderConfig(image_dims=(64, 64), base_step=1.0 / 64.0,
                         max_requests_per_frame=512, traversal_start_level=2),
            [ChannelSettings(slot=0, tf=grayscale_ramp_tf(threshold=40.0))],
            orbit_pose(0.7))


def _session(transport, **kw):
    from paper_2309_04393_b200 import Session
    e, r, c, _ = _cfg()
    return Session(transport, e, r, c, **kw)


class _Flaky:
    """Fails every brick fetch `failures` times before serving it."""

    def __init__(self, inner, failures):
        self.inner, self.failures, self.seen = inner, failures, {}
        self.metadata_supported = True

    @property
    def manifest(self):
        return self.inner.manifest

    def fetch_brick(self, c, l, coord):
        from paper_2309_04393_b200.volume import TransportError
        n = self.seen.get((c, l, coord), 0)
        if n < self.failures:
            self.seen[(c, l, coord)] = n + 1
            raise TransportError("synthetic drop")
        return self.inner.fetch_brick(c, l, coord)

    def fetch_metadata(self, c, l, box):
        return self.inner.fetch_metadata(c, l, box)

    def close(self):
        pass


def test_channel_slot_validated():
    """test_session.py:24-27"""
    from paper_2309_04393_b200 import (ChannelSettings, LocalTransport, Session,
                                       grayscale_ramp_tf)
    from paper_2309_04393_b200.session import SessionError
    e, r, _, _ = _cfg()
    with pytest.raises(SessionError):
        Session(LocalTransport(scenes.store("shell64")), e, r,
                [ChannelSettings(slot=5, tf=grayscale_ramp_tf(40.0))])


def test_converges_with_working_set():
    """test_session.py:30-45"""
    from paper_2309_04393_b200 import LocalTransport
    pose = _cfg()[3]
    s = _session(LocalTransport(scenes.store("shell64")))
    recs = s.run_until_converged(pose)
    assert s.converged and len(recs) < 50
    assert recs[0].output.stats.requests_issued > 0
    assert recs[-1].output.stats.requests_issued == 0
    assert recs[-1].image_digest == recs[-2].image_digest
    assert recs[-1].output.image[..., 3].max() > 0.5
    ws = s.working_set()
    assert ws["resident_bricks"] > 0 and ws["resident_bytes"] == ws["resident_bricks"] * 16 ** 3
    s.close()


def test_plain_file_metadata_fallback_is_nearly_identical():
    """test_session.py:60-79: metadata from bricks (coarser, undilated
    footprint) culls slightly differently at node borders only."""
    from paper_2309_04393_b200 import LocalTransport
    from paper_2309_04393_b200.volume import TransportError
    pose = _cfg()[3]

    class Plain(LocalTransport):
        metadata_supported = False

        def fetch_metadata(self, c, l, box):
            raise TransportError("501")

    plain = _session(Plain(scenes.store("shell64")))
    plain.run_until_converged(pose)
    assert plain.converged and sum(r.metadata_applied for r in plain.history) > 0
    full = _session(LocalTransport(scenes.store("shell64")))
    full.run_until_converged(pose)
    a, b = plain.history[-1].output.image, full.history[-1].output.image
    assert np.abs(a - b).mean() < 1e-3
    assert (np.abs(a - b).max(axis=-1) > 1e-6).mean() < 0.01
    plain.close()
    full.close()


def test_retries_recover_and_persistent_failures_drop():
    """test_session.py:109-125"""
    from paper_2309_04393_b200 import LocalTransport
    pose = _cfg()[3]
    st = scenes.store("shell64")
    s = _session(_Flaky(LocalTransport(st), failures=2), retries=3, backoff=0.0)
    recs = s.run_until_converged(pose)
    clean = _session(LocalTransport(st))
    clean.run_until_converged(pose)
    assert s.converged
    assert np.array_equal(recs[-1].output.image, clean.history[-1].output.image)
    bad = _session(_Flaky(LocalTransport(st), failures=10), retries=2, backoff=0.0)
    rec = bad.step_frame(pose)
    assert rec.bricks_applied == 0
    assert rec.requests_dropped >= len(rec.output.brick_requests)
    for x in (s, clean, bad):
        x.close()


def test_set_channels_rerenders():
    """test_session.py:144-152"""
    from paper_2309_04393_b200 import ChannelSettings, LocalTransport, grayscale_ramp_tf
    pose = _cfg()[3]
    s = _session(LocalTransport(scenes.store("shell64")))
    s.run_until_converged(pose)
    before = s.history[-1].output.image.copy()
    s.set_channels([ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0, max_alpha=0.3))])
    assert not s.converged
    s.run_until_converged(pose)
    assert not np.array_equal(before, s.history[-1].output.image)
    s.close()


def test_png_roundtrip():
    """test_session.py:155-164 (decoded with zlib instead of PIL)."""
    from paper_2309_04393_b200.session import image_to_png_bytes
    img = np.random.default_rng(0).random((16, 24, 4)).astype(np.float32)
    png = image_to_png_bytes(img)
    assert png[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat, w = 8, b"", 0
    while pos < len(png):
        n = struct.unpack(">I", png[pos:pos + 4])[0]
        tag, data = png[pos + 4:pos + 8], png[pos + 8:pos + 8 + n]
        if tag == b"IHDR":
            w, h = struct.unpack(">II", data[:8])
        elif tag == b"IDAT":
            idat += data
        pos += 12 + n
    rows = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(h, 1 + 4 * w)
    back = rows[:, 1:].reshape(h, w, 4)
    assert back.shape == (16, 24, 4)
    assert np.array_equal(back, np.clip(np.rint(img * 255), 0, 255).astype(np.uint8))


def test_held_frame_outputs_are_never_overwritten():
    """render_frame recycles its pinned result buffers only once every array
    of an earlier FrameOutput is dropped: outputs a caller keeps (the
    session history does) stay intact across later frames."""
    from paper_2309_04393_b200 import (ChannelSettings, methods, orbit_pose, render_frame,
                                       grayscale_ramp_tf)
    from paper_2309_04393_b200.render import RenderConfig
    st = scenes.store("shell64")
    eng = methods.prepare_engine(st, {0: 0}, methods.full_engine_config(st, 1, 3))
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0))]
    cfg = RenderConfig(image_dims=(64, 48), base_step=1.0 / 64.0)
    outs, snaps = [], []
    for a in (0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 0.5):
        o = render_frame(eng.paging, eng.octree, chans, orbit_pose(a), cfg)
        outs.append(o)
        snaps.append((o.image.copy(), o.required_mask.copy(), o.pixel_required.copy()))
    for o, (img, req, pix) in zip(outs, snaps):
        assert np.array_equal(o.image, img)
        assert np.array_equal(o.required_mask, req)
        assert np.array_equal(o.pixel_required, pix)
    assert not np.array_equal(snaps[0][0], snaps[3][0])   # poses differ
    # held outputs beyond the pool depth came from the staging set (copies)
    from paper_2309_04393_b200 import render as R
    assert max(R._RESULTS._count.values()) <= R._RESULTS.depth
    # dropped outputs are recycled: the steady state allocates nothing new
    import gc
    del outs, o
    gc.collect()
    before = dict(R._RESULTS._count)
    for _ in range(5):
        render_frame(eng.paging, eng.octree, chans, orbit_pose(0.2), cfg)
    assert R._RESULTS._count == before
