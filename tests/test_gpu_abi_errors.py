"""Error paths of the C ABI: invalid arguments return RO_EINVAL (or another
negative code) with a message from ro_last_error(), never a crash or a
silent success; the context stays usable afterwards."""

import ctypes as C

import numpy as np
import pytest

from conftest import cuda_ok
import scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def _err(rc):
    from paper_2309_04393_b200 import _native as N
    assert rc < 0, rc
    msg = N.lib().ro_last_error().decode()
    assert msg, "missing error message"
    return msg


def test_gpu_abi_rejects_bad_arguments():
    from paper_2309_04393_b200 import (ChannelSettings, Engine, EngineConfig, RenderConfig,
                                       grayscale_ramp_tf, orbit_pose, render_frame)
    from paper_2309_04393_b200 import _native as N
    from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass
    lib = N.lib()
    st = scenes.store("mc64")
    eng = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=2))
    p = eng.paging
    ctx = p.ctx
    state = p.state()
    s = N.stream_ptr()
    # layout validation
    bad = p.layout()
    bad.k = 0
    h = C.c_void_p()
    assert "k" in _err(lib.ro_create(C.byref(bad), C.byref(h)))
    # null context / state pointers
    assert _err(lib.ro_sync(None, s))
    empty = N.State()
    assert "state" in _err(lib.ro_note_sampled(ctx, C.byref(empty), None, 1, s))
    # brick ids outside the layout
    ids = np.array([(1 << 32) + 5], dtype=np.int64)
    pay = np.zeros((1, 16, 16, 16), np.uint8)
    assert _err(lib.ro_apply_bricks(ctx, C.byref(state), ids.ctypes.data, 1, pay.ctypes.data,
                                    0, 1, 1, None, None, s))
    ids = np.array([p.encode(0, 0, (0, 0, 0)) | (7 << 24)], dtype=np.int64)  # slot >= m
    assert _err(lib.ro_apply_bricks(ctx, C.byref(state), ids.ctypes.data, 1, pay.ctypes.data,
                                    0, 1, 1, None, None, s))
    # metadata: min > max, slot out of range
    node = np.array([3], np.int64)
    sl, mn, mx = np.array([0], np.int32), np.array([9], np.int32), np.array([3], np.int32)
    assert _err(lib.ro_apply_metadata(ctx, C.byref(state), node.ctypes.data, sl.ctypes.data,
                                      mn.ctypes.data, mx.ctypes.data, 1, s))
    sl[0], mn[0], mx[0] = 5, 1, 2
    assert _err(lib.ro_apply_metadata(ctx, C.byref(state), node.ctypes.data, sl.ctypes.data,
                                      mn.ctypes.data, mx.ctypes.data, 1, s))
    # swap / level metadata on bad slots
    assert _err(lib.ro_swap_channel(ctx, C.byref(state), 7, 1, s))
    # render: bad mode, bad partition, n_ch, TF points, classic without metadata
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(40.0))]
    cfg = RenderConfig(image_dims=(16, 12), base_step=1 / 64, max_requests_per_frame=16)
    fp = FramePass(MODE_RESIDENCY, p, eng.octree, chans, orbit_pose(0.5), cfg)
    for field, value, expect in (("mode", 9, "mode"), ("n_parts", 0, "partition"),
                                 ("n_ch", 0, "n_ch"), ("width", 0, "image"),
                                 ("mode", 3, "classic")):
        old = getattr(fp.frame, field)
        setattr(fp.frame, field, value)
        msg = _err(lib.ro_render(ctx, C.byref(fp.frame), C.byref(fp.state),
                                 C.byref(fp.buf.outputs), s))
        assert expect in msg, (field, msg)
        setattr(fp.frame, field, old)
    fp.frame.ch[0].npoints = 99
    assert "transfer" in _err(lib.ro_render(ctx, C.byref(fp.frame), C.byref(fp.state),
                                            C.byref(fp.buf.outputs), s))
    fp.frame.ch[0].npoints = len(chans[0].tf.points)
    # pageable host memory is not a valid image target
    host = np.zeros((16 * 12, 4), np.float32)
    outs = N.Outputs(host.ctypes.data, fp.buf.required.data_ptr(), fp.buf.pix_required.data_ptr(),
                     fp.buf.hist.data_ptr(), fp.buf.counters.data_ptr())
    assert "pinned" in _err(lib.ro_render(ctx, C.byref(fp.frame), C.byref(fp.state),
                                          C.byref(outs), s))
    # LZ4: a frame that does not decode to one brick
    from paper_2309_04393_b200 import ingest
    f = ingest.compress(bytes(100))
    buf, offs = ingest.pack_frames([f])
    ids = np.array([p.encode(0, 0, (0, 0, 0))], np.int64)
    msg = _err(lib.ro_apply_bricks_lz4(ctx, C.byref(state), ids.ctypes.data, 1, buf.ctypes.data,
                                       offs.ctypes.data, 0, 1, 1, None, None, s))
    assert "size" in msg
    # the context is still usable: a normal frame renders
    out = render_frame(p, eng.octree, chans, orbit_pose(0.5), cfg)
    assert out.image.shape == (12, 16, 4)
    p.check_bijection()


def test_gpu_abi_pinned_payload_error_leaves_context_usable():
    """ro_apply_bricks with page-locked payloads (direct DMA from the
    caller's buffer) and a brick id outside the layout: error code +
    message, nothing inserted, and the same pinned buffer then uploads a
    valid batch correctly."""
    import torch
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200 import _native as N
    lib = N.lib()
    st = scenes.store("mc64")
    eng = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=2))
    p = eng.paging
    state = p.state()
    s = N.stream_ptr()
    pay = torch.empty((2, 16, 16, 16), dtype=torch.uint8, pin_memory=True)
    pay.copy_(torch.arange(2 * 16 ** 3, dtype=torch.int64).remainder(251).to(torch.uint8)
              .view(2, 16, 16, 16))
    good = p.encode(0, 0, (0, 0, 0))
    ids = np.array([good, (1 << 32) + 5], dtype=np.int64)
    assert _err(lib.ro_apply_bricks(p.ctx, C.byref(state), ids.ctypes.data, 2,
                                    pay.data_ptr(), 0, 1, 1, None, None, s))
    assert p.resident_slot(good) is None
    ids = np.array([good, p.encode(1, 0, (1, 0, 0))], dtype=np.int64)
    eng.advance_frame()
    eng.apply_bricks(ids, pay)
    for i, bid in enumerate(ids):
        slot = p.resident_slot(int(bid))
        assert slot is not None
        assert np.array_equal(p.cache[slot], pay[i].numpy())


def test_gpu_abi_pageable_payload_error_leaves_feedback_intact():
    """ro_apply_bricks with PAGEABLE payloads (staged through the handle's
    pinned buffer, uploaded into their own scratch slot) and a bad id: the
    call fails before any copy is queued, nothing is inserted, and the next
    frame's request ordering and a following valid batch are unaffected
    (no late DMA can land in another call's scratch)."""
    from paper_2309_04393_b200 import (ChannelSettings, Engine, EngineConfig, RenderConfig,
                                       grayscale_ramp_tf, orbit_pose, render_frame)
    from paper_2309_04393_b200 import _native as N
    lib = N.lib()
    st = scenes.store("mc64")
    eng = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=2))
    p = eng.paging
    state = p.state()
    s = N.stream_ptr()
    pay = (np.arange(3 * 16 ** 3, dtype=np.int64) % 249).astype(np.uint8).reshape(3, 16, 16, 16)
    good = p.encode(0, 0, (0, 0, 0))
    ids = np.array([good, p.encode(1, 0, (1, 0, 0)), (1 << 33) + 7], dtype=np.int64)
    msg = _err(lib.ro_apply_bricks(p.ctx, C.byref(state), ids.ctypes.data, 3,
                                   pay.ctypes.data, 0, 1, 1, None, None, s))
    assert "index 2" in msg
    assert p.resident_slot(good) is None
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(20.0))]
    cfg = RenderConfig(image_dims=(16, 12), base_step=1 / 64, max_requests_per_frame=64)
    a = render_frame(p, eng.octree, chans, orbit_pose(0.5), cfg)
    b = render_frame(p, eng.octree, chans, orbit_pose(0.5), cfg)
    assert a.brick_requests == b.brick_requests and a.metadata_requests == b.metadata_requests
    eng.advance_frame()
    eng.apply_bricks(ids[:2], pay[:2])
    for i, bid in enumerate(ids[:2]):
        slot = p.resident_slot(int(bid))
        assert slot is not None and np.array_equal(p.cache[slot], pay[i])


def test_gpu_render_without_collect_leaves_no_stale_requests():
    """A ray-cast pass whose requests were never collected (ro_render alone,
    render_frame_device(collect=False)) must not leak its first-seen keys
    into the next frame's ordered lists."""
    from paper_2309_04393_b200 import (ChannelSettings, Engine, EngineConfig, RenderConfig,
                                       grayscale_ramp_tf, orbit_pose, render_frame)
    from paper_2309_04393_b200.render import MODE_RESIDENCY, render_frame_device
    st = scenes.store("mc64")
    eng = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=2))
    chans = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(20.0)),
             ChannelSettings(slot=1, tf=grayscale_ramp_tf(30.0))]
    cfg = RenderConfig(image_dims=(24, 16), base_step=1 / 64, max_requests_per_frame=64)
    want = render_frame(eng.paging, eng.octree, chans, orbit_pose(2.5), cfg)
    render_frame_device(MODE_RESIDENCY, eng.paging, eng.octree, chans, orbit_pose(0.4), cfg,
                        collect=False)
    got = render_frame(eng.paging, eng.octree, chans, orbit_pose(2.5), cfg)
    assert got.brick_requests == want.brick_requests
    assert got.metadata_requests == want.metadata_requests
