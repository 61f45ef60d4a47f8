"""Frame streaming: the viewer protocol state
machine over a GPU session, restating the socket tests of the reference's
test_viewer_protocol.py:80-160 against SessionDriver directly (the socket
server itself is networking, not rebuilt)."""

import base64
import struct
import zlib

import numpy as np
import pytest

from conftest import cuda_ok
import scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

RAMP = [[40.0, [0, 0, 0, 0]], [255.0, [1, 1, 1, 1]]]
CAMERA = {"type": "set_camera", "position": [2.0, 0.85, 1.9]}
CHANNELS = {"type": "set_channels", "channels": [{"slot": 0, "channel": 0, "tf": RAMP}]}
FRAME_KEYS = {"type", "frameId", "pngBytes"}
STATS_KEYS = {"type", "frameId", "requests", "residentBricks", "residentBytes",
              "converged", "renderMs"}


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


@pytest.fixture()
def driver():
    from paper_2309_04393_b200 import EngineConfig, LocalTransport, RenderConfig
    from paper_2309_04393_b200.viewer import SessionDriver
    d = SessionDriver(LocalTransport(scenes.store("shell64")),
                      EngineConfig(octree_depth=3, cache_slots=(8, 8, 8), channel_slots=2),
                      RenderConfig(image_dims=(48, 48), base_step=1.0 / 64.0,
                                   max_requests_per_frame=512, traversal_start_level=2))
    yield d
    d.close()


def send(driver, *msgs):
    out = []
    for m in msgs:
        out.extend(driver.handle(m))
    return out


def decode_png(b64):
    png = base64.b64decode(b64)
    assert png[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat = 8, b""
    while pos < len(png):
        n = struct.unpack(">I", png[pos:pos + 4])[0]
        tag, data = png[pos + 4:pos + 8], png[pos + 8:pos + 8 + n]
        if tag == b"IHDR":
            w, h, depth, ctype = struct.unpack(">IIBB", data[:10])
            assert depth == 8 and ctype == 6            # 8-bit RGBA
        elif tag == b"IDAT":
            idat += data
        pos += 12 + n
    rows = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(h, 1 + 4 * w)
    return rows[:, 1:].reshape(h, w, 4)


def test_streams_schema_valid_frames_until_converged(driver):
    replies = send(driver, CHANNELS, CAMERA)
    frames = [r for r in replies if r["type"] == "frame"]
    stats = [r for r in replies if r["type"] == "stats"]
    assert frames and len(frames) == len(stats)
    assert all(set(f) == FRAME_KEYS for f in frames)
    assert all(set(s) == STATS_KEYS for s in stats)
    ids = [f["frameId"] for f in frames]
    assert ids == sorted(set(ids)) and [s["frameId"] for s in stats] == ids
    for s in stats:
        assert isinstance(s["converged"], bool)
        assert s["residentBytes"] == s["residentBricks"] * 16 ** 3
    assert stats[-1]["converged"] and stats[-1]["requests"] == 0
    assert not any(s["converged"] for s in stats[:-1])


def test_frames_are_rgba_pngs_of_the_rendered_image(driver):
    replies = send(driver, CHANNELS, CAMERA)
    img = decode_png([r for r in replies if r["type"] == "frame"][-1]["pngBytes"])
    assert img.shape == (48, 48, 4) and img[..., 3].max() > 0
    last = driver.session.history[-1].output.image
    assert np.array_equal(img, np.clip(np.rint(last * 255), 0, 255).astype(np.uint8))


def test_camera_alone_renders_with_the_default_channel(driver):
    assert any(r["type"] == "frame" for r in send(driver, CAMERA))


def test_state_changes_restream_with_later_frame_ids(driver):
    first = send(driver, CHANNELS, CAMERA)
    last_id = [r for r in first if r["type"] == "frame"][-1]["frameId"]
    dim = {"type": "set_channels", "channels": [
        {"slot": 0, "channel": 0, "tf": [[40.0, [0, 0, 0, 0]], [255.0, [1, 1, 1, 0.3]]]}]}
    second = send(driver, dim)
    ids = [r["frameId"] for r in second if r["type"] == "frame"]
    assert ids and min(ids) > last_id
    assert [r for r in first if r["type"] == "frame"][-1]["pngBytes"] != \
        [r for r in second if r["type"] == "frame"][-1]["pngBytes"]
    replies = send(driver, {"type": "set_config", "imageDims": [32, 24]})
    img = decode_png([r for r in replies if r["type"] == "frame"][-1]["pngBytes"])
    assert img.shape == (24, 32, 4)


def test_bad_messages_reply_errors_and_keep_the_session(driver):
    for bad in ("not a dict", {"no": "type"}, {"type": "bogus"},
                {"type": "set_camera", "position": [0.5, 0.5, 0.5]},
                {"type": "set_channels", "channels": [{"slot": 0}]}):
        replies = driver.handle(bad)
        assert len(replies) == 1 and replies[0]["type"] == "error"
    assert "bogus" in driver.handle({"type": "bogus"})[0]["message"]
    assert any(r["type"] == "frame" for r in send(driver, CHANNELS, CAMERA))
