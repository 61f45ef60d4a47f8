"""Viewer protocol message parsing (viewer_service.py:39-72), CPU only;
restates the parsing half of the reference's test_viewer_protocol.py."""

import pytest

from paper_2309_04393_b200.engine import EngineConfig
from paper_2309_04393_b200.viewer import ProtocolError, parse_camera, parse_channels, parse_tf

RAMP = [[40.0, [0, 0, 0, 0]], [255.0, [1, 1, 1, 1]]]


def test_tf_messages():
    assert parse_tf(RAMP).opacity(255.0) == 1.0 and parse_tf(RAMP).opacity(40.0) == 0.0
    for bad in ([["x", [0, 0, 0, 0]]], "nope", [[1.0]], None):
        with pytest.raises(ProtocolError):
            parse_tf(bad)


def test_camera_messages():
    cam = parse_camera({"position": [0, 0, 3]})
    assert cam.target == (0.5, 0.5, 0.5) and cam.up == (0.0, 1.0, 0.0)
    assert cam.fov_deg == 45.0
    cam = parse_camera({"position": [1, 2, 3], "target": [0, 0, 0], "fov": 30})
    assert cam.position == (1.0, 2.0, 3.0) and cam.fov_deg == 30.0
    for bad in ({}, {"position": "abc"}, {"position": [0.5, 0.5, 0.5]},
                {"position": [0, 0, 3], "fov": 200}):
        with pytest.raises(ProtocolError):
            parse_camera(bad)


def test_channel_messages():
    chans, mapping = parse_channels(
        [{"slot": 1, "channel": 3, "tf": RAMP, "levelRange": [2, 2]},
         {"slot": 0, "tf": RAMP}], EngineConfig(channel_slots=2))
    assert [c.slot for c in chans] == [1, 0]
    assert chans[0].level_range == (2, 2) and chans[1].level_range == (0, 15)
    assert mapping == {1: 3}
