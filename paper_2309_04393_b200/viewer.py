"""Frame streaming for interactive viewers.

The reference's viewer protocol (viewer_service.py:1-141): JSON messages
change the viewing state (camera, channels, render config); after each
change the session steps its render / download loop until the image
converges (bounded per update) and streams, per step, a PNG frame and a
stats message.  This module is that protocol state machine, transport
agnostic (the reference drives it from a FastAPI WebSocket; a socket
server is networking, out of scope here -- any host loop can feed
``SessionDriver.handle`` and forward its replies).  Every frame is rendered
by the CUDA ray caster through ``Session``; PNG encoding is
``session.image_to_png_bytes``.

Messages in:  set_camera {position, target?, up?, fov?}
              set_channels {channels: [{slot, channel?, tf, levelRange?}]}
              set_config {imageDims?, baseStep?, maxRequests?}
Messages out: frame {frameId, pngBytes (base64)}
              stats {frameId, requests, residentBricks, residentBytes,
                     converged, renderMs}
              error {message}
"""

from __future__ import annotations

import base64
from dataclasses import replace

from .camera import Camera
from .engine import EngineConfig
from .render import ChannelSettings, RenderConfig
from .session import Session, image_to_png_bytes
from .transfer import TransferFunction, grayscale_ramp_tf


class ProtocolError(ValueError):
    pass


def parse_tf(points) -> TransferFunction:
    """[[scalar, [r, g, b, a]], ...] -> TransferFunction (viewer_service.py:39-45)."""
    try:
        knots = tuple((float(p[0]), tuple(float(c) for c in p[1])) for p in points)
    except (TypeError, ValueError, IndexError) as exc:
        raise ProtocolError(f"malformed transfer function: {exc}") from exc
    return TransferFunction(points=knots)


def parse_channels(spec, engine_config: EngineConfig):
    """viewer_service.py:48-61: the visible channels and the requested
    slot -> dataset channel mapping ({} when no entry names a channel)."""
    channels, mapping = [], {}
    for entry in spec:
        slot = int(entry["slot"])
        lo, hi = entry.get("levelRange", (0, 15))
        channels.append(ChannelSettings(slot=slot, tf=parse_tf(entry["tf"]),
                                        level_range=(int(lo), int(hi))))
        if "channel" in entry:
            mapping[slot] = int(entry["channel"])
    return channels, mapping


def parse_camera(msg) -> Camera:
    """viewer_service.py:64-72 (target / up / fov default to the orbit view)."""
    try:
        vec = lambda key, default: tuple(float(v) for v in msg.get(key, default))  # noqa: E731
        return Camera(position=tuple(float(v) for v in msg["position"]),
                      target=vec("target", (0.5, 0.5, 0.5)),
                      up=vec("up", (0.0, 1.0, 0.0)),
                      fov_deg=float(msg.get("fov", 45.0)))
    except (KeyError, TypeError, ValueError) as exc:
        raise ProtocolError(f"malformed camera: {exc}") from exc


class SessionDriver:
    """One viewer connection's session (viewer_service.py:75-141)."""

    def __init__(self, transport, engine_config: EngineConfig,
                 render_config: RenderConfig, channels=None,
                 max_frames_per_update: int = 50, **session_kw):
        if channels is None:
            channels = [ChannelSettings(slot=0, tf=grayscale_ramp_tf(1.0))]
        self.session = Session(transport, engine_config, render_config, channels,
                               **session_kw)
        self.camera: Camera | None = None
        self.max_frames = int(max_frames_per_update)
        self._handlers = {"set_camera": self._set_camera,
                          "set_channels": self._set_channels,
                          "set_config": self._set_config}

    # -- message handlers -----------------------------------------------------

    def _set_camera(self, msg):
        self.camera = parse_camera(msg)

    def _set_channels(self, msg):
        channels, mapping = parse_channels(msg["channels"], self.session.engine.config)
        current = self.session.engine.paging.channel_mapping
        for slot, dataset_channel in mapping.items():
            if current[slot] != dataset_channel:
                self.session.swap_channel(slot, dataset_channel)
        self.session.set_channels(channels)

    def _set_config(self, msg):
        cfg = self.session.render_config
        if "imageDims" in msg:
            cfg = replace(cfg, image_dims=tuple(int(v) for v in msg["imageDims"]))
        if "baseStep" in msg:
            cfg = replace(cfg, base_step=float(msg["baseStep"]))
        if "maxRequests" in msg:
            cfg = replace(cfg, max_requests_per_frame=int(msg["maxRequests"]))
        self.session.set_render_config(cfg)

    def handle(self, msg) -> list:
        """Apply one message, then stream until converged; returns the
        outgoing messages (a single error message if the input is bad)."""
        if not isinstance(msg, dict) or "type" not in msg:
            return [{"type": "error", "message": "message needs a type"}]
        handler = self._handlers.get(msg["type"])
        if handler is None:
            return [{"type": "error", "message": f"unknown message type {msg['type']!r}"}]
        try:
            handler(msg)
        except (ProtocolError, KeyError, TypeError, ValueError) as exc:
            return [{"type": "error", "message": str(exc)}]
        return self.render_until_converged()

    def _messages(self, rec) -> tuple:
        """The frame + stats pair streamed for one session step."""
        ws = self.session.working_set()
        st = rec.output.stats
        frame = dict(type="frame", frameId=rec.frame_id,
                     pngBytes=base64.b64encode(image_to_png_bytes(rec.output.image))
                     .decode("ascii"))
        stats = dict(type="stats", frameId=rec.frame_id, requests=st.requests_issued,
                     residentBricks=ws["resident_bricks"], residentBytes=ws["resident_bytes"],
                     converged=self.session.converged, renderMs=st.render_ms)
        return frame, stats

    def render_until_converged(self) -> list:
        """viewer_service.py:123-141: at most max_frames session steps,
        stopping after the first converged one; nothing before a camera."""
        out = []
        steps = self.max_frames if self.camera is not None else 0
        while steps > 0:
            steps -= 1
            out.extend(self._messages(self.session.step_frame(self.camera)))
            if self.session.converged:
                break
        return out

    def close(self):
        self.session.close()
