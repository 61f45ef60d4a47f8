"""B200-native residency-octree render path (arXiv 2309.04393).

Drop-in for the reference ``resoctree`` render path: same Python API
(``render_frame``, ``render_reference``, ``Engine``, ``Session``,
``MultiChannelPaging``, ``ResidencyOctree``), state resident in HBM, and the
work done by hand-written sm_100a kernels in ``libresoct.so`` (C ABI:
``include/resoct.h``).  There is no CPU fallback.
"""

from .camera import Camera, generate_rays, orbit_path, orbit_pose  # noqa: F401
from .engine import Engine, EngineConfig, EngineError  # noqa: F401
from .octree import (INVALID_WORD, NodeAddress, OctreeConfig,  # noqa: F401
                     OctreeError, ResidencyOctree, level_offset, node_from_index,
                     total_nodes)
from .paging import (EMPTY, MAPPED, UNMAPPED, MultiChannelPaging,  # noqa: F401
                     PagingConfig, PagingError, decode_brick_id, encode_brick_id)
from .render import (ChannelSettings, ClassicMetadata, FrameOutput,  # noqa: F401
                     FrameStats, RenderConfig, RenderError, SampleProbe, probe_sample,
                     render_classic_octree, render_frame, render_frame_part,
                     render_pagetable_only, render_reference)
from .session import FrameRecord, Session  # noqa: F401
from .viewer import ProtocolError, SessionDriver  # noqa: F401
from .transfer import (TransferFunction, grayscale_ramp_tf,  # noqa: F401
                       transparent_tf)
from .volume import LocalTransport, VolumeStore  # noqa: F401

__version__ = "0.1.0"
