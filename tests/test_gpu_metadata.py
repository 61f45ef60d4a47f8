"""GPU culling-metadata producer against the
reference's definitions: per-node region_min_max over the dilated
metadata_box (service.py:102-115, engine.py:109-127) and the per-level
_box_minmax_grid (engine.py:186-219; restated in volume.box_minmax_grid and
pinned through the golden octree-word hashes)."""

import numpy as np
import pytest

from conftest import cuda_ok, load_golden
import scenes
from gpu_helpers import device_state_hashes, diff_hashes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module", autouse=True)
def _lib(native_lib):
    return native_lib


def _region_min_max(vol, box):
    """service.py:102-115, restated."""
    nz, ny, nx = vol.shape
    x0, y0, z0, x1, y1, z1 = box
    x0, y0, z0 = max(0, x0), max(0, y0), max(0, z0)
    x1, y1, z1 = min(nx, x1), min(ny, y1), min(nz, z1)
    if x0 >= x1 or y0 >= y1 or z0 >= z1:
        return 0, 0
    part = vol[z0:z1, y0:y1, x0:x1]
    return int(part.min()), int(part.max())


@pytest.mark.parametrize("shape,pad", [((64, 64, 64), 6), ((37, 50, 21), 3), ((9, 130, 17), 0),
                                       ((5, 5, 5), 20)])
def test_gpu_node_minmax_equals_region_min_max(shape, pad):
    from paper_2309_04393_b200.metadata import node_minmax
    from paper_2309_04393_b200.volume import box_minmax_grid
    rng = np.random.default_rng(sum(shape) + pad)
    vol = rng.integers(0, 256, size=shape, dtype=np.uint8)
    vol[:, :, : shape[2] // 3] //= 7   # uneven ranges
    nz, ny, nx = shape
    for d in range(0, 5):
        side = 1 << d
        mn, mx = (t.cpu().numpy().reshape(side, side, side) for t in node_minmax(vol, d, pad))
        gm, gx = box_minmax_grid(vol, side, pad)
        assert np.array_equal(mn, gm) and np.array_equal(mx, gx), d
        # spot-check against the per-request definition
        for _ in range(20):
            x, y, z = (int(v) for v in rng.integers(0, side, 3))
            box = []
            for a, n in ((x, nx), (y, ny), (z, nz)):
                box.append((a * n) // side - pad)
            for a, n in ((x, nx), (y, ny), (z, nz)):
                box.append(-((-(a + 1) * n) // side) + pad)
            assert (int(mn[z, y, x]), int(mx[z, y, x])) == _region_min_max(vol, box)


def test_gpu_session_device_metadata_matches_reference():
    """session_mc64 golden (cold start dominated by metadata requests) with
    the requests answered from the GPU min/max pyramid."""
    from paper_2309_04393_b200 import Camera, EngineConfig, LocalTransport, Session
    meta, rec = load_golden("session_mc64")
    e = meta["engine"]
    sess = Session(LocalTransport(scenes.store("mc64")),
                   EngineConfig(octree_depth=e["depth"], cache_slots=tuple(e["cache_slots"]),
                                channel_slots=e["m"]),
                   scenes.render_config(meta["render"]),
                   scenes.product_channels(meta["channels"]), device_metadata=True,
                   compressed_transfer=True)
    assert sess.device_metadata
    for item in meta["script"]:
        if "swap" in item:
            for s, c in item["swap"]:
                sess.swap_channel(s, c)
            continue
        pos, tgt, up, fov = item["pose"]
        r = sess.step_frame(Camera(position=tuple(pos), target=tuple(tgt), up=tuple(up),
                                   fov_deg=fov))
        i = item["frame"]
        assert np.array_equal(r.output.image, rec[f"f{i}_image"].reshape(r.output.image.shape))
        assert r.metadata_applied == item["metadata_applied"]
        assert not diff_hashes(device_state_hashes(sess.engine), item["after"]), i
    sess.close()


def test_gpu_fill_metadata_from_device_volume():
    """fill_metadata_from_volumes with a device tensor == with the numpy
    volume == the golden prepared state (words hash)."""
    import torch
    from paper_2309_04393_b200 import methods
    meta, _ = load_golden("vessel256_full")
    st = scenes.store("vessel256")
    econf = methods.full_engine_config(st, 1, depth=meta["engine"]["depth"])
    eng = methods.prepare_engine(st, {0: 0}, econf)
    assert not diff_hashes(device_state_hashes(eng), meta["state"])
    eng.octree.words_dev[:] = eng.octree.words_dev & 0xFFFF
    eng.fill_metadata_from_volumes({0: torch.from_numpy(st.level_array(0, 0)).cuda()})
    assert not diff_hashes(device_state_hashes(eng), meta["state"])
