"""GPU brick ingest against its oracles.

* LZ4: the reference's own frames (golden) and liblz4-produced frames under
  every frame option decode bit-exactly; corrupt / truncated / trailing /
  mis-sized frames are rejected wherever liblz4 (lz4io.decompress) rejects
  them.
* apply_bricks_lz4: a Session fetching LZ4 frames and decoding them into the
  cache on the GPU reproduces the reference's golden session frame by frame.
* normalize_to_u8 / downsample_box / build_pyramid / extract_bricks equal
  the numpy restatement (volume.py), itself pinned to the reference's
  pyramids (test_restated_ingest_matches_reference_pyramids).
"""

import hashlib

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


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_gpu_lz4_decodes_reference_frames():
    from paper_2309_04393_b200 import ingest
    meta, rec = load_golden("lz4_frames")
    by_size = {}
    for i, item in enumerate(meta["items"]):
        by_size.setdefault(tuple(item["brick"]), []).append(i)
    for size, idx in by_size.items():
        frames = [rec[f"frame{i}"].tobytes() for i in idx]
        out, st = ingest.decompress_bricks(frames, size)
        assert (st == 0).all()
        got = out.cpu().numpy()
        for j, i in enumerate(idx):
            assert _sha(got[j]) == meta["items"][i]["payload_sha"], meta["items"][i]["kind"]


def _payloads(rng, n, size):
    """Bricks of very different compressibility: runs, small-period patterns
    (overlapping matches), sparse spikes, smooth ramps, pure noise."""
    bx, by, bz = size
    out = []
    for i in range(n):
        kind = i % 5
        if kind == 0:
            p = np.repeat(rng.integers(0, 256, size=(bx * by * bz) // 64 + 1,
                                       dtype=np.uint8), 64)[:bx * by * bz]
        elif kind == 1:
            period = int(rng.integers(1, 40))
            p = np.resize(rng.integers(0, 256, size=period, dtype=np.uint8), bx * by * bz)
        elif kind == 2:
            p = np.zeros(bx * by * bz, np.uint8)
            idx = rng.integers(0, bx * by * bz, size=50)
            p[idx] = rng.integers(1, 256, size=50)
        elif kind == 3:
            p = (np.arange(bx * by * bz) // int(rng.integers(1, 300))).astype(np.uint8)
        else:
            p = rng.integers(0, 256, size=bx * by * bz, dtype=np.uint8)
        out.append(p.reshape(bz, by, bx))
    return out


@pytest.mark.parametrize("opts", [
    dict(),
    dict(linked=True),
    dict(content_checksum=True, block_checksum=True, content_size=True),
    dict(block_size_id=5, linked=True, level=9),
    dict(block_size_id=6, level=3, content_checksum=True),
    dict(block_size_id=7, linked=True, content_size=True),
])
@pytest.mark.parametrize("size", [(32, 32, 32), (16, 16, 16), (64, 64, 64)])
def test_gpu_lz4_frame_options(opts, size):
    from oracle import lz4_ref
    from paper_2309_04393_b200 import ingest
    rng = np.random.default_rng(hash((str(opts), size)) % 2**32)
    pays = _payloads(rng, 10, size)
    frames = [lz4_ref.prefs_frame(p.tobytes(), **opts) for p in pays]
    out, st = ingest.decompress_bricks(frames, size)
    assert (st == 0).all(), st
    got = out.cpu().numpy()
    for j, p in enumerate(pays):
        assert np.array_equal(got[j], p), (opts, j)


@pytest.mark.parametrize("level", [0, 9])
def test_gpu_lz4_map_decoder_corpus(level):
    """One wave of 32^3 frames (148: the one-CTA map decoder's batch) of
    every compressibility class plus noise-floor bricks (values 0..k: tens
    of thousands of short matches, deep match chains for the pointer
    jumping) and mixed bricks (noise + runs, offsets up to 64 KB), compared
    with liblz4's decode byte for byte."""
    from oracle import lz4_ref
    from paper_2309_04393_b200 import ingest
    rng = np.random.default_rng(7 + level)
    size = (32, 32, 32)
    n = 32 * 32 * 32
    pays = _payloads(rng, 60, size)
    for i in range(60):
        kind = i % 3
        if kind == 0:   # noise floor
            p = rng.integers(0, 1 + i % 5, size=n, dtype=np.uint8)
        elif kind == 1:  # noise floor with bright blobs
            p = rng.integers(0, 3, size=n, dtype=np.uint8)
            for _ in range(8):
                a = int(rng.integers(0, n - 900))
                p[a:a + int(rng.integers(10, 900))] = rng.integers(100, 256, dtype=np.uint8)
        else:           # repeats of an earlier region (long offsets) + noise
            p = rng.integers(0, 256, size=n, dtype=np.uint8)
            for _ in range(20):
                a, b = sorted(int(v) for v in rng.integers(0, n - 600, size=2))
                L = int(rng.integers(4, 600))
                p[b:b + L] = p[a:a + L]
        pays.append(p.reshape(32, 32, 32))
    pays = pays[:148] + [np.zeros(size, np.uint8)] * (148 - len(pays))
    frames = [lz4_ref.prefs_frame(p.tobytes(), level=level) for p in pays]
    out, st = ingest.decompress_bricks(frames, size)
    assert (st == 0).all(), st
    got = out.cpu().numpy()
    for j, f in enumerate(frames):
        want = np.frombuffer(lz4_ref.decompress(f, expected_size=n), np.uint8)
        assert np.array_equal(got[j].reshape(-1), want), j


def test_gpu_lz4_rejects_what_liblz4_rejects():
    """Mutated frames: whenever liblz4 (lz4io.decompress semantics) rejects a
    frame the GPU status is non-zero; whenever liblz4 accepts it the GPU
    decodes the same bytes.  Content + block checksums make almost every
    payload mutation detectable; truncation, trailing bytes, bad magic and
    wrong sizes are covered explicitly."""
    from oracle import lz4_ref
    from paper_2309_04393_b200 import ingest
    size = (32, 32, 32)
    bvox = 32 * 32 * 32
    rng = np.random.default_rng(11)
    pays = _payloads(rng, 5, size)
    cases = []
    for p in pays:
        for opts in (dict(), dict(content_checksum=True, block_checksum=True)):
            f = bytearray(lz4_ref.prefs_frame(p.tobytes(), **opts))
            cases += [bytes(f[:-1]), bytes(f) + b"\0", b"\x05" + bytes(f[1:]), bytes(f[:9])]
            for _ in range(30):
                g = bytearray(f)
                k = int(rng.integers(0, len(g)))
                g[k] ^= int(rng.integers(1, 256))
                cases.append(bytes(g))
    cases.append(lz4_ref.prefs_frame(bytes(bvox - 1)))            # one byte short
    cases.append(lz4_ref.prefs_frame(bytes(bvox + 7)))            # too long
    cases.append(lz4_ref.prefs_frame(bytes(bvox), content_size=True))
    out, st = ingest.decompress_bricks(cases, size, raise_on_error=False)
    got = out.cpu().numpy()
    n_rej = 0
    for j, c in enumerate(cases):
        try:
            ref = lz4_ref.decompress(c, expected_size=bvox)
        except lz4_ref.Lz4DecodeError:
            ref = None
        if ref is None:
            assert st[j] != 0, (j, len(c))
            n_rej += 1
        else:
            assert st[j] == 0, (j, int(st[j]))
            assert got[j].tobytes() == ref, j
    assert n_rej >= 40


def test_gpu_session_lz4_transfer_matches_reference():
    """session_mc64 golden (cold start, LRU pressure, mid-stream swap) with
    bricks fetched as LZ4 frames and decoded on the GPU into the cache."""
    from paper_2309_04393_b200 import (Camera, EngineConfig, LocalTransport, Session)
    meta, rec = load_golden("session_mc64")
    e = meta["engine"]
    sess = Session(LocalTransport(scenes.store("mc64")),
                   EngineConfig(octree_depth=e["depth"], cache_slots=tuple(e["cache_slots"]),
                                channel_slots=e["m"]),
                   scenes.render_config(meta["render"]),
                   scenes.product_channels(meta["channels"]), compressed_transfer=True)
    assert sess.compressed_transfer
    for item in meta["script"]:
        if "swap" in item:
            for s, c in item["swap"]:
                sess.swap_channel(s, c)
            assert not diff_hashes(device_state_hashes(sess.engine), item["after_swap"])
            continue
        pos, tgt, up, fov = item["pose"]
        r = sess.step_frame(Camera(position=tuple(pos), target=tuple(tgt), up=tuple(up),
                                   fov_deg=fov))
        i = item["frame"]
        assert np.array_equal(r.output.image, rec[f"f{i}_image"].reshape(r.output.image.shape))
        assert r.bricks_applied == item["bricks_applied"]
        assert not diff_hashes(device_state_hashes(sess.engine), item["after"]), i
    sess.close()


def test_gpu_apply_bricks_lz4_rejects_batch_atomically():
    from paper_2309_04393_b200 import Engine, EngineConfig
    from paper_2309_04393_b200 import ingest
    from paper_2309_04393_b200._native import NativeError
    st = scenes.store("mc64")
    eng = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=4))
    ids = [eng.paging.encode(0, 0, (x, 0, 0)) for x in range(3)]
    frames = [st.brick_bytes(0, 0, (x, 0, 0)) for x in range(3)]
    before = device_state_hashes(eng)
    bad = list(frames)
    bad[1] = bad[1][:-3]
    with pytest.raises(NativeError, match="brick 1 of the batch"):
        eng.apply_bricks_lz4(ids, bad)
    assert not diff_hashes(device_state_hashes(eng), before)
    eng.apply_bricks_lz4(ids, frames)
    ref = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                           channel_slots=4))
    ref.apply_bricks(ids, np.stack([st.brick(0, 0, (x, 0, 0)) for x in range(3)]))
    assert device_state_hashes(eng) == device_state_hashes(ref)
    # device-resident frames (already uploaded) take the same path
    buf, offs = ingest.pack_frames(frames)
    import torch
    eng2 = Engine(st.manifest, EngineConfig(octree_depth=3, cache_slots=(4, 4, 4),
                                            channel_slots=4))
    eng2.apply_bricks_lz4(ids, (torch.from_numpy(buf).cuda(), offs))
    assert device_state_hashes(eng2) == device_state_hashes(ref)


@pytest.mark.parametrize("shape", [(37, 50, 21), (64, 64, 64), (9, 1, 30)])
@pytest.mark.parametrize("dtype", ["u8", "u16", "u32", "f32"])
def test_gpu_normalize_to_u8(shape, dtype):
    import torch
    from paper_2309_04393_b200 import ingest
    from paper_2309_04393_b200.volume import normalize_to_u8
    rng = np.random.default_rng(7)
    if dtype == "f32":
        raw = (rng.standard_normal(shape) * 1000.0).astype(np.float32)
    else:
        hi = {"u8": 256, "u16": 65536, "u32": 2**32}[dtype]
        raw = rng.integers(0, hi, size=shape, dtype={"u8": np.uint8, "u16": np.uint16,
                                                     "u32": np.uint32}[dtype])
    got = ingest.normalize_to_u8(torch.from_numpy(raw).cuda()).cpu().numpy()
    assert np.array_equal(got, normalize_to_u8(raw))
    flat = np.full(shape, 7, dtype=raw.dtype)
    assert not ingest.normalize_to_u8(torch.from_numpy(flat).cuda()).cpu().numpy().any()


@pytest.mark.parametrize("shape", [(33, 50, 21), (64, 64, 64), (1, 7, 2)])
@pytest.mark.parametrize("factors", [(2, 2, 2), (2, 2, 1), (1, 2, 2), (2, 1, 1)])
def test_gpu_downsample_box(shape, factors):
    import torch
    from paper_2309_04393_b200 import ingest
    from paper_2309_04393_b200.volume import downsample_box
    rng = np.random.default_rng(1)
    lvl = rng.integers(0, 256, size=shape, dtype=np.uint8)
    got = ingest.downsample_box(torch.from_numpy(lvl).cuda(), factors).cpu().numpy()
    assert np.array_equal(got, downsample_box(lvl, factors))


def test_gpu_pyramid_and_bricks_match_store():
    """Device pyramid + bricks of every level == the restated host store
    (pinned to the reference's pyramids by pyramid_sha)."""
    import torch
    from paper_2309_04393_b200 import ingest
    from paper_2309_04393_b200 import volume as V
    raw = V.sparse_multichannel(64, channels=2)
    st = scenes.store("mc64")
    for c in range(2):
        u8 = ingest.normalize_to_u8(torch.from_numpy(np.ascontiguousarray(raw[c])).cuda())
        pyr = ingest.build_pyramid(u8, st.manifest.levels)
        for lev, arr in enumerate(pyr):
            assert np.array_equal(arr.cpu().numpy(), st.level_array(c, lev)), (c, lev)
            bricks = ingest.extract_bricks(arr, st.manifest.brick_size).cpu().numpy()
            gx, gy, gz = st.manifest.levels[lev].brick_grid_dims
            i = 0
            for z in range(gz):
                for y in range(gy):
                    for x in range(gx):
                        assert np.array_equal(bricks[i], st.brick(c, lev, (x, y, z)))
                        i += 1


# -- known answers of the reference's ingest / lz4io tests ---------------------

def test_gpu_normalize_known_answers():
    """test_ingest.py:13-31: full [0, 255] range, order kept, constant
    volume -> 0, and the midpoint rounds half up (1 of [0, 2] -> 128)."""
    import torch
    from paper_2309_04393_b200 import ingest
    raw = np.array([[[10, 20], [30, 40]], [[50, 60], [70, 90]]], dtype=np.uint16)
    out = ingest.normalize_to_u8(torch.from_numpy(raw).cuda()).cpu().numpy()
    assert out.dtype == np.uint8 and out.min() == 0 and out.max() == 255
    assert np.array_equal(np.argsort(raw.ravel()), np.argsort(out.ravel()))
    mid = np.array([0, 1, 2], dtype=np.float32).reshape(1, 1, 3)
    assert ingest.normalize_to_u8(torch.from_numpy(mid).cuda()).cpu().numpy().ravel() \
        .tolist() == [0, 128, 255]


def test_gpu_edge_bricks_replicate_the_nearest_voxel():
    """test_ingest.py:74-84: interior bricks are plain crops, edge bricks
    repeat the last in-volume voxel along each clipped axis."""
    import torch
    from paper_2309_04393_b200 import ingest
    data = np.arange(5 * 6 * 7, dtype=np.uint8).reshape(5, 6, 7)
    bricks = ingest.extract_bricks(torch.from_numpy(data).cuda(), (4, 4, 4)).cpu().numpy()
    assert bricks.shape == (2 * 2 * 2, 4, 4, 4)
    assert np.array_equal(bricks[0], data[:4, :4, :4])
    edge = bricks[7]                                   # grid (1, 1, 1): origin (4, 4, 4)
    assert edge[0, 0, 0] == data[4, 4, 4] and edge[1, 0, 0] == data[4, 4, 4]
    assert edge[0, 0, 2] == data[4, 4, 6] and edge[0, 0, 3] == data[4, 4, 6]
    want = data[np.minimum(np.arange(4, 8), 4)][:, np.minimum(np.arange(4, 8), 5)][
        :, :, np.minimum(np.arange(4, 8), 6)]
    assert np.array_equal(edge, want)


def test_gpu_lz4_error_known_answers():
    """test_lz4io.py:24-52: a zero brick compresses below 1 %; a size
    mismatch, a truncated or corrupted frame, garbage and an empty input are
    all rejected (per frame, the others in the batch still decode)."""
    from paper_2309_04393_b200 import ingest
    zero = ingest.compress(bytes(32 ** 3))
    assert len(zero) < 32 ** 3 // 100
    good = ingest.compress(bytes(range(256)) * 16)           # 4096 bytes = 16^3
    corrupt = bytearray(good)
    corrupt[4] ^= 0xFF
    frames = [good, ingest.compress(b"abcdef"), good[:len(good) // 2], bytes(corrupt),
              b"not lz4 data at all", b"", good]
    out, st = ingest.decompress_bricks(frames, (16, 16, 16), raise_on_error=False)
    assert st[0] == 0 and st[-1] == 0 and all(st[1:-1] != 0)
    assert bytes(out[0].cpu().numpy().tobytes()) == bytes(range(256)) * 16
    with pytest.raises(ingest.IngestError):
        ingest.decompress_bricks(frames[1:2], (16, 16, 16))
