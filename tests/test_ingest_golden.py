"""Wire format + ingest restatements against the reference (CPU, no GPU).

The LZ4 oracle is liblz4 itself, called the way lz4io.py:69-110 does; the
golden frames were produced by the reference's own compress_brick
(tests/golden/make_golden.py lz4_frames)."""

import hashlib

import numpy as np

from conftest import load_golden


def _sha(b) -> str:
    return hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest()


def test_lz4_oracle_decodes_reference_frames():
    from oracle import lz4_ref
    meta, rec = load_golden("lz4_frames")
    for i, item in enumerate(meta["items"]):
        bx, by, bz = item["brick"]
        frame = rec[f"frame{i}"].tobytes()
        assert len(frame) == item["bytes"]
        out = lz4_ref.decompress(frame, expected_size=bx * by * bz)
        assert _sha(np.frombuffer(out, np.uint8)) == item["payload_sha"], item["kind"]


def test_server_side_compression_matches_reference_bytes():
    """ingest.compress_brick (host liblz4, default preferences) reproduces
    the reference's frames byte for byte."""
    from oracle import lz4_ref
    from paper_2309_04393_b200 import ingest
    meta, rec = load_golden("lz4_frames")
    for i, item in enumerate(meta["items"]):
        bx, by, bz = item["brick"]
        frame = rec[f"frame{i}"].tobytes()
        payload = np.frombuffer(lz4_ref.decompress(frame, bx * by * bz), np.uint8)
        assert ingest.compress_brick(payload) == frame, item["kind"]


def test_lz4_oracle_error_behaviour():
    """lz4io.decompress raises on truncation, trailing bytes, bad magic and
    size mismatch -- the cases the GPU decoder must also reject."""
    import pytest
    from oracle import lz4_ref
    from paper_2309_04393_b200 import ingest
    data = bytes(range(256)) * 128
    f = ingest.compress(data)
    assert lz4_ref.decompress(f, len(data)) == data
    for bad in (f[:-1], f + b"\0", b"\x00" + f[1:], f[:10]):
        with pytest.raises(lz4_ref.Lz4DecodeError):
            lz4_ref.decompress(bad, len(data))
    with pytest.raises(lz4_ref.Lz4DecodeError):
        lz4_ref.decompress(f, len(data) + 1)
