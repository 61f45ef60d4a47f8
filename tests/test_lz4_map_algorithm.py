"""CPU restatement of the one-CTA LZ4 map decoder's algorithm
(csrc/ingest.cu k_lz4_decode_map: seq_at / block_fast / pointer jumping),
checked against liblz4 on frames of every compressibility class.  The
phases are written out with numpy / loops exactly as the kernel splits
them, so a flaw in the idea (the all-positions parse, the next4 chain walk
with group marks, the per-group placement by prefix sums, the pointer
jumping over match references) shows up here without a GPU."""
import numpy as np
import pytest

ERR = 0x7FFF


def seq_at(b, bl, p, cap):
    """(lit_at, lit, off, ml, nx, last) of a sequence starting at p, or None."""
    token = b[p]
    q = p + 1
    lit = token >> 4
    if lit == 15:
        while True:
            if q >= bl or lit > cap:
                return None
            x = b[q]
            q += 1
            lit += x
            if x != 255:
                break
    if lit > cap or q + lit > bl:
        return None
    lit_at = q
    q += lit
    if q == bl:
        return lit_at, lit, 0, 0, bl, True
    if q + 2 > bl:
        return None
    off = b[q] | (b[q + 1] << 8)
    q += 2
    ml = token & 15
    if ml == 15:
        while True:
            if q >= bl or ml > cap:
                return None
            x = b[q]
            q += 1
            ml += x
            if x != 255:
                break
    ml += 4
    if lit + ml > cap or q >= bl:
        return None
    return lit_at, lit, off, ml, q, False


def block_map(b, cap):
    """Phases A-C of block_fast: the source map of one compressed block
    (literal refs as -1 - frame_index, match refs as output indices), or
    None where the kernel falls back to the serial parser."""
    bl = len(b)
    nx1 = np.full(bl, ERR, np.int64)
    for p in range(bl):                       # A: every position
        s = seq_at(b, bl, p, cap)
        if s is not None:
            nx1[p] = s[4]
    nxt = lambda arr, q: arr[q] if q < bl else q  # noqa: E731 (bl / ERR propagate)
    nx2 = np.array([nxt(nx1, int(q)) for q in nx1], np.int64)
    nx4 = np.array([nxt(nx2, int(q)) for q in nx2], np.int64)
    marks = []                                # B: the chain, four per load
    s = 0
    while True:
        a4 = int(nx4[s])
        marks.append(s)
        if a4 >= bl:
            c = s
            for _ in range(4):
                c = int(nx1[c])
                if c >= bl:
                    break
            if c != bl:
                return None
            break
        s = a4
    lens = []                                 # C: group lengths, prefix sums
    for p in marks:
        c, n = p, 0
        for _ in range(4):
            _, lit, _, ml, nx, last = seq_at(b, bl, c, cap)
            n += lit + ml
            if last:
                break
            c = nx
        lens.append(n)
    total = sum(lens)
    if total > cap:
        return None
    m = np.zeros(total, np.int64)
    o = 0
    for p in marks:
        c = p
        for _ in range(4):
            lit_at, lit, off, ml, nx, last = seq_at(b, bl, c, cap)
            m[o:o + lit] = -1 - np.arange(lit_at, lit_at + lit)
            o += lit
            if last:
                break
            if off == 0 or off > o:
                return None
            m[o:o + ml] = np.arange(o, o + ml) - off
            o += ml
            c = nx
    return m


def decode(frame: bytes, cap: int):
    """Frames of one compressed block (the kernel's fast path) -> bytes."""
    f = np.frombuffer(frame, np.uint8)
    assert int.from_bytes(frame[:4], "little") == 0x184D2204
    flg = f[4]
    pos = 7 + (8 if flg & 0x08 else 0) + (4 if flg & 0x01 else 0)
    bs = int.from_bytes(frame[pos:pos + 4], "little")
    pos += 4
    raw, bl = bs >> 31, bs & 0x7FFFFFFF
    block = f[pos:pos + bl].astype(np.int64)
    if raw:
        return block.astype(np.uint8).tobytes()
    m = block_map(block, cap)
    assert m is not None
    while True:                               # D: pointer jumping
        ref = m >= 0
        if not ref.any():
            break
        m[ref] = m[m[ref]]
    return block[-1 - m].astype(np.uint8).tobytes()


def _payloads(rng, n):
    out = []
    for i in range(n):
        kind = i % 6
        if kind == 0:
            p = rng.integers(0, 256, n_vox, dtype=np.uint8)
        elif kind == 1:
            p = rng.integers(0, 1 + i % 4, n_vox, dtype=np.uint8)
        elif kind == 2:
            p = np.resize(rng.integers(0, 256, int(rng.integers(1, 30)), dtype=np.uint8), n_vox)
        elif kind == 3:
            p = np.zeros(n_vox, np.uint8)
            p[rng.integers(0, n_vox, 40)] = 200
        elif kind == 4:
            p = (np.arange(n_vox) // int(rng.integers(1, 200))).astype(np.uint8)
        else:
            p = rng.integers(0, 3, n_vox, dtype=np.uint8)
            for _ in range(6):
                a, b = sorted(int(v) for v in rng.integers(0, n_vox - 300, 2))
                L = int(rng.integers(4, 300))
                p[b:b + L] = p[a:a + L]
        out.append(p)
    return out


n_vox = 16 * 16 * 16


@pytest.mark.parametrize("level", [0, 9])
def test_map_decoder_algorithm_matches_liblz4(level):
    from oracle import lz4_ref
    rng = np.random.default_rng(31 + level)
    for p in _payloads(rng, 12):
        frame = lz4_ref.prefs_frame(p.tobytes(), level=level)
        want = lz4_ref.decompress(frame, expected_size=n_vox)
        assert decode(frame, n_vox) == want
