"""CPU restatement of the residency walk's per-frame node classes
(csrc/raycast.cu k_classify + the path-class skip in k_raycast's channel
loop), checked against a node-by-node walk: for random octree words, TF
transparency tables and homogeneity thresholds, every (depth-dt node,
cursor depth, channel) must give the same terminal node / visit count, and
the ZERO shortcut (<= 4 channels) must fire exactly on transparent
terminals.  The GPU parity tests check the kernel itself; this pins the bit
logic (byte-per-channel packing, ffs of the inverted run, 4-channel ZERO
bytes) without a GPU."""
import numpy as np
import pytest


def level_offset(d):
    return ((1 << (3 * d)) - 1) // 7


def node_kind(w, eb, eps_i):
    """'plain' / 'zero' / 'other' of one word for one channel (kernels.py:444-517)."""
    mn, mx = (w >> 16) & 0xFF, (w >> 24) & 0xFF
    if mn == 255 and mx == 0:
        return "other"           # INVALID: metadata request
    if mx < eb[mn]:
        return "zero"            # K_ZERO
    if mx - mn <= eps_i:
        return "other"           # K_CONST
    return "plain" if (w & 0xFFFF) else "other"   # else K_MISSU


def classify(words, D, n_ch, ebs, eps_i):
    """k_classify top-down: path[x] byte ci = plain bits of ci along root->x,
    bytes 4+ci the ZERO bits when n_ch <= 4; fast[x] bit0 / bit1."""
    n = level_offset(D + 1)
    path = np.zeros(n, np.uint64)
    fast = np.zeros(n, np.uint8)
    for d in range(D + 1):
        side = 1 << d
        for local in range(side ** 3):
            x = level_offset(d) + local
            gx, gy, gz = local % side, (local // side) % side, local // (side * side)
            if d:
                par = level_offset(d - 1) + ((gz >> 1) * (side // 2) + (gy >> 1)) * (side // 2) + (gx >> 1)
                pp, ch0 = int(path[par]), (int(fast[par]) >> 1) & 1
            else:
                pp, ch0 = 0, 1
            kinds = [node_kind(int(words[x, ci]), ebs[ci], eps_i) for ci in range(n_ch)]
            for ci, kd in enumerate(kinds):
                if kd == "plain":
                    pp |= 1 << (8 * ci + d)
                if kd == "zero" and n_ch <= 4:
                    pp |= 1 << (32 + 8 * ci + d)
            ch0 &= int(kinds[0] == "plain")
            allp = all(kd == "plain" for kd in kinds)
            path[x] = pp
            fast[x] = (1 if (allp and ch0) else 0) | (ch0 << 1)
    return path, fast


def ancestor(leaf_local, dt, d):
    side = 1 << dt
    gx, gy, gz = leaf_local % side, (leaf_local // side) % side, leaf_local // (side * side)
    sh, s2 = dt - d, 1 << d
    return level_offset(d) + ((gz >> sh) * s2 + (gy >> sh)) * s2 + (gx >> sh)


@pytest.mark.parametrize("n_ch", [1, 3, 4, 6, 8])
def test_path_class_skip_equals_node_walk(n_ch):
    rng = np.random.default_rng(n_ch)
    D = 3
    n = level_offset(D + 1)
    words = np.zeros((n, n_ch), np.uint64)
    for ci in range(n_ch):
        mn = rng.integers(0, 200, n)
        mx = np.minimum(255, mn + rng.integers(0, 60, n))
        mask = np.where(rng.random(n) < 0.2, 0, rng.integers(1, 1 << 7, n))
        w = (mx.astype(np.uint64) << 24) | (mn.astype(np.uint64) << 16) | mask.astype(np.uint64)
        inv = rng.random(n) < 0.08
        w[inv] = (w[inv] & 0xFFFF) | (0xFF << 16)
        words[:, ci] = w
    ebs = [np.sort(rng.integers(0, 120, 256)) for _ in range(n_ch)]
    eps_i = int(rng.integers(-1, 4))
    path, fast = classify(words, D, n_ch, ebs, eps_i)
    for dt in range(D + 1):
        for leaf_local in rng.integers(0, 1 << (3 * dt), 40):
            leaf = level_offset(dt) + int(leaf_local)
            pc = int(path[leaf])
            for d in range(dt + 1):
                for ci in range(n_ch):
                    # node-by-node: step through plain nodes from d
                    e = d
                    while e < dt and node_kind(int(words[ancestor(int(leaf_local), dt, e), ci]),
                                               ebs[ci], eps_i) == "plain":
                        e += 1
                    # path class: first zero bit of ci's byte at/after d, capped at dt
                    pm = (pc >> (8 * ci)) & 0xFF
                    inv = ~(pm >> d) & 0xFFFFFFFF
                    t = d + ((inv & -inv).bit_length() - 1)
                    t = min(t, dt)
                    assert t == e, (dt, d, ci)
                    kind_t = node_kind(int(words[ancestor(int(leaf_local), dt, t), ci]), ebs[ci], eps_i)
                    if n_ch <= 4:
                        assert bool((pc >> (32 + 8 * ci + t)) & 1) == (kind_t == "zero")
            # fast: every channel plain at dt and channel 0 plain from the root
            want_fast = all(node_kind(int(words[leaf, ci]), ebs[ci], eps_i) == "plain"
                            for ci in range(n_ch)) and all(
                node_kind(int(words[ancestor(int(leaf_local), dt, a), 0]), ebs[0], eps_i) == "plain"
                for a in range(dt + 1))
            assert bool(fast[leaf] & 1) == want_fast
