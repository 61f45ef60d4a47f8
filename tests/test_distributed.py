"""Sort-first exchange over torch.distributed (gloo, world size 2, CPU).

Each rank renders its round-robin row blocks with the CPU oracle, turns its
blocks' first-seen request lists into (key, id) pairs, and runs the same
``distributed.exchange`` the GPU ranks run over NCCL.  The merged frame must
equal a single full-frame pass exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden
import scenes

TILE = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from oracle.session import OracleSession
    meta, _ = load_golden("session_mc64")
    e = meta["engine"]
    kw = scenes.render_kw(meta["render"])
    kw["image_dims"] = (40, 37)
    kw["budget"] = 30
    sess = OracleSession(scenes.store("mc64"), e["m"], e["depth"], e["cache_slots"],
                         scenes.oracle_channels(meta["channels"]), kw, e["pad"])
    cam = tuple(meta["script"][0]["pose"])
    for _ in range(2):
        sess.step_frame(cam)
    return sess, cam, kw


def _local_part(sess, cam, kw, world, rank):
    from paper_2309_04393_b200.distributed import part_rows
    w, h = kw["image_dims"]
    m = sess.st.m
    rows = part_rows(h, world, rank, TILE)
    image = np.zeros((len(rows) * w, 4), dtype=np.float32)
    pixreq = np.zeros(len(rows) * w, dtype=np.int32)
    req = None
    hist = None
    counters = np.zeros(8, dtype=np.int64)
    first_b, first_m = {}, {}
    pos = 0
    blocks = (h + TILE - 1) // TILE
    for b in range(rank, blocks, world):
        r0, r1 = b * TILE, min((b + 1) * TILE, h)
        out = sess.render(cam, rows=(r0, r1))
        n = (r1 - r0) * w
        image[pos:pos + n] = out.image[r0:r1].reshape(-1, 4)
        pixreq[pos:pos + n] = out.pixel_required[r0 * w:r1 * w]
        pos += n
        for i, bid in enumerate(out.all_brick_requests):
            first_b.setdefault(bid, (b << 32) | i)
        for i, (node, slot) in enumerate(out.all_metadata_requests):
            first_m.setdefault(node * m + slot, (b << 32) | i)
        req = out.required_mask.copy() if req is None else (req | out.required_mask)
        hist = out.level_histogram.copy() if hist is None else hist + out.level_histogram
        counters[:5] += out.counters
    budget = kw["budget"]
    fb = np.zeros((4, budget), dtype=np.int64)
    bl = sorted((k, v) for v, k in first_b.items())[:budget]
    ml = sorted((k, v) for v, k in first_m.items())[:budget]
    for j, (k, v) in enumerate(bl):
        fb[0, j], fb[1, j] = k, v
    for j, (k, v) in enumerate(ml):
        fb[2, j], fb[3, j] = k, v
    counts = np.array([len(first_b), len(first_m), len(bl), len(ml)], dtype=np.int64)
    return dict(image=torch.from_numpy(image), required=torch.from_numpy(req),
                pix_required=torch.from_numpy(pixreq), hist=torch.from_numpy(hist),
                counters=torch.from_numpy(counters), fb=torch.from_numpy(fb), counts=counts)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04393_b200.distributed import exchange
        sess, cam, kw = _scene()
        local = _local_part(sess, cam, kw, world, rank)
        out = exchange(local, kw["image_dims"], TILE, kw["budget"], sess.st.m)
        res = {"bricks": out["bricks"], "metas": out["metas"],
               "required": out["required"].numpy(), "hist": out["hist"].numpy(),
               "counters": out["counters"].numpy()}
        if rank == 0:
            res["image"] = out["image"].numpy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sort_first_exchange_gloo_world2(oracle_lib):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sess, cam, kw = _scene()
    full = sess.render(cam)
    for r in range(world):
        res = results[r]
        assert res["bricks"] == full.brick_requests
        assert res["metas"] == full.metadata_requests
        assert np.array_equal(res["required"], full.required_mask)
        assert np.array_equal(res["hist"], full.level_histogram)
        assert list(res["counters"][:5]) == list(full.counters)
    assert np.array_equal(results[0]["image"], full.image)


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_04393_b200.distributed import gather_image, part_rows
    w, h = 11, 37
    full = np.arange(h * w * 4, dtype=np.float32).reshape(h, w, 4)
    local = full[part_rows(h, world, rank, TILE)]
    got = gather_image(local, (w, h), TILE)
    if rank == 0:
        q.put(bool(np.array_equal(got, full)))
    else:
        q.put(got is None)
    dist.destroy_process_group()


def test_gather_image_assembles_capacity_mode_tiles():
    """distributed.gather_image (capacity-mode frame assembly) over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res), res
