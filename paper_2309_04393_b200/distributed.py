"""Sort-first multi-GPU frames.

Rows are cut in blocks of ``tile_rows``; block b is rendered by part
b % n_parts (round-robin, so every GPU gets a fair share of the dense middle
of the image).  Every GPU holds its own replica of the render state (octree
words, page tables, brick cache) and renders its rows with the same kernel.

One exchange step per frame, over NCCL / NVLink:
  * image tiles      -> gathered to rank 0 (f32 RGBA, 33 MB at 1080p)
  * request lists    -> all-gathered (key, id) pairs, <= budget per rank;
                        merged by key = (pixel << 32 | event), keep-first,
                        bricks-first budget -- identical on every rank, so
                        every replica applies the same uploads (parity mode)
  * usage mask       -> all-reduce MAX (u8), then note_sampled everywhere
  * counters / hist  -> all-reduce SUM
The merged result is bit-identical to a single-GPU frame (tested in
tests/test_gpu_parity.py and, for the exchange itself, with gloo on CPU in
tests/test_distributed.py).

Capacity mode (``Session(partition=...)``): every GPU keeps its own cache,
LRU and octree for its own rows only (no feedback exchange, so per-GPU cache
capacity adds up); ``gather_image`` collects the tiles on rank 0.  Images
equal the single-GPU ones once the parts have converged (every desired brick
resident), like the reference's full-residency image.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def part_rows(height: int, n_parts: int, part: int, tile_rows: int) -> list:
    rows = []
    blocks = (height + tile_rows - 1) // tile_rows
    for b in range(part, blocks, n_parts):
        rows.extend(range(b * tile_rows, min((b + 1) * tile_rows, height)))
    return rows


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _gather_stacked(x: torch.Tensor) -> torch.Tensor:
    """All-gather into one (world, *x.shape) tensor (a single NCCL
    all-gather; per-rank views for other backends)."""
    world = dist.get_world_size()
    out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, x.contiguous())
    else:
        dist.all_gather(list(out.unbind(0)), x.contiguous())
    return out


def merge_feedback(key_id_lists, budget: int, m: int):
    """key_id_lists: [(bkeys, bids, mkeys, mids)] per part (numpy).

    Returns (bricks, metas) exactly as one full-frame pass would."""
    def merge(keys, ids):
        if not keys:
            return []
        k = np.concatenate(keys)
        v = np.concatenate(ids)
        order = np.argsort(k, kind="stable")
        out, seen = [], set()
        for i in order:
            x = int(v[i])
            if x not in seen:
                seen.add(x)
                out.append(x)
        return out

    bricks = merge([p[0] for p in key_id_lists], [p[1] for p in key_id_lists])[:budget]
    metas = merge([p[2] for p in key_id_lists], [p[3] for p in key_id_lists])
    metas = [(v // m, v % m) for v in metas[:budget - len(bricks)]]
    return bricks, metas


def merge_parts(parts, image_dims, n_parts, tile_rows, budget, m) -> dict:
    """Assemble per-part device/host results into the full-frame outputs."""
    w, h = image_dims
    image = np.zeros((h, w, 4), dtype=np.float32)
    pixreq = np.zeros(h * w, dtype=np.int32)
    lists = []
    required = None
    hist = None
    counters = None
    for p, part in enumerate(parts):
        rows = part_rows(h, n_parts, p, tile_rows)
        img = _np(part["image"]).reshape(-1, w, 4)[:len(rows)]
        image[rows] = img
        pr = _np(part["pix_required"]).reshape(-1, w)[:len(rows)]
        pixreq.reshape(h, w)[rows] = pr
        counts = _np(part["counts"])
        fb = _np(part["fb"])
        nb, nm = int(counts[2]), int(counts[3])
        lists.append((fb[0][:nb], fb[1][:nb], fb[2][:nm], fb[3][:nm]))
        r = _np(part["required"])
        required = r.copy() if required is None else (required | r)
        hs = _np(part["hist"])
        hist = hs.copy() if hist is None else hist + hs
        c = _np(part["counters"])
        counters = c.copy() if counters is None else counters + c
    bricks, metas = merge_feedback(lists, budget, m)
    return dict(image=image, pix_required=pixreq, bricks=bricks, metas=metas,
                required=required, hist=hist, counters=counters)


def exchange(local: dict, image_dims, tile_rows: int, budget: int, m: int,
             gather_image: bool = True, paging=None) -> dict:
    """One frame's collective step; every rank returns the merged feedback,
    rank 0 also the assembled image.

    local: image (local_rows*w, 4), required (E,) u8, pix_required, hist,
    counters (tensors on this rank's device), fb (4, budget) i64 tensor,
    counts (4,) host array (or counts_dev, a (4,) device tensor).

    With ``paging`` (a GPU replica) the whole step stays on the device:
    the gathered request blocks are folded into the replica's first-seen
    key arrays (ro_feedback_merge) and ordered by ro_feedback_collect, and
    the image is assembled by ro_gather_rows -- no host round trip until
    the caller reads the lists.  Without it (CPU / gloo checks) the same
    merge runs on the host (merge_feedback)."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    w, h = image_dims
    dev = local["required"].device
    # usage mask, histogram, counters
    required = local["required"].clone()
    dist.all_reduce(required, op=dist.ReduceOp.MAX)
    hist = local["hist"].clone()
    dist.all_reduce(hist)
    counters = local["counters"].clone()
    dist.all_reduce(counters)
    # request lists: fixed-size (4, budget) blocks + counts
    fb = local["fb"].contiguous()
    if local.get("counts_dev") is not None:
        counts = local["counts_dev"].contiguous()
    else:
        counts = torch.as_tensor(np.asarray(local["counts"], dtype=np.int64), device=dev)
    fbs = _gather_stacked(fb)
    cts = _gather_stacked(counts)
    if paging is not None:
        from . import _native as N
        import ctypes as C
        merged = torch.zeros((4, max(budget, 1)), dtype=torch.int64, device=dev)
        mcounts = torch.zeros(4, dtype=torch.int64, device=dev)
        N.check(N.lib().ro_feedback_merge(paging.ctx, fbs.data_ptr(), cts.data_ptr(), world,
                                          budget, N.stream_ptr()))
        fbd = N.Feedback(merged[0].data_ptr(), merged[1].data_ptr(), merged[2].data_ptr(),
                         merged[3].data_ptr(), None, mcounts.data_ptr())
        N.check(N.lib().ro_feedback_collect(paging.ctx, budget, 1, C.byref(fbd),
                                            N.stream_ptr()))
        host = torch.cat([mcounts, merged.reshape(-1)]).cpu().numpy()  # one read-back
        nb, nm = int(host[2]), int(host[3])
        blk = host[4:].reshape(4, -1)
        bricks = [int(v) for v in blk[1][:nb]]
        metas = [(int(v) // m, int(v) % m) for v in blk[3][:nm]]
    else:
        lists = []
        for f, c in zip(fbs, cts):
            f = f.cpu().numpy()
            c = c.cpu().numpy()
            nb, nm = int(c[2]), int(c[3])
            lists.append((f[0][:nb], f[1][:nb], f[2][:nm], f[3][:nm]))
        bricks, metas = merge_feedback(lists, budget, m)
    out = dict(bricks=bricks, metas=metas, required=required, hist=hist,
               counters=counters)
    if gather_image:
        max_rows = max(len(part_rows(h, world, p, tile_rows)) for p in range(world))
        img = torch.zeros((max_rows * w, 4), dtype=torch.float32, device=dev)
        img[:local["image"].shape[0]] = local["image"]
        # NCCL: gather to rank 0; other backends (gloo, CPU tests): all-gather.
        # The choice depends only on the backend, so every rank takes the
        # same collective.
        if dist.get_backend() == "nccl":
            parts = [torch.empty_like(img) for _ in range(world)] if rank == 0 else None
            dist.gather(img, parts, dst=0)
        else:
            parts = [torch.empty_like(img) for _ in range(world)]
            dist.all_gather(parts, img)
        if rank == 0:
            full = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
            if paging is not None:
                from . import _native as N
                stacked = torch.stack(parts)
                N.check(N.lib().ro_gather_rows(stacked.data_ptr(), world, max_rows * w * 4, h, w,
                                               tile_rows, full.data_ptr(), N.stream_ptr()))
            else:
                for p in range(world):
                    rows = part_rows(h, world, p, tile_rows)
                    idx = torch.as_tensor(rows, device=dev, dtype=torch.long)
                    full.index_copy_(0, idx, parts[p][:len(rows) * w].reshape(len(rows), w, 4))
            out["image"] = full
    return out


def gather_image(local_rows_image, image_dims, tile_rows: int):
    """Gather every rank's rows (local_rows, w, 4) into the full (h, w, 4)
    frame on rank 0 (None elsewhere).  NCCL: gather to rank 0; other
    backends: all-gather (the choice depends only on the backend)."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    w, h = image_dims
    local = torch.as_tensor(local_rows_image)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")
    max_rows = max(len(part_rows(h, world, p, tile_rows)) for p in range(world))
    buf = torch.zeros((max_rows * w, 4), dtype=torch.float32, device=dev)
    flat = local.reshape(-1, 4).to(dev)
    buf[:flat.shape[0]] = flat
    if dist.get_backend() == "nccl":
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, parts, dst=0)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
    if rank != 0:
        return None
    full = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
    for p in range(world):
        rows = part_rows(h, world, p, tile_rows)
        idx = torch.as_tensor(rows, device=dev, dtype=torch.long)
        full.index_copy_(0, idx, parts[p][:len(rows) * w].reshape(len(rows), w, 4))
    return full.cpu().numpy()


# ---------------------------------------------------------------------------
# sort-first over peer memory (fused render + exchange)
# ---------------------------------------------------------------------------

class PeerFrame:
    """Sort-first frames whose exchange is done by the ray caster itself.

    Rank 0 (the owner) allocates the full-frame outputs -- image, per-pixel
    brick counts, usage mask, histogram, counters -- and the first-seen
    request-key arrays, and shares them with every rank through CUDA IPC
    (torch's reductions; on an NVLink/NVSwitch box the mappings are peer
    memory).  Each rank's ``ro_render`` (``shared_outputs = 1``) then writes
    its pixels at their global rows, ORs its usage marks, adds its histogram
    / counters and issues its RED.MIN request atomics straight into the
    owner's buffers while it ray-casts: the image gather, the usage
    all-reduce and the request all-gather + merge of ``exchange`` all
    disappear.  One barrier later the owner's ``ro_feedback_collect`` yields
    exactly the single-GPU request lists (same keys, same atomics), which are
    broadcast (<= budget ids) so every replica applies the same uploads.
    """

    def __init__(self, paging, octree, n_ch: int, image_dims):
        from torch.multiprocessing.reductions import reduce_tensor
        from . import _native as N
        self.N = N
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.paging = paging
        w, h = image_dims
        k, m = paging.config.k, paging.config.m
        dev = paging.device
        n_meta = octree.num_nodes * m
        names = ("image", "pix_required", "required", "hist", "counters", "bkeys", "mkeys")
        if self.rank == 0:
            bufs = dict(
                image=torch.zeros((h * w, 4), dtype=torch.float32, device=dev),
                pix_required=torch.zeros(h * w, dtype=torch.int32, device=dev),
                required=torch.zeros(paging.total_entries, dtype=torch.uint8, device=dev),
                hist=torch.zeros((n_ch, k), dtype=torch.int64, device=dev),
                counters=torch.zeros(N.RO_NUM_COUNTERS, dtype=torch.int64, device=dev),
                bkeys=torch.full((paging.total_entries,), -1, dtype=torch.int64, device=dev),
                mkeys=torch.full((n_meta,), -1, dtype=torch.int64, device=dev))
            torch.cuda.synchronize(dev)
            shared = [reduce_tensor(bufs[n]) for n in names]
        else:
            shared = None
        box = [shared]
        dist.broadcast_object_list(box, src=0)
        if self.rank != 0:
            bufs = {n: fn(*args) for n, (fn, args) in zip(names, box[0])}
            owner_dev = bufs["image"].device.index
            with torch.cuda.device(dev):   # this rank's kernels reach the owner's GPU
                N.check(N.lib().ro_enable_peer_access(owner_dev))
        self.bufs = bufs
        self.nccl = dist.get_backend() == "nccl"
        self._tok = torch.zeros(1, dtype=torch.int32, device=dev if self.nccl else "cpu")
        N.check(N.lib().ro_set_feedback_buffers(paging.ctx, bufs["bkeys"].data_ptr(),
                                                bufs["mkeys"].data_ptr()))
        self.outputs = N.Outputs(bufs["image"].data_ptr(), bufs["required"].data_ptr(),
                                 bufs["pix_required"].data_ptr(), bufs["hist"].data_ptr(),
                                 bufs["counters"].data_ptr())
        # no trailing collective: a rank that failed after the broadcast must
        # meet the others at the caller's next collective (bench.py agrees on
        # peer vs NCCL exchange with one all-reduce)

    def _token(self):
        """A rank-wide rendezvous.  NCCL: a one-element all-reduce on the
        current stream -- every later launch on this stream is ordered after
        every rank reached it, without blocking the host.  Other backends
        (the one-GPU gloo check): the host waits for the stream, then meets
        the other ranks."""
        if self.nccl:
            dist.all_reduce(self._tok)
        else:
            torch.cuda.current_stream().synchronize()
            dist.all_reduce(self._tok)

    def frame(self, fp, budget: int, m: int, events=None):
        """One sort-first frame: ``fp`` is this rank's FramePass (its
        partition set, bricks_first=True).  Returns (bricks, metas) on every
        rank; the full-frame image / usage / histogram / counters are
        ``self.bufs`` (complete on every rank after the call, valid until the
        next ``frame`` call).

        Stream-ordered (NCCL): owner clears the accumulators -> token ->
        every part ray-casts into the owner's buffers -> token -> owner
        orders the requests on the device -> the ordered block (<= budget
        entries + counts) is broadcast -> one host read.  The host waits
        once per frame, for the lists it must return."""
        N = self.N
        stream = torch.cuda.current_stream()
        if self.rank == 0:
            for n in ("required", "hist", "counters"):
                self.bufs[n].zero_()
        # (the previous frame's broadcast already ordered every rank's
        # previous render before this clear)
        self._token()                      # accumulators clear before any part writes
        fp.frame.shared_outputs = 1
        if events:
            events[0].record(stream)
        fp.render(self.outputs)
        if events:
            events[1].record(stream)
        self._token()                      # every part's writes / atomics landed
        b = fp.buf
        if self.rank == 0:
            fp.collect(asynchronous=True)  # owner's keys hold every part's requests
        block = b.small[b.hist.numel() + b.counters.numel():]   # lists + counts
        if self.nccl:
            dist.broadcast(block, src=0)
            host = block.cpu().numpy()
        else:
            host_t = block.cpu()
            dist.broadcast(host_t, src=0)
            host = host_t.numpy()
        nb, nm = int(host[-2]), int(host[-1])
        fbh = host[:-4].reshape(4, -1)
        return ([int(v) for v in fbh[1][:nb]], [(int(v) // m, int(v) % m) for v in fbh[3][:nm]])

    def close(self):
        self.N.check(self.N.lib().ro_set_feedback_buffers(self.paging.ctx, None, None))
        dist.barrier()
        self.bufs = None
