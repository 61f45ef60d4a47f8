// feedback.cu -- kernel 3a: request ordering + budget, and the LRU touch.
//
// The ray caster leaves, per touched brick / metadata entry, the smallest
// (pixel << 32 | event) key of any request for it (raycast.cu, RED.MIN).
// Ordering the touched entries by that key reproduces the reference's
// single-threaded first-seen append order (kernels.py:457-517, seen_brick /
// seen_meta); the bricks-first budget is render.py:210-215.
//
// One cooperative kernel (k_feedback) does the whole frame's ordering, with
// no host round trip and no library call:
//   A. a streaming pass over both key arrays compacts the touched (key,
//      entry) pairs and resets the keys for the next frame (warp-aggregated
//      appends), and finds the largest pixel and event index;       grid sync
//   B. keys are repacked order-preservingly as q = pixel << ev_bits | event;
//      only the `keep` smallest survive the budget, so instead of sorting
//      every touched entry the kernel radix-SELECTS the keep-th smallest q
//      (8-bit digits from the top, one histogram pass per digit over the
//      candidates, grid sync per digit) -- skipped when everything survives;
//   C. the survivors (q <= threshold) are gathered into the output range and
//      one CTA sorts them in shared memory (bitonic, <= kChunk pairs) and
//      writes the unpacked keys and the decoded BrickIDs.
// Budgets above kChunk are cut into consecutive rank chunks, each selected
// and sorted the same way.  Nothing synchronises the host: the counts land
// in device memory (and, for the synchronous API, in host memory after one
// final copy).
#include "internal.cuh"
#include "topk.cuh"

namespace cg = cooperative_groups;

namespace ro {

namespace {

constexpr int kFbThreads = 1024;
constexpr int kChunk = topk::kChunk;  // pairs sorted per CTA in shared memory (96 KB)
constexpr size_t kFbSmem = topk::kSortSmem;

// ctl block (u32, zeroed before the launch):
//   [0] touched bricks  [1] touched metas  [2] max pixel  [3] max event
//   [8 ..)          gather counters, one per chunk
//   [kHistOff ..)   3 x 256 digit histograms (a ring, see topk::select_kth)
constexpr int kMaxChunks = 1024;
constexpr int kHistOff = 8 + kMaxChunks;
constexpr int kCtlWords = kHistOff + 3 * 256;

struct FbArgs {
    DevLayout L;
    unsigned long long *bkeys;  // [E] first-seen keys (~0 = untouched)
    int64_t nbk;
    unsigned long long *mkeys;  // [n_meta] (may be null)
    int64_t nmk;
    unsigned long long *cand_k;  // [E + n_meta] compacted keys (bricks, then metas at +E)
    int32_t *cand_v;             // [E + n_meta] entries
    uint32_t *ctl;
    int64_t budget;
    int32_t bricks_first;
    int64_t *out_bkeys, *out_bids, *out_mkeys, *out_mids;  // [budget] each
    int64_t *counts;  // [4] device: touched bricks, touched metas, emitted, emitted
};

__device__ __forceinline__ int bit_len(unsigned v) { return v ? 32 - __clz(v) : 0; }

// with ev < 2^ev_bits: order-preserving, injective repack of (pixel << 32 | event)

// phase A: one list's key array -> compacted candidates
__device__ void compact(unsigned long long *__restrict__ keys, int64_t n,
                        unsigned long long *__restrict__ out_k, int32_t *__restrict__ out_v,
                        uint32_t *count, unsigned &mpix, unsigned &mev) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wb = warp * 64; wb < n; wb += nwarps * 64) {  // warp-uniform trip count
        const int64_t base = wb + 2 * lane;
        unsigned long long k0 = ~0ull, k1 = ~0ull;
        if (base + 1 < n) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(keys + base);
            k0 = v.x;
            k1 = v.y;
        } else if (base < n) {
            k0 = keys[base];
        }
        const bool t0 = k0 != ~0ull, t1 = k1 != ~0ull;
        if (t0) { mpix = max(mpix, (unsigned)(k0 >> 32)); mev = max(mev, (unsigned)k0); }
        if (t1) { mpix = max(mpix, (unsigned)(k1 >> 32)); mev = max(mev, (unsigned)k1); }
        const unsigned b0 = __ballot_sync(0xffffffffu, t0), b1 = __ballot_sync(0xffffffffu, t1);
        const int total = __popc(b0) + __popc(b1);
        if (total == 0) continue;
        uint32_t basepos = 0;
        if (lane == 0) basepos = atomicAdd(count, (uint32_t)total);
        basepos = __shfl_sync(0xffffffffu, basepos, 0);
        const unsigned below = (1u << lane) - 1u;
        uint32_t pos = basepos + __popc(b0 & below) + __popc(b1 & below);
        if (t0) {
            out_k[pos] = k0;
            out_v[pos] = (int32_t)base;
            keys[base] = ~0ull;
            ++pos;
        }
        if (t1) {
            out_k[pos] = k1;
            out_v[pos] = (int32_t)(base + 1);
            keys[base + 1] = ~0ull;
        }
    }
}

__device__ __forceinline__ unsigned long long pack(unsigned long long k, int ev_bits) {
    return ((k >> 32) << ev_bits) | (k & 0xFFFFFFFFull);
}
__device__ __forceinline__ unsigned long long unpack(unsigned long long q, int ev_bits) {
    return ((q >> ev_bits) << 32) | (q & ((1ull << ev_bits) - 1ull));
}

// one CTA: sort the gathered [0, w) (q in okeys, entry in oids) and write
// the unpacked keys / decoded ids back
__device__ void sort_emit(const DevLayout &L, bool bricks, int64_t *okeys, int64_t *oids,
                          int64_t w, int ev_bits, unsigned char *smem) {
    auto *sk = reinterpret_cast<unsigned long long *>(smem);
    auto *sv = reinterpret_cast<int32_t *>(sk + kChunk);
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        sk[i] = (unsigned long long)__ldcg(okeys + i);
        sv[i] = (int32_t)__ldcg(oids + i);
    }
    topk::sort_pairs(sk, sv, (int)w);
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        okeys[i] = (int64_t)unpack(sk[i], ev_bits);
        oids[i] = bricks ? entry_to_id(L, sv[i]) : (int64_t)sv[i];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kFbThreads, 1) k_feedback(const __grid_constant__ FbArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_hist[256];
    cg::grid_group grid = cg::this_grid();
    uint32_t *ctl = A.ctl;

    // ---- A: compaction ----
    unsigned mpix = 0, mev = 0;
    compact(A.bkeys, A.nbk, A.cand_k, A.cand_v, &ctl[0], mpix, mev);
    if (A.mkeys) compact(A.mkeys, A.nmk, A.cand_k + A.nbk, A.cand_v + A.nbk, &ctl[1], mpix, mev);
    mpix = __reduce_max_sync(0xffffffffu, mpix);
    mev = __reduce_max_sync(0xffffffffu, mev);
    if ((threadIdx.x & 31) == 0 && (mpix | mev)) {
        atomicMax(&ctl[2], mpix);
        atomicMax(&ctl[3], mev);
    }
    grid.sync();

    const int64_t nb = __ldcg(&ctl[0]), nm = __ldcg(&ctl[1]);
    const int ev_bits = bit_len(__ldcg(&ctl[3]));
    const int tb = bit_len(__ldcg(&ctl[2])) + ev_bits;
    const int top_shift = tb > 8 ? ((tb + 7) / 8 - 1) * 8 : 0;
    const int64_t kb = nb < A.budget ? nb : A.budget;
    const int64_t rest = A.bricks_first ? A.budget - kb : A.budget;
    const int64_t km = nm < rest ? nm : rest;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.counts[0] = nb;
        A.counts[1] = nm;
        A.counts[2] = kb;
        A.counts[3] = km;
    }

    // ---- B + C per list, in rank chunks ----
    uint32_t g = 0;   // histogram ring step (identical in every CTA)
    int chunk = 0;    // gather counter index (identical in every CTA)
    for (int list = 0; list < 2; ++list) {
        const bool bricks = list == 0;
        const int64_t n = bricks ? nb : nm;
        const int64_t keep = bricks ? kb : km;
        const unsigned long long *cand = A.cand_k + (bricks ? 0 : A.nbk);
        const int32_t *candv = A.cand_v + (bricks ? 0 : A.nbk);
        int64_t *okeys = bricks ? A.out_bkeys : A.out_mkeys;
        int64_t *oids = bricks ? A.out_bids : A.out_mids;
        bool has_lo = false;
        unsigned long long lo = 0;
        for (int64_t done = 0; done < keep; done += kChunk, ++chunk) {
            const int64_t w = keep - done < kChunk ? keep - done : kChunk;
            // threshold: the w-th smallest above lo, or everything left
            unsigned long long hi = ~0ull;
            if (done + w < n) {
                auto key_of = [&](int64_t i, unsigned long long &q) {
                    q = pack(__ldcg(cand + i), ev_bits);
                    return true;
                };
                hi = topk::select_kth(grid, n, key_of, has_lo, lo, w, top_shift,
                                      ctl + kHistOff, g, s_hist);
            }
            uint32_t *cnt = &ctl[8 + (chunk % kMaxChunks)];
            for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
                 i += (int64_t)gridDim.x * blockDim.x) {
                const unsigned long long q = pack(__ldcg(cand + i), ev_bits);
                if ((has_lo && q <= lo) || q > hi) continue;
                const uint32_t pos = atomicAdd(cnt, 1u);
                okeys[done + pos] = (int64_t)q;
                oids[done + pos] = __ldcg(candv + i);
            }
            grid.sync();
            // one CTA per chunk sorts it; the others go on selecting
            if (blockIdx.x == (unsigned)(chunk % gridDim.x))
                sort_emit(A.L, bricks, okeys + done, oids + done, w, ev_bits, smem);
            has_lo = true;
            lo = hi;
        }
    }
}

// Sort-first merge: every part's ordered (key, id) lists
// -- each already cut to the budget, which keeps every entry of the global
// first `budget` -- are scattered back into the first-seen key arrays with
// the ray caster's own RED.MIN rule (the smallest key of an entry wins);
// ro_feedback_collect then orders them exactly like one full-frame pass.
__global__ void k_merge_requests(const DevLayout L, int32_t n_parts, int64_t budget,
                                 const int64_t *__restrict__ blocks,  // [n_parts][4][budget]
                                 const int64_t *__restrict__ counts,  // [n_parts][4]
                                 unsigned long long *__restrict__ bkeys,
                                 unsigned long long *__restrict__ mkeys) {
    const int64_t per = 2 * budget;  // brick slots then meta slots of one part
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_parts * per;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = (int32_t)(j / per);
        const int64_t r = j - p * per;
        const bool meta = r >= budget;
        const int64_t i = meta ? r - budget : r;
        if (i >= counts[p * 4 + (meta ? 3 : 2)]) continue;
        const int64_t *blk = blocks + (int64_t)p * 4 * budget;
        const unsigned long long key = (unsigned long long)blk[(meta ? 2 : 0) * budget + i];
        const int64_t id = blk[(meta ? 3 : 1) * budget + i];
        if (meta) {
            atomicMin(mkeys + id, key);
        } else {
            const Decoded d = decode_id(L, id);
            if (d.ok) atomicMin(bkeys + entry_index(L, d.slot, d.lev, d.x, d.y, d.z), key);
        }
    }
}

// engine.py:72-81: every sampled entry that is MAPPED stamps its slot
__global__ void k_note_sampled(const uint8_t *__restrict__ required,
                               const int32_t *__restrict__ pt, int64_t E,
                               int64_t *__restrict__ last_used, int64_t frame) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride) {
        if (required[e]) {
            int32_t s = pt[e];
            if (s >= 0) last_used[s] = frame;
        }
    }
}

}  // namespace

int feedback_collect(ro_ctx *c, int64_t budget, int32_t bricks_first,
                     const ro_feedback *fb, cudaStream_t s) {
    if (budget < 0) return fail(RO_EINVAL, "negative budget");
    if (budget > (int64_t)kChunk * (kMaxChunks / 2 - 1))
        return fail(RO_EINVAL, "request budget above 4M entries");
    const int64_t n_meta = meta_keys(c) ? c->n_meta : 0;
    void *p0, *p2, *pc;
    int rc;
    // compacted candidates: bricks at [0, E), metas at [E, E + n_meta)
    if ((rc = scratch(c, 0, sizeof(unsigned long long) * (c->E + n_meta), &p0))) return rc;
    if ((rc = scratch(c, 2, sizeof(int32_t) * (c->E + n_meta), &p2))) return rc;
    if ((rc = scratch(c, 11, sizeof(uint32_t) * kCtlWords + sizeof(int64_t) * 8, &pc))) return rc;
    auto *ctl = (uint32_t *)pc;
    auto *dcounts = fb->counts_dev ? fb->counts_dev
                                   : reinterpret_cast<int64_t *>(ctl + kCtlWords + (kCtlWords & 1));
    static int64_t dummy[1];
    FbArgs A;
    A.L = c->dl;
    A.bkeys = brick_keys(c);
    A.nbk = c->E;
    A.mkeys = n_meta ? meta_keys(c) : nullptr;
    A.nmk = n_meta;
    A.cand_k = (unsigned long long *)p0;
    A.cand_v = (int32_t *)p2;
    A.ctl = ctl;
    A.budget = budget;
    A.bricks_first = bricks_first;
    // outputs may be null with budget 0 (nothing is written then)
    A.out_bkeys = fb->brick_keys ? fb->brick_keys : dummy;
    A.out_bids = fb->brick_ids ? fb->brick_ids : dummy;
    A.out_mkeys = fb->meta_keys ? fb->meta_keys : dummy;
    A.out_mids = fb->meta_ids ? fb->meta_ids : dummy;
    A.counts = dcounts;
    static int grid = 0;
    if (grid == 0) {
        RO_CUDA(cudaFuncSetAttribute(k_feedback, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kFbSmem));
        int dev = 0, sms = 0, per_sm = 0;
        RO_CUDA(cudaGetDevice(&dev));
        RO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        RO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_feedback, kFbThreads,
                                                              kFbSmem));
        if (per_sm < 1) return fail(RO_ECUDA, "feedback kernel cannot be resident");
        grid = sms;  // one CTA per SM
    }
    RO_CUDA(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * kCtlWords, s));
    c->keys_dirty = false;  // this pass resets every key it reads
    void *args[] = {&A};
    RO_CUDA(cudaLaunchCooperativeKernel((const void *)k_feedback, dim3(grid), dim3(kFbThreads),
                                        args, kFbSmem, s));
    if (fb->counts) {  // synchronous form: counts on the host when the call returns
        int64_t *h = c->pinned_small + 8;
        RO_CUDA(cudaMemcpyAsync(h, dcounts, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RO_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < 4; ++i) fb->counts[i] = h[i];
    }
    return RO_OK;
}

int feedback_merge(ro_ctx *c, const int64_t *blocks, const int64_t *counts, int32_t n_parts,
                   int64_t budget, cudaStream_t s) {
    if (n_parts < 1 || budget < 0) return fail(RO_EINVAL, "bad part count / budget");
    if (budget == 0) return RO_OK;
    if (!meta_keys(c)) {
        int rc = ensure_meta_keys(c);
        if (rc) return rc;
    }
    const int64_t total = 2 * budget * n_parts;
    int64_t blocks_n = (total + 255) / 256;
    if (blocks_n > 148 * 8) blocks_n = 148 * 8;
    k_merge_requests<<<(unsigned)blocks_n, 256, 0, s>>>(c->dl, n_parts, budget, blocks, counts,
                                                        brick_keys(c), meta_keys(c));
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

// one-time costs ahead of the first frame: key arrays, the compaction /
// control scratch, the kernel's shared-memory attribute and module load
int feedback_reserve(ro_ctx *c) {
    int rc;
    if (!c->meta_key && (rc = ensure_meta_keys(c))) return rc;
    const int64_t n_meta = c->n_meta;
    void *p;
    if ((rc = scratch(c, 0, sizeof(unsigned long long) * (c->E + n_meta), &p))) return rc;
    if ((rc = scratch(c, 2, sizeof(int32_t) * (c->E + n_meta), &p))) return rc;
    if ((rc = scratch(c, 11, sizeof(uint32_t) * kCtlWords + sizeof(int64_t) * 8, &p))) return rc;
    RO_CUDA(cudaFuncSetAttribute(k_feedback, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kFbSmem));
    cudaFuncAttributes fa;
    RO_CUDA(cudaFuncGetAttributes(&fa, k_feedback));
    RO_CUDA(cudaFuncGetAttributes(&fa, k_note_sampled));
    RO_CUDA(cudaFuncGetAttributes(&fa, k_merge_requests));
    return RO_OK;
}

int note_sampled(ro_ctx *c, const ro_state *st, const uint8_t *required,
                 int64_t frame, cudaStream_t s) {
    int64_t blocks = (c->E + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_note_sampled<<<(unsigned)blocks, 256, 0, s>>>(required, st->pt, c->E,
                                                    st->slot_last_used, frame);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

}  // namespace ro
