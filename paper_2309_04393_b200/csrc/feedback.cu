// feedback.cu -- kernel 3a: request ordering + budget, and the LRU touch.
//
// The ray caster leaves, per touched brick / metadata entry, the smallest
// (pixel << 32 | event) key of any request for it (raycast.cu, RED.MIN).
// Sorting the touched entries by that key reproduces the reference's
// single-threaded first-seen append order (kernels.py:457-517, seen_brick /
// seen_meta); the bricks-first budget is render.py:210-215.
//
// Touched entries are found by one streaming pass over the key arrays
// (E u64 for bricks, N*m u64 for metadata: 0.6 MB + 9.6 MB at config 2),
// which also resets them for the next frame -- cheaper than making every
// request wait for an atomic's return value in the ray caster.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace ro {

namespace {

constexpr unsigned kScanBlocks = 148 * 4;

// compact (key, entry) of every touched entry, reset the key; warp-aggregated
// slot allocation
// (also the largest pixel and event index among the touched keys, so the
// sort only has to order the bits those need)
__global__ void __launch_bounds__(256) k_compact(unsigned long long *__restrict__ keys,
                                                 int64_t n,
                                                 unsigned long long *__restrict__ out_keys,
                                                 int32_t *__restrict__ out_vals,
                                                 int32_t *__restrict__ count,
                                                 unsigned *__restrict__ maxes) {
    unsigned mpix = 0, mev = 0;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // warp-uniform trip count (the shuffles need all 32 lanes)
    for (int64_t wb = warp * 64; wb < n; wb += nwarps * 64) {
        const int64_t base = wb + 2 * lane;
        // two entries per lane: 16-byte loads
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
        const int mine = (int)t0 + (int)t1;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        int basepos = 0;
        if (lane == 31 && total) basepos = atomicAdd(count, total);
        basepos = __shfl_sync(0xffffffffu, basepos, 31);
        int pos = basepos + incl - mine;
        if (t0) {
            out_keys[pos] = k0;
            out_vals[pos] = (int32_t)base;
            keys[base] = ~0ull;
            ++pos;
        }
        if (t1) {
            out_keys[pos] = k1;
            out_vals[pos] = (int32_t)(base + 1);
            keys[base + 1] = ~0ull;
        }
    }
    mpix = __reduce_max_sync(0xffffffffu, mpix);
    mev = __reduce_max_sync(0xffffffffu, mev);
    if (lane == 0 && (mpix | mev)) {
        atomicMax(&maxes[0], mpix);
        atomicMax(&maxes[1], mev);
    }
}

// (pixel << 32 | event) -> (pixel << ev_bits | event): order-preserving and
// injective while pixel < 2^pix_bits and event < 2^ev_bits
__global__ void k_pack_keys(const unsigned long long *__restrict__ in, int32_t n, int ev_bits,
                            uint32_t *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = in[i];
    out[i] = ((uint32_t)(k >> 32) << ev_bits) | (uint32_t)k;
}

__device__ __forceinline__ unsigned long long unpack_key(uint32_t k, int ev_bits) {
    return ((unsigned long long)(k >> ev_bits) << 32) | (k & ((1u << ev_bits) - 1u));
}

__global__ void k_emit_bricks(const DevLayout L,
                              const unsigned long long *__restrict__ keys,
                              const uint32_t *__restrict__ keys32, int ev_bits,
                              const int32_t *__restrict__ vals, int32_t n,
                              int64_t *__restrict__ out_keys,
                              int64_t *__restrict__ out_ids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out_keys[i] = (int64_t)(keys32 ? unpack_key(keys32[i], ev_bits) : keys[i]);
    out_ids[i] = entry_to_id(L, vals[i]);
}

__global__ void k_emit_metas(const unsigned long long *__restrict__ keys,
                             const uint32_t *__restrict__ keys32, int ev_bits,
                             const int32_t *__restrict__ vals, int32_t n,
                             int64_t *__restrict__ out_keys,
                             int64_t *__restrict__ out_ids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out_keys[i] = (int64_t)(keys32 ? unpack_key(keys32[i], ev_bits) : keys[i]);
    out_ids[i] = vals[i];
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

inline unsigned scan_blocks(int64_t n) {
    int64_t b = (n + 511) / 512;
    if (b < 1) b = 1;
    if (b > kScanBlocks) b = kScanBlocks;
    return (unsigned)b;
}

inline int bit_length(unsigned v) { return v ? 32 - __builtin_clz(v) : 0; }

// sort the n compacted (key, entry) pairs and emit the first `keep`.  Only
// the key bits in use are ordered: (pixel, event) packed into 32 bits when
// they fit (4 radix passes instead of 8), else the 64-bit key up to the top
// pixel bit.
int sort_and_emit(ro_ctx *c, unsigned long long *k_in, int32_t *v_in, int32_t n,
                  int32_t keep, bool bricks, int pix_bits, int ev_bits,
                  int64_t *out_keys, int64_t *out_ids, cudaStream_t s) {
    if (n <= 0 || keep <= 0) return RO_OK;
    void *p1, *p3, *tmp;
    int rc;
    if ((rc = scratch(c, 3, sizeof(int32_t) * n, &p3))) return rc;
    auto *v_out = (int32_t *)p3;
    size_t tmp_bytes = 0;
    const unsigned long long *k64 = nullptr;
    const uint32_t *k32 = nullptr;
    if (pix_bits + ev_bits <= 32) {
        void *p5, *p6;
        if ((rc = scratch(c, 5, sizeof(uint32_t) * n, &p5))) return rc;
        if ((rc = scratch(c, 6, sizeof(uint32_t) * n, &p6))) return rc;
        auto *q_in = (uint32_t *)p5, *q_out = (uint32_t *)p6;
        k_pack_keys<<<(n + 255) / 256, 256, 0, s>>>(k_in, n, ev_bits, q_in);
        const int end_bit = pix_bits + ev_bits > 0 ? pix_bits + ev_bits : 1;
        RO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, q_in, q_out, v_in, v_out, n,
                                                0, end_bit, s));
        if ((rc = scratch(c, 4, tmp_bytes, &tmp))) return rc;
        RO_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, q_in, q_out, v_in, v_out, n, 0,
                                                end_bit, s));
        k32 = q_out;
    } else {
        if ((rc = scratch(c, 1, sizeof(unsigned long long) * n, &p1))) return rc;
        auto *k_out = (unsigned long long *)p1;
        const int end_bit = 32 + pix_bits;
        RO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, v_out, n,
                                                0, end_bit, s));
        if ((rc = scratch(c, 4, tmp_bytes, &tmp))) return rc;
        RO_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, v_out, n, 0,
                                                end_bit, s));
        k64 = k_out;
    }
    if (bricks)
        k_emit_bricks<<<(keep + 255) / 256, 256, 0, s>>>(c->dl, k64, k32, ev_bits, v_out, keep,
                                                          out_keys, out_ids);
    else
        k_emit_metas<<<(keep + 255) / 256, 256, 0, s>>>(k64, k32, ev_bits, v_out, keep, out_keys,
                                                         out_ids);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

}  // namespace

int feedback_collect(ro_ctx *c, int64_t budget, int32_t bricks_first,
                     const ro_feedback *fb, cudaStream_t s) {
    if (budget < 0) return fail(RO_EINVAL, "negative budget");
    const int64_t n_meta = meta_keys(c) ? c->n_meta : 0;
    void *p0, *p2;
    int rc;
    // compacted arrays: bricks at [0, E), metas at [E, E + n_meta)
    if ((rc = scratch(c, 0, sizeof(unsigned long long) * (c->E + n_meta), &p0))) return rc;
    if ((rc = scratch(c, 2, sizeof(int32_t) * (c->E + n_meta), &p2))) return rc;
    auto *ck = (unsigned long long *)p0;
    auto *cv = (int32_t *)p2;
    // touched_n: [0] bricks, [1] metas, [2] max pixel, [3] max event
    RO_CUDA(cudaMemsetAsync(c->touched_n, 0, 4 * sizeof(int32_t), s));
    auto *maxes = reinterpret_cast<unsigned *>(c->touched_n + 2);
    k_compact<<<scan_blocks(c->E), 256, 0, s>>>(brick_keys(c), c->E, ck, cv, c->touched_n,
                                                maxes);
    if (n_meta)
        k_compact<<<scan_blocks(n_meta), 256, 0, s>>>(meta_keys(c), n_meta, ck + c->E,
                                                      cv + c->E, c->touched_n + 1, maxes);
    RO_CUDA(cudaGetLastError());
    int32_t *hn = reinterpret_cast<int32_t *>(c->pinned_small);
    RO_CUDA(cudaMemcpyAsync(hn, c->touched_n, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaStreamSynchronize(s));
    const int32_t nb = hn[0], nm = hn[1];
    const int pix_bits = bit_length((unsigned)hn[2]), ev_bits = bit_length((unsigned)hn[3]);
    const int32_t kb = (int32_t)(nb < budget ? nb : budget);
    const int64_t rest = bricks_first ? budget - kb : budget;
    const int32_t km = (int32_t)(nm < rest ? nm : rest);
    rc = sort_and_emit(c, ck, cv, nb, kb, true, pix_bits, ev_bits, fb->brick_keys,
                       fb->brick_ids, s);
    if (rc) return rc;
    rc = sort_and_emit(c, ck + c->E, cv + c->E, nm, km, false, pix_bits, ev_bits,
                       fb->meta_keys, fb->meta_ids, s);
    if (rc) return rc;
    fb->counts[0] = nb;
    fb->counts[1] = nm;
    fb->counts[2] = kb;
    fb->counts[3] = km;
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
