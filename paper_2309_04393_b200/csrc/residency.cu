// residency.cu -- kernels 2 and 3b: LRU slot assignment, page-table and
// cache updates, and the octree residency-bitmask update pass.
//
// LRU (paging.py:187-239).  A frame's ordered batch of n unique, unmapped
// bricks is assigned in three phases that reproduce n sequential
// insert_brick calls exactly:
//   (i)   the first min(n, |free|) pop the LIFO free list from the top;
//   (ii)  the next take the slots occupied at batch start with
//         last_used < frame, in (last_used, slot) order -- the argmin
//         victims of the sequential loop;
//   (iii) once those run out (every slot stamped `frame`), each further
//         insert evicts slot 0, the argmin tie-break, i.e. the previous
//         phase-(iii) brick.
// Batches that break the precondition (duplicates, already-mapped ids) run
// the literal sequential loop in one thread instead.
//
// Octree (octree.py:193-246).  Masks are a pure function of the resident
// set (leaf ground truth + OR closure, octree.py:355-395), so after a batch
// every leaf overlapped by a changed brick is recomputed for that brick's
// (slot, level) from the final page table, then ancestors are re-ORed level
// by level.  Metadata bits (16..31) are never touched here.
#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "internal.cuh"
#include "topk.cuh"

namespace ro {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr unsigned kGridStride = 148 * 8;

__global__ void k_check_batch(const DevLayout L, const int64_t *__restrict__ ids,
                              int32_t n, const int32_t *__restrict__ pt,
                              uint32_t *__restrict__ claim, uint32_t epoch,
                              int32_t *__restrict__ flag,
                              int64_t *__restrict__ entries) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Decoded d = decode_id(L, ids[i]);
    if (!d.ok) { atomicOr(flag, 2); entries[i] = -1; return; }
    int64_t e = entry_index(L, d.slot, d.lev, d.x, d.y, d.z);
    entries[i] = e;
    if (pt[e] >= 0) atomicOr(flag, 1);
    if (atomicExch(claim + e, epoch) == epoch) atomicOr(flag, 1);
}

// copy payloads of final occupants into their cache slots (16-byte lanes)
__global__ void k_copy_payloads(int32_t n, int64_t bvox,
                                const uint8_t *__restrict__ src,
                                const int32_t *__restrict__ slots,
                                const uint8_t *__restrict__ final_flag,
                                uint8_t *__restrict__ cache) {
    const int64_t nv = bvox / 16;  // bricks are powers of two >= 8 voxels
    const int64_t total = nv * n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = j / nv, q = j - i * nv;
        if (!final_flag[i]) continue;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src + i * bvox);
        uint4 *d4 = reinterpret_cast<uint4 *>(cache + (int64_t)slots[i] * bvox);
        d4[q] = s4[q];
    }
}

// per-slot 8^3 sub-block maxima, dilated by one voxel (ro_state.sub_max):
// one CTA per batch brick, one thread per sub-block
__global__ void k_sub_max(int32_t n, int bx, int by, int bz, const uint8_t *__restrict__ src,
                          const int32_t *__restrict__ slots,
                          const uint8_t *__restrict__ final_flag, uint8_t *__restrict__ sub_max) {
    const int i = blockIdx.x;
    if (i >= n || !final_flag[i]) return;
    const int nx = bx >> RO_SUB_LOG, ny = by >> RO_SUB_LOG, nz = bz >> RO_SUB_LOG,
              nsb = nx * ny * nz;
    constexpr int E = RO_SUB_E;
    const int64_t bvox = (int64_t)bx * by * bz;
    const uint8_t *b = src ? src + (int64_t)i * bvox : nullptr;
    for (int q = threadIdx.x; q < nsb; q += blockDim.x) {
        unsigned mx = 255;
        if (b) {
            const int sx = q % nx, sy = (q / nx) % ny, sz = q / (nx * ny);
            const int x0 = max(E * sx - 1, 0), x1 = min(E * sx + E + 1, bx);
            const int y0 = max(E * sy - 1, 0), y1 = min(E * sy + E + 1, by);
            const int z0 = max(E * sz - 1, 0), z1 = min(E * sz + E + 1, bz);
            mx = 0;
            for (int z = z0; z < z1; ++z)
                for (int y = y0; y < y1; ++y) {
                    const uint8_t *row = b + ((int64_t)z * by + y) * bx;
                    for (int x = x0; x < x1; ++x) mx = max(mx, (unsigned)row[x]);
                }
        }
        sub_max[(int64_t)slots[i] * nsb + q] = (uint8_t)mx;
    }
}

// The same maxima for bricks up to 32 KiB: the brick is staged in shared
// memory and the dilated box max is separable -- x windows, then y, then z
// (each sub-block's window is [4s - 1, 4s + 4] clipped to the brick).
constexpr int kSubMaxThreads = 256;
__global__ void __launch_bounds__(kSubMaxThreads)
k_sub_max_smem(int32_t n, int bx, int by, int bz, const uint8_t *__restrict__ src,
               const int32_t *__restrict__ slots, const uint8_t *__restrict__ final_flag,
               uint8_t *__restrict__ sub_max, uint8_t *__restrict__ cache) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int i = blockIdx.x;
    if (i >= n || !final_flag[i]) return;
    constexpr int E = RO_SUB_E;
    const int nx = bx >> RO_SUB_LOG, ny = by >> RO_SUB_LOG, nz = bz >> RO_SUB_LOG,
              nsb = nx * ny * nz;
    const int bvox = bx * by * bz;
    uint8_t *v = sm;                      // [bz][by][bx]
    uint8_t *tx = v + bvox;               // [bz][by][nx]
    uint8_t *ty = tx + bz * by * nx;      // [bz][ny][nx]
    uint8_t *out = sub_max + (int64_t)slots[i] * nsb;
    if (!src) {  // payload unknown: "may be anything"
        for (int q = threadIdx.x; q < nsb; q += blockDim.x) out[q] = 255;
        return;
    }
    const uint8_t *b = src + (int64_t)i * bvox;
    if ((((uintptr_t)b) & 15) == 0 && (bvox & 15) == 0) {
        // (cache != null: the brick also lands in its cache slot from here,
        // the caller guarantees 16-byte alignment)
        uint4 *c4 = cache ? reinterpret_cast<uint4 *>(cache + (int64_t)slots[i] * bvox) : nullptr;
        for (int j = threadIdx.x; j < bvox / 16; j += blockDim.x) {
            const uint4 w = reinterpret_cast<const uint4 *>(b)[j];
            reinterpret_cast<uint4 *>(v)[j] = w;
            if (c4) c4[j] = w;
        }
    } else {
        for (int j = threadIdx.x; j < bvox; j += blockDim.x) v[j] = b[j];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < bz * by * nx; j += blockDim.x) {
        const int sx = j % nx, row = j / nx;
        const uint8_t *r = v + row * bx;
        unsigned m = 0;
        for (int x = max(E * sx - 1, 0); x < min(E * sx + E + 1, bx); ++x) m = max(m, (unsigned)r[x]);
        tx[j] = (uint8_t)m;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < bz * ny * nx; j += blockDim.x) {
        const int sx = j % nx, sy = (j / nx) % ny, z = j / (nx * ny);
        unsigned m = 0;
        for (int y = max(E * sy - 1, 0); y < min(E * sy + E + 1, by); ++y)
            m = max(m, (unsigned)tx[(z * by + y) * nx + sx]);
        ty[j] = (uint8_t)m;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nsb; q += blockDim.x) {
        const int sx = q % nx, sy = (q / nx) % ny, sz = q / (nx * ny);
        unsigned m = 0;
        for (int z = max(E * sz - 1, 0); z < min(E * sz + E + 1, bz); ++z)
            m = max(m, (unsigned)ty[(z * ny + sy) * nx + sx]);
        out[q] = (uint8_t)m;
    }
}

__global__ void k_copy_payloads_bytes(int32_t n, int64_t bvox,
                                      const uint8_t *__restrict__ src,
                                      const int32_t *__restrict__ slots,
                                      const uint8_t *__restrict__ final_flag,
                                      uint8_t *__restrict__ cache) {
    const int64_t total = bvox * n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = j / bvox, q = j - i * bvox;
        if (final_flag[i]) cache[(int64_t)slots[i] * bvox + q] = src[i * bvox + q];
    }
}

// literal sequential insert_brick loop (one thread) for irregular batches
__device__ void sequential_insert(const DevLayout L, int32_t n,
                                    const int64_t *__restrict__ ids,
                                    int32_t *__restrict__ pt,
                                    int64_t *__restrict__ slot_brick,
                                    int64_t *__restrict__ last_used,
                                    int32_t *__restrict__ free_stack,
                                    int32_t *__restrict__ free_count,
                                    int64_t frame, int32_t *__restrict__ slots,
                                    int64_t *__restrict__ evicted,
                                    uint8_t *__restrict__ final_flag) {
    for (int i = 0; i < n; ++i) {
        Decoded d = decode_id(L, ids[i]);
        int64_t e = entry_index(L, d.slot, d.lev, d.x, d.y, d.z);
        final_flag[i] = 0;
        evicted[i] = -1;
        if (pt[e] >= 0) { slots[i] = pt[e]; continue; }  // no-op re-insert
        int32_t lin;
        if (*free_count > 0) {
            lin = free_stack[--(*free_count)];
        } else {
            lin = -1;
            int64_t best = 0;
            for (int64_t s = 0; s < L.num_slots; ++s) {
                if (slot_brick[s] < 0) continue;
                if (lin < 0 || last_used[s] < best) { lin = (int32_t)s; best = last_used[s]; }
            }
            int64_t ev = slot_brick[lin];
            evicted[i] = ev;
            Decoded de = decode_id(L, ev);
            pt[entry_index(L, de.slot, de.lev, de.x, de.y, de.z)] = RO_PT_UNMAPPED;
            for (int q = 0; q < i; ++q)  // its payload never lands
                if (slots[q] == lin) final_flag[q] = 0;
        }
        slot_brick[lin] = ids[i];
        last_used[lin] = frame;
        pt[e] = lin;
        slots[i] = lin;
        final_flag[i] = 1;
    }
}

// sub_max of every slot from the cache (ro_upload_state)
__global__ void k_sub_max_all(int64_t S, int bx, int by, int bz, const uint8_t *__restrict__ cache,
                              const int64_t *__restrict__ slot_brick,
                              uint8_t *__restrict__ sub_max) {
    const int nx = bx >> RO_SUB_LOG, ny = by >> RO_SUB_LOG, nz = bz >> RO_SUB_LOG,
              nsb = nx * ny * nz;
    constexpr int E = RO_SUB_E;
    const int64_t bvox = (int64_t)bx * by * bz;
    for (int64_t i = blockIdx.x; i < S; i += gridDim.x) {
        const uint8_t *b = cache + i * bvox;
        const bool occupied = slot_brick[i] >= 0;
        for (int q = threadIdx.x; q < nsb; q += blockDim.x) {
            unsigned mx = 255;
            if (occupied) {
                const int sx = q % nx, sy = (q / nx) % ny, sz = q / (nx * ny);
                mx = 0;
                for (int z = max(E * sz - 1, 0); z < min(E * sz + E + 1, bz); ++z)
                    for (int y = max(E * sy - 1, 0); y < min(E * sy + E + 1, by); ++y)
                        for (int x = max(E * sx - 1, 0); x < min(E * sx + E + 1, bx); ++x)
                            mx = max(mx, (unsigned)b[((int64_t)z * by + y) * bx + x]);
            }
            sub_max[i * nsb + q] = (uint8_t)mx;
        }
    }
}

// explicit eviction / mark_empty (sequential: duplicates are no-ops)
__global__ void k_release(const DevLayout L, int32_t n, const int64_t *__restrict__ ids,
                          int32_t new_status, int32_t *__restrict__ pt,
                          int64_t *__restrict__ slot_brick,
                          int64_t *__restrict__ last_used,
                          int32_t *__restrict__ free_stack,
                          int32_t *__restrict__ free_count) {
    for (int i = 0; i < n; ++i) {
        Decoded d = decode_id(L, ids[i]);
        int64_t e = entry_index(L, d.slot, d.lev, d.x, d.y, d.z);
        int32_t lin = pt[e];
        if (lin >= 0) {
            slot_brick[lin] = -1;
            last_used[lin] = 0;
            free_stack[(*free_count)++] = lin;
        }
        if (new_status == RO_PT_EMPTY || lin >= 0) pt[e] = new_status;
    }
}

// ---- full rebuild (verification) ----
__global__ void k_rebuild_leaves(const DevLayout L, const int32_t *__restrict__ pt,
                                 uint32_t *__restrict__ words) {
    const int D = L.depth;
    const int64_t side = int64_t(1) << D;
    const int64_t nleaf = side * side * side;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nleaf * L.m;
         j += (int64_t)gridDim.x * blockDim.x) {
        int slot = (int)(j % L.m);
        int64_t leaf = j / L.m;
        int lx = (int)(leaf % side), ly = (int)((leaf / side) % side), lz = (int)(leaf / (side * side));
        uint32_t mask = 0;
        for (int lev = 0; lev < L.k; ++lev) {
            Box3 bb = brick_box(L, D, lx, ly, lz, lev);
            if (bb.empty) continue;
            bool backed = false;
            for (int z = bb.lo[2]; z <= bb.hi[2] && !backed; ++z)
                for (int y = bb.lo[1]; y <= bb.hi[1] && !backed; ++y)
                    for (int x = bb.lo[0]; x <= bb.hi[0]; ++x)
                        if (pt[entry_index(L, slot, lev, x, y, z)] >= 0) { backed = true; break; }
            if (backed) mask |= 1u << lev;
        }
        uint32_t *wp = words + (level_offset(D) + leaf) * L.m + slot;
        *wp = (*wp & 0xFFFF0000u) | mask;
    }
}

__global__ void k_rebuild_level(const DevLayout L, int dd, uint32_t *__restrict__ words) {
    const int64_t side = int64_t(1) << dd;
    const int64_t nn = side * side * side;
    const int64_t cside = side * 2;
    const int64_t cbase = level_offset(dd + 1);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn * L.m;
         j += (int64_t)gridDim.x * blockDim.x) {
        int slot = (int)(j % L.m);
        int64_t node = j / L.m;
        int64_t nx = node % side, ny = (node / side) % side, nz = node / (side * side);
        uint32_t mask = 0;
        for (int c = 0; c < 8; ++c) {
            int64_t cx = 2 * nx + (c & 1), cy = 2 * ny + ((c >> 1) & 1), cz = 2 * nz + (c >> 2);
            mask |= words[(cbase + (cz * cside + cy) * cside + cx) * L.m + slot] & 0xFFFFu;
        }
        uint32_t *wp = words + (level_offset(dd) + node) * L.m + slot;
        *wp = (*wp & 0xFFFF0000u) | mask;
    }
}

__global__ void k_set_metadata(const DevLayout L, int32_t n,
                               const int64_t *__restrict__ node,
                               const int32_t *__restrict__ slot,
                               const int32_t *__restrict__ mn,
                               const int32_t *__restrict__ mx,
                               uint32_t *__restrict__ words) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t *wp = words + node[i] * L.m + slot[i];
    *wp = (*wp & 0xFFFFu) | ((uint32_t)mn[i] << 16) | ((uint32_t)mx[i] << 24);
}

__global__ void k_level_metadata(const DevLayout L, int slot, int dd,
                                 const uint8_t *__restrict__ mins,
                                 const uint8_t *__restrict__ maxs,
                                 uint32_t *__restrict__ words) {
    const int64_t side = int64_t(1) << dd;
    const int64_t nn = side * side * side;
    const int64_t base = level_offset(dd);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nn;
         j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t *wp = words + (base + j) * L.m + slot;
        *wp = (*wp & 0xFFFFu) | ((uint32_t)mins[j] << 16) | ((uint32_t)maxs[j] << 24);
    }
}

__global__ void k_reset_range(int32_t *__restrict__ pt, int64_t lo, int64_t hi) {
    for (int64_t e = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < hi;
         e += (int64_t)gridDim.x * blockDim.x)
        pt[e] = RO_PT_UNMAPPED;
}

// Engine.swap_channel's release (paging.py:280-283): every slot holding a
// brick of channel slot cs is freed and pushed on the free list in
// ascending slot order.  Cooperative: each CTA owns a contiguous slot range,
// counts its slots, and after one grid sync appends them in order at its
// offset (block-wide ballot scan).
__global__ void __launch_bounds__(1024, 1) k_swap_release(const DevLayout L, int32_t cs,
                                                          int64_t *__restrict__ slot_brick,
                                                          int64_t *__restrict__ last_used,
                                                          int32_t *__restrict__ free_stack,
                                                          int32_t *__restrict__ free_count,
                                                          uint32_t *__restrict__ cta_counts) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_total;
    cg::grid_group grid = cg::this_grid();
    const int64_t S = L.num_slots;
    const int64_t per = (S + gridDim.x - 1) / gridDim.x;
    const int64_t s0 = blockIdx.x * per, s1 = min(S, s0 + per);
    auto mine = [&](int64_t sl) {
        if (sl >= s1) return false;
        const int64_t b = slot_brick[sl];
        return b >= 0 && (int)(((b >> 24) & 0xFF) / L.k) == cs;
    };
    uint32_t cnt = 0;
    for (int64_t sl = s0 + threadIdx.x; sl < s1; sl += blockDim.x) cnt += mine(sl) ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_warp[w];
        cta_counts[blockIdx.x] = t;
    }
    const int32_t base = *free_count;
    grid.sync();
    int64_t off = base;
    for (unsigned c = 0; c < blockIdx.x; ++c) off += __ldcg(cta_counts + c);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t0 = s0; t0 < s1; t0 += blockDim.x) {
        const int64_t sl = t0 + threadIdx.x;
        const bool f = mine(sl);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        __syncthreads();
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const uint32_t c = s_warp[w];
                s_warp[w] = run;
                run += c;
            }
            s_total = run;
        }
        __syncthreads();
        if (f) {
            free_stack[off + s_warp[warp] + __popc(bal & ((1u << lane) - 1u))] = (int32_t)sl;
            slot_brick[sl] = -1;
            last_used[sl] = 0;
        }
        off += s_total;
    }
    grid.sync();
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *free_count = (int32_t)off;
}

__global__ void k_invalidate(const DevLayout L, int32_t slot, uint32_t *__restrict__ words) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.num_nodes;
         i += (int64_t)gridDim.x * blockDim.x)
        words[i * L.m + slot] = 0x00FF0000u;
}

// ---- LRU batch: phases (i)-(iii), page-table map / unmap, one launch ----
constexpr int kCoopThreads = 1024;
constexpr int kLruMaxChunks = 1024;
// ctl (u32, zeroed before the launch): [0] stale count, [1] max stale
// last_used, [8, 8 + kLruMaxChunks) gather counters, then the select ring
constexpr int kLruHist = 8 + kLruMaxChunks;
constexpr int kLruCtlWords = kLruHist + topk::kHistWords;

struct LruArgs {
    DevLayout L;
    int32_t n;
    const int64_t *ids, *entries;
    const int32_t *flag;  // k_check_batch: 0 = regular batch
    int32_t *pt;
    int64_t *slot_brick, *last_used;
    int32_t *free_stack, *free_count;
    int64_t S, frame;
    int32_t *slots;
    int64_t *evicted;
    uint8_t *final_flag;
    unsigned long long *gather;  // [n] victim keys
    uint32_t *ctl;
};

// stale occupant of slot s: key (last_used << 32 | s), the argmin order of
// paging.py:205-206 (min last_used, ties to the lower slot)
__device__ __forceinline__ bool stale_key(const LruArgs &A, int64_t s, unsigned long long &q) {
    const int64_t lu = __ldcg(A.last_used + s);
    if (__ldcg(A.slot_brick + s) < 0 || lu >= A.frame) return false;
    q = ((unsigned long long)lu << 32) | (unsigned long long)s;
    return true;
}

__global__ void __launch_bounds__(kCoopThreads, 1) k_lru_batch(const __grid_constant__ LruArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_hist[256];
    cg::grid_group grid = cg::this_grid();
    const int32_t n = A.n;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    if (__ldcg(A.flag) != 0) {  // duplicates / mapped ids: the literal loop
        if (gtid == 0)
            sequential_insert(A.L, n, A.ids, A.pt, A.slot_brick, A.last_used, A.free_stack,
                              A.free_count, A.frame, A.slots, A.evicted, A.final_flag);
        return;
    }
    const int32_t fc = __ldcg(A.free_count);
    const int32_t n1 = n < fc ? n : fc;
    // (i) pop the free list top-first
    for (int64_t i = gtid; i < n1; i += gstride) {
        A.slots[i] = __ldcg(A.free_stack + fc - 1 - i);
        A.evicted[i] = -1;
    }
    const int32_t want = n - n1;
    int32_t n2 = 0;
    if (want > 0) {
        // (ii) the `want` stalest occupants at batch start, in (last_used, slot) order
        uint32_t cnt = 0, mx = 0;
        for (int64_t s = gtid; s < A.S; s += gstride) {
            unsigned long long q;
            if (stale_key(A, s, q)) {
                ++cnt;
                mx = max(mx, (uint32_t)(q >> 32));
            }
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if ((threadIdx.x & 31) == 0 && cnt) {
            atomicAdd(&A.ctl[0], cnt);
            atomicMax(&A.ctl[1], mx);
        }
        grid.sync();
        const int64_t n_stale = __ldcg(&A.ctl[0]);
        n2 = (int32_t)(want < n_stale ? want : n_stale);
        const int bits = 32 + topk::bit_len64(__ldcg(&A.ctl[1]));
        const int top_shift = ((bits + 7) / 8 - 1) * 8;
        auto key_of = [&](int64_t s, unsigned long long &q) { return stale_key(A, s, q); };
        uint32_t g = 0;
        bool has_lo = false;
        unsigned long long lo = 0;
        int chunk = 0;
        for (int64_t done = 0; done < n2; done += topk::kChunk, ++chunk) {
            const int64_t w = n2 - done < topk::kChunk ? n2 - done : topk::kChunk;
            unsigned long long hi = ~0ull;
            if (done + w < n_stale)
                hi = topk::select_kth(grid, A.S, key_of, has_lo, lo, w, top_shift,
                                      A.ctl + kLruHist, g, s_hist);
            uint32_t *cntp = &A.ctl[8 + chunk % kLruMaxChunks];
            for (int64_t s = gtid; s < A.S; s += gstride) {
                unsigned long long q;
                if (!stale_key(A, s, q) || (has_lo && q <= lo) || q > hi) continue;
                A.gather[done + atomicAdd(cntp, 1u)] = q;
            }
            grid.sync();
            if (blockIdx.x == (unsigned)(chunk % gridDim.x)) {
                auto *sk = reinterpret_cast<unsigned long long *>(smem);
                auto *sv = reinterpret_cast<int32_t *>(sk + topk::kChunk);
                for (int j = threadIdx.x; j < w; j += blockDim.x) {
                    sk[j] = __ldcg(A.gather + done + j);
                    sv[j] = 0;
                }
                topk::sort_pairs(sk, sv, (int)w);
                for (int j = threadIdx.x; j < w; j += blockDim.x) {
                    const int32_t slot = (int32_t)(sk[j] & 0xFFFFFFFFull);
                    A.slots[n1 + done + j] = slot;
                    A.evicted[n1 + done + j] = __ldcg(A.slot_brick + slot);
                }
                __syncthreads();
            }
            has_lo = true;
            lo = hi;
        }
    }
    // (iii) cache full of this frame's bricks: every further insert takes slot 0
    const int32_t p3 = n1 + n2;
    for (int64_t i = p3 + gtid; i < n; i += gstride) {
        A.slots[i] = 0;
        A.evicted[i] = i == p3 ? -2 : A.ids[i - 1];
    }
    grid.sync();
    if (p3 < n && gtid == 0) {  // slot 0's occupant when phase (iii) starts
        int64_t occ = __ldcg(A.slot_brick);
        for (int32_t i = p3 - 1; i >= 0; --i)
            if (__ldcg(A.slots + i) == 0) { occ = A.ids[i]; break; }
        A.evicted[p3] = occ;
    }
    grid.sync();
    // map the batch; final occupants own their slot
    for (int64_t i = gtid; i < n; i += gstride) {
        const int32_t s = __ldcg(A.slots + i);
        A.pt[A.entries[i]] = s;
        const bool fin = p3 >= n || s != 0 || i == n - 1;
        A.final_flag[i] = fin ? 1 : 0;
        if (fin) A.slot_brick[s] = A.ids[i];
        A.last_used[s] = A.frame;
    }
    grid.sync();
    for (int64_t i = gtid; i < n; i += gstride) {
        const int64_t v = __ldcg(A.evicted + i);
        if (v < 0) continue;
        const Decoded d = decode_id(A.L, v);
        A.pt[entry_index(A.L, d.slot, d.lev, d.x, d.y, d.z)] = RO_PT_UNMAPPED;
    }
    if (gtid == 0) *A.free_count = fc - n1;
}

// ---- octree update: every level of the changed bricks, one launch ----
// a changed brick, decoded once: its (slot, level) and its leaf box at
// depth D (lev < 0: skipped / empty)
struct BrickInfo {
    int lo[3], hi[3];
    int slot, lev;
};

struct OctArgs {
    DevLayout L;
    int32_t n;
    const int64_t *ids;  // changed bricks (< 0: skip)
    const int32_t *pt;
    uint32_t *words;
    int64_t *offs;     // [n + 1] per-level exclusive scan of node counts
    BrickInfo *info;   // [n]
};

// nodes of brick i's leaf box at depth dd (0 for skipped / empty)
__device__ __forceinline__ int64_t level_count(const BrickInfo &b, int D, int dd) {
    if (b.lev < 0) return 0;
    const int sh = D - dd;
    int64_t c = 1;
    for (int a = 0; a < 3; ++a) c *= (int64_t)((b.hi[a] >> sh) - (b.lo[a] >> sh) + 1);
    return c;
}

// bricks of `lev` overlapping leaf (x, y, z) -- octree.py:161-189 at depth
// D: the divisor 2^D * B is a power of two, so the exact floor / ceil
// divisions of brick_box are shifts
__device__ __forceinline__ Box3 leaf_bricks(const DevLayout &L, int lx, int ly, int lz, int lev) {
    Box3 b;
    b.empty = false;
    const int n[3] = {lx, ly, lz};
    const int B[3] = {L.bx, L.by, L.bz};
    for (int a = 0; a < 3; ++a) {
        const int shift = L.depth + (__ffs(B[a]) - 1);
        const int64_t dim = L.dims[lev][a];
        const int64_t lo = ((int64_t)n[a] * dim) >> shift;
        int64_t hi = ((((int64_t)n[a] + 1) * dim + (int64_t(1) << shift) - 1) >> shift) - 1;
        if (hi > L.grids[lev][a] - 1) hi = L.grids[lev][a] - 1;
        if (lo > hi) b.empty = true;
        b.lo[a] = (int)lo;
        b.hi[a] = (int)hi;
    }
    return b;
}

__global__ void __launch_bounds__(kCoopThreads, 1) k_octree_update(const __grid_constant__ OctArgs A) {
    __shared__ int64_t s_part[kCoopThreads];
    cg::grid_group grid = cg::this_grid();
    const int D = A.L.depth;
    const int32_t n = A.n;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    // decode every changed brick once (its leaf box costs six 64-bit divisions)
    for (int64_t i = gtid; i < n; i += gstride) {
        BrickInfo bi;
        bi.lev = -1;
        bi.slot = 0;
        const int64_t id = A.ids[i];
        if (id >= 0) {
            const Decoded d = decode_id(A.L, id);
            if (d.ok) {
                const Box3 b = leaf_box(A.L, d.lev, d.x, d.y, d.z);
                if (!b.empty) {
                    for (int a = 0; a < 3; ++a) {
                        bi.lo[a] = b.lo[a];
                        bi.hi[a] = b.hi[a];
                    }
                    bi.slot = d.slot;
                    bi.lev = d.lev;
                }
            }
        }
        A.info[i] = bi;
    }
    grid.sync();
    for (int dd = D; dd >= 0; --dd) {
        // CTA 0: exclusive scan of the per-brick node counts at this depth
        if (blockIdx.x == 0) {
            const int32_t per = (n + kCoopThreads - 1) / kCoopThreads;
            const int32_t b0 = threadIdx.x * per, b1 = min(n, b0 + per);
            int64_t sum = 0;
            for (int32_t i = b0; i < b1; ++i) sum += level_count(A.info[i], D, dd);
            s_part[threadIdx.x] = sum;
            __syncthreads();
            for (int o = 1; o < kCoopThreads; o <<= 1) {  // Hillis-Steele inclusive scan
                const int64_t y = threadIdx.x >= o ? s_part[threadIdx.x - o] : 0;
                __syncthreads();
                s_part[threadIdx.x] += y;
                __syncthreads();
            }
            int64_t run = s_part[threadIdx.x] - sum;
            for (int32_t i = b0; i < b1; ++i) {
                A.offs[i] = run;
                run += level_count(A.info[i], D, dd);
            }
            if (threadIdx.x == kCoopThreads - 1) A.offs[n] = s_part[threadIdx.x];
        }
        grid.sync();
        const int64_t total = __ldcg(A.offs + n);
        const int sh = D - dd;
        for (int64_t j = gtid; j < total; j += gstride) {
            // brick owning work item j: last i with offs[i] <= j
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldcg(A.offs + mid) <= j) lo = mid; else hi = mid - 1;
            }
            const int32_t i = lo;
            const BrickInfo b = A.info[i];
            struct { int slot, lev; } d = {b.slot, b.lev};
            const int lo0 = b.lo[0] >> sh, lo1 = b.lo[1] >> sh, lo2 = b.lo[2] >> sh;
            const int w = (b.hi[0] >> sh) - lo0 + 1, h = (b.hi[1] >> sh) - lo1 + 1;
            const int64_t r = j - __ldcg(A.offs + i);
            const int nx = lo0 + (int)(r % w);
            const int ny = lo1 + (int)((r / w) % h);
            const int nz = lo2 + (int)(r / ((int64_t)w * h));
            const int64_t side = int64_t(1) << dd;
            uint32_t *wp = A.words +
                           (level_offset(dd) + ((int64_t)nz * side + ny) * side + nx) * A.L.m + d.slot;
            if (dd == D) {
                // leaf: this (slot, level) bit = some MAPPED brick of that level
                // overlaps the leaf (octree.py:221-226 _leaf_backed)
                const Box3 bb = leaf_bricks(A.L, nx, ny, nz, d.lev);
                bool backed = false;
                if (!bb.empty) {
                    for (int z = bb.lo[2]; z <= bb.hi[2] && !backed; ++z)
                        for (int y = bb.lo[1]; y <= bb.hi[1] && !backed; ++y)
                            for (int x = bb.lo[0]; x <= bb.hi[0]; ++x)
                                if (A.pt[entry_index(A.L, d.slot, d.lev, x, y, z)] >= 0) {
                                    backed = true;
                                    break;
                                }
                }
                const uint32_t bit = 1u << d.lev;
                if (backed) atomicOr(wp, bit);
                else atomicAnd(wp, ~bit);
            } else {
                // inner node: OR of the 8 children's masks (octree.py:228-246)
                const int64_t cside = side * 2, cbase = level_offset(dd + 1);
                uint32_t mask = 0;
                for (int c = 0; c < 8; ++c) {
                    const int64_t cx = 2 * nx + (c & 1), cy = 2 * ny + ((c >> 1) & 1),
                                  cz = 2 * nz + (c >> 2);
                    mask |= __ldcg(A.words + (cbase + (cz * cside + cy) * cside + cx) * A.L.m +
                                   d.slot) & 0xFFFFu;
                }
                const uint32_t old = __ldcg(wp);
                const uint32_t nw = (old & 0xFFFF0000u) | mask;
                if (nw != old) *wp = nw;
            }
        }
        grid.sync();
    }
}

// one CTA per SM (cooperative kernels above)
int coop_grid(const void *kern, size_t smem, int *out) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        RO_CUDA(cudaGetDevice(&dev));
        RO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int per_sm = 0;
    RO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCoopThreads, smem));
    if (per_sm < 1) return fail(RO_ECUDA, "cooperative kernel cannot be resident");
    *out = sms;
    return RO_OK;
}

inline unsigned blocks_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > kGridStride) b = kGridStride;
    return (unsigned)b;
}

}  // namespace

// octree update for a device list of changed brick ids (entries < 0 skipped)
int octree_update(ro_ctx *c, const ro_state *st, const int64_t *ids, int32_t n,
                  cudaStream_t s) {
    if (st->words == nullptr || n <= 0) return RO_OK;
    void *po;
    int rc;
    if ((rc = scratch(c, 6, sizeof(int64_t) * ((size_t)n + 2) + sizeof(BrickInfo) * (size_t)n, &po)))
        return rc;
    OctArgs A;
    A.L = c->dl;
    A.n = n;
    A.ids = ids;
    A.pt = st->pt;
    A.words = st->words;
    A.offs = (int64_t *)po;
    A.info = reinterpret_cast<BrickInfo *>(A.offs + n + 2);
    int grid = 0;
    if ((rc = coop_grid((const void *)k_octree_update, 0, &grid))) return rc;
    // a grid sync costs microseconds per level: batches of a few hundred
    // bricks (a few thousand node updates per level) run on fewer CTAs
    grid = (int)std::min<int64_t>(grid, std::max<int64_t>(1, n / 8));
    void *args[] = {&A};
    RO_CUDA(cudaLaunchCooperativeKernel((const void *)k_octree_update, dim3(grid),
                                        dim3(kCoopThreads), args, 0, s));
    return RO_OK;
}

int apply_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n64,
                 const void *payloads, int32_t on_device, int64_t frame,
                 int32_t update_octree, int32_t *slots_out, int64_t *evicted_out,
                 cudaStream_t s) {
    if (n64 <= 0) return RO_OK;
    if (n64 > (int64_t)1 << 30) return fail(RO_EINVAL, "batch too large");
    if (frame < 0 || frame >= ((int64_t)1 << 31)) return fail(RO_EINVAL, "frame out of range");
    const int32_t n = (int32_t)n64;
    const int64_t bvox = c->bvox;
    // ids are validated on the host: nothing is queued for a bad batch
    for (int32_t i = 0; i < n; ++i) {
        if (!decode_id(c->dl, ids_h[i]).ok) {
            char msg[160];
            snprintf(msg, sizeof msg, "brick id outside the layout (index %d of %d, id %lld)",
                     i, n, (long long)ids_h[i]);
            return fail(RO_EINVAL, msg);
        }
    }
    int rc;
    void *p, *pl;
    // ids | evicted | entries | gather | slots | final | flag  (ids + evicted
    // contiguous: together they are the changed set of the octree pass)
    size_t need = sizeof(int64_t) * 4 * n + sizeof(int32_t) * n + n + 64;
    if ((rc = scratch(c, 1, need, &p))) return rc;
    int64_t *d_ids = (int64_t *)p;
    int64_t *d_evicted = d_ids + n;
    int64_t *d_entries = d_evicted + n;
    auto *d_gather = (unsigned long long *)(d_entries + n);
    int32_t *d_slots = (int32_t *)(d_gather + n);
    uint8_t *d_final = (uint8_t *)(d_slots + n);
    int32_t *d_flag = (int32_t *)(((uintptr_t)(d_final + n) + 15) & ~(uintptr_t)15);
    if ((rc = scratch(c, 13, sizeof(uint32_t) * kLruCtlWords, &pl))) return rc;
    auto *d_ctl = (uint32_t *)pl;
    int grid = 0;
    RO_CUDA(cudaFuncSetAttribute(k_lru_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)topk::kSortSmem));
    if ((rc = coop_grid((const void *)k_lru_batch, topk::kSortSmem, &grid))) return rc;
    void *dp = nullptr;
    const size_t bytes = (size_t)bvox * n;
    if (payloads && !on_device) {
        // the upload has a scratch slot of its own: nothing else on the
        // stream can reuse it while the DMA may still run
        if ((rc = scratch(c, 12, bytes, &dp))) return rc;
    }

    // payload upload on the side stream (overlaps the checks, the LRU, the
    // octree update and -- chunk by chunk -- the cache copy)
    const uint8_t *d_payload = nullptr;
    const int32_t chunk = std::max<int32_t>(256, (n + ro_ctx::kUploadChunks - 1) /
                                                     ro_ctx::kUploadChunks);
    const int n_chunks = (int)((n + chunk - 1) / chunk);
    bool queued = false, caller_pinned = false;
    // once the DMA is queued, every return makes the stream wait for it, and
    // a caller-pinned source buffer is released only when the DMA is done
    struct UploadGuard {
        ro_ctx *c;
        cudaStream_t s;
        const bool *queued, *pinned;
        ~UploadGuard() {
            if (*queued) cudaStreamWaitEvent(s, c->upload_done, 0);
            if (*queued && *pinned) cudaEventSynchronize(c->upload_done);
        }
    } guard{c, s, &queued, &caller_pinned};
    if (payloads) {
        if (on_device) {
            d_payload = (const uint8_t *)payloads;
        } else {
            cudaPointerAttributes pa;
            if (cudaPointerGetAttributes(&pa, payloads) != cudaSuccess) {
                cudaGetLastError();
                pa.type = cudaMemoryTypeUnregistered;
            }
            caller_pinned = pa.type == cudaMemoryTypeHost;
            const void *src = payloads;
            if (!caller_pinned) {
                // pageable payloads: one host copy into the handle's pinned staging
                if (c->staging_bytes < bytes) {
                    RO_CUDA(cudaEventSynchronize(c->upload_done));
                    if (c->staging) cudaFreeHost(c->staging);
                    c->staging = nullptr;
                    c->staging_bytes = 0;
                    RO_CUDA(cudaMallocHost(&c->staging, bytes));
                    c->staging_bytes = bytes;
                }
                // the previous upload must have finished before we overwrite staging
                RO_CUDA(cudaEventSynchronize(c->upload_done));
                if (payloads != c->staging) memcpy(c->staging, payloads, bytes);
                src = c->staging;
            }
            RO_CUDA(cudaEventRecord(c->host_done, s));
            RO_CUDA(cudaStreamWaitEvent(c->upload, c->host_done, 0));
            // in chunks: each chunk's cache copy / sub-block maxima start as
            // soon as it has landed, under the rest of the DMA
            for (int q = 0; q < n_chunks; ++q) {
                const int64_t b0 = (int64_t)q * chunk, nb = std::min<int64_t>(chunk, n - b0);
                RO_CUDA(cudaMemcpyAsync((uint8_t *)dp + b0 * bvox,
                                        (const uint8_t *)src + b0 * bvox, (size_t)(nb * bvox),
                                        cudaMemcpyHostToDevice, c->upload));
                RO_CUDA(cudaEventRecord(c->chunk_done[q], c->upload));
            }
            RO_CUDA(cudaEventRecord(c->upload_done, c->upload));
            queued = true;
            d_payload = (const uint8_t *)dp;
        }
    }
    RO_CUDA(cudaMemcpyAsync(d_ids, ids_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), s));
    RO_CUDA(cudaMemsetAsync(d_ctl, 0, sizeof(uint32_t) * kLruCtlWords, s));
    if (++c->epoch == 0) {  // stamp wrap: clear claims
        RO_CUDA(cudaMemsetAsync(c->claim, 0, sizeof(uint32_t) * c->E, s));
        c->epoch = 1;
    }
    k_check_batch<<<(n + 255) / 256, 256, 0, s>>>(c->dl, d_ids, n, st->pt, c->claim,
                                                  c->epoch, d_flag, d_entries);
    RO_CUDA(cudaGetLastError());
    // LRU assignment + page-table map / unmap: one cooperative launch, the
    // regular / sequential choice made on the device (no host round trip)
    LruArgs A;
    A.L = c->dl;
    A.n = n;
    A.ids = d_ids;
    A.entries = d_entries;
    A.flag = d_flag;
    A.pt = st->pt;
    A.slot_brick = st->slot_brick;
    A.last_used = st->slot_last_used;
    A.free_stack = st->free_stack;
    A.free_count = st->free_count;
    A.S = c->S;
    A.frame = frame;
    A.slots = d_slots;
    A.evicted = d_evicted;
    A.final_flag = d_final;
    A.gather = d_gather;
    A.ctl = d_ctl;
    void *args[] = {&A};
    RO_CUDA(cudaLaunchCooperativeKernel((const void *)k_lru_batch, dim3(grid),
                                        dim3(kCoopThreads), args, topk::kSortSmem, s));
    // the octree update needs the ids / evictions only: it runs while the
    // payloads are still crossing PCIe
    if (update_octree && st->words) {
        // changed = batch bricks + evicted residents
        rc = octree_update(c, st, d_ids, 2 * n, s);
        if (rc) return rc;
    }
    const bool sub_ok = st->sub_max && c->layout.brick[0] >= RO_SUB_E &&
                        c->layout.brick[1] >= RO_SUB_E && c->layout.brick[2] >= RO_SUB_E;
    const int bx = c->layout.brick[0], by = c->layout.brick[1], bz = c->layout.brick[2];
    const size_t sub_smem = (size_t)bx * by * bz + (size_t)bz * by * (bx >> RO_SUB_LOG) +
                            (size_t)bz * (by >> RO_SUB_LOG) * (bx >> RO_SUB_LOG);
    const bool aligned = bvox % 16 == 0 && ((uintptr_t)d_payload & 15) == 0 &&
                         ((uintptr_t)st->cache & 15) == 0;
    // the sub-block maxima kernel stages each brick in shared memory anyway:
    // it also stores it into the cache slot (one read of the payload)
    const bool fused = sub_ok && sub_smem <= 48 * 1024 && aligned;
    if (d_payload) {
        const int nq = queued ? n_chunks : 1;
        const int32_t cq = queued ? chunk : n;
        for (int q = 0; q < nq; ++q) {
            const int32_t b0 = q * cq, nb = std::min<int32_t>(cq, n - b0);
            if (queued) RO_CUDA(cudaStreamWaitEvent(s, c->chunk_done[q], 0));
            const uint8_t *pq = d_payload + (int64_t)b0 * bvox;
            if (fused) {
                k_sub_max_smem<<<nb, kSubMaxThreads, sub_smem, s>>>(
                    nb, bx, by, bz, pq, d_slots + b0, d_final + b0, st->sub_max, st->cache);
            } else {
                if (aligned)
                    k_copy_payloads<<<blocks_for((bvox / 16) * nb), kThreads, 0, s>>>(
                        nb, bvox, pq, d_slots + b0, d_final + b0, st->cache);
                else
                    k_copy_payloads_bytes<<<blocks_for(bvox * nb), kThreads, 0, s>>>(
                        nb, bvox, pq, d_slots + b0, d_final + b0, st->cache);
                if (sub_ok) {
                    if (sub_smem <= 48 * 1024)
                        k_sub_max_smem<<<nb, kSubMaxThreads, sub_smem, s>>>(
                            nb, bx, by, bz, pq, d_slots + b0, d_final + b0, st->sub_max,
                            nullptr);
                    else
                        k_sub_max<<<nb, 128, 0, s>>>(nb, bx, by, bz, pq, d_slots + b0,
                                                     d_final + b0, st->sub_max);
                }
            }
            RO_CUDA(cudaGetLastError());
        }
    } else if (sub_ok) {  // payload unknown: "may be anything" (255) rows
        if (sub_smem <= 48 * 1024)
            k_sub_max_smem<<<n, kSubMaxThreads, sub_smem, s>>>(n, bx, by, bz, nullptr, d_slots,
                                                               d_final, st->sub_max, nullptr);
        else
            k_sub_max<<<n, 128, 0, s>>>(n, bx, by, bz, nullptr, d_slots, d_final,
                                        st->sub_max);
        RO_CUDA(cudaGetLastError());
    }
    if (slots_out) RO_CUDA(cudaMemcpyAsync(slots_out, d_slots, sizeof(int32_t) * n,
                                           cudaMemcpyDeviceToHost, s));
    if (evicted_out) RO_CUDA(cudaMemcpyAsync(evicted_out, d_evicted, sizeof(int64_t) * n,
                                             cudaMemcpyDeviceToHost, s));
    if (slots_out || evicted_out) RO_CUDA(cudaStreamSynchronize(s));
    return RO_OK;
}

// one-time costs of batches up to max_batch bricks: the batch / LRU /
// octree scratch, the payload upload slot, the pinned staging of pageable
// payloads, and every kernel of this file loaded
int lru_reserve(ro_ctx *c, int64_t max_batch) {
    if (max_batch < 1) return RO_OK;
    if (max_batch > (int64_t)1 << 30) return fail(RO_EINVAL, "batch too large");
    const int64_t n = max_batch;
    void *p;
    int rc;
    if ((rc = scratch(c, 1, sizeof(int64_t) * 4 * n + sizeof(int32_t) * n + n + 64, &p))) return rc;
    if ((rc = scratch(c, 13, sizeof(uint32_t) * kLruCtlWords, &p))) return rc;
    if ((rc = scratch(c, 6, sizeof(int64_t) * (2 * (size_t)n + 2) + sizeof(BrickInfo) * 2 * (size_t)n,
                      &p)))
        return rc;
    if ((rc = scratch(c, 12, (size_t)c->bvox * n, &p))) return rc;
    const size_t bytes = (size_t)c->bvox * n;
    if (c->staging_bytes < bytes) {
        RO_CUDA(cudaEventSynchronize(c->upload_done));
        if (c->staging) cudaFreeHost(c->staging);
        c->staging = nullptr;
        c->staging_bytes = 0;
        RO_CUDA(cudaMallocHost(&c->staging, bytes));
        c->staging_bytes = bytes;
    }
    RO_CUDA(cudaFuncSetAttribute(k_lru_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)topk::kSortSmem));
    const void *kernels[] = {(const void *)k_check_batch, (const void *)k_copy_payloads,
                             (const void *)k_copy_payloads_bytes, (const void *)k_sub_max,
                             (const void *)k_sub_max_smem,
                             (const void *)k_sub_max_all, (const void *)k_release,
                             (const void *)k_lru_batch, (const void *)k_octree_update,
                             (const void *)k_swap_release, (const void *)k_invalidate,
                             (const void *)k_set_metadata, (const void *)k_level_metadata,
                             (const void *)k_reset_range, (const void *)k_rebuild_leaves,
                             (const void *)k_rebuild_level};
    cudaFuncAttributes fa;
    for (const void *k : kernels) RO_CUDA(cudaFuncGetAttributes(&fa, k));
    int grid;
    if ((rc = coop_grid((const void *)k_lru_batch, topk::kSortSmem, &grid))) return rc;
    if ((rc = coop_grid((const void *)k_octree_update, 0, &grid))) return rc;
    return RO_OK;
}

int release_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n64,
                   int32_t status, int32_t update_octree, cudaStream_t s) {
    if (n64 <= 0) return RO_OK;
    const int32_t n = (int32_t)n64;
    for (int32_t i = 0; i < n; ++i) {
        Decoded d = decode_id(c->dl, ids_h[i]);
        if (!d.ok) return fail(RO_EINVAL, "brick id outside the layout");
    }
    void *p;
    int rc;
    if ((rc = scratch(c, 2, sizeof(int64_t) * n, &p))) return rc;
    int64_t *d_ids = (int64_t *)p;
    RO_CUDA(cudaMemcpyAsync(d_ids, ids_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    k_release<<<1, 1, 0, s>>>(c->dl, n, d_ids, status, st->pt, st->slot_brick,
                              st->slot_last_used, st->free_stack, st->free_count);
    RO_CUDA(cudaGetLastError());
    if (update_octree && st->words) return octree_update(c, st, d_ids, n, s);
    return RO_OK;
}

int apply_metadata(ro_ctx *c, const ro_state *st, const int64_t *node_h,
                   const int32_t *slot_h, const int32_t *mn_h, const int32_t *mx_h,
                   int64_t n64, cudaStream_t s) {
    if (n64 <= 0) return RO_OK;
    if (!st->words) return fail(RO_EINVAL, "no octree words");
    int32_t n = (int32_t)n64;
    for (int32_t i = 0; i < n; ++i) {
        if (node_h[i] < 0 || node_h[i] >= c->num_nodes)
            return fail(RO_EINVAL, "node index beyond tree depth");
        if (slot_h[i] < 0 || slot_h[i] >= c->layout.m) return fail(RO_EINVAL, "slot out of range");
        if (!(0 <= mn_h[i] && mn_h[i] <= mx_h[i] && mx_h[i] <= 255))
            return fail(RO_EINVAL, "need 0 <= min <= max <= 255");
    }
    // duplicates: later entries win (sequential semantics); drop earlier ones
    std::vector<int32_t> keep;
    {
        std::unordered_map<int64_t, int32_t> last;
        last.reserve((size_t)n * 2);
        for (int32_t i = 0; i < n; ++i) last[node_h[i] * c->layout.m + slot_h[i]] = i;
        keep.reserve(last.size());
        for (int32_t i = 0; i < n; ++i)
            if (last[node_h[i] * c->layout.m + slot_h[i]] == i) keep.push_back(i);
    }
    std::vector<int64_t> nodes(keep.size());
    std::vector<int32_t> slots(keep.size()), mns(keep.size()), mxs(keep.size());
    for (size_t j = 0; j < keep.size(); ++j) {
        nodes[j] = node_h[keep[j]];
        slots[j] = slot_h[keep[j]];
        mns[j] = mn_h[keep[j]];
        mxs[j] = mx_h[keep[j]];
    }
    node_h = nodes.data();
    slot_h = slots.data();
    mn_h = mns.data();
    mx_h = mxs.data();
    const int32_t n_in = n;
    (void)n_in;
    n = (int32_t)keep.size();
    void *p;
    int rc;
    size_t bytes = (sizeof(int64_t) + 3 * sizeof(int32_t)) * n;
    if ((rc = scratch(c, 2, bytes, &p))) return rc;
    int64_t *d_node = (int64_t *)p;
    int32_t *d_slot = (int32_t *)(d_node + n), *d_mn = d_slot + n, *d_mx = d_mn + n;
    RO_CUDA(cudaMemcpyAsync(d_node, node_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemcpyAsync(d_slot, slot_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemcpyAsync(d_mn, mn_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemcpyAsync(d_mx, mx_h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    k_set_metadata<<<(n + 255) / 256, 256, 0, s>>>(c->dl, n, d_node, d_slot, d_mn, d_mx,
                                                   st->words);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int write_level_metadata(ro_ctx *c, const ro_state *st, int32_t slot, int32_t d,
                         const uint8_t *mins, const uint8_t *maxs, cudaStream_t s) {
    if (!st->words) return fail(RO_EINVAL, "no octree words");
    if (slot < 0 || slot >= c->layout.m || d < 0 || d > c->layout.depth)
        return fail(RO_EINVAL, "slot/depth out of range");
    int64_t nn = int64_t(1) << (3 * d);
    k_level_metadata<<<blocks_for(nn), kThreads, 0, s>>>(c->dl, slot, d, mins, maxs, st->words);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int swap_channel(ro_ctx *c, const ro_state *st, int32_t cs, int32_t invalidate,
                 cudaStream_t s) {
    if (cs < 0 || cs >= c->layout.m) return fail(RO_EINVAL, "channel slot out of range");
    const int k = c->layout.k;
    const int64_t lo = c->layout.pt_offsets[cs * k], hi = c->layout.pt_offsets[cs * k + k];
    if (hi > lo) k_reset_range<<<blocks_for(hi - lo), kThreads, 0, s>>>(st->pt, lo, hi);
    void *pc;
    int rc, grid = 0;
    if ((rc = coop_grid((const void *)k_swap_release, 0, &grid))) return rc;
    if ((rc = scratch(c, 14, sizeof(uint32_t) * grid, &pc))) return rc;
    DevLayout L = c->dl;
    int32_t cs_ = cs;
    int64_t *sb = st->slot_brick, *lu = st->slot_last_used;
    int32_t *fs = st->free_stack, *fc = st->free_count;
    uint32_t *cnt = (uint32_t *)pc;
    void *args[] = {&L, &cs_, &sb, &lu, &fs, &fc, &cnt};
    RO_CUDA(cudaLaunchCooperativeKernel((const void *)k_swap_release, dim3(grid),
                                        dim3(kCoopThreads), args, 0, s));
    if (invalidate && st->words)
        k_invalidate<<<blocks_for(c->num_nodes), kThreads, 0, s>>>(c->dl, cs, st->words);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int octree_update_host(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n64,
                       cudaStream_t s) {
    if (n64 <= 0) return RO_OK;
    const int32_t n = (int32_t)n64;
    for (int32_t i = 0; i < n; ++i)
        if (!decode_id(c->dl, ids_h[i]).ok) return fail(RO_EINVAL, "brick id outside the layout");
    void *p;
    int rc;
    if ((rc = scratch(c, 2, sizeof(int64_t) * n, &p))) return rc;
    RO_CUDA(cudaMemcpyAsync(p, ids_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    return octree_update(c, st, (const int64_t *)p, n, s);
}

int rebuild_masks(ro_ctx *c, const ro_state *st, cudaStream_t s) {
    if (!st->words) return fail(RO_EINVAL, "no octree words");
    const int D = c->layout.depth;
    k_rebuild_leaves<<<kGridStride, kThreads, 0, s>>>(c->dl, st->pt, st->words);
    for (int dd = D - 1; dd >= 0; --dd)
        k_rebuild_level<<<kGridStride, kThreads, 0, s>>>(c->dl, dd, st->words);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int rebuild_sub_max(ro_ctx *c, const ro_state *st, cudaStream_t s) {
    if (!st->sub_max || c->layout.brick[0] < RO_SUB_E || c->layout.brick[1] < RO_SUB_E ||
        c->layout.brick[2] < RO_SUB_E)
        return RO_OK;
    const int64_t S = c->S;
    const unsigned g = (unsigned)(S < 148 * 64 ? S : 148 * 64);
    k_sub_max_all<<<g, 128, 0, s>>>(S, c->layout.brick[0], c->layout.brick[1],
                                    c->layout.brick[2], st->cache, st->slot_brick, st->sub_max);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

}  // namespace ro
