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
#include <cub/cub.cuh>

#include <cstring>
#include <unordered_map>
#include <vector>

#include "internal.cuh"

namespace ro {

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

// phase (i): pop the free list top-first
__global__ void k_assign_free(int32_t n1, const int32_t *__restrict__ free_stack,
                              int32_t free_count, int32_t *__restrict__ slots,
                              int64_t *__restrict__ evicted) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n1) return;
    slots[i] = free_stack[free_count - 1 - i];
    evicted[i] = -1;
}

// stale keys: (last_used << 32 | slot) for occupied slots with last_used < frame
__global__ void k_stale_keys(const int64_t *__restrict__ slot_brick,
                             const int64_t *__restrict__ last_used, int64_t S,
                             int64_t frame, unsigned long long *__restrict__ keys,
                             int32_t *__restrict__ count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += stride) {
        if (slot_brick[s] >= 0 && last_used[s] < frame) {
            int pos = atomicAdd(count, 1);
            keys[pos] = ((unsigned long long)last_used[s] << 32) | (unsigned long long)s;
        }
    }
}

// phases (ii) and (iii)
__global__ void k_assign_victims(int32_t n1, int32_t n, int32_t n2,
                                 const unsigned long long *__restrict__ sorted,
                                 const int64_t *__restrict__ slot_brick,
                                 const int64_t *__restrict__ ids,
                                 int32_t *__restrict__ slots,
                                 int64_t *__restrict__ evicted) {
    int i = n1 + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int j = i - n1;
    if (j < n2) {
        int32_t s = (int32_t)(sorted[j] & 0xFFFFFFFFull);
        slots[i] = s;
        evicted[i] = slot_brick[s];
    } else {
        slots[i] = 0;
        // first phase-(iii) insert: fixed up by k_phase3_first
        evicted[i] = (i == n1 + n2) ? -2 : ids[i - 1];
    }
}

// occupant of slot 0 when phase (iii) starts
__global__ void k_phase3_first(int32_t p3, const int32_t *__restrict__ slots,
                               const int64_t *__restrict__ ids,
                               const int64_t *__restrict__ slot_brick,
                               int64_t *__restrict__ evicted) {
    int64_t occ = slot_brick[0];
    for (int i = p3 - 1; i >= 0; --i) {
        if (slots[i] == 0) { occ = ids[i]; break; }
    }
    evicted[p3] = occ;
}

// map batch bricks; final occupants own their slot
__global__ void k_map_batch(const DevLayout L, int32_t n, int32_t p3,
                            const int64_t *__restrict__ ids,
                            const int64_t *__restrict__ entries,
                            const int32_t *__restrict__ slots,
                            int32_t *__restrict__ pt,
                            int64_t *__restrict__ slot_brick,
                            int64_t *__restrict__ last_used, int64_t frame,
                            uint8_t *__restrict__ final_flag) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t s = slots[i];
    pt[entries[i]] = s;
    bool final_occ = (p3 >= n) ? true : (s == 0 ? i == n - 1 : true);
    final_flag[i] = final_occ ? 1 : 0;
    if (final_occ) slot_brick[s] = ids[i];
    last_used[s] = frame;
}

__global__ void k_unmap_evicted(const DevLayout L, int32_t n,
                                const int64_t *__restrict__ evicted,
                                int32_t *__restrict__ pt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t v = evicted[i];
    if (v < 0) return;
    Decoded d = decode_id(L, v);
    pt[entry_index(L, d.slot, d.lev, d.x, d.y, d.z)] = RO_PT_UNMAPPED;
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
__global__ void k_sequential_insert(const DevLayout L, int32_t n,
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

// ---- octree: per changed brick, node boxes at every depth ----
struct BrickBoxes {
    int slot, lev;
    int lo[3], hi[3];  // leaf box at depth D
    bool empty;
};

__global__ void k_brick_counts(const DevLayout L, int32_t n,
                               const int64_t *__restrict__ ids,
                               int64_t *__restrict__ counts /* [(D+1)*n] */) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t id = ids[i];
    Box3 b;
    b.empty = true;
    if (id >= 0) {
        Decoded d = decode_id(L, id);
        if (d.ok) b = leaf_box(L, d.lev, d.x, d.y, d.z);
    }
    for (int dd = 0; dd <= L.depth; ++dd) {
        int64_t c = 0;
        if (!b.empty) {
            int sh = L.depth - dd;
            c = 1;
            for (int a = 0; a < 3; ++a) c *= (int64_t)((b.hi[a] >> sh) - (b.lo[a] >> sh) + 1);
        }
        counts[(int64_t)dd * n + i] = c;
    }
}

__device__ __forceinline__ int find_seg(const int64_t *__restrict__ off, int n, int64_t j) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// depth D: recompute the (slot, level) bit of each overlapped leaf
__global__ void k_update_leaves(const DevLayout L, int32_t n,
                                const int64_t *__restrict__ ids,
                                const int64_t *__restrict__ off /* level D seg */,
                                const int64_t *__restrict__ total_p,
                                const int32_t *__restrict__ pt,
                                uint32_t *__restrict__ words) {
    const int64_t total = *total_p;
    const int D = L.depth;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        int i = find_seg(off, n, j);
        Decoded d = decode_id(L, ids[i]);
        Box3 b = leaf_box(L, d.lev, d.x, d.y, d.z);
        int64_t r = j - off[i];
        int w = b.hi[0] - b.lo[0] + 1, h = b.hi[1] - b.lo[1] + 1;
        int lx = b.lo[0] + (int)(r % w);
        int lyy = b.lo[1] + (int)((r / w) % h);
        int lz = b.lo[2] + (int)(r / ((int64_t)w * h));
        Box3 bb = brick_box(L, D, lx, lyy, lz, d.lev);
        bool backed = false;
        if (!bb.empty) {
            for (int z = bb.lo[2]; z <= bb.hi[2] && !backed; ++z)
                for (int y = bb.lo[1]; y <= bb.hi[1] && !backed; ++y)
                    for (int x = bb.lo[0]; x <= bb.hi[0]; ++x)
                        if (pt[entry_index(L, d.slot, d.lev, x, y, z)] >= 0) { backed = true; break; }
        }
        int64_t side = int64_t(1) << D;
        int64_t nidx = level_offset(D) + ((int64_t)lz * side + lyy) * side + lx;
        uint32_t bit = 1u << d.lev;
        if (backed) atomicOr(words + nidx * L.m + d.slot, bit);
        else atomicAnd(words + nidx * L.m + d.slot, ~bit);
    }
}

// depth dd < D: mask = OR of the 8 children's masks
__global__ void k_update_parents(const DevLayout L, int32_t n, int dd,
                                 const int64_t *__restrict__ ids,
                                 const int64_t *__restrict__ off,
                                 const int64_t *__restrict__ total_p,
                                 uint32_t *__restrict__ words) {
    const int64_t total = *total_p;
    const int sh = L.depth - dd;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
         j += (int64_t)gridDim.x * blockDim.x) {
        int i = find_seg(off, n, j);
        Decoded d = decode_id(L, ids[i]);
        Box3 b = leaf_box(L, d.lev, d.x, d.y, d.z);
        int lo0 = b.lo[0] >> sh, lo1 = b.lo[1] >> sh, lo2 = b.lo[2] >> sh;
        int w = (b.hi[0] >> sh) - lo0 + 1, h = (b.hi[1] >> sh) - lo1 + 1;
        int64_t r = j - off[i];
        int nx = lo0 + (int)(r % w);
        int ny = lo1 + (int)((r / w) % h);
        int nz = lo2 + (int)(r / ((int64_t)w * h));
        int64_t cside = int64_t(1) << (dd + 1);
        int64_t cbase = level_offset(dd + 1);
        uint32_t mask = 0;
        for (int c = 0; c < 8; ++c) {
            int64_t cx = 2 * nx + (c & 1), cy = 2 * ny + ((c >> 1) & 1), cz = 2 * nz + (c >> 2);
            mask |= words[(cbase + (cz * cside + cy) * cside + cx) * L.m + d.slot] & 0xFFFFu;
        }
        int64_t side = int64_t(1) << dd;
        uint32_t *wp = words + (level_offset(dd) + ((int64_t)nz * side + ny) * side + nx) * L.m + d.slot;
        uint32_t old = *wp;
        uint32_t nw = (old & 0xFFFF0000u) | mask;
        if (nw != old) *wp = nw;
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

__global__ void k_swap_flags(const DevLayout L, const int64_t *__restrict__ slot_brick,
                             int32_t cs, int32_t *__restrict__ flags) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L.num_slots;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = slot_brick[s];
        flags[s] = (b >= 0 && (int)(((b >> 24) & 0xFF) / L.k) == cs) ? 1 : 0;
    }
}

// push released slots onto the free list in ascending slot order
__global__ void k_swap_release(const DevLayout L, const int32_t *__restrict__ flags,
                               const int32_t *__restrict__ pos,
                               int64_t *__restrict__ slot_brick,
                               int64_t *__restrict__ last_used,
                               int32_t *__restrict__ free_stack,
                               const int32_t *__restrict__ free_count) {
    const int32_t base = *free_count;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L.num_slots;
         s += (int64_t)gridDim.x * blockDim.x) {
        if (flags[s]) {
            slot_brick[s] = -1;
            last_used[s] = 0;
            free_stack[base + pos[s]] = (int32_t)s;
        }
    }
}

__global__ void k_swap_count(const DevLayout L, const int32_t *__restrict__ flags,
                             const int32_t *__restrict__ pos,
                             int32_t *__restrict__ free_count) {
    int64_t last = L.num_slots - 1;
    *free_count += pos[last] + flags[last];
}

__global__ void k_invalidate(const DevLayout L, int32_t slot, uint32_t *__restrict__ words) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.num_nodes;
         i += (int64_t)gridDim.x * blockDim.x)
        words[i * L.m + slot] = 0x00FF0000u;
}

__global__ void k_sub_free(int32_t *free_count, int32_t n1) { *free_count -= n1; }

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
    const int D = c->layout.depth;
    const int64_t nseg = (int64_t)(D + 1) * n;
    void *pc, *po, *tmp;
    int rc;
    if ((rc = scratch(c, 5, sizeof(int64_t) * (nseg + D + 1), &pc))) return rc;
    if ((rc = scratch(c, 6, sizeof(int64_t) * (nseg + D + 1), &po))) return rc;
    int64_t *counts = (int64_t *)pc, *offs = (int64_t *)po;
    k_brick_counts<<<(n + 255) / 256, 256, 0, s>>>(c->dl, n, ids, counts);
    RO_CUDA(cudaGetLastError());
    // per-level exclusive scans; the level total is stored after the segments
    size_t tb = 0, tb2 = 0;
    RO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, offs, (int)n, s));
    RO_CUDA(cub::DeviceReduce::Sum(nullptr, tb2, counts, offs, (int)n, s));
    if (tb2 > tb) tb = tb2;
    if ((rc = scratch(c, 7, tb, &tmp))) return rc;
    int64_t *totals = offs + nseg;
    for (int dd = D; dd >= 0; --dd) {
        int64_t *cseg = counts + (int64_t)dd * n, *oseg = offs + (int64_t)dd * n;
        RO_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cseg, oseg, (int)n, s));
        // total = off[n-1] + count[n-1]: folded into the kernels via a tiny add
        RO_CUDA(cub::DeviceReduce::Sum(tmp, tb, cseg, totals + dd, (int)n, s));
        if (dd == D)
            k_update_leaves<<<kGridStride, kThreads, 0, s>>>(c->dl, n, ids, oseg,
                                                             totals + dd, st->pt, st->words);
        else
            k_update_parents<<<kGridStride, kThreads, 0, s>>>(c->dl, n, dd, ids, oseg,
                                                              totals + dd, st->words);
        RO_CUDA(cudaGetLastError());
    }
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
    int rc;
    void *p;
    // device scratch layout (slot 0..4 are feedback's; use a dedicated pool)
    // ids | evicted | entries | slots | final | flag   (ids+evicted contiguous:
    // together they are the changed set of the octree pass)
    size_t need = sizeof(int64_t) * 3 * n + sizeof(int32_t) * n + n + 64;
    if ((rc = scratch(c, 1, need, &p))) return rc;
    int64_t *d_ids = (int64_t *)p;
    int64_t *d_evicted = d_ids + n;
    int64_t *d_entries = d_evicted + n;
    int32_t *d_slots = (int32_t *)(d_entries + n);
    uint8_t *d_final = (uint8_t *)(d_slots + n);
    int32_t *d_flag = (int32_t *)(((uintptr_t)(d_final + n) + 15) & ~(uintptr_t)15);

    // payload upload on the side stream (overlaps the checks)
    const uint8_t *d_payload = nullptr;
    bool caller_pinned = false;
    // a DMA from the caller's pinned buffer completes before any return
    struct UploadWait {
        ro_ctx *c;
        const bool *on;
        ~UploadWait() { if (*on) cudaEventSynchronize(c->upload_done); }
    } upload_wait{c, &caller_pinned};
    if (payloads) {
        if (on_device) {
            d_payload = (const uint8_t *)payloads;
        } else {
            void *dp;
            if ((rc = scratch(c, 2, (size_t)bvox * n, &dp))) return rc;
            size_t bytes = (size_t)bvox * n;
            // payloads already in pinned memory are DMA'd straight from the
            // caller's buffer (waited for before returning); pageable ones go
            // through the handle's pinned staging buffer
            cudaPointerAttributes pa;
            if (cudaPointerGetAttributes(&pa, payloads) != cudaSuccess) {
                cudaGetLastError();
                pa.type = cudaMemoryTypeUnregistered;
            }
            caller_pinned = pa.type == cudaMemoryTypeHost;
            const void *src = payloads;
            if (!caller_pinned) {
                if (c->staging_bytes < bytes) {
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
            RO_CUDA(cudaMemcpyAsync(dp, src, bytes, cudaMemcpyHostToDevice, c->upload));
            RO_CUDA(cudaEventRecord(c->upload_done, c->upload));
            d_payload = (const uint8_t *)dp;
        }
    }
    RO_CUDA(cudaMemcpyAsync(d_ids, ids_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), s));
    if (++c->epoch == 0) {  // stamp wrap: clear claims
        RO_CUDA(cudaMemsetAsync(c->claim, 0, sizeof(uint32_t) * c->E, s));
        c->epoch = 1;
    }
    k_check_batch<<<(n + 255) / 256, 256, 0, s>>>(c->dl, d_ids, n, st->pt, c->claim,
                                                  c->epoch, d_flag, d_entries);
    RO_CUDA(cudaGetLastError());
    int32_t *h = reinterpret_cast<int32_t *>(c->pinned_small);
    RO_CUDA(cudaMemcpyAsync(h, d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaMemcpyAsync(h + 1, st->free_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaStreamSynchronize(s));
    const int32_t flag = h[0], free_count = h[1];
    if (flag & 2) {
        std::vector<int64_t> back(n), ent(n);
        cudaMemcpy(back.data(), d_ids, sizeof(int64_t) * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(ent.data(), d_entries, sizeof(int64_t) * n, cudaMemcpyDeviceToHost);
        int32_t bad = -1;
        for (int32_t i = 0; i < n; ++i)
            if (ent[i] < 0) { bad = i; break; }
        char msg[256];
        snprintf(msg, sizeof msg,
                 "brick id outside the layout (flag %d, n %d, first bad index %d, "
                 "device id %lld, host id %lld)", flag, n, bad,
                 bad >= 0 ? (long long)back[bad] : -1LL,
                 bad >= 0 ? (long long)ids_h[bad] : -1LL);
        return fail(RO_EINVAL, msg);
    }

    int32_t p3 = n;  // first phase-(iii) index
    if (flag == 0) {
        const int32_t n1 = n < free_count ? n : free_count;
        if (n1 > 0) {
            k_assign_free<<<(n1 + 255) / 256, 256, 0, s>>>(n1, st->free_stack, free_count,
                                                           d_slots, d_evicted);
            k_sub_free<<<1, 1, 0, s>>>(st->free_count, n1);
        }
        if (n > n1) {
            void *pk, *pk2, *ptmp;
            const int64_t S = c->S;
            if ((rc = scratch(c, 3, sizeof(unsigned long long) * S + 16, &pk))) return rc;
            if ((rc = scratch(c, 0, sizeof(unsigned long long) * S, &pk2))) return rc;
            auto *keys = (unsigned long long *)pk, *sorted = (unsigned long long *)pk2;
            int32_t *d_cnt = (int32_t *)(keys + S);
            RO_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int32_t), s));
            k_stale_keys<<<blocks_for(S), kThreads, 0, s>>>(st->slot_brick, st->slot_last_used,
                                                             S, frame, keys, d_cnt);
            RO_CUDA(cudaMemcpyAsync(h + 2, d_cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            RO_CUDA(cudaStreamSynchronize(s));
            const int32_t n_stale = h[2];
            const int32_t want = n - n1;
            const int32_t n2 = want < n_stale ? want : n_stale;
            if (n_stale > 0) {
                size_t tb = 0;
                RO_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, n_stale, 0, 64, s));
                if ((rc = scratch(c, 4, tb, &ptmp))) return rc;
                RO_CUDA(cub::DeviceRadixSort::SortKeys(ptmp, tb, keys, sorted, n_stale, 0, 64, s));
            }
            k_assign_victims<<<(want + 255) / 256, 256, 0, s>>>(n1, n, n2, sorted, st->slot_brick,
                                                                d_ids, d_slots, d_evicted);
            RO_CUDA(cudaGetLastError());
            if (n1 + n2 < n) {
                p3 = n1 + n2;
                k_phase3_first<<<1, 1, 0, s>>>(p3, d_slots, d_ids, st->slot_brick, d_evicted);
            }
        }
        k_map_batch<<<(n + 255) / 256, 256, 0, s>>>(c->dl, n, p3, d_ids, d_entries, d_slots,
                                                    st->pt, st->slot_brick, st->slot_last_used,
                                                    frame, d_final);
        k_unmap_evicted<<<(n + 255) / 256, 256, 0, s>>>(c->dl, n, d_evicted, st->pt);
        RO_CUDA(cudaGetLastError());
    } else {
        k_sequential_insert<<<1, 1, 0, s>>>(c->dl, n, d_ids, st->pt, st->slot_brick,
                                            st->slot_last_used, st->free_stack, st->free_count,
                                            frame, d_slots, d_evicted, d_final);
        RO_CUDA(cudaGetLastError());
    }
    if (d_payload) {
        if (!on_device) RO_CUDA(cudaStreamWaitEvent(s, c->upload_done, 0));
        if (bvox % 16 == 0 && ((uintptr_t)d_payload & 15) == 0 &&
            ((uintptr_t)st->cache & 15) == 0)
            k_copy_payloads<<<blocks_for((bvox / 16) * n), kThreads, 0, s>>>(
                n, bvox, d_payload, d_slots, d_final, st->cache);
        else
            k_copy_payloads_bytes<<<blocks_for(bvox * n), kThreads, 0, s>>>(
                n, bvox, d_payload, d_slots, d_final, st->cache);
        RO_CUDA(cudaGetLastError());
    }
    if (st->sub_max && c->layout.brick[0] >= RO_SUB_E && c->layout.brick[1] >= RO_SUB_E &&
        c->layout.brick[2] >= RO_SUB_E) {
        k_sub_max<<<n, 128, 0, s>>>(n, c->layout.brick[0], c->layout.brick[1],
                                    c->layout.brick[2], d_payload, d_slots, d_final,
                                    st->sub_max);
        RO_CUDA(cudaGetLastError());
    }
    if (update_octree && st->words) {
        // changed = batch bricks + evicted residents
        rc = octree_update(c, st, d_ids, 2 * n, s);
        if (rc) return rc;
    }
    if (slots_out) RO_CUDA(cudaMemcpyAsync(slots_out, d_slots, sizeof(int32_t) * n,
                                           cudaMemcpyDeviceToHost, s));
    if (evicted_out) RO_CUDA(cudaMemcpyAsync(evicted_out, d_evicted, sizeof(int64_t) * n,
                                             cudaMemcpyDeviceToHost, s));
    if (slots_out || evicted_out) RO_CUDA(cudaStreamSynchronize(s));
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
    const int64_t S = c->S;
    void *pf, *pp, *tmp;
    int rc;
    if ((rc = scratch(c, 2, sizeof(int32_t) * S, &pf))) return rc;
    if ((rc = scratch(c, 3, sizeof(int32_t) * S, &pp))) return rc;
    int32_t *flags = (int32_t *)pf, *pos = (int32_t *)pp;
    k_swap_flags<<<blocks_for(S), kThreads, 0, s>>>(c->dl, st->slot_brick, cs, flags);
    size_t tb = 0;
    RO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, pos, (int)S, s));
    if ((rc = scratch(c, 4, tb, &tmp))) return rc;
    RO_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, pos, (int)S, s));
    k_swap_release<<<blocks_for(S), kThreads, 0, s>>>(c->dl, flags, pos, st->slot_brick,
                                                       st->slot_last_used, st->free_stack,
                                                       st->free_count);
    k_swap_count<<<1, 1, 0, s>>>(c->dl, flags, pos, st->free_count);
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
