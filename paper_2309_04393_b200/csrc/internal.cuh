// internal.cuh -- shared device helpers and the context of libresoct.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/resoct.h"

#define RO_BVOX_MAX (1 << 21)

// edge of the sub-blocks of ro_state.sub_max (RO_SUB_E^3 voxels)
#ifndef RO_SUB_LOG
#define RO_SUB_LOG 2  // 4^3 sub-blocks: measured 8 % faster ray cast than 8^3, same as 2^3
#endif
#define RO_SUB_E (1 << RO_SUB_LOG)  // == RO_SUB_EDGE of resoct.h in the default build

namespace ro {

// thread-local last error (ro_last_error)
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define RO_CUDA(call)                                                    \
    do {                                                                 \
        cudaError_t _e = (call);                                         \
        if (_e != cudaSuccess) return ro::cuda_fail(_e, #call);          \
    } while (0)

// ---------------------------------------------------------------------------
// geometry helpers (device + host), all integer
// ---------------------------------------------------------------------------

__host__ __device__ inline int64_t level_offset(int d) {
    return ((int64_t(1) << (3 * d)) - 1) / 7;
}

__host__ __device__ inline int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) {
    return -floor_div(-a, b);
}

// Device copy of the layout (passed by value into kernels).
struct DevLayout {
    int32_t m, k, depth, npt;
    int32_t bx, by, bz, _pad;
    int32_t dims[RO_MAX_LEVELS][3];
    int32_t grids[RO_MAX_LEVELS][3];
    int64_t pt_off[RO_MAX_PT + 1];
    int64_t num_slots, E, num_nodes, bvox;
};

// page-table entry index of (slot, level, coord) -- kernels.py:187-191
__host__ __device__ inline int64_t entry_index(const DevLayout &L, int slot,
                                               int lev, int cx, int cy, int cz) {
    int gx = L.grids[lev][0], gy = L.grids[lev][1];
    return L.pt_off[slot * L.k + lev] + ((int64_t)cz * gy + cy) * gx + cx;
}

// brick id codec -- paging.py:43-61
__host__ __device__ inline int64_t encode_id(const DevLayout &L, int slot,
                                             int lev, int cx, int cy, int cz) {
    return ((int64_t)(slot * L.k + lev) << 24) | ((int64_t)cz << 16) |
           ((int64_t)cy << 8) | (int64_t)cx;
}

struct Decoded {
    int slot, lev, x, y, z;
    bool ok;
};

__host__ __device__ inline Decoded decode_id(const DevLayout &L, int64_t id) {
    Decoded d;
    d.ok = id >= 0 && id < (int64_t(1) << 32);
    int pt = (int)((id >> 24) & 0xFF);
    d.slot = pt / L.k;
    d.lev = pt % L.k;
    d.x = (int)(id & 0xFF);
    d.y = (int)((id >> 8) & 0xFF);
    d.z = (int)((id >> 16) & 0xFF);
    if (d.slot >= L.m) d.ok = false;
    if (d.ok) {
        if (d.x >= L.grids[d.lev][0] || d.y >= L.grids[d.lev][1] ||
            d.z >= L.grids[d.lev][2])
            d.ok = false;
    }
    return d;
}

// entry index -> brick id (inverse of entry_index)
__host__ __device__ inline int64_t entry_to_id(const DevLayout &L, int64_t e) {
    int lo = 0, hi = L.npt - 1;  // find pt with pt_off[pt] <= e < pt_off[pt+1]
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (L.pt_off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    int pt = lo;
    int lev = pt % L.k;
    int64_t local = e - L.pt_off[pt];
    int gx = L.grids[lev][0], gy = L.grids[lev][1];
    int x = (int)(local % gx);
    int y = (int)((local / gx) % gy);
    int z = (int)(local / ((int64_t)gx * gy));
    return ((int64_t)pt << 24) | ((int64_t)z << 16) | ((int64_t)y << 8) | x;
}

// leaves (depth D) overlapping a brick's open box -- octree.py:126-159
struct Box3 {
    int lo[3], hi[3];
    bool empty;
};

__host__ __device__ inline Box3 leaf_box(const DevLayout &L, int lev, int cx,
                                         int cy, int cz) {
    Box3 b;
    b.empty = false;
    int64_t side = int64_t(1) << L.depth;
    int c[3] = {cx, cy, cz};
    int B[3] = {L.bx, L.by, L.bz};
    for (int a = 0; a < 3; ++a) {
        int64_t dim = L.dims[lev][a];
        int64_t lo = floor_div((int64_t)c[a] * B[a] * side, dim);
        int64_t hi = ceil_div((int64_t)(c[a] + 1) * B[a] * side, dim) - 1;
        if (lo < 0) lo = 0;
        if (hi > side - 1) hi = side - 1;
        if (lo > hi) b.empty = true;
        b.lo[a] = (int)lo;
        b.hi[a] = (int)hi;
    }
    return b;
}

// bricks of `lev` overlapping node (d, x, y, z) -- octree.py:161-189
__host__ __device__ inline Box3 brick_box(const DevLayout &L, int d, int nx,
                                          int ny, int nz, int lev) {
    Box3 b;
    b.empty = false;
    int64_t side = int64_t(1) << d;
    int n[3] = {nx, ny, nz};
    int B[3] = {L.bx, L.by, L.bz};
    for (int a = 0; a < 3; ++a) {
        int64_t dim = L.dims[lev][a];
        int64_t grid = L.grids[lev][a];
        int64_t lo = floor_div((int64_t)n[a] * dim, side * B[a]);
        int64_t hi = ceil_div((int64_t)(n[a] + 1) * dim, side * B[a]) - 1;
        if (lo < 0) lo = 0;
        if (hi > grid - 1) hi = grid - 1;
        if (lo > hi) b.empty = true;
        b.lo[a] = (int)lo;
        b.hi[a] = (int)hi;
    }
    return b;
}

}  // namespace ro

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------

struct ro_ctx {
    ro_layout layout;
    ro::DevLayout dl;
    int64_t E, num_nodes, n_meta, S, bvox;

    // feedback: first-seen keys + touched lists (render -> collect)
    unsigned long long *brick_key = nullptr;  // [E]
    unsigned long long *meta_key = nullptr;   // [n_meta] (lazy, needs words)
    int32_t *brick_touched = nullptr;         // [E]
    int32_t *meta_touched = nullptr;          // [n_meta]
    int32_t *touched_n = nullptr;             // [2] device
    int64_t *pinned_small = nullptr;          // host pinned scratch [64]

    // generic grow-only device scratch
    // 0-7 feedback / octree / ingest / metadata passes, 11 feedback control,
    // 12 brick-payload upload (its own: a DMA may still be running into it),
    // 13 LRU control, 14 swap counts
    void *scratch[16] = {nullptr};
    size_t scratch_bytes[16] = {0};
    // pinned host staging for payload uploads
    void *staging = nullptr;
    size_t staging_bytes = 0;
    cudaStream_t upload = nullptr;
    cudaEvent_t upload_done = nullptr;
    // the payload upload in chunks: chunk q landed (apply_bricks)
    static constexpr int kUploadChunks = 8;
    cudaEvent_t chunk_done[kUploadChunks] = {};
    cudaEvent_t host_done = nullptr;
    uint32_t *claim = nullptr;  // [E] batch dedupe stamps
    // caller-owned key arrays (ro_set_feedback_buffers; possibly another
    // process's over peer memory) replacing brick_key / meta_key when set
    unsigned long long *brick_key_ext = nullptr;
    unsigned long long *meta_key_ext = nullptr;
    uint32_t epoch = 0;
    // per-frame node classes of the ray caster's residency walk (raycast.cu
    // k_classify_nodes): [num_nodes] bytes, allocated with the context
    // per-frame node classes (k_classify): fast flags, path classes (depth <= 7)
    uint8_t *node_fast = nullptr;
    uint64_t *node_path = nullptr;
    // a ray-cast pass left first-seen keys that no ro_feedback_collect has
    // consumed (and reset) yet
    bool keys_dirty = false;
};

namespace ro {
// first-seen key arrays in use (external ones when set)
inline unsigned long long *brick_keys(ro_ctx *c) {
    return c->brick_key_ext ? c->brick_key_ext : c->brick_key;
}
inline unsigned long long *meta_keys(ro_ctx *c) {
    return c->meta_key_ext ? c->meta_key_ext : c->meta_key;
}
// grow-only scratch buffer i of at least `bytes`
int scratch(ro_ctx *c, int i, size_t bytes, void **out);
int ensure_meta_keys(ro_ctx *c);
}  // namespace ro
