// api.cu -- the extern "C" boundary of libresoct.so (include/resoct.h).
#include <cstdio>
#include <cstring>
#include <string>

#include <vector>

#include "internal.cuh"

namespace ro {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? RO_ENOMEM : RO_ECUDA;
}

int scratch(ro_ctx *c, int i, size_t bytes, void **out) {
    if (bytes == 0) bytes = 16;
    if (c->scratch_bytes[i] < bytes) {
        if (c->scratch[i]) cudaFree(c->scratch[i]);
        c->scratch[i] = nullptr;
        c->scratch_bytes[i] = 0;
        size_t want = bytes + bytes / 4;
        RO_CUDA(cudaMalloc(&c->scratch[i], want));
        c->scratch_bytes[i] = want;
    }
    *out = c->scratch[i];
    return RO_OK;
}

int ensure_meta_keys(ro_ctx *c) {
    if (c->meta_key) return RO_OK;
    RO_CUDA(cudaMalloc(&c->meta_key, sizeof(unsigned long long) * c->n_meta));
    RO_CUDA(cudaMemset(c->meta_key, 0xFF, sizeof(unsigned long long) * c->n_meta));
    RO_CUDA(cudaMalloc(&c->meta_touched, sizeof(int32_t) * c->n_meta));
    return RO_OK;
}

int render(ro_ctx *c, const ro_frame *F, const ro_state *st, const ro_outputs *out,
           cudaStream_t s);
int feedback_collect(ro_ctx *c, int64_t budget, int32_t bricks_first,
                     const ro_feedback *fb, cudaStream_t s);
int note_sampled(ro_ctx *c, const ro_state *st, const uint8_t *required,
                 int64_t frame, cudaStream_t s);
int feedback_merge(ro_ctx *c, const int64_t *blocks, const int64_t *counts, int32_t n_parts,
                   int64_t budget, cudaStream_t s);
int gather_rows(const float *parts, int32_t n_parts, int64_t part_stride, int32_t height,
                int32_t width, int32_t tile_rows, float *full, cudaStream_t s);
int apply_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                 const void *payloads, int32_t on_device, int64_t frame,
                 int32_t update_octree, int32_t *slots_out, int64_t *evicted_out,
                 cudaStream_t s);
int release_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                   int32_t status, int32_t update_octree, cudaStream_t s);
int apply_metadata(ro_ctx *c, const ro_state *st, const int64_t *node_h,
                   const int32_t *slot_h, const int32_t *mn_h, const int32_t *mx_h,
                   int64_t n, cudaStream_t s);
int write_level_metadata(ro_ctx *c, const ro_state *st, int32_t slot, int32_t d,
                         const uint8_t *mins, const uint8_t *maxs, cudaStream_t s);
int swap_channel(ro_ctx *c, const ro_state *st, int32_t cs, int32_t invalidate,
                 cudaStream_t s);
int rebuild_masks(ro_ctx *c, const ro_state *st, cudaStream_t s);
int octree_update_host(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                       cudaStream_t s);

int lz4_decode(ro_ctx *c, const uint8_t *src, const int64_t *off, int64_t n, uint8_t *dst,
               int64_t stride, int64_t expected, int32_t *status, int32_t *first_bad,
               cudaStream_t s);
int apply_bricks_lz4(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                     const uint8_t *frames, const int64_t *off_h, int32_t on_device,
                     int64_t frame, int32_t update_octree, int32_t *slots_out,
                     int64_t *evicted_out, cudaStream_t s);
int normalize_to_u8(ro_ctx *c, const void *src, int32_t dtype, int64_t n, uint8_t *dst,
                    cudaStream_t s);
int downsample_box(const uint8_t *src, int32_t dx, int32_t dy, int32_t dz, int32_t fx,
                   int32_t fy, int32_t fz, uint8_t *dst, cudaStream_t s);
int extract_bricks(const uint8_t *level, int32_t dx, int32_t dy, int32_t dz, int32_t bx,
                   int32_t by, int32_t bz, uint8_t *dst, cudaStream_t s);

int node_minmax(ro_ctx *c, const uint8_t *vol, int32_t dx, int32_t dy, int32_t dz, int32_t d,
                int32_t pad, uint8_t *mins, uint8_t *maxs, cudaStream_t s);
int fill_metadata(ro_ctx *c, const ro_state *st, int32_t slot, const uint8_t *vol, int32_t dx,
                  int32_t dy, int32_t dz, int32_t pad, cudaStream_t s);
int bricks_box_minmax(const uint8_t *bricks, const int32_t *boxes, int64_t n, int32_t bx,
                      int32_t by, int32_t bz, uint8_t *mins, uint8_t *maxs, cudaStream_t s);
int rebuild_sub_max(ro_ctx *c, const ro_state *st, cudaStream_t s);
int feedback_reserve(ro_ctx *c);
int lru_reserve(ro_ctx *c, int64_t max_batch);
int raycast_warm(ro_ctx *c);

static int check_state(const ro_ctx *c, const ro_state *st) {
    if (!c) return fail(RO_EINVAL, "null context");
    if (!st || !st->pt || !st->slot_brick || !st->slot_last_used || !st->free_stack ||
        !st->free_count)
        return fail(RO_EINVAL, "incomplete state pointers");
    return RO_OK;
}

}  // namespace ro

using namespace ro;

extern "C" {

int ro_abi_version(void) { return RO_ABI_VERSION; }

const char *ro_last_error(void) { return g_err.c_str(); }

int64_t ro_local_rows(int32_t height, int32_t n_parts, int32_t part, int32_t tile_rows) {
    if (height <= 0 || n_parts < 1 || part < 0 || part >= n_parts || tile_rows < 1) return 0;
    int64_t blocks = (height + tile_rows - 1) / tile_rows;
    int64_t rows = 0;
    for (int64_t b = part; b < blocks; b += n_parts) {
        int64_t r0 = b * tile_rows, r1 = r0 + tile_rows;
        if (r1 > height) r1 = height;
        rows += r1 - r0;
    }
    // local row index is (local block * tile_rows + row in block); a partial
    // last block still reserves whole tile rows only up to its real size
    return rows;
}

int ro_create(const ro_layout *layout, ro_ctx **out) {
    if (!layout || !out) return fail(RO_EINVAL, "null argument");
    const ro_layout &L = *layout;
    if (L.m < 1 || L.k < 1 || L.k > RO_MAX_LEVELS || L.m * L.k > RO_MAX_PT)
        return fail(RO_EINVAL, "need 1 <= k <= 16 and m*k <= 256");
    if (L.depth < 0 || L.depth > 15) return fail(RO_EINVAL, "depth must be in [0, 15]");
    if (L.num_slots < 1 || L.num_slots >= (int64_t(1) << 31))
        return fail(RO_EINVAL, "cache slot count out of range");
    for (int a = 0; a < 3; ++a)
        if (L.brick[a] < 2 || (L.brick[a] & (L.brick[a] - 1)))
            return fail(RO_EINVAL, "brick size must be a power of two >= 2");
    for (int l = 0; l < L.k; ++l)
        for (int a = 0; a < 3; ++a)
            if (L.level_grids[l][a] < 1 || L.level_grids[l][a] > 256 || L.level_dims[l][a] < 1)
                return fail(RO_EINVAL, "level grid outside [1, 256]");
    ro_ctx *c = new ro_ctx();
    c->layout = L;
    DevLayout &d = c->dl;
    memset(&d, 0, sizeof(d));
    d.m = L.m;
    d.k = L.k;
    d.depth = L.depth;
    d.npt = L.m * L.k;
    d.bx = L.brick[0];
    d.by = L.brick[1];
    d.bz = L.brick[2];
    memcpy(d.dims, L.level_dims, sizeof(d.dims));
    memcpy(d.grids, L.level_grids, sizeof(d.grids));
    memcpy(d.pt_off, L.pt_offsets, sizeof(d.pt_off));
    d.num_slots = L.num_slots;
    d.E = L.pt_offsets[L.m * L.k];
    d.num_nodes = level_offset(L.depth + 1);
    d.bvox = (int64_t)L.brick[0] * L.brick[1] * L.brick[2];
    c->E = d.E;
    c->num_nodes = d.num_nodes;
    c->n_meta = d.num_nodes * L.m;
    c->S = L.num_slots;
    c->bvox = d.bvox;
    if (c->E < 1 || c->E >= (int64_t(1) << 31) || c->n_meta >= (int64_t(1) << 31)) {
        delete c;
        return fail(RO_EINVAL, "page table / octree too large for 32-bit entry lists");
    }
    cudaError_t e;
#define TRY(call)                                   \
    do {                                            \
        e = (call);                                 \
        if (e != cudaSuccess) {                     \
            ro_destroy(c);                          \
            return cuda_fail(e, #call);             \
        }                                           \
    } while (0)
    TRY(cudaMalloc(&c->brick_key, sizeof(unsigned long long) * c->E));
    TRY(cudaMemset(c->brick_key, 0xFF, sizeof(unsigned long long) * c->E));
    TRY(cudaMalloc(&c->brick_touched, sizeof(int32_t) * c->E));
    // [0..1] feedback counts, [2] ray-cast tile counter
    TRY(cudaMalloc(&c->touched_n, sizeof(int32_t) * 4));
    TRY(cudaMemset(c->touched_n, 0, sizeof(int32_t) * 4));
    TRY(cudaMalloc(&c->claim, sizeof(uint32_t) * c->E));
    TRY(cudaMemset(c->claim, 0, sizeof(uint32_t) * c->E));
    TRY(cudaMallocHost(&c->pinned_small, sizeof(int64_t) * 64));
    if (L.depth <= 9) {
        TRY(cudaMalloc(&c->node_fast, (size_t)c->num_nodes));
    }
    if (L.depth <= 7) TRY(cudaMalloc(&c->node_path, sizeof(uint64_t) * c->num_nodes));
    TRY(cudaStreamCreateWithFlags(&c->upload, cudaStreamNonBlocking));
    TRY(cudaEventCreateWithFlags(&c->upload_done, cudaEventDisableTiming));
    for (auto &ev : c->chunk_done) TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TRY(cudaEventCreateWithFlags(&c->host_done, cudaEventDisableTiming));
    TRY(cudaDeviceSynchronize());
#undef TRY
    *out = c;
    return RO_OK;
}

int ro_destroy(ro_ctx *c) {
    if (!c) return RO_OK;
    cudaDeviceSynchronize();
    cudaFree(c->brick_key);
    cudaFree(c->meta_key);
    cudaFree(c->brick_touched);
    cudaFree(c->meta_touched);
    cudaFree(c->touched_n);
    cudaFree(c->claim);
    cudaFree(c->node_fast);
    cudaFree(c->node_path);
    for (int i = 0; i < 16; ++i) cudaFree(c->scratch[i]);
    if (c->pinned_small) cudaFreeHost(c->pinned_small);
    if (c->staging) cudaFreeHost(c->staging);
    if (c->upload) cudaStreamDestroy(c->upload);
    if (c->upload_done) cudaEventDestroy(c->upload_done);
    for (auto &ev : c->chunk_done)
        if (ev) cudaEventDestroy(ev);
    if (c->host_done) cudaEventDestroy(c->host_done);
    delete c;
    return RO_OK;
}

int ro_reserve(ro_ctx *c, int64_t max_batch) {
    if (!c) return fail(RO_EINVAL, "null context");
    if (max_batch < 0) return fail(RO_EINVAL, "negative batch size");
    int rc;
    if ((rc = feedback_reserve(c))) return rc;
    if ((rc = lru_reserve(c, max_batch))) return rc;
    if ((rc = raycast_warm(c))) return rc;
    RO_CUDA(cudaDeviceSynchronize());
    return RO_OK;
}

int ro_render(ro_ctx *c, const ro_frame *frame, const ro_state *st, const ro_outputs *out,
              void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!frame || !out || !out->image || !out->required || !out->pix_required || !out->hist ||
        !out->counters || !st->cache)
        return fail(RO_EINVAL, "null output / state pointer");
    return render(c, frame, st, out, (cudaStream_t)stream);
}

int ro_feedback_collect(ro_ctx *c, int64_t budget, int32_t bricks_first,
                        const ro_feedback *fb, void *stream) {
    if (!c || !fb || (!fb->counts && !fb->counts_dev)) return fail(RO_EINVAL, "null argument");
    if (budget > 0 && (!fb->brick_keys || !fb->brick_ids || !fb->meta_keys || !fb->meta_ids))
        return fail(RO_EINVAL, "null feedback buffer");
    return feedback_collect(c, budget, bricks_first, fb, (cudaStream_t)stream);
}

int ro_feedback_merge(ro_ctx *c, const int64_t *blocks, const int64_t *counts,
                      int32_t n_parts, int64_t budget, void *stream) {
    if (!c) return fail(RO_EINVAL, "null context");
    if (budget > 0 && (!blocks || !counts)) return fail(RO_EINVAL, "null request blocks");
    return feedback_merge(c, blocks, counts, n_parts, budget, (cudaStream_t)stream);
}

int ro_gather_rows(const float *parts, int32_t n_parts, int64_t part_stride, int32_t height,
                   int32_t width, int32_t tile_rows, float *full, void *stream) {
    if (!parts || !full) return fail(RO_EINVAL, "null image");
    if (n_parts < 1 || tile_rows < 1 || height < 1 || width < 1)
        return fail(RO_EINVAL, "bad partition");
    return gather_rows(parts, n_parts, part_stride, height, width, tile_rows, full,
                       (cudaStream_t)stream);
}

int ro_note_sampled(ro_ctx *c, const ro_state *st, const uint8_t *required, int64_t frame,
                    void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!required) return fail(RO_EINVAL, "null mask");
    return note_sampled(c, st, required, frame, (cudaStream_t)stream);
}

int ro_apply_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids, int64_t n,
                    const void *payloads, int32_t payload_on_device, int64_t frame,
                    int32_t update_octree, int32_t *slots_out, int64_t *evicted_out,
                    void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (n > 0 && !ids) return fail(RO_EINVAL, "null ids");
    if (payloads && !st->cache) return fail(RO_EINVAL, "null cache");
    return apply_bricks(c, st, ids, n, payloads, payload_on_device, frame, update_octree,
                        slots_out, evicted_out, (cudaStream_t)stream);
}

int ro_apply_bricks_lz4(ro_ctx *c, const ro_state *st, const int64_t *ids, int64_t n,
                        const uint8_t *frames, const int64_t *frame_offsets,
                        int32_t frames_on_device, int64_t frame, int32_t update_octree,
                        int32_t *slots_out, int64_t *evicted_out, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!st->cache) return fail(RO_EINVAL, "null cache");
    return apply_bricks_lz4(c, st, ids, n, frames, frame_offsets, frames_on_device, frame,
                            update_octree, slots_out, evicted_out, (cudaStream_t)stream);
}

int ro_lz4_decode(ro_ctx *c, const uint8_t *src, const int64_t *src_offsets, int64_t n,
                  uint8_t *dst, int64_t dst_stride, int64_t expected_size, int32_t *status,
                  void *stream) {
    if (!c) return fail(RO_EINVAL, "null context");
    if (n > 0 && (!src || !src_offsets || !dst || !status)) return fail(RO_EINVAL, "null array");
    if (dst_stride < 1) return fail(RO_EINVAL, "dst_stride must be >= 1");
    return lz4_decode(c, src, src_offsets, n, dst, dst_stride, expected_size, status, nullptr,
                      (cudaStream_t)stream);
}

int ro_normalize_to_u8(ro_ctx *c, const void *src, int32_t dtype, int64_t n, uint8_t *dst,
                       void *stream) {
    if (!c) return fail(RO_EINVAL, "null context");
    if (n > 0 && (!src || !dst)) return fail(RO_EINVAL, "null array");
    return normalize_to_u8(c, src, dtype, n, dst, (cudaStream_t)stream);
}

int ro_downsample_box(const uint8_t *src, int32_t dx, int32_t dy, int32_t dz, int32_t fx,
                      int32_t fy, int32_t fz, uint8_t *dst, void *stream) {
    if (!src || !dst) return fail(RO_EINVAL, "null array");
    return downsample_box(src, dx, dy, dz, fx, fy, fz, dst, (cudaStream_t)stream);
}

int ro_extract_bricks(const uint8_t *level, int32_t dx, int32_t dy, int32_t dz, int32_t bx,
                      int32_t by, int32_t bz, uint8_t *dst, void *stream) {
    if (!level || !dst) return fail(RO_EINVAL, "null array");
    return extract_bricks(level, dx, dy, dz, bx, by, bz, dst, (cudaStream_t)stream);
}

int ro_node_minmax(ro_ctx *c, const uint8_t *volume, int32_t dx, int32_t dy, int32_t dz,
                   int32_t d, int32_t pad, uint8_t *mins, uint8_t *maxs, void *stream) {
    if (!c) return fail(RO_EINVAL, "null context");
    return node_minmax(c, volume, dx, dy, dz, d, pad, mins, maxs, (cudaStream_t)stream);
}

int ro_fill_metadata(ro_ctx *c, const ro_state *st, int32_t slot, const uint8_t *volume,
                     int32_t dx, int32_t dy, int32_t dz, int32_t pad, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!volume) return fail(RO_EINVAL, "null volume");
    if (dx != c->layout.level_dims[0][0] || dy != c->layout.level_dims[0][1] ||
        dz != c->layout.level_dims[0][2])
        return fail(RO_EINVAL, "volume dims differ from level 0 of the layout");
    return fill_metadata(c, st, slot, volume, dx, dy, dz, pad, (cudaStream_t)stream);
}

int ro_bricks_box_minmax(const uint8_t *bricks, const int32_t *boxes, int64_t n, int32_t bx,
                         int32_t by, int32_t bz, uint8_t *mins, uint8_t *maxs, void *stream) {
    return bricks_box_minmax(bricks, boxes, n, bx, by, bz, mins, maxs, (cudaStream_t)stream);
}

int ro_evict_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids, int64_t n,
                    int32_t update_octree, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (n > 0 && !ids) return fail(RO_EINVAL, "null ids");
    return release_bricks(c, st, ids, n, RO_PT_UNMAPPED, update_octree, (cudaStream_t)stream);
}

int ro_mark_empty(ro_ctx *c, const ro_state *st, const int64_t *ids, int64_t n, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (n > 0 && !ids) return fail(RO_EINVAL, "null ids");
    return release_bricks(c, st, ids, n, RO_PT_EMPTY, 0, (cudaStream_t)stream);
}

int ro_apply_metadata(ro_ctx *c, const ro_state *st, const int64_t *node_idx,
                      const int32_t *slot, const int32_t *mn, const int32_t *mx, int64_t n,
                      void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (n > 0 && (!node_idx || !slot || !mn || !mx)) return fail(RO_EINVAL, "null array");
    return apply_metadata(c, st, node_idx, slot, mn, mx, n, (cudaStream_t)stream);
}

int ro_write_level_metadata(ro_ctx *c, const ro_state *st, int32_t slot, int32_t d,
                            const uint8_t *mins, const uint8_t *maxs, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!mins || !maxs) return fail(RO_EINVAL, "null grid");
    return write_level_metadata(c, st, slot, d, mins, maxs, (cudaStream_t)stream);
}

int ro_swap_channel(ro_ctx *c, const ro_state *st, int32_t channel_slot,
                    int32_t invalidate_octree, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    return swap_channel(c, st, channel_slot, invalidate_octree, (cudaStream_t)stream);
}

int ro_octree_update(ro_ctx *c, const ro_state *st, const int64_t *ids, int64_t n,
                     void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!st->words) return fail(RO_EINVAL, "no octree words");
    if (n > 0 && !ids) return fail(RO_EINVAL, "null ids");
    return octree_update_host(c, st, ids, n, (cudaStream_t)stream);
}

int ro_rebuild_masks(ro_ctx *c, const ro_state *st, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    return rebuild_masks(c, st, (cudaStream_t)stream);
}

int ro_upload_state(ro_ctx *c, const ro_host_state *h, const ro_state *st, void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    if (!h || !h->pt_status || !h->pt_slot || !h->slot_brick || !h->slot_last_used ||
        (h->free_count > 0 && !h->free_list))
        return fail(RO_EINVAL, "incomplete host state");
    if (h->free_count < 0 || h->free_count > c->S) return fail(RO_EINVAL, "bad free count");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<int32_t> pt((size_t)c->E);
    for (int64_t e = 0; e < c->E; ++e) {
        const int8_t stt = h->pt_status[e];
        if (stt == 1) {
            if (h->pt_slot[e] < 0 || h->pt_slot[e] >= c->S)
                return fail(RO_EINVAL, "MAPPED entry with a slot outside the cache");
            pt[(size_t)e] = h->pt_slot[e];
        } else if (stt == 2) {
            pt[(size_t)e] = RO_PT_EMPTY;
        } else if (stt == 0) {
            pt[(size_t)e] = RO_PT_UNMAPPED;
        } else {
            return fail(RO_EINVAL, "pt_status must be 0, 1 or 2");
        }
    }
    RO_CUDA(cudaMemcpyAsync(st->pt, pt.data(), sizeof(int32_t) * c->E, cudaMemcpyHostToDevice, s));
    if (h->words && st->words)
        RO_CUDA(cudaMemcpyAsync(st->words, h->words, sizeof(uint32_t) * c->num_nodes * c->layout.m,
                                cudaMemcpyHostToDevice, s));
    if (h->cache && st->cache)
        RO_CUDA(cudaMemcpyAsync(st->cache, h->cache, (size_t)c->S * c->bvox,
                                cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemcpyAsync(st->slot_brick, h->slot_brick, sizeof(int64_t) * c->S,
                            cudaMemcpyHostToDevice, s));
    RO_CUDA(cudaMemcpyAsync(st->slot_last_used, h->slot_last_used, sizeof(int64_t) * c->S,
                            cudaMemcpyHostToDevice, s));
    if (h->free_count > 0)
        RO_CUDA(cudaMemcpyAsync(st->free_stack, h->free_list, sizeof(int32_t) * h->free_count,
                                cudaMemcpyHostToDevice, s));
    const int32_t fc = (int32_t)h->free_count;
    RO_CUDA(cudaMemcpyAsync(st->free_count, &fc, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (h->cache && st->cache && (rc = rebuild_sub_max(c, st, s))) return rc;
    RO_CUDA(cudaStreamSynchronize(s));
    return RO_OK;
}

int ro_download_state(ro_ctx *c, const ro_state *st, int8_t *pt_status, int32_t *pt_slot,
                      uint32_t *words, uint8_t *cache, int64_t *slot_brick,
                      int64_t *slot_last_used, int32_t *free_list, int64_t *free_count_out,
                      void *stream) {
    int rc = check_state(c, st);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<int32_t> pt((size_t)c->E);
    int32_t fc = 0;
    RO_CUDA(cudaMemcpyAsync(pt.data(), st->pt, sizeof(int32_t) * c->E, cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaMemcpyAsync(&fc, st->free_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (words && st->words)
        RO_CUDA(cudaMemcpyAsync(words, st->words, sizeof(uint32_t) * c->num_nodes * c->layout.m,
                                cudaMemcpyDeviceToHost, s));
    if (cache && st->cache)
        RO_CUDA(cudaMemcpyAsync(cache, st->cache, (size_t)c->S * c->bvox, cudaMemcpyDeviceToHost,
                                s));
    if (slot_brick)
        RO_CUDA(cudaMemcpyAsync(slot_brick, st->slot_brick, sizeof(int64_t) * c->S,
                                cudaMemcpyDeviceToHost, s));
    if (slot_last_used)
        RO_CUDA(cudaMemcpyAsync(slot_last_used, st->slot_last_used, sizeof(int64_t) * c->S,
                                cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaStreamSynchronize(s));
    if (free_list && fc > 0)
        RO_CUDA(cudaMemcpy(free_list, st->free_stack, sizeof(int32_t) * fc, cudaMemcpyDeviceToHost));
    if (free_count_out) *free_count_out = fc;
    for (int64_t e = 0; e < c->E; ++e) {
        const int32_t v = pt[(size_t)e];
        if (pt_status) pt_status[e] = v >= 0 ? 1 : (v == RO_PT_EMPTY ? 2 : 0);
        if (pt_slot) pt_slot[e] = v >= 0 ? v : -1;
    }
    return RO_OK;
}

int ro_set_feedback_buffers(ro_ctx *c, unsigned long long *bk, unsigned long long *mk) {
    if (!c) return fail(RO_EINVAL, "null context");
    if ((bk == nullptr) != (mk == nullptr))
        return fail(RO_EINVAL, "set both key arrays or neither");
    c->brick_key_ext = bk;
    c->meta_key_ext = mk;
    return RO_OK;
}

int ro_enable_peer_access(int32_t peer_device) {
    int cur = 0;
    RO_CUDA(cudaGetDevice(&cur));
    if (peer_device == cur) return RO_OK;
    int can = 0;
    RO_CUDA(cudaDeviceCanAccessPeer(&can, cur, peer_device));
    if (!can) return fail(RO_EINVAL, "device cannot access the peer device's memory");
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return RO_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    return RO_OK;
}

int ro_sync(ro_ctx *c, void *stream) {
    if (!c) return fail(RO_EINVAL, "null context");
    RO_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

}  // extern "C"
