// feedback.cu -- kernel 3a: request ordering + budget, and the LRU touch.
//
// The ray caster leaves, per touched brick / metadata entry, the smallest
// (pixel << 32 | event) key of any request for it (raycast.cu).  Sorting the
// touched entries by that key reproduces the reference's single-threaded
// first-seen append order (kernels.py:457-517, seen_brick / seen_meta); the
// bricks-first budget is render.py:210-215.  Keys are reset in the same pass
// so the next frame starts clean without an O(E) memset.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace ro {

namespace {

__global__ void k_gather_keys(const int32_t *__restrict__ touched, int32_t n,
                              unsigned long long *__restrict__ keys,
                              unsigned long long *__restrict__ out_keys,
                              int32_t *__restrict__ out_vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t e = touched[i];
    out_keys[i] = keys[e];
    out_vals[i] = e;
    keys[e] = ~0ull;
}

__global__ void k_emit_bricks(const DevLayout L,
                              const unsigned long long *__restrict__ keys,
                              const int32_t *__restrict__ vals, int32_t n,
                              int64_t *__restrict__ out_keys,
                              int64_t *__restrict__ out_ids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out_keys[i] = (int64_t)keys[i];
    out_ids[i] = entry_to_id(L, vals[i]);
}

__global__ void k_emit_metas(const unsigned long long *__restrict__ keys,
                             const int32_t *__restrict__ vals, int32_t n,
                             int64_t *__restrict__ out_keys,
                             int64_t *__restrict__ out_ids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out_keys[i] = (int64_t)keys[i];
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

// sort n (key, value) pairs held at ctx scratch and emit the first `keep`
int sort_and_emit(ro_ctx *c, unsigned long long *key_arr, const int32_t *touched,
                  int32_t n, int32_t keep, bool bricks, int64_t *out_keys,
                  int64_t *out_ids, cudaStream_t s) {
    if (n <= 0) return RO_OK;
    void *p0, *p1, *p2, *p3, *tmp;
    int rc;
    if ((rc = scratch(c, 0, sizeof(unsigned long long) * n, &p0))) return rc;
    if ((rc = scratch(c, 1, sizeof(unsigned long long) * n, &p1))) return rc;
    if ((rc = scratch(c, 2, sizeof(int32_t) * n, &p2))) return rc;
    if ((rc = scratch(c, 3, sizeof(int32_t) * n, &p3))) return rc;
    auto *k_in = (unsigned long long *)p0, *k_out = (unsigned long long *)p1;
    auto *v_in = (int32_t *)p2, *v_out = (int32_t *)p3;
    k_gather_keys<<<(n + 255) / 256, 256, 0, s>>>(touched, n, key_arr, k_in, v_in);
    RO_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    RO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in,
                                            v_out, n, 0, 64, s));
    if ((rc = scratch(c, 4, tmp_bytes, &tmp))) return rc;
    RO_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in,
                                            v_out, n, 0, 64, s));
    if (keep > 0) {
        if (bricks)
            k_emit_bricks<<<(keep + 255) / 256, 256, 0, s>>>(c->dl, k_out, v_out, keep,
                                                              out_keys, out_ids);
        else
            k_emit_metas<<<(keep + 255) / 256, 256, 0, s>>>(k_out, v_out, keep,
                                                             out_keys, out_ids);
        RO_CUDA(cudaGetLastError());
    }
    return RO_OK;
}

}  // namespace

int feedback_collect(ro_ctx *c, int64_t budget, int32_t bricks_first,
                     const ro_feedback *fb, cudaStream_t s) {
    if (budget < 0) return fail(RO_EINVAL, "negative budget");
    int32_t *hn = reinterpret_cast<int32_t *>(c->pinned_small);
    RO_CUDA(cudaMemcpyAsync(hn, c->touched_n, 2 * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaStreamSynchronize(s));
    const int32_t nb = hn[0], nm = hn[1];
    const int32_t kb = (int32_t)(nb < budget ? nb : budget);
    int64_t rest = bricks_first ? budget - kb : budget;
    const int32_t km = (int32_t)(nm < rest ? nm : rest);
    int rc = sort_and_emit(c, c->brick_key, c->brick_touched, nb, kb, true,
                           fb->brick_keys, fb->brick_ids, s);
    if (rc) return rc;
    if (nm > 0) {
        rc = sort_and_emit(c, c->meta_key, c->meta_touched, nm, km, false,
                           fb->meta_keys, fb->meta_ids, s);
        if (rc) return rc;
    }
    RO_CUDA(cudaMemsetAsync(c->touched_n, 0, 2 * sizeof(int32_t), s));
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
