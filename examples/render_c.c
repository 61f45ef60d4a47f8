/*
 * render_c.c -- a C host driving libresoct.so through include/resoct.h only
 * (no Python, no torch): one channel, 64^3 voxels in 16^3 bricks, 2 levels,
 * octree depth 3.  It inserts every brick (batched LRU insert + octree
 * update), fills the culling metadata from the level-0 volume, packs a frame
 * with ro_pack_frame, ray-casts it, orders the feedback, and writes
 *   <out>.img  : f32 RGBA image (h*w*4)
 *   <out>.txt  : counters, request counts and the ordered brick requests
 * tests/test_gpu_c_host.py builds the same scene through the Python API and
 * compares both bit for bit.
 *
 *   gcc -O2 examples/render_c.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2309_04393_b200 -lresoct -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2309_04393_b200 -o render_c && ./render_c out
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "resoct.h"

#define CHECK(x)                                                              \
    do {                                                                      \
        int rc_ = (x);                                                        \
        if (rc_ != 0) {                                                       \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, ro_last_error()); \
            exit(1);                                                          \
        }                                                                     \
    } while (0)
#define CUDA(x)                                                        \
    do {                                                               \
        cudaError_t e_ = (x);                                          \
        if (e_ != cudaSuccess) {                                       \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));  \
            exit(1);                                                   \
        }                                                              \
    } while (0)

/* the scene's voxel value at level-0 voxel (x, y, z): a spherical shell of
   200 over a low-valued pattern (integers only, mirrored by the test) */
static uint8_t voxel(int x, int y, int z) {
    const int dx = 2 * x + 1 - 64, dy = 2 * y + 1 - 64, dz = 2 * z + 1 - 64;
    const int d2 = dx * dx + dy * dy + dz * dz;
    if (d2 > 1600 && d2 < 2400) return 200;
    return (uint8_t)((x * 7 + y * 13 + z * 3) % 23);
}

int main(int argc, char **argv) {
    const char *out = argc > 1 ? argv[1] : "render_c_out";
    const int B = 16, K = 2, DEPTH = 3, S = 125, W = 40, H = 32, BUDGET = 64;
    const int dims[2] = {64, 32}, grids[2] = {4, 2};
    ro_layout L;
    memset(&L, 0, sizeof L);
    L.m = 1;
    L.k = K;
    L.depth = DEPTH;
    L.brick[0] = L.brick[1] = L.brick[2] = B;
    for (int l = 0; l < K; ++l)
        for (int a = 0; a < 3; ++a) {
            L.level_dims[l][a] = dims[l];
            L.level_grids[l][a] = grids[l];
        }
    L.pt_offsets[0] = 0;
    L.pt_offsets[1] = 64;
    L.pt_offsets[2] = 72;
    L.num_slots = S;
    ro_ctx *ctx = NULL;
    CHECK(ro_create(&L, &ctx));

    /* device state (caller-owned) */
    const int64_t E = 72, N = 585, bvox = (int64_t)B * B * B;
    ro_state st;
    memset(&st, 0, sizeof st);
    CUDA(cudaMalloc((void **)&st.words, sizeof(uint32_t) * N));
    CUDA(cudaMalloc((void **)&st.pt, sizeof(int32_t) * E));
    CUDA(cudaMalloc((void **)&st.cache, (size_t)(S + 1) * bvox));  /* + one brick of padding */
    CUDA(cudaMalloc((void **)&st.slot_brick, sizeof(int64_t) * S));
    CUDA(cudaMalloc((void **)&st.slot_last_used, sizeof(int64_t) * S));
    CUDA(cudaMalloc((void **)&st.free_stack, sizeof(int32_t) * S));
    CUDA(cudaMalloc((void **)&st.free_count, sizeof(int32_t)));
    CUDA(cudaMalloc((void **)&st.sub_max, (size_t)S * (B / 4) * (B / 4) * (B / 4)));
    {
        uint32_t *w = malloc(sizeof(uint32_t) * N);
        for (int64_t i = 0; i < N; ++i) w[i] = 0x00FF0000u; /* INVALID, no residency */
        CUDA(cudaMemcpy(st.words, w, sizeof(uint32_t) * N, cudaMemcpyHostToDevice));
        free(w);
        int32_t *pt = malloc(sizeof(int32_t) * E);
        for (int64_t i = 0; i < E; ++i) pt[i] = RO_PT_UNMAPPED;
        CUDA(cudaMemcpy(st.pt, pt, sizeof(int32_t) * E, cudaMemcpyHostToDevice));
        free(pt);
        int64_t *sb = malloc(sizeof(int64_t) * S);
        int32_t *fs = malloc(sizeof(int32_t) * S);
        for (int i = 0; i < S; ++i) {
            sb[i] = -1;
            fs[i] = S - 1 - i; /* LIFO: slot 0 on top */
        }
        CUDA(cudaMemcpy(st.slot_brick, sb, sizeof(int64_t) * S, cudaMemcpyHostToDevice));
        CUDA(cudaMemset(st.slot_last_used, 0, sizeof(int64_t) * S));
        CUDA(cudaMemcpy(st.free_stack, fs, sizeof(int32_t) * S, cudaMemcpyHostToDevice));
        const int32_t fc = S;
        CUDA(cudaMemcpy(st.free_count, &fc, sizeof(int32_t), cudaMemcpyHostToDevice));
        CUDA(cudaMemset(st.sub_max, 255, (size_t)S * (B / 4) * (B / 4) * (B / 4)));
        CUDA(cudaMemset(st.cache, 0, (size_t)(S + 1) * bvox));
        free(sb);
        free(fs);
    }

    /* every brick of both levels in (level, z, y, x) order */
    int64_t ids[72];
    uint8_t *pay = malloc((size_t)72 * bvox);
    int n = 0;
    for (int l = 0; l < K; ++l)
        for (int bz = 0; bz < grids[l]; ++bz)
            for (int by = 0; by < grids[l]; ++by)
                for (int bx = 0; bx < grids[l]; ++bx) {
                    ids[n] = ((int64_t)l << 24) | (bz << 16) | (by << 8) | bx;
                    uint8_t *p = pay + (size_t)n * bvox;
                    for (int z = 0; z < B; ++z)
                        for (int y = 0; y < B; ++y)
                            for (int x = 0; x < B; ++x) {
                                const int s = 1 << l; /* level-l voxel -> level-0 coords */
                                p[(z * B + y) * B + x] = voxel((bx * B + x) * s, (by * B + y) * s,
                                                               (bz * B + z) * s);
                            }
                    ++n;
                }
    CHECK(ro_apply_bricks(ctx, &st, ids, n, pay, 0, 0, 1, NULL, NULL, NULL));
    free(pay);

    /* culling metadata from the level-0 volume, pad = ceil(1.5 * 2^(k-1)) */
    uint8_t *vol = malloc(64 * 64 * 64), *dvol = NULL;
    for (int z = 0; z < 64; ++z)
        for (int y = 0; y < 64; ++y)
            for (int x = 0; x < 64; ++x) vol[(z * 64 + y) * 64 + x] = voxel(x, y, z);
    CUDA(cudaMalloc((void **)&dvol, 64 * 64 * 64));
    CUDA(cudaMemcpy(dvol, vol, 64 * 64 * 64, cudaMemcpyHostToDevice));
    CHECK(ro_fill_metadata(ctx, &st, 0, dvol, 64, 64, 64, 3, NULL));
    free(vol);

    /* frame: grayscale ramp above 40, orbit-like camera */
    ro_camera cam = {{2.1, 1.2, 1.4}, {0.5, 0.5, 0.5}, {0.0, 1.0, 0.0}, 45.0};
    ro_render_config cfg = {W, H, 1.0 / 64.0, 1.0, 0.99, 2, 0};
    ro_channel_desc ch;
    memset(&ch, 0, sizeof ch);
    ch.slot = 0;
    ch.level_lo = 0;
    ch.level_hi = 15;
    ch.npoints = 3;
    ch.x[0] = 0.0;
    ch.x[1] = 40.0;
    ch.x[2] = 255.0;
    for (int q = 0; q < 4; ++q) ch.rgba[2][q] = 1.0;
    ro_frame F;
    CHECK(ro_pack_frame(K, 1, DEPTH, RO_MODE_RESIDENCY, &cam, &cfg, &ch, 1, 0.0, &F));

    ro_outputs o;
    CUDA(cudaMalloc((void **)&o.image, sizeof(float) * W * H * 4));
    CUDA(cudaMalloc((void **)&o.required, E));
    CUDA(cudaMalloc((void **)&o.pix_required, sizeof(int32_t) * W * H));
    CUDA(cudaMalloc((void **)&o.hist, sizeof(int64_t) * K));
    CUDA(cudaMalloc((void **)&o.counters, sizeof(int64_t) * RO_NUM_COUNTERS));
    CHECK(ro_render(ctx, &F, &st, &o, NULL));
    ro_feedback fb;
    int64_t counts[4];
    CUDA(cudaMalloc((void **)&fb.brick_keys, sizeof(int64_t) * BUDGET));
    CUDA(cudaMalloc((void **)&fb.brick_ids, sizeof(int64_t) * BUDGET));
    CUDA(cudaMalloc((void **)&fb.meta_keys, sizeof(int64_t) * BUDGET));
    CUDA(cudaMalloc((void **)&fb.meta_ids, sizeof(int64_t) * BUDGET));
    fb.counts = counts;
    fb.counts_dev = NULL;
    CHECK(ro_feedback_collect(ctx, BUDGET, 1, &fb, NULL));
    CHECK(ro_sync(ctx, NULL));

    float *img = malloc(sizeof(float) * W * H * 4);
    int64_t ctr[RO_NUM_COUNTERS], bids[64];
    CUDA(cudaMemcpy(img, o.image, sizeof(float) * W * H * 4, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(ctr, o.counters, sizeof ctr, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(bids, fb.brick_ids, sizeof(int64_t) * counts[2], cudaMemcpyDeviceToHost));
    char path[512];
    snprintf(path, sizeof path, "%s.img", out);
    FILE *f = fopen(path, "wb");
    fwrite(img, sizeof(float), (size_t)W * H * 4, f);
    fclose(f);
    snprintf(path, sizeof path, "%s.txt", out);
    f = fopen(path, "w");
    fprintf(f, "%lld %lld %lld %lld\n", (long long)ctr[0], (long long)ctr[1], (long long)ctr[2],
            (long long)ctr[3]);
    fprintf(f, "%lld %lld\n", (long long)counts[2], (long long)counts[3]);
    for (int64_t i = 0; i < counts[2]; ++i) fprintf(f, "%lld\n", (long long)bids[i]);
    fclose(f);
    printf("rendered %dx%d: %lld samples evaluated, %lld brick / %lld metadata requests\n", W, H,
           (long long)ctr[1], (long long)counts[2], (long long)counts[3]);
    free(img);
    CHECK(ro_destroy(ctx));
    return 0;
}
