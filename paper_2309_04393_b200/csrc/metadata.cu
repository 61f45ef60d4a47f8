// metadata.cu -- the culling-metadata producer on the GPU (SURVEY.md §8(f)
// row 3).
//
// A node's metadata is the min / max of the level-0 volume over the node's
// extent dilated by `pad` voxels (engine.py:109-127 metadata_box), computed
// by the server per request (service.py:102-115 region_min_max, requested by
// session.py:140-158) or for a whole tree level at once
// (engine.py:138-152 fill_metadata_from_volumes via _box_minmax_grid,
// engine.py:186-219).  Here one tree level of one channel is three separable
// window reductions over the device-resident volume:
//
//   x: [dz][dy][dx] u8      -> [dz][dy][side]   (min, max) pairs
//   y: [dz][dy][side]       -> [dz][side][side]
//   z: [dz][side][side]     -> [side]^3 mins, maxs  ([z][y][x] node order)
//
// with the reference's per-axis windows [max(0, floor(i*n/side) - pad),
// min(n, ceil((i+1)*n/side) + pad)).  Min / max are order-independent, so
// the result equals the reference's per-node box reduction exactly; a window
// that is empty on any axis yields (0, 0) like the reference.
#include "internal.cuh"

namespace ro {

int write_level_metadata(ro_ctx *c, const ro_state *st, int32_t slot, int32_t d,
                         const uint8_t *mins, const uint8_t *maxs, cudaStream_t s);

namespace {

__device__ __forceinline__ void window(int i, int n, int side, int pad, int &lo, int &hi) {
    const int64_t v0 = ((int64_t)i * n) / side - pad;
    const int64_t v1 = ((int64_t)(i + 1) * n + side - 1) / side + pad;  // ceil((i+1)n/side) + pad
    lo = v0 < 0 ? 0 : (int)v0;
    hi = v1 > n ? n : (int)v1;
}

// x pass: one thread per (row, ix); 16-byte loads over the aligned interior
__global__ void k_minmax_x(const uint8_t *__restrict__ vol, int dx, int64_t rows, int side,
                           int pad, uchar2 *__restrict__ out) {
    const int64_t total = rows * side;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(t % side);
        const int64_t row = t / side;
        int lo, hi;
        window(ix, dx, side, pad, lo, hi);
        const uint8_t *p = vol + row * dx;
        unsigned mn = 255, mx = 0;
        int x = lo;
        for (; x < hi && ((reinterpret_cast<uintptr_t>(p + x)) & 15); ++x) {
            mn = min(mn, (unsigned)p[x]);
            mx = max(mx, (unsigned)p[x]);
        }
        for (; x + 16 <= hi; x += 16) {
            const uint4 v = *reinterpret_cast<const uint4 *>(p + x);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                // byte-wise min / max of 4 packed bytes
                const unsigned a = w[q];
                const unsigned m1 = __vminu4(a, a >> 16), M1 = __vmaxu4(a, a >> 16);
                const unsigned m2 = __vminu4(m1, m1 >> 8), M2 = __vmaxu4(M1, M1 >> 8);
                mn = min(mn, m2 & 0xFFu);
                mx = max(mx, M2 & 0xFFu);
            }
        }
        for (; x < hi; ++x) {
            mn = min(mn, (unsigned)p[x]);
            mx = max(mx, (unsigned)p[x]);
        }
        out[t] = make_uchar2((unsigned char)mn, (unsigned char)mx);
    }
}

// y pass: [dz][dy][side] -> [dz][side][side]
__global__ void k_minmax_y(const uchar2 *__restrict__ in, int dy, int dz, int side, int pad,
                           uchar2 *__restrict__ out) {
    const int64_t total = (int64_t)dz * side * side;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(t % side);
        const int iy = (int)((t / side) % side);
        const int64_t z = t / ((int64_t)side * side);
        int lo, hi;
        window(iy, dy, side, pad, lo, hi);
        unsigned mn = 255, mx = 0;
        for (int y = lo; y < hi; ++y) {
            const uchar2 v = in[(z * dy + y) * side + ix];
            mn = min(mn, (unsigned)v.x);
            mx = max(mx, (unsigned)v.y);
        }
        out[t] = make_uchar2((unsigned char)mn, (unsigned char)mx);
    }
}

// z pass: [dz][side][side] -> mins / maxs [side]^3
__global__ void k_minmax_z(const uchar2 *__restrict__ in, int dz, int side, int pad,
                           uint8_t *__restrict__ mins, uint8_t *__restrict__ maxs) {
    const int64_t plane = (int64_t)side * side;
    const int64_t total = plane * side;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t yx = t % plane;
        const int iz = (int)(t / plane);
        int lo, hi;
        window(iz, dz, side, pad, lo, hi);
        unsigned mn = 255, mx = 0;
        for (int z = lo; z < hi; ++z) {
            const uchar2 v = in[z * plane + yx];
            mn = min(mn, (unsigned)v.x);
            mx = max(mx, (unsigned)v.y);
        }
        if (mn > mx) mn = mx = 0;  // an empty window on some axis
        mins[t] = (uint8_t)mn;
        maxs[t] = (uint8_t)mx;
    }
}

// octree.py:275-306 compute_node_metadata_from_bricks, the min / max part:
// brick i contributes the voxels of its sub-box boxes[i] = x0,y0,z0,x1,y1,z1
// (half-open, brick-local); one CTA per brick, block reduction.
__global__ void k_brick_box_minmax(int64_t n, const uint8_t *__restrict__ bricks, int bx,
                                   int by, int bz, const int32_t *__restrict__ boxes,
                                   uint8_t *__restrict__ mins, uint8_t *__restrict__ maxs) {
    __shared__ unsigned red[2][32];
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const int32_t *b = boxes + i * 6;
    const int x0 = b[0], y0 = b[1], z0 = b[2], x1 = b[3], y1 = b[4], z1 = b[5];
    const int nx = max(x1 - x0, 0), ny = max(y1 - y0, 0), nz = max(z1 - z0, 0);
    const int64_t cnt = (int64_t)nx * ny * nz;
    const uint8_t *p = bricks + i * (int64_t)bx * by * bz;
    unsigned mn = 255, mx = 0;
    for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int x = x0 + (int)(j % nx), y = y0 + (int)((j / nx) % ny),
                  z = z0 + (int)(j / ((int64_t)nx * ny));
        const unsigned v = p[((int64_t)z * by + y) * bx + x];
        mn = min(mn, v);
        mx = max(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = mn;
        red[1][w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
            mn = min(mn, red[0][q]);
            mx = max(mx, red[1][q]);
        }
        mins[i] = (uint8_t)mn;  // 255 / 0 for an empty sub-box
        maxs[i] = (uint8_t)mx;
    }
}

unsigned grid_of(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

int node_minmax(ro_ctx *c, const uint8_t *vol, int32_t dx, int32_t dy, int32_t dz, int32_t d,
                int32_t pad, uint8_t *mins, uint8_t *maxs, cudaStream_t s) {
    if (!vol || !mins || !maxs) return fail(RO_EINVAL, "null array");
    if (dx < 1 || dy < 1 || dz < 1) return fail(RO_EINVAL, "empty volume");
    if (d < 0 || d > 10) return fail(RO_EINVAL, "tree depth outside [0, 10]");
    if (pad < 0) return fail(RO_EINVAL, "negative pad");
    const int side = 1 << d;
    void *pa, *pb;
    int rc;
    const int64_t rows = (int64_t)dz * dy;
    if ((rc = scratch(c, 8, sizeof(uchar2) * rows * side, &pa))) return rc;
    if ((rc = scratch(c, 9, sizeof(uchar2) * (int64_t)dz * side * side, &pb))) return rc;
    k_minmax_x<<<grid_of(rows * side), 256, 0, s>>>(vol, dx, rows, side, pad, (uchar2 *)pa);
    k_minmax_y<<<grid_of((int64_t)dz * side * side), 256, 0, s>>>((const uchar2 *)pa, dy, dz,
                                                                  side, pad, (uchar2 *)pb);
    k_minmax_z<<<grid_of((int64_t)side * side * side), 256, 0, s>>>((const uchar2 *)pb, dz, side,
                                                                    pad, mins, maxs);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int bricks_box_minmax(const uint8_t *bricks, const int32_t *boxes, int64_t n, int32_t bx,
                      int32_t by, int32_t bz, uint8_t *mins, uint8_t *maxs, cudaStream_t s) {
    if (n <= 0) return RO_OK;
    if (!bricks || !boxes || !mins || !maxs) return fail(RO_EINVAL, "null array");
    if (n > 0x7FFFFFFF) return fail(RO_EINVAL, "too many bricks");
    k_brick_box_minmax<<<(unsigned)n, 256, 0, s>>>(n, bricks, bx, by, bz, boxes, mins, maxs);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

// engine.py:138-152 for one slot: every tree level from the level-0 volume
int fill_metadata(ro_ctx *c, const ro_state *st, int32_t slot, const uint8_t *vol, int32_t dx,
                  int32_t dy, int32_t dz, int32_t pad, cudaStream_t s) {
    if (!st->words) return fail(RO_EINVAL, "no octree words");
    if (slot < 0 || slot >= c->layout.m) return fail(RO_EINVAL, "slot out of range");
    const int D = c->layout.depth;
    const int64_t nodes = ((int64_t)1 << (3 * D));
    void *p;
    int rc;
    if ((rc = scratch(c, 10, 2 * nodes, &p))) return rc;
    uint8_t *mins = (uint8_t *)p, *maxs = mins + nodes;
    for (int d = 0; d <= D; ++d) {
        if ((rc = node_minmax(c, vol, dx, dy, dz, d, pad, mins, maxs, s))) return rc;
        if ((rc = write_level_metadata(c, st, slot, d, mins, maxs, s))) return rc;
    }
    return RO_OK;
}

}  // namespace ro
