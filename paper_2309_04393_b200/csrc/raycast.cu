// raycast.cu -- kernel 1: the per-pixel residency-octree ray caster.
//
// Restates /root/reference/pkg/src/resoctree/kernels.py:209-704
// (raycast_frame) for MODE_RESIDENCY (431-558) and MODE_REFERENCE (301-314)
// with the skip loop (561-635), single-sample compositing (637-694) and the
// skip audit (595-625, 644-655, 707-723).
//
// B200 design:
//  * one thread per pixel, each warp an 8x4 pixel packet so neighbouring
//    rays walk the same octree nodes / bricks (L1 hits for words, page-table
//    entries and trilinear taps); 128-thread CTAs;
//  * rays are generated in-kernel from the camera basis (bit-exact with
//    camera.py:32-51, no 50 MB/frame ray upload);
//  * per-channel TF tables, emptiness thresholds and page-table offsets are
//    staged in shared memory once per CTA;
//  * each channel is composited the moment the shared cursor resolves it
//    (same channel order and arithmetic as the reference's two-pass form),
//    so no per-channel outcome arrays live in local memory;
//  * request recording keeps the reference's first-seen order without a
//    serial buffer: every request event carries key = (pixel << 32 | event
//    index within the pixel) and an atomicMin per brick / metadata entry
//    keeps the smallest key; the first toucher appends the entry to a
//    compact list (feedback.cu sorts it);
//  * fp64 throughout on the decision path, compiled with -fmad=false so
//    every operation rounds like numba's unfused code.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace ro {

namespace {

constexpr int kBlock = 128;  // 4 warps, 16x8 pixels
constexpr int kTileW = 16;
constexpr int kTileH = 8;
constexpr double kClampHi = 1.0 - 1e-9;

struct FrameSmem {
    double tf_x[RO_MAX_CH][RO_MAX_TF_POINTS];
    double tf_rgba[RO_MAX_CH][RO_MAX_TF_POINTS][4];
    uint16_t empty_below[RO_MAX_CH][256];
    int64_t ptoff[RO_MAX_CH][RO_MAX_LEVELS];  // pt_offsets[slot*k + lev]
    int64_t lvl_off[RO_MAX_LEVELS];
    double lod_thr[RO_MAX_LEVELS + 1];
    double step_tab[RO_MAX_LEVELS];
    int32_t maxlev[RO_MAX_LEVELS];
    int32_t dt_tab[RO_MAX_LEVELS];
    int32_t dims[RO_MAX_LEVELS][3];
    int32_t grids[RO_MAX_LEVELS][3];
    int32_t slot[RO_MAX_CH], lo[RO_MAX_CH], hi[RO_MAX_CH], np[RO_MAX_CH];
    unsigned long long red[RO_NUM_COUNTERS];
};

struct RayArgs {
    DevLayout L;
    const uint32_t *words;
    const int32_t *pt;
    const uint8_t *cache;
    float *image;
    uint8_t *required;
    int32_t *pix_required;
    unsigned long long *hist;      // [n_ch*k] as u64
    unsigned long long *counters;  // [RO_NUM_COUNTERS]
    unsigned long long *brick_key;
    unsigned long long *meta_key;
    int32_t *brick_touched;
    int32_t *meta_touched;
    int32_t *touched_n;
    int32_t local_rows;
};

__device__ __forceinline__ double lerp(double a, double b, double t) {
    return a + (b - a) * t;
}

// (1-alpha)^(2^j): the reference calls libm pow with ratio = step/base_step,
// always an exact power of two.  Repeated squaring in double-double gives
// the correctly rounded power (glibc pow is within 0.52 ulp, so the two
// agree except in vanishingly rare near-midpoint cases).
__device__ __forceinline__ double pow_pow2(double x, int j) {
    double hi = x, lo = 0.0;
    for (int i = 0; i < j; ++i) {
        double p = __dmul_rn(hi, hi);
        double e = __fma_rn(hi, hi, -p);
        e = __dadd_rn(e, __dmul_rn(__dmul_rn(2.0, hi), lo));
        double s = __dadd_rn(p, e);
        lo = __dsub_rn(e, __dsub_rn(s, p));
        hi = s;
    }
    return hi;
}

// raw LOD level (kernels.py:43-54 before the per-channel clamp); levels
// above 15 clamp identically for every channel (hi <= k-1 <= 15).
__device__ __forceinline__ int lod_raw(double t, double t0, const FrameSmem &S) {
    double ratio = t / t0;
    if (ratio < 1.0) return 0;
    int e = ilogb(ratio);
    if (e >= RO_MAX_LEVELS - 1) return RO_MAX_LEVELS - 1;
    int lev = e;
    if (ratio >= S.lod_thr[lev + 1]) lev += 1;
    else if (lev >= 1 && ratio < S.lod_thr[lev]) lev -= 1;
    return lev;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// kernels.py:177-184
__device__ __forceinline__ int brick_axis(double p, int dim, int b, int grid) {
    int c = (int)(p * (double)dim / (double)b);
    if (c < 0) c = 0;
    if (c > grid - 1) c = grid - 1;
    return c;
}

// kernels.py:119-133
__device__ __forceinline__ void tf_eval(const FrameSmem &S, int ci, double v,
                                        double &r, double &g, double &b,
                                        double &a) {
    r = g = b = a = 0.0;
    const int n = S.np[ci];
    if (v < S.tf_x[ci][0] || v > S.tf_x[ci][n - 1]) return;
    for (int i = 0; i < n - 1; ++i) {
        double x0 = S.tf_x[ci][i], x1 = S.tf_x[ci][i + 1];
        if (x0 <= v && v <= x1) {
            double t = (x1 == x0) ? 0.0 : (v - x0) / (x1 - x0);
            r = lerp(S.tf_rgba[ci][i][0], S.tf_rgba[ci][i + 1][0], t);
            g = lerp(S.tf_rgba[ci][i][1], S.tf_rgba[ci][i + 1][1], t);
            b = lerp(S.tf_rgba[ci][i][2], S.tf_rgba[ci][i + 1][2], t);
            a = lerp(S.tf_rgba[ci][i][3], S.tf_rgba[ci][i + 1][3], t);
            return;
        }
    }
}

// kernels.py:136-174
__device__ __forceinline__ double trilinear(const uint8_t *__restrict__ brick,
                                            double lx, double ly, double lz,
                                            int bx, int by, int bz) {
    double fx = lx - 0.5, fy = ly - 0.5, fz = lz - 0.5;
    if (fx < 0.0) fx = 0.0;
    if (fy < 0.0) fy = 0.0;
    if (fz < 0.0) fz = 0.0;
    if (fx > bx - 1.0) fx = bx - 1.0;
    if (fy > by - 1.0) fy = by - 1.0;
    if (fz > bz - 1.0) fz = bz - 1.0;
    int x0 = (int)fx, y0 = (int)fy, z0 = (int)fz;
    int x1 = x0 + 1 < bx ? x0 + 1 : bx - 1;
    int y1 = y0 + 1 < by ? y0 + 1 : by - 1;
    int z1 = z0 + 1 < bz ? z0 + 1 : bz - 1;
    double tx = fx - x0, ty = fy - y0, tz = fz - z0;
    const int r00 = (z0 * by + y0) * bx, r10 = (z0 * by + y1) * bx;
    const int r01 = (z1 * by + y0) * bx, r11 = (z1 * by + y1) * bx;
    double v000 = __ldg(brick + r00 + x0), v001 = __ldg(brick + r00 + x1);
    double v010 = __ldg(brick + r10 + x0), v011 = __ldg(brick + r10 + x1);
    double v100 = __ldg(brick + r01 + x0), v101 = __ldg(brick + r01 + x1);
    double v110 = __ldg(brick + r11 + x0), v111 = __ldg(brick + r11 + x1);
    double c00 = lerp(v000, v001, tx);
    double c10 = lerp(v010, v011, tx);
    double c01 = lerp(v100, v101, tx);
    double c11 = lerp(v110, v111, tx);
    return lerp(lerp(c00, c10, ty), lerp(c01, c11, ty), tz);
}

// kernels.py:97-116
__device__ __forceinline__ double box_exit(double ox, double oy, double oz,
                                           double dx, double dy, double dz,
                                           double lx, double ly, double lz,
                                           double hx, double hy, double hz) {
    double te = 1e30, t;
    if (dx > 1e-12) { t = (hx - ox) / dx; if (t < te) te = t; }
    else if (dx < -1e-12) { t = (lx - ox) / dx; if (t < te) te = t; }
    if (dy > 1e-12) { t = (hy - oy) / dy; if (t < te) te = t; }
    else if (dy < -1e-12) { t = (ly - oy) / dy; if (t < te) te = t; }
    if (dz > 1e-12) { t = (hz - oz) / dz; if (t < te) te = t; }
    else if (dz < -1e-12) { t = (lz - oz) / dz; if (t < te) te = t; }
    return te;
}

__device__ __forceinline__ void axis_box(double o, double d, double &tmin,
                                         double &tmax, bool &miss) {
    if (fabs(d) < 1e-12) {
        if (o < 0.0 || o > 1.0) miss = true;
    } else {
        double inv = 1.0 / d;
        double t0 = (0.0 - o) * inv;
        double t1 = (1.0 - o) * inv;
        if (t0 > t1) { double s = t0; t0 = t1; t1 = s; }
        if (t0 > tmin) tmin = t0;
        if (t1 < tmax) tmax = t1;
    }
}

// first-seen request: keep the minimum (pixel, event) key per entry and list
// each touched entry once.
__device__ __forceinline__ void request(unsigned long long *keys,
                                        int32_t *touched, int32_t *touched_n,
                                        int64_t entry,
                                        unsigned long long key) {
    unsigned long long old = atomicMin(keys + entry, key);
    if (old == ~0ull) {
        int pos = atomicAdd(touched_n, 1);
        touched[pos] = (int32_t)entry;
    }
}

template <int MODE, bool CHECK>
__global__ void __launch_bounds__(kBlock)
k_raycast(const __grid_constant__ ro_frame F, const __grid_constant__ RayArgs A) {
    __shared__ FrameSmem S;
    extern __shared__ int32_t dyn[];  // per-thread channel state
    const int tid = threadIdx.x;
    const int n_ch = F.n_ch;
    const int k = A.L.k;
    const int m = A.L.m;

    // ---- stage frame tables ----
    for (int i = tid; i < n_ch * RO_MAX_TF_POINTS; i += kBlock) {
        int c = i / RO_MAX_TF_POINTS, p = i % RO_MAX_TF_POINTS;
        S.tf_x[c][p] = F.ch[c].tf_x[p];
        for (int q = 0; q < 4; ++q) S.tf_rgba[c][p][q] = F.ch[c].tf_rgba[p][q];
    }
    for (int i = tid; i < n_ch * 256; i += kBlock)
        S.empty_below[i / 256][i % 256] = F.ch[i / 256].empty_below[i % 256];
    for (int i = tid; i < n_ch * RO_MAX_LEVELS; i += kBlock) {
        int c = i / RO_MAX_LEVELS, l = i % RO_MAX_LEVELS;
        S.ptoff[c][l] = l < k ? A.L.pt_off[F.ch[c].slot * k + l] : 0;
    }
    if (tid < RO_MAX_LEVELS) {
        S.lvl_off[tid] = level_offset(tid);
        S.step_tab[tid] = F.step_tab[tid];
        S.maxlev[tid] = F.maxlev_tab[tid];
        S.dt_tab[tid] = F.dt_tab[tid];
        for (int a = 0; a < 3; ++a) {
            S.dims[tid][a] = A.L.dims[tid][a];
            S.grids[tid][a] = A.L.grids[tid][a];
        }
    }
    if (tid <= RO_MAX_LEVELS) S.lod_thr[tid] = F.lod_threshold[tid];
    if (tid < RO_MAX_CH) {
        S.slot[tid] = F.ch[tid].slot;
        S.lo[tid] = F.ch[tid].lo;
        S.hi[tid] = F.ch[tid].hi;
        S.np[tid] = F.ch[tid].npoints;
    }
    if (tid < RO_NUM_COUNTERS) S.red[tid] = 0;
    // per-thread arrays: [ci*kBlock + tid]
    int32_t *prev_brick = dyn;                        // n_ch
    int32_t *last_breq = prev_brick + n_ch * kBlock;  // n_ch
    int32_t *last_mreq = last_breq + n_ch * kBlock;   // n_ch
    uint32_t *hist_t = reinterpret_cast<uint32_t *>(last_mreq + n_ch * kBlock);
    for (int i = 0; i < n_ch; ++i) {
        prev_brick[i * kBlock + tid] = -1;
        last_breq[i * kBlock + tid] = -1;
        last_mreq[i * kBlock + tid] = -1;
    }
    for (int i = 0; i < n_ch * k; ++i) hist_t[i * kBlock + tid] = 0;
    __syncthreads();

    // ---- pixel of this thread: warp = 8x4 packet ----
    const int lane = tid & 31, warp = tid >> 5;
    const int x = blockIdx.x * kTileW + (warp & 1) * 8 + (lane & 7);
    const int ly = blockIdx.y * kTileH + (warp >> 1) * 4 + (lane >> 3);
    const int tr = F.tile_rows;
    const int gy = ((ly / tr) * F.n_parts + F.part) * tr + (ly % tr);
    const bool active = x < F.width && ly < A.local_rows && gy < F.height;

    unsigned long long c_steps = 0, c_eval = 0, c_skip = 0, c_viol = 0,
                       c_live = 0;

    if (active) {
        const int bx = A.L.bx, by = A.L.by, bz = A.L.bz;
        const int64_t bvox = (int64_t)bx * by * bz;
        const int D = A.L.depth;
        const int64_t pix = (int64_t)gy * F.width + x;
        const int64_t lpix = (int64_t)ly * F.width + x;

        // camera.py:32-51, same operation order as the numpy code
        const double u = (((double)x + 0.5) / (double)F.width * 2.0 - 1.0) *
                         F.tan_half * F.aspect;
        const double v = (1.0 - ((double)gy + 0.5) / (double)F.height * 2.0) *
                         F.tan_half;
        double dx = (F.cam_fwd[0] + u * F.cam_right[0]) + v * F.cam_up[0];
        double dy = (F.cam_fwd[1] + u * F.cam_right[1]) + v * F.cam_up[1];
        double dz = (F.cam_fwd[2] + u * F.cam_right[2]) + v * F.cam_up[2];
        const double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
        dx = dx / nrm;
        dy = dy / nrm;
        dz = dz / nrm;
        const double ox = F.cam_pos[0], oy = F.cam_pos[1], oz = F.cam_pos[2];

        // kernels.py:69-94
        double tnear = -1e30, tfar = 1e30;
        bool miss = false;
        axis_box(ox, dx, tnear, tfar, miss);
        if (!miss) axis_box(oy, dy, tnear, tfar, miss);
        if (!miss) axis_box(oz, dz, tnear, tfar, miss);
        if (miss) { tnear = 1.0; tfar = -1.0; }

        double accR = 0.0, accG = 0.0, accB = 0.0, accA = 0.0;
        double t = tnear > 0.0 ? tnear : 0.0;
        int prev_depth = F.start_level;
        int stall = 0;
        uint32_t ev = 0;  // request event index within this pixel
        int32_t pixreq = 0;

        while (t < tfar && accA < F.early_alpha) {
            double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
            if (px < 0.0) px = 0.0;
            if (py < 0.0) py = 0.0;
            if (pz < 0.0) pz = 0.0;
            if (px > kClampHi) px = kClampHi;
            if (py > kClampHi) py = kClampHi;
            if (pz > kClampHi) pz = kClampHi;

            const int raw = lod_raw(t, F.t0, S);
            double step = S.step_tab[raw];
            int jexp = S.maxlev[raw];
            const int dt_ = S.dt_tab[raw];

            double sR = 0.0, sG = 0.0, sB = 0.0, trans = 1.0;
            bool any_const = false;
            uint32_t zero_mask = 0;
            bool skippable = false;
            double skip_exit = -1.0;
            int end_depth = prev_depth;

            // sample one resolved channel: trilinear + usage + composite input
            auto sample = [&](int ci, int lev, int cbx, int cby, int cbz,
                              int slot_lin, int64_t e) {
                const double lx = px * S.dims[lev][0] - (double)(cbx * bx);
                const double lyy = py * S.dims[lev][1] - (double)(cby * by);
                const double lz = pz * S.dims[lev][2] - (double)(cbz * bz);
                const double val = trilinear(A.cache + (int64_t)slot_lin * bvox,
                                             lx, lyy, lz, bx, by, bz);
                int32_t &pb = prev_brick[ci * kBlock + tid];
                if ((int32_t)e != pb) {
                    pb = (int32_t)e;
                    pixreq += 1;
                    A.required[e] = 1;
                }
                hist_t[(ci * k + lev) * kBlock + tid] += 1;
                double r, g, b, a;
                tf_eval(S, ci, val, r, g, b, a);
                sR += r * a;
                sG += g * a;
                sB += b * a;
                trans *= (1.0 - a);
            };

            if (MODE == RO_MODE_REFERENCE) {
                for (int ci = 0; ci < n_ch; ++ci) {
                    const int lev = clampi(raw, S.lo[ci], S.hi[ci]);
                    const int cbx = brick_axis(px, S.dims[lev][0], bx, S.grids[lev][0]);
                    const int cby = brick_axis(py, S.dims[lev][1], by, S.grids[lev][1]);
                    const int cbz = brick_axis(pz, S.dims[lev][2], bz, S.grids[lev][2]);
                    const int64_t e = S.ptoff[ci][lev] +
                        ((int64_t)cbz * S.grids[lev][1] + cby) * S.grids[lev][0] + cbx;
                    const int pv = __ldg(A.pt + e);
                    if (pv >= 0) sample(ci, lev, cbx, cby, cbz, pv, e);
                }
            } else {
                // kernels.py:431-558 -- one cursor shared by all channels
                int d = prev_depth - 1;
                if (d < 0) d = 0;
                if (F.start_level < d) d = F.start_level;
                if (d > dt_) d = dt_;
                int ci = 0;
                bool all_cz = true;
                int ix = 0, iy = 0, iz = 0;
                while (ci < n_ch) {
                    const int side = 1 << d;
                    ix = (int)(px * (double)side);
                    iy = (int)(py * (double)side);
                    iz = (int)(pz * (double)side);
                    const int64_t nidx = S.lvl_off[d] +
                        ((int64_t)iz * side + iy) * side + ix;
                    c_steps += 1;
                    const int slot = S.slot[ci];
                    const uint32_t w = __ldg(A.words + nidx * m + slot);
                    const int mn = (w >> 16) & 0xFF, mx = (w >> 24) & 0xFF;
                    const uint32_t mask = w & 0xFFFF;
                    if (mn == 255 && mx == 0) {  // INVALID: metadata request
                        const int64_t mid = nidx * m + slot;
                        const unsigned long long key =
                            ((unsigned long long)pix << 32) | ev++;
                        int32_t &lm = last_mreq[ci * kBlock + tid];
                        if ((int32_t)mid != lm) {
                            lm = (int32_t)mid;
                            request(A.meta_key, A.meta_touched, A.touched_n + 1,
                                    mid, key);
                        }
                    } else {
                        if (mx < (int)S.empty_below[ci][mn]) {  // K_ZERO
                            zero_mask |= 1u << ci;
                            ci += 1;
                            continue;
                        }
                        if ((double)(mx - mn) <= F.eps_h) {  // K_CONST
                            double r, g, b, a;
                            tf_eval(S, ci, (double)mn, r, g, b, a);
                            sR += r * a;
                            sG += g * a;
                            sB += b * a;
                            trans *= (1.0 - a);
                            any_const = true;
                            ci += 1;
                            continue;
                        }
                    }
                    const int lev = clampi(raw, S.lo[ci], S.hi[ci]);
                    if (mask == 0) {  // K_MISSU: request the desired brick
                        const int cbx = brick_axis(px, S.dims[lev][0], bx, S.grids[lev][0]);
                        const int cby = brick_axis(py, S.dims[lev][1], by, S.grids[lev][1]);
                        const int cbz = brick_axis(pz, S.dims[lev][2], bz, S.grids[lev][2]);
                        const int64_t gb = S.ptoff[ci][lev] +
                            ((int64_t)cbz * S.grids[lev][1] + cby) * S.grids[lev][0] + cbx;
                        const unsigned long long key =
                            ((unsigned long long)pix << 32) | ev++;
                        int32_t &lb = last_breq[ci * kBlock + tid];
                        if ((int32_t)gb != lb) {
                            lb = (int32_t)gb;
                            request(A.brick_key, A.brick_touched, A.touched_n, gb, key);
                        }
                        ci += 1;
                        continue;
                    }
                    if (d < dt_) {
                        d += 1;
                        continue;
                    }
                    // at traversal depth: probe the desired brick
                    const int cbx = brick_axis(px, S.dims[lev][0], bx, S.grids[lev][0]);
                    const int cby = brick_axis(py, S.dims[lev][1], by, S.grids[lev][1]);
                    const int cbz = brick_axis(pz, S.dims[lev][2], bz, S.grids[lev][2]);
                    const int64_t e = S.ptoff[ci][lev] +
                        ((int64_t)cbz * S.grids[lev][1] + cby) * S.grids[lev][0] + cbx;
                    const int pv = __ldg(A.pt + e);
                    if (pv >= 0) {
                        sample(ci, lev, cbx, cby, cbz, pv, e);
                    } else {
                        const unsigned long long key =
                            ((unsigned long long)pix << 32) | ev++;
                        int32_t &lb = last_breq[ci * kBlock + tid];
                        if ((int32_t)e != lb) {
                            lb = (int32_t)e;
                            request(A.brick_key, A.brick_touched, A.touched_n, e, key);
                        }
                        // nearest resident level in this node, coarser first
                        bool found = false;
                        for (int delta = 1; delta < k && !found; ++delta) {
                            for (int sgn = 0; sgn < 2; ++sgn) {
                                const int cand = sgn == 0 ? lev + delta : lev - delta;
                                if (cand < 0 || cand >= k) continue;
                                if (!((mask >> cand) & 1u)) continue;
                                const int abx = brick_axis(px, S.dims[cand][0], bx, S.grids[cand][0]);
                                const int aby = brick_axis(py, S.dims[cand][1], by, S.grids[cand][1]);
                                const int abz = brick_axis(pz, S.dims[cand][2], bz, S.grids[cand][2]);
                                const int64_t e2 = S.ptoff[ci][cand] +
                                    ((int64_t)abz * S.grids[cand][1] + aby) * S.grids[cand][0] + abx;
                                const int pv2 = __ldg(A.pt + e2);
                                if (pv2 >= 0) {
                                    sample(ci, cand, abx, aby, abz, pv2, e2);
                                    found = true;
                                    break;
                                }
                            }
                        }
                    }
                    all_cz = false;
                    ci += 1;
                }
                end_depth = d;
                if (all_cz) {
                    skippable = true;
                    const double s = 1.0 / (double)(1 << d);
                    skip_exit = box_exit(ox, oy, oz, dx, dy, dz, ix * s, iy * s,
                                         iz * s, (ix + 1) * s, (iy + 1) * s,
                                         (iz + 1) * s);
                }
            }

            if (skippable) {  // kernels.py:561-635
                const double limit = skip_exit < tfar ? skip_exit : tfar;
                const double t_before = t;
                const double alpha = 1.0 - trans;
                while (t < limit && accA < F.early_alpha) {
                    if (any_const) {
                        if (alpha > 0.0) {
                            const double corr = 1.0 - pow_pow2(1.0 - alpha, jexp);
                            const double scale = corr / alpha;
                            const double wgt = 1.0 - accA;
                            accR += wgt * sR * scale;
                            accG += wgt * sG * scale;
                            accB += wgt * sB * scale;
                            accA += wgt * corr;
                        }
                        c_eval += 1;
                    } else {
                        c_skip += 1;
                        if (CHECK && zero_mask) {
                            double qx = ox + t * dx, qy = oy + t * dy, qz = oz + t * dz;
                            if (qx < 0.0) qx = 0.0;
                            if (qy < 0.0) qy = 0.0;
                            if (qz < 0.0) qz = 0.0;
                            if (qx > kClampHi) qx = kClampHi;
                            if (qy > kClampHi) qy = kClampHi;
                            if (qz > kClampHi) qz = kClampHi;
                            const int raw2 = lod_raw(t, F.t0, S);
                            for (int ci = 0; ci < n_ch; ++ci) {
                                if (!((zero_mask >> ci) & 1u)) continue;
                                const int lev = clampi(raw2, S.lo[ci], S.hi[ci]);
                                const int cbx = brick_axis(qx, S.dims[lev][0], bx, S.grids[lev][0]);
                                const int cby = brick_axis(qy, S.dims[lev][1], by, S.grids[lev][1]);
                                const int cbz = brick_axis(qz, S.dims[lev][2], bz, S.grids[lev][2]);
                                const int64_t e = S.ptoff[ci][lev] +
                                    ((int64_t)cbz * S.grids[lev][1] + cby) * S.grids[lev][0] + cbx;
                                const int rp = F.ref_pt[e];
                                if (rp < 0) continue;
                                const double rv = trilinear(
                                    F.ref_cache + (int64_t)rp * bvox,
                                    qx * S.dims[lev][0] - (double)(cbx * bx),
                                    qy * S.dims[lev][1] - (double)(cby * by),
                                    qz * S.dims[lev][2] - (double)(cbz * bz), bx, by, bz);
                                double r, g, b, a;
                                tf_eval(S, ci, rv, r, g, b, a);
                                if (a > 0.0) c_viol += 1;
                            }
                        }
                    }
                    const int raw2 = lod_raw(t, F.t0, S);
                    step = S.step_tab[raw2];
                    jexp = S.maxlev[raw2];
                    t += step;
                }
                prev_depth = end_depth;
                if (t == t_before) {
                    if (++stall > D + 2) { c_live += 1; break; }
                } else {
                    stall = 0;
                }
                continue;
            }
            stall = 0;

            if (CHECK && zero_mask) {  // kernels.py:644-655
                for (int ci = 0; ci < n_ch; ++ci) {
                    if (!((zero_mask >> ci) & 1u)) continue;
                    const int lev = clampi(raw, S.lo[ci], S.hi[ci]);
                    const int cbx = brick_axis(px, S.dims[lev][0], bx, S.grids[lev][0]);
                    const int cby = brick_axis(py, S.dims[lev][1], by, S.grids[lev][1]);
                    const int cbz = brick_axis(pz, S.dims[lev][2], bz, S.grids[lev][2]);
                    const int64_t e = S.ptoff[ci][lev] +
                        ((int64_t)cbz * S.grids[lev][1] + cby) * S.grids[lev][0] + cbx;
                    const int rp = F.ref_pt[e];
                    if (rp < 0) continue;
                    const double rv = trilinear(
                        F.ref_cache + (int64_t)rp * bvox,
                        px * S.dims[lev][0] - (double)(cbx * bx),
                        py * S.dims[lev][1] - (double)(cby * by),
                        pz * S.dims[lev][2] - (double)(cbz * bz), bx, by, bz);
                    double r, g, b, a;
                    tf_eval(S, ci, rv, r, g, b, a);
                    if (a > 0.0) c_viol += 1;
                }
            }
            const double alpha = 1.0 - trans;
            if (alpha > 0.0) {
                const double corr = 1.0 - pow_pow2(1.0 - alpha, jexp);
                const double scale = corr / alpha;
                const double wgt = 1.0 - accA;
                accR += wgt * sR * scale;
                accG += wgt * sG * scale;
                accB += wgt * sB * scale;
                accA += wgt * corr;
            }
            c_eval += 1;
            t += step;
            prev_depth = end_depth;
        }
        float4 px4 = make_float4(__double2float_rn(accR), __double2float_rn(accG),
                                 __double2float_rn(accB), __double2float_rn(accA));
        reinterpret_cast<float4 *>(A.image)[lpix] = px4;
        A.pix_required[lpix] = pixreq;
    }

    // ---- block reductions ----
    unsigned long long vals[5] = {c_steps, c_eval, c_skip, c_viol, c_live};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        unsigned long long v = vals[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&S.red[i], v);
    }
    __syncthreads();
    if (tid < 5 && S.red[tid]) atomicAdd(A.counters + tid, S.red[tid]);
    for (int i = tid; i < n_ch * k; i += kBlock) {
        unsigned long long s = 0;
        for (int j = 0; j < kBlock; ++j) s += hist_t[i * kBlock + j];
        if (s) atomicAdd(A.hist + i, s);
    }
}

template <int MODE, bool CHECK>
cudaError_t launch(const ro_frame &F, const RayArgs &A, cudaStream_t s) {
    dim3 grid((F.width + kTileW - 1) / kTileW,
              (A.local_rows + kTileH - 1) / kTileH);
    size_t dyn = (size_t)F.n_ch * kBlock * 4 * 3 + (size_t)F.n_ch * A.L.k * kBlock * 4;
    auto kern = k_raycast<MODE, CHECK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return e;
    kern<<<grid, kBlock, dyn, s>>>(F, A);
    return cudaGetLastError();
}

}  // namespace

int render(ro_ctx *c, const ro_frame *F, const ro_state *st,
           const ro_outputs *out, cudaStream_t s) {
    if (F->n_ch < 1 || F->n_ch > RO_MAX_CH) return fail(RO_EINVAL, "n_ch outside [1, 8]");
    if (F->width < 1 || F->height < 1) return fail(RO_EINVAL, "empty image");
    if (F->n_parts < 1 || F->part < 0 || F->part >= F->n_parts || F->tile_rows < 1)
        return fail(RO_EINVAL, "bad partition");
    if ((int64_t)F->width * F->height >= (int64_t(1) << 31))
        return fail(RO_EINVAL, "image too large");
    for (int i = 0; i < F->n_ch; ++i) {
        const ro_channel &ch = F->ch[i];
        if (ch.slot < 0 || ch.slot >= c->layout.m) return fail(RO_EINVAL, "channel slot out of range");
        if (ch.lo < 0 || ch.hi >= c->layout.k || ch.lo > ch.hi)
            return fail(RO_EINVAL, "channel level range invalid");
        if (ch.npoints < 1 || ch.npoints > RO_MAX_TF_POINTS)
            return fail(RO_EINVAL, "transfer function point count outside [1, 16]");
    }
    if (F->mode == RO_MODE_RESIDENCY && st->words == nullptr)
        return fail(RO_EINVAL, "residency mode needs octree words");
    if (F->check_skips && (F->ref_pt == nullptr || F->ref_cache == nullptr))
        return fail(RO_EINVAL, "check_skips needs reference paging");
    if (F->mode == RO_MODE_RESIDENCY) {
        int rc = ensure_meta_keys(c);
        if (rc) return rc;
    }
    RayArgs A;
    A.L = c->dl;
    A.words = st->words;
    A.pt = st->pt;
    A.cache = st->cache;
    A.image = out->image;
    A.required = out->required;
    A.pix_required = out->pix_required;
    A.hist = reinterpret_cast<unsigned long long *>(out->hist);
    A.counters = reinterpret_cast<unsigned long long *>(out->counters);
    A.brick_key = c->brick_key;
    A.meta_key = c->meta_key;
    A.brick_touched = c->brick_touched;
    A.meta_touched = c->meta_touched;
    A.touched_n = c->touched_n;
    A.local_rows = (int32_t)ro_local_rows(F->height, F->n_parts, F->part, F->tile_rows);
    RO_CUDA(cudaMemsetAsync(out->required, 0, (size_t)c->E, s));
    RO_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(int64_t) * F->n_ch * c->layout.k, s));
    RO_CUDA(cudaMemsetAsync(out->counters, 0, sizeof(int64_t) * RO_NUM_COUNTERS, s));
    if (A.local_rows == 0) return RO_OK;
    cudaError_t e;
    if (F->mode == RO_MODE_REFERENCE) {
        e = launch<RO_MODE_REFERENCE, false>(*F, A, s);
    } else if (F->check_skips) {
        e = launch<RO_MODE_RESIDENCY, true>(*F, A, s);
    } else {
        e = launch<RO_MODE_RESIDENCY, false>(*F, A, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "k_raycast launch");
    return RO_OK;
}

}  // namespace ro
