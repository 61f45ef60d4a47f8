/*
 * resoct_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference ray-cast frame kernel
 *   /root/reference/pkg/src/resoctree/kernels.py:209-704 (raycast_frame)
 * for MODE_RESIDENCY (kernels.py:431-558), MODE_REFERENCE (301-314) and
 * the two baseline methods MODE_PAGETABLE (316-357) / MODE_CLASSIC (359-429),
 * including the skip loop (561-635), single-sample compositing (637-694)
 * and the skip audit (`check_skips`, 595-625 / 644-655 / 707-723).
 *
 * It takes the reference's own array layouts (pt_status i8 + pt_slot i32,
 * words u32[N, m], cache u8[S, bz, by, bx]) so reference state can be fed
 * to it unchanged.  Arithmetic follows the numba code operation by
 * operation in IEEE fp64 with NO contraction (build with -ffp-contract=off);
 * log2 and pow come from the system libm exactly like numba's calls
 * (kernels.py:49,61,585,685).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library.  The product path never calls it.
 *
 * Deviation (documented): the reference livelocks when a skip exit does not
 * advance t (SURVEY.md §7 hard part 4).  Here a ray whose state repeats
 * (no progress for depth+2 consecutive samples) is terminated and counted in
 * counters[4]; parity is undefined for such rays (the reference never
 * returns).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define K_ZERO 0
#define K_CONST 1
#define K_SAMPLE 2
#define K_MISSU 3
#define K_MISSP 4
#define ST_MAPPED 1
#define ST_EMPTY 2
#define MODE_RESIDENCY 0
#define MODE_REFERENCE 1
#define MODE_PAGETABLE 2
#define MODE_CLASSIC 3
#define MAXC 64

static const double CLAMP_HI = 1.0 - 1e-9;

typedef struct oracle_frame {
    int64_t mode;
    int64_t npix;
    const double *origins; /* [npix*3] */
    const double *dirs;    /* [npix*3] */
    int64_t n_ch;
    const int64_t *ch_slot, *ch_lo, *ch_hi; /* [n_ch] */
    int64_t npoints;
    const double *tf_x;    /* [n_ch*npoints] */
    const double *tf_rgba; /* [n_ch*npoints*4] */
    const int64_t *tf_np;  /* [n_ch] */
    const double *tf_f, *tf_op; /* [n_ch*256] */
    double base_step, t0, early_alpha, eps_h;
    int64_t start_level, depth_d, k, m;
    const int64_t *lvl_off; /* [depth+1] */
    const uint32_t *words;  /* [N*m] */
    const int32_t *dims, *grids; /* [k*3] (x,y,z) */
    int64_t bx, by, bz;
    const int64_t *pt_offsets; /* [m*k+1] */
    const int8_t *pt_status;
    const int32_t *pt_slot;
    const uint8_t *cache;
    int64_t check_skips;
    const int8_t *ref_status;
    const int32_t *ref_slot;
    const uint8_t *ref_cache;
    /* classic-octree baseline metadata (render.py:271-315), MODE_CLASSIC only */
    const uint8_t *cls_min, *cls_max; /* [n_nodes*m] */
    int64_t cls_depth;
    const int64_t *cls_lvl_off;       /* [cls_depth+1] */
    /* outputs */
    float *image;             /* [npix*4] */
    int64_t *brick_req, *brick_req_n;
    int64_t *meta_req, *meta_req_n;
    int64_t req_cap;
    uint8_t *seen_brick, *seen_meta, *required;
    int32_t *pix_required;    /* [npix] */
    int64_t *hist;            /* [n_ch*k] */
    int64_t *counters;        /* [5]: steps, evaluated, skipped, violations, livelocks */
    int64_t pix_begin, pix_end;
    /* optional [S*bvox]: every cache byte a trilinear fetch reads is set to
       1 (fixture generation: which voxels a frame depends on) */
    uint8_t *touched;
} oracle_frame;

static inline double lerp(double a, double b, double t) { return a + (b - a) * t; }

/* kernels.py:43-54 */
static int64_t lod_level(double t, double t0, int64_t lo, int64_t hi) {
    double ratio = t / t0;
    int64_t lev;
    if (ratio < 1.0) lev = 0;
    else lev = (int64_t)floor(log2(ratio));
    if (lev < lo) lev = lo;
    if (lev > hi) lev = hi;
    return lev;
}

/* kernels.py:57-66 */
static int64_t traversal_depth(double step, int64_t max_depth) {
    if (step >= 1.0) return 0;
    int64_t d = (int64_t)floor(log2(1.0 / step));
    if (d < 0) d = 0;
    if (d > max_depth) d = max_depth;
    return d;
}

/* kernels.py:69-94 */
static void ray_box_unit(double ox, double oy, double oz, double dx, double dy,
                         double dz, double *tn, double *tf) {
    double tmin = -1e30, tmax = 1e30;
    double o3[3] = {ox, oy, oz}, d3[3] = {dx, dy, dz};
    for (int a = 0; a < 3; ++a) {
        double o = o3[a], d = d3[a];
        if (fabs(d) < 1e-12) {
            if (o < 0.0 || o > 1.0) { *tn = 1.0; *tf = -1.0; return; }
        } else {
            double inv = 1.0 / d;
            double t0 = (0.0 - o) * inv;
            double t1 = (1.0 - o) * inv;
            if (t0 > t1) { double s = t0; t0 = t1; t1 = s; }
            if (t0 > tmin) tmin = t0;
            if (t1 < tmax) tmax = t1;
        }
    }
    *tn = tmin; *tf = tmax;
}

/* kernels.py:97-116 */
static double box_exit(double ox, double oy, double oz, double dx, double dy,
                       double dz, double lx, double ly, double lz, double hx,
                       double hy, double hz) {
    double te = 1e30;
    double o3[3] = {ox, oy, oz}, d3[3] = {dx, dy, dz};
    double l3[3] = {lx, ly, lz}, h3[3] = {hx, hy, hz};
    for (int a = 0; a < 3; ++a) {
        double t;
        if (d3[a] > 1e-12) t = (h3[a] - o3[a]) / d3[a];
        else if (d3[a] < -1e-12) t = (l3[a] - o3[a]) / d3[a];
        else continue;
        if (t < te) te = t;
    }
    return te;
}

/* kernels.py:119-133 */
static void tf_eval(const oracle_frame *f, int64_t ci, double v, double *r,
                    double *g, double *b, double *a) {
    const double *x = f->tf_x + ci * f->npoints;
    const double *c = f->tf_rgba + ci * f->npoints * 4;
    int64_t n = f->tf_np[ci];
    *r = *g = *b = *a = 0.0;
    if (v < x[0] || v > x[n - 1]) return;
    for (int64_t i = 0; i < n - 1; ++i) {
        double x0 = x[i], x1 = x[i + 1];
        if (x0 <= v && v <= x1) {
            double t = (x1 == x0) ? 0.0 : (v - x0) / (x1 - x0);
            *r = lerp(c[i * 4 + 0], c[(i + 1) * 4 + 0], t);
            *g = lerp(c[i * 4 + 1], c[(i + 1) * 4 + 1], t);
            *b = lerp(c[i * 4 + 2], c[(i + 1) * 4 + 2], t);
            *a = lerp(c[i * 4 + 3], c[(i + 1) * 4 + 3], t);
            return;
        }
    }
}

/* kernels.py:136-174 */
static double trilinear_brick(const uint8_t *cache, int64_t slot_lin, double lx,
                              double ly, double lz, int64_t bx, int64_t by,
                              int64_t bz, uint8_t *touched) {
    double fx = lx - 0.5, fy = ly - 0.5, fz = lz - 0.5;
    if (fx < 0.0) fx = 0.0;
    if (fy < 0.0) fy = 0.0;
    if (fz < 0.0) fz = 0.0;
    if (fx > bx - 1.0) fx = bx - 1.0;
    if (fy > by - 1.0) fy = by - 1.0;
    if (fz > bz - 1.0) fz = bz - 1.0;
    int64_t x0 = (int64_t)fx, y0 = (int64_t)fy, z0 = (int64_t)fz;
    int64_t x1 = x0 + 1 < bx ? x0 + 1 : bx - 1;
    int64_t y1 = y0 + 1 < by ? y0 + 1 : by - 1;
    int64_t z1 = z0 + 1 < bz ? z0 + 1 : bz - 1;
    double tx = fx - x0, ty = fy - y0, tz = fz - z0;
    const uint8_t *c = cache + slot_lin * bx * by * bz;
    if (touched) {
        uint8_t *tc = touched + slot_lin * bx * by * bz;
        const int64_t zs[2] = {z0, z1}, ys[2] = {y0, y1}, xs[2] = {x0, x1};
        for (int a = 0; a < 2; ++a)
            for (int b2 = 0; b2 < 2; ++b2)
                for (int c2 = 0; c2 < 2; ++c2) tc[(zs[a] * by + ys[b2]) * bx + xs[c2]] = 1;
    }
#define V(z, y, x) ((double)c[((z) * by + (y)) * bx + (x)])
    double c00 = lerp(V(z0, y0, x0), V(z0, y0, x1), tx);
    double c10 = lerp(V(z0, y1, x0), V(z0, y1, x1), tx);
    double c01 = lerp(V(z1, y0, x0), V(z1, y0, x1), tx);
    double c11 = lerp(V(z1, y1, x0), V(z1, y1, x1), tx);
#undef V
    return lerp(lerp(c00, c10, ty), lerp(c01, c11, ty), tz);
}

/* kernels.py:177-184 */
static inline int64_t brick_axis(double p, int32_t dim, int64_t b, int32_t grid) {
    int64_t c = (int64_t)(p * (double)dim / (double)b);
    if (c < 0) c = 0;
    if (c > grid - 1) c = grid - 1;
    return c;
}

/* kernels.py:187-198 */
static inline int64_t entry_index(const oracle_frame *f, int64_t slot, int64_t lev,
                                  int64_t cx, int64_t cy, int64_t cz) {
    int64_t gx = f->grids[lev * 3 + 0], gy = f->grids[lev * 3 + 1];
    return f->pt_offsets[slot * f->k + lev] + (cz * gy + cy) * gx + cx;
}

/* kernels.py:201-206 */
static inline int is_empty_meta(const oracle_frame *f, int64_t ci, int64_t mn, int64_t mx) {
    double fv = f->tf_f[ci * 256 + mn];
    if (fv > (double)mx) return 1;
    return fv == (double)mx && f->tf_op[ci * 256 + mx] == 0.0;
}

/* kernels.py:707-723 */
static double ref_value(const oracle_frame *f, int64_t slot, int64_t lev,
                        double px, double py, double pz) {
    int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], f->bx, f->grids[lev * 3 + 0]);
    int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], f->by, f->grids[lev * 3 + 1]);
    int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], f->bz, f->grids[lev * 3 + 2]);
    int64_t e = entry_index(f, slot, lev, cbx, cby, cbz);
    if (f->ref_status[e] != ST_MAPPED) return -1.0;
    double lx = px * f->dims[lev * 3 + 0] - (double)(cbx * f->bx);
    double ly = py * f->dims[lev * 3 + 1] - (double)(cby * f->by);
    double lz = pz * f->dims[lev * 3 + 2] - (double)(cbz * f->bz);
    return trilinear_brick(f->ref_cache, f->ref_slot[e], lx, ly, lz, f->bx, f->by, f->bz,
                           NULL);
}

static inline void push_req(int64_t *buf, int64_t *n, int64_t cap, int64_t v) {
    int64_t nn = *n;
    if (nn < cap) { buf[nn] = v; *n = nn + 1; }
}

static inline int64_t brick_id(int64_t slot, int64_t k, int64_t lev, int64_t cx,
                               int64_t cy, int64_t cz) {
    return ((slot * k + lev) << 24) | (cz << 16) | (cy << 8) | cx;
}

/* kernels.py:209-704 over pixels [pix_begin, pix_end) */
int oracle_raycast(const oracle_frame *f) {
    const int64_t n_ch = f->n_ch, k = f->k, m = f->m;
    const int64_t bx = f->bx, by = f->by, bz = f->bz;
    if (n_ch < 1 || n_ch > MAXC) return -1;
    int64_t desired[MAXC], out_kind[MAXC], out_slot[MAXC], out_level[MAXC];
    int64_t prev_brick[MAXC];
    double out_val[MAXC];
    int64_t steps_total = 0, evaluated = 0, skipped = 0, violations = 0, livelocks = 0;

    for (int64_t pix = f->pix_begin; pix < f->pix_end; ++pix) {
        const double ox = f->origins[pix * 3 + 0], oy = f->origins[pix * 3 + 1],
                     oz = f->origins[pix * 3 + 2];
        const double dx = f->dirs[pix * 3 + 0], dy = f->dirs[pix * 3 + 1],
                     dz = f->dirs[pix * 3 + 2];
        double tnear, tfar;
        ray_box_unit(ox, oy, oz, dx, dy, dz, &tnear, &tfar);
        double accR = 0.0, accG = 0.0, accB = 0.0, accA = 0.0;
        double t = tnear > 0.0 ? tnear : 0.0;
        for (int64_t ci = 0; ci < n_ch; ++ci) prev_brick[ci] = -1;
        int64_t prev_depth = f->start_level;
        int64_t stall = 0; /* livelock guard, see header */

        while (t < tfar && accA < f->early_alpha) {
            double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
            if (px < 0.0) px = 0.0;
            if (py < 0.0) py = 0.0;
            if (pz < 0.0) pz = 0.0;
            if (px > CLAMP_HI) px = CLAMP_HI;
            if (py > CLAMP_HI) py = CLAMP_HI;
            if (pz > CLAMP_HI) pz = CLAMP_HI;

            int64_t maxlev = 0;
            for (int64_t ci = 0; ci < n_ch; ++ci) {
                int64_t lev = lod_level(t, f->t0, f->ch_lo[ci], f->ch_hi[ci]);
                desired[ci] = lev;
                if (lev > maxlev) maxlev = lev;
            }
            double step = f->base_step * (double)((int64_t)1 << maxlev);
            int64_t dt_ = traversal_depth(step, f->depth_d);

            int skippable = 0;
            double skip_exit = -1.0;
            int64_t end_depth = prev_depth;

            if (f->mode == MODE_REFERENCE) {
                for (int64_t ci = 0; ci < n_ch; ++ci) {
                    int64_t lev = desired[ci];
                    int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], bx, f->grids[lev * 3 + 0]);
                    int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], by, f->grids[lev * 3 + 1]);
                    int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], bz, f->grids[lev * 3 + 2]);
                    int64_t e = entry_index(f, f->ch_slot[ci], lev, cbx, cby, cbz);
                    if (f->pt_status[e] == ST_MAPPED) {
                        out_kind[ci] = K_SAMPLE;
                        out_slot[ci] = f->pt_slot[e];
                        out_level[ci] = lev;
                    } else {
                        out_kind[ci] = K_MISSP;
                    }
                }
            } else if (f->mode == MODE_PAGETABLE) { /* kernels.py:316-357 */
                int all_empty = 1;
                skip_exit = 1e30;
                for (int64_t ci = 0; ci < n_ch; ++ci) {
                    int64_t lev = desired[ci];
                    int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], bx, f->grids[lev * 3 + 0]);
                    int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], by, f->grids[lev * 3 + 1]);
                    int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], bz, f->grids[lev * 3 + 2]);
                    int64_t slot = f->ch_slot[ci];
                    int64_t e = entry_index(f, slot, lev, cbx, cby, cbz);
                    int st = f->pt_status[e];
                    if (st == ST_MAPPED) {
                        out_kind[ci] = K_SAMPLE;
                        out_slot[ci] = f->pt_slot[e];
                        out_level[ci] = lev;
                        all_empty = 0;
                    } else if (st == ST_EMPTY) {
                        out_kind[ci] = K_ZERO;
                        double dxl = (double)f->dims[lev * 3 + 0], dyl = (double)f->dims[lev * 3 + 1],
                               dzl = (double)f->dims[lev * 3 + 2];
                        double ex = box_exit(ox, oy, oz, dx, dy, dz,
                                             (double)(cbx * bx) / dxl, (double)(cby * by) / dyl,
                                             (double)(cbz * bz) / dzl,
                                             (double)((cbx + 1) * bx) / dxl,
                                             (double)((cby + 1) * by) / dyl,
                                             (double)((cbz + 1) * bz) / dzl);
                        if (ex < skip_exit) skip_exit = ex;
                    } else {
                        out_kind[ci] = K_MISSP;
                        if (f->seen_brick[e] == 0) {
                            f->seen_brick[e] = 1;
                            push_req(f->brick_req, f->brick_req_n, f->req_cap,
                                     brick_id(slot, k, lev, cbx, cby, cbz));
                        }
                        all_empty = 0;
                    }
                }
                skippable = all_empty;
            } else if (f->mode == MODE_CLASSIC) { /* kernels.py:359-429 */
                int all_empty = 1;
                int64_t deep_d = -1, dix = 0, diy = 0, diz = 0;
                for (int64_t ci = 0; ci < n_ch; ++ci) {
                    int64_t lev = desired[ci];
                    int64_t slot = f->ch_slot[ci];
                    int64_t d_target = f->cls_depth - lev;
                    if (d_target < 0) d_target = 0;
                    int64_t d = 0, last_slot = -1, last_lev = -1;
                    while (1) {
                        steps_total += 1;
                        int64_t side = (int64_t)1 << d;
                        int64_t ix = (int64_t)(px * (double)side);
                        int64_t iy = (int64_t)(py * (double)side);
                        int64_t iz = (int64_t)(pz * (double)side);
                        int64_t nidx = f->cls_lvl_off[d] + (iz * side + iy) * side + ix;
                        int64_t mn = f->cls_min[nidx * m + slot], mx = f->cls_max[nidx * m + slot];
                        if (is_empty_meta(f, ci, mn, mx)) {
                            out_kind[ci] = K_ZERO;
                            if (d > deep_d) { deep_d = d; dix = ix; diy = iy; diz = iz; }
                            break;
                        }
                        int64_t lev_d = f->cls_depth - d;
                        int64_t e = entry_index(f, slot, lev_d, ix, iy, iz);
                        f->required[e] = 1;
                        if (f->pt_status[e] != ST_MAPPED) {
                            if (f->seen_brick[e] == 0) {
                                f->seen_brick[e] = 1;
                                push_req(f->brick_req, f->brick_req_n, f->req_cap,
                                         brick_id(slot, k, lev_d, ix, iy, iz));
                            }
                            /* descent blocked: deepest resident ancestor */
                            if (last_slot >= 0) {
                                out_kind[ci] = K_SAMPLE;
                                out_slot[ci] = last_slot;
                                out_level[ci] = last_lev;
                            } else {
                                out_kind[ci] = K_MISSP;
                            }
                            all_empty = 0;
                            break;
                        }
                        last_slot = f->pt_slot[e];
                        last_lev = lev_d;
                        if (d == d_target) {
                            out_kind[ci] = K_SAMPLE;
                            out_slot[ci] = last_slot;
                            out_level[ci] = last_lev;
                            all_empty = 0;
                            break;
                        }
                        d += 1;
                    }
                }
                if (all_empty && deep_d >= 0) {
                    skippable = 1;
                    double s = 1.0 / (double)((int64_t)1 << deep_d);
                    skip_exit = box_exit(ox, oy, oz, dx, dy, dz, dix * s, diy * s, diz * s,
                                         (dix + 1) * s, (diy + 1) * s, (diz + 1) * s);
                }
            } else { /* MODE_RESIDENCY, kernels.py:431-558 */
                int64_t d = prev_depth - 1;
                if (d < 0) d = 0;
                if (f->start_level < d) d = f->start_level;
                if (d > dt_) d = dt_;
                int64_t ci = 0;
                int all_cz = 1;
                int64_t ix = 0, iy = 0, iz = 0;
                while (ci < n_ch) {
                    int64_t side = (int64_t)1 << d;
                    ix = (int64_t)(px * (double)side);
                    iy = (int64_t)(py * (double)side);
                    iz = (int64_t)(pz * (double)side);
                    int64_t nidx = f->lvl_off[d] + (iz * side + iy) * side + ix;
                    steps_total += 1;
                    int64_t slot = f->ch_slot[ci];
                    int64_t w = (int64_t)f->words[nidx * m + slot];
                    int64_t mn = (w >> 16) & 0xFF, mx = (w >> 24) & 0xFF, mask = w & 0xFFFF;
                    int valid = !(mn == 255 && mx == 0);
                    if (!valid) {
                        int64_t mid = nidx * m + slot;
                        if (f->seen_meta[mid] == 0) {
                            f->seen_meta[mid] = 1;
                            push_req(f->meta_req, f->meta_req_n, f->req_cap, mid);
                        }
                    } else {
                        if (is_empty_meta(f, ci, mn, mx)) {
                            out_kind[ci] = K_ZERO;
                            ci += 1;
                            continue;
                        }
                        if ((double)(mx - mn) <= f->eps_h) {
                            out_kind[ci] = K_CONST;
                            out_val[ci] = (double)mn;
                            ci += 1;
                            continue;
                        }
                    }
                    if (mask == 0) {
                        out_kind[ci] = K_MISSU;
                        int64_t lev = desired[ci];
                        int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], bx, f->grids[lev * 3 + 0]);
                        int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], by, f->grids[lev * 3 + 1]);
                        int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], bz, f->grids[lev * 3 + 2]);
                        int64_t gb = entry_index(f, slot, lev, cbx, cby, cbz);
                        if (f->seen_brick[gb] == 0) {
                            f->seen_brick[gb] = 1;
                            push_req(f->brick_req, f->brick_req_n, f->req_cap,
                                     brick_id(slot, k, lev, cbx, cby, cbz));
                        }
                        ci += 1;
                        continue;
                    }
                    if (d < dt_) {
                        d += 1;
                        continue;
                    }
                    int64_t lev = desired[ci];
                    int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], bx, f->grids[lev * 3 + 0]);
                    int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], by, f->grids[lev * 3 + 1]);
                    int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], bz, f->grids[lev * 3 + 2]);
                    int64_t e = entry_index(f, slot, lev, cbx, cby, cbz);
                    if (f->pt_status[e] == ST_MAPPED) {
                        out_kind[ci] = K_SAMPLE;
                        out_slot[ci] = f->pt_slot[e];
                        out_level[ci] = lev;
                        all_cz = 0;
                    } else {
                        if (f->seen_brick[e] == 0) {
                            f->seen_brick[e] = 1;
                            push_req(f->brick_req, f->brick_req_n, f->req_cap,
                                     brick_id(slot, k, lev, cbx, cby, cbz));
                        }
                        int found = 0;
                        for (int64_t delta = 1; delta < k && !found; ++delta) {
                            for (int sgn = 0; sgn < 2; ++sgn) {
                                int64_t cand = sgn == 0 ? lev + delta : lev - delta;
                                if (cand < 0 || cand >= k) continue;
                                if (!((mask >> cand) & 1)) continue;
                                int64_t abx = brick_axis(px, f->dims[cand * 3 + 0], bx, f->grids[cand * 3 + 0]);
                                int64_t aby = brick_axis(py, f->dims[cand * 3 + 1], by, f->grids[cand * 3 + 1]);
                                int64_t abz = brick_axis(pz, f->dims[cand * 3 + 2], bz, f->grids[cand * 3 + 2]);
                                int64_t e2 = entry_index(f, slot, cand, abx, aby, abz);
                                if (f->pt_status[e2] == ST_MAPPED) {
                                    out_kind[ci] = K_SAMPLE;
                                    out_slot[ci] = f->pt_slot[e2];
                                    out_level[ci] = cand;
                                    found = 1;
                                    break;
                                }
                            }
                        }
                        if (!found) out_kind[ci] = K_MISSP;
                        all_cz = 0;
                    }
                    ci += 1;
                }
                end_depth = d;
                if (all_cz) {
                    skippable = 1;
                    double s = 1.0 / (double)((int64_t)1 << d);
                    skip_exit = box_exit(ox, oy, oz, dx, dy, dz, ix * s, iy * s, iz * s,
                                         (ix + 1) * s, (iy + 1) * s, (iz + 1) * s);
                }
            }

            if (skippable) { /* kernels.py:561-635 */
                int any_const = 0;
                for (int64_t ci = 0; ci < n_ch; ++ci)
                    if (out_kind[ci] == K_CONST) any_const = 1;
                double limit = skip_exit < tfar ? skip_exit : tfar;
                double t_before = t;
                while (t < limit && accA < f->early_alpha) {
                    if (any_const) {
                        double sR = 0.0, sG = 0.0, sB = 0.0, trans = 1.0;
                        for (int64_t ci = 0; ci < n_ch; ++ci) {
                            if (out_kind[ci] != K_CONST) continue;
                            double r, g, b, a;
                            tf_eval(f, ci, out_val[ci], &r, &g, &b, &a);
                            sR += r * a; sG += g * a; sB += b * a;
                            trans *= (1.0 - a);
                        }
                        double alpha = 1.0 - trans;
                        if (alpha > 0.0) {
                            double ratio = step / f->base_step;
                            double corr = 1.0 - pow(1.0 - alpha, ratio);
                            double scale = corr / alpha;
                            double wgt = 1.0 - accA;
                            accR += wgt * sR * scale;
                            accG += wgt * sG * scale;
                            accB += wgt * sB * scale;
                            accA += wgt * corr;
                        }
                        evaluated += 1;
                    } else {
                        skipped += 1;
                        if (f->check_skips) {
                            double qx = ox + t * dx, qy = oy + t * dy, qz = oz + t * dz;
                            if (qx < 0.0) qx = 0.0;
                            if (qy < 0.0) qy = 0.0;
                            if (qz < 0.0) qz = 0.0;
                            if (qx > CLAMP_HI) qx = CLAMP_HI;
                            if (qy > CLAMP_HI) qy = CLAMP_HI;
                            if (qz > CLAMP_HI) qz = CLAMP_HI;
                            for (int64_t ci = 0; ci < n_ch; ++ci) {
                                if (out_kind[ci] != K_ZERO) continue;
                                int64_t lev = lod_level(t, f->t0, f->ch_lo[ci], f->ch_hi[ci]);
                                double rv = ref_value(f, f->ch_slot[ci], lev, qx, qy, qz);
                                if (rv >= 0.0) {
                                    double r, g, b, a;
                                    tf_eval(f, ci, rv, &r, &g, &b, &a);
                                    if (a > 0.0) violations += 1;
                                }
                            }
                        }
                    }
                    int64_t ml = 0;
                    for (int64_t ci = 0; ci < n_ch; ++ci) {
                        int64_t lev = lod_level(t, f->t0, f->ch_lo[ci], f->ch_hi[ci]);
                        if (lev > ml) ml = lev;
                    }
                    step = f->base_step * (double)((int64_t)1 << ml);
                    t += step;
                }
                prev_depth = end_depth;
                if (t == t_before) {
                    if (++stall > f->depth_d + 2) { livelocks += 1; break; }
                } else {
                    stall = 0;
                }
                continue;
            }
            stall = 0;

            /* single-sample evaluation, kernels.py:637-694 */
            double sR = 0.0, sG = 0.0, sB = 0.0, trans = 1.0;
            for (int64_t ci = 0; ci < n_ch; ++ci) {
                int64_t kind = out_kind[ci];
                if (kind == K_ZERO) {
                    if (f->check_skips) {
                        int64_t lev = lod_level(t, f->t0, f->ch_lo[ci], f->ch_hi[ci]);
                        double rv = ref_value(f, f->ch_slot[ci], lev, px, py, pz);
                        if (rv >= 0.0) {
                            double r, g, b, a0;
                            tf_eval(f, ci, rv, &r, &g, &b, &a0);
                            if (a0 > 0.0) violations += 1;
                        }
                    }
                    continue;
                }
                if (kind == K_MISSU || kind == K_MISSP) continue;
                double v;
                if (kind == K_CONST) {
                    v = out_val[ci];
                } else {
                    int64_t lev = out_level[ci];
                    int64_t cbx = brick_axis(px, f->dims[lev * 3 + 0], bx, f->grids[lev * 3 + 0]);
                    int64_t cby = brick_axis(py, f->dims[lev * 3 + 1], by, f->grids[lev * 3 + 1]);
                    int64_t cbz = brick_axis(pz, f->dims[lev * 3 + 2], bz, f->grids[lev * 3 + 2]);
                    double lx = px * f->dims[lev * 3 + 0] - (double)(cbx * bx);
                    double ly = py * f->dims[lev * 3 + 1] - (double)(cby * by);
                    double lz = pz * f->dims[lev * 3 + 2] - (double)(cbz * bz);
                    v = trilinear_brick(f->cache, out_slot[ci], lx, ly, lz, bx, by, bz,
                                        f->touched);
                    int64_t gb = entry_index(f, f->ch_slot[ci], lev, cbx, cby, cbz);
                    f->required[gb] = 1;
                    f->hist[ci * k + lev] += 1;
                    if (gb != prev_brick[ci]) {
                        prev_brick[ci] = gb;
                        f->pix_required[pix] += 1;
                    }
                }
                double r, g, b, a;
                tf_eval(f, ci, v, &r, &g, &b, &a);
                sR += r * a; sG += g * a; sB += b * a;
                trans *= (1.0 - a);
            }
            double alpha = 1.0 - trans;
            if (alpha > 0.0) {
                double ratio = step / f->base_step;
                double corr = 1.0 - pow(1.0 - alpha, ratio);
                double scale = corr / alpha;
                double wgt = 1.0 - accA;
                accR += wgt * sR * scale;
                accG += wgt * sG * scale;
                accB += wgt * sB * scale;
                accA += wgt * corr;
            }
            evaluated += 1;
            t += step;
            prev_depth = end_depth;
        }
        f->image[pix * 4 + 0] = (float)accR;
        f->image[pix * 4 + 1] = (float)accG;
        f->image[pix * 4 + 2] = (float)accB;
        f->image[pix * 4 + 3] = (float)accA;
    }
    f->counters[0] += steps_total;
    f->counters[1] += evaluated;
    f->counters[2] += skipped;
    f->counters[3] += violations;
    f->counters[4] += livelocks;
    return 0;
}

/*
 * Multi-threaded driver for the CPU baseline: pixels are cut into bands,
 * each band renders with private request buffers / seen flags / usage mask /
 * counters, and the bands are merged in scanline order with keep-first
 * dedupe (the merge rule of SURVEY.md §8(d) "CPU baseline timing").  The
 * result is identical to one single-threaded oracle_raycast over the same
 * pixel range.  `n_entries` = total page-table entries, `n_meta` = N*m.
 */
int oracle_raycast_parallel(const oracle_frame *f, int64_t n_entries,
                            int64_t n_meta, int64_t n_threads) {
    int64_t npix = f->pix_end - f->pix_begin;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > npix) n_threads = npix > 0 ? npix : 1;
    int64_t nb = n_threads * 8; /* bands: a few per thread for balance */
    if (nb > npix) nb = npix > 0 ? npix : 1;
    oracle_frame *bands = (oracle_frame *)calloc((size_t)nb, sizeof(oracle_frame));
    int64_t cap = f->req_cap;
    int64_t nhist = f->n_ch * f->k;
    for (int64_t b = 0; b < nb; ++b) {
        oracle_frame *g = &bands[b];
        *g = *f;
        g->pix_begin = f->pix_begin + npix * b / nb;
        g->pix_end = f->pix_begin + npix * (b + 1) / nb;
        g->brick_req = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
        g->meta_req = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
        g->brick_req_n = (int64_t *)calloc(1, sizeof(int64_t));
        g->meta_req_n = (int64_t *)calloc(1, sizeof(int64_t));
        g->seen_brick = (uint8_t *)calloc((size_t)n_entries, 1);
        g->seen_meta = (uint8_t *)calloc((size_t)(n_meta > 0 ? n_meta : 1), 1);
        g->required = (uint8_t *)calloc((size_t)n_entries, 1);
        g->hist = (int64_t *)calloc((size_t)nhist, sizeof(int64_t));
        g->counters = (int64_t *)calloc(5, sizeof(int64_t));
    }
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
    for (int64_t b = 0; b < nb; ++b) oracle_raycast(&bands[b]);
    for (int64_t b = 0; b < nb; ++b) {
        oracle_frame *g = &bands[b];
        for (int64_t i = 0; i < *g->brick_req_n; ++i) {
            int64_t bid = g->brick_req[i];
            /* dedupe by page-table entry: recompute it from the id */
            int64_t pt = (bid >> 24) & 0xFF, lev = pt % f->k, slot = pt / f->k;
            int64_t cx = bid & 0xFF, cy = (bid >> 8) & 0xFF, cz = (bid >> 16) & 0xFF;
            int64_t e = entry_index(f, slot, lev, cx, cy, cz);
            if (!f->seen_brick[e]) {
                f->seen_brick[e] = 1;
                push_req(f->brick_req, f->brick_req_n, cap, bid);
            }
        }
        for (int64_t i = 0; i < *g->meta_req_n; ++i) {
            int64_t mid = g->meta_req[i];
            if (!f->seen_meta[mid]) {
                f->seen_meta[mid] = 1;
                push_req(f->meta_req, f->meta_req_n, cap, mid);
            }
        }
        for (int64_t e = 0; e < n_entries; ++e) f->required[e] |= g->required[e];
        for (int64_t i = 0; i < nhist; ++i) f->hist[i] += g->hist[i];
        for (int i = 0; i < 5; ++i) f->counters[i] += g->counters[i];
        free(g->brick_req); free(g->meta_req); free(g->brick_req_n); free(g->meta_req_n);
        free(g->seen_brick); free(g->seen_meta); free(g->required); free(g->hist);
        free(g->counters);
    }
    free(bands);
    return 0;
}
