// pack.cu -- host-side frame packing for C / C++ hosts (ro_pack_frame).
//
// Fills an ro_frame exactly like the Python mirror (render._pack_frame,
// camera.ray_basis, transfer.TransferFunction.empty_below), byte for byte:
//   * camera basis: numpy's camera.py:35-44 arithmetic (np.linalg.norm of a
//     3-vector as BLAS ddot computes it, np.cross component order);
//   * LOD thresholds: T[L] = smallest ratio >= 1 with floor(log2(ratio)) >= L,
//     found with the platform libm log2 the reference calls (kernels.py:49);
//   * per raw level: maxlev over the channels' clamped ranges, step =
//     base_step * 2^maxlev, traversal depth (kernels.py:57-66);
//   * per channel: clamped level range, TF knots, and the emptiness table
//     E[mn] (interval (mn, mx) transparent <=> mx < E[mn]) restating
//     transfer.py:38-120 (support intervals, first support at or after v).
// No CUDA calls: usable without a device.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace ro {
namespace {

// ---- transfer-function queries (transfer.py:38-120 semantics) ----------
// A TF is n knots (x strictly increasing, RGBA each); every query below is a
// function of the knots alone and is exported for the host mirror
// (transfer.TransferFunction keeps only the validated knot tuple).
struct TF {
    int n;
    const double *x;
    const double (*c)[4];
};

// RGBA at v: linear on the first knot segment containing v (a shared knot
// belongs to the segment on its left -- same value either way), transparent
// outside [x_0, x_{n-1}].  The reference rounds t = (v - x0) / (x1 - x0)
// and c0 + (c1 - c0) * t unfused; this file is compiled with
// -ffp-contract=off so the host values equal the kernel's bit for bit.
void tf_rgba_at(const TF &tf, double v, double out[4]) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    // (a single knot has no segment: transparent everywhere, like the reference)
    if (tf.n < 2 || v < tf.x[0] || v > tf.x[tf.n - 1]) return;
    int i = 0;
    while (i + 2 < tf.n && tf.x[i + 1] < v) ++i;
    const double x0 = tf.x[i], x1 = tf.x[i + 1];
    const double t = (x1 == x0) ? 0.0 : (v - x0) / (x1 - x0);
    for (int j = 0; j < 4; ++j) out[j] = tf.c[i][j] + (tf.c[i + 1][j] - tf.c[i][j]) * t;
}

double tf_alpha_at(const TF &tf, double v) {
    double o[4];
    tf_rgba_at(tf, v, o);
    return o[3];
}

// segment i carries opacity somewhere iff one of its knots is opaque; its
// opaque part is the closed segment minus each end whose knot alpha is 0
inline bool seg_opaque(const TF &tf, int i) { return tf.c[i][3] > 0.0 || tf.c[i + 1][3] > 0.0; }

// inf{x >= a : alpha(x) > 0}, +inf when the TF is transparent from a on.
// A segment's opaque part meets [a, inf) iff its right end lies beyond a,
// or at a with an opaque right knot; it then starts at max(x_i, a).
double tf_first_support(const TF &tf, double a) {
    if (tf_alpha_at(tf, a) > 0.0) return a;
    double best = INFINITY;
    for (int i = 0; i + 1 < tf.n; ++i) {
        if (!seg_opaque(tf, i)) continue;
        const double x1 = tf.x[i + 1];
        if (x1 > a || (x1 == a && tf.c[i + 1][3] > 0.0)) best = std::fmin(best, std::fmax(tf.x[i], a));
    }
    return best;
}

// maximal runs of opaque segments as (start, end, end_closed)
int tf_support_runs(const TF &tf, double *out) {
    int n = 0;
    for (int i = 0; i + 1 < tf.n;) {
        if (!seg_opaque(tf, i)) { ++i; continue; }
        int j = i;
        while (j + 2 < tf.n && seg_opaque(tf, j + 1)) ++j;
        out[3 * n + 0] = tf.x[i];
        out[3 * n + 1] = tf.x[j + 1];
        out[3 * n + 2] = tf.c[j + 1][3] > 0.0 ? 1.0 : 0.0;
        ++n;
        i = j + 1;
    }
    return n;
}

// integer scalars: first support (inf -> 1e30) and opacity, plus the
// kernel's emptiness threshold E[mn]: metadata (mn, mx) is transparent
// (kernels.py:201-206: f > mx, or f == mx with alpha(mx) == 0) iff mx < E[mn]
void tf_tables(const TF &tf, double f[256], double op[256], uint16_t eb[256]) {
    for (int v = 0; v < 256; ++v) op[v] = tf_alpha_at(tf, (double)v);
    for (int v = 0; v < 256; ++v) {
        const double fs = tf_first_support(tf, (double)v);
        f[v] = std::isfinite(fs) ? fs : 1e30;
        int e;
        if (fs >= 256.0) {
            e = 256;  // transparent on [v, 255]
        } else if (fs == std::floor(fs)) {
            // mx = fs is empty only when the support is open at fs
            e = op[(int)fs] == 0.0 ? (int)fs + 1 : (int)fs;
        } else {
            e = (int)std::ceil(fs);
        }
        eb[v] = (uint16_t)(e < 256 ? e : 256);
    }
}

// largest integer v with alpha(u) == 0 for every u <= v (-1: none; 255: all):
// the sampled value lies below the first opaque knot segment's support
int tf_zero_upto(const TF &tf) {
    for (int i = 0; i + 1 < tf.n; ++i) {
        if (tf.c[i][3] > 0.0) return (int)std::ceil(tf.x[i]) - 1;
        if (tf.c[i + 1][3] > 0.0) return (int)std::floor(tf.x[i]);
    }
    return 255;  // transparent everywhere (a single knot evaluates to 0 off it)
}

// kernel search start per integer scalar j: the first segment whose right
// knot is >= j
void tf_seg_start(const TF &tf, uint8_t out[256]) {
    int s = 0;
    for (int j = 0; j < 256; ++j) {
        while (s < tf.n - 2 && tf.x[s + 1] < (double)j) ++s;
        out[j] = (uint8_t)s;
    }
}

// render.py:lod_thresholds
void lod_thresholds(double out[RO_MAX_LEVELS + 1]) {
    out[0] = 1.0;
    for (int L = 1; L < RO_MAX_LEVELS; ++L) {
        double r = std::ldexp(1.0, L);
        while (true) {
            const double p = std::nextafter(r, 0.0);
            if (std::floor(std::log2(p)) >= L) r = p;
            else break;
        }
        out[L] = r;
    }
    out[RO_MAX_LEVELS] = INFINITY;
}

// kernels.py:57-66
int traversal_depth(double step, int max_depth) {
    if (step >= 1.0) return 0;
    int d = (int)std::floor(std::log2(1.0 / step));
    if (d < 0) d = 0;
    return d > max_depth ? max_depth : d;
}

// numpy.linalg.norm of a 3-vector = sqrt(x.dot(x)); the BLAS ddot in this
// image accumulates with fused multiply-adds in index order (measured:
// identical to np.linalg.norm on every tested vector)
double norm3(const double v[3]) {
    return std::sqrt(std::fma(v[2], v[2], std::fma(v[1], v[1], v[0] * v[0])));
}

void cross3(const double a[3], const double b[3], double out[3]) {
    out[0] = a[1] * b[2] - a[2] * b[1];
    out[1] = a[2] * b[0] - a[0] * b[2];
    out[2] = a[0] * b[1] - a[1] * b[0];
}

int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

}  // namespace
}  // namespace ro

using namespace ro;

extern "C" int ro_pack_frame(int32_t k, int32_t m, int32_t depth, int32_t mode,
                             const ro_camera *cam, const ro_render_config *cfg,
                             const ro_channel_desc *channels, int32_t n_ch, double eps_h,
                             ro_frame *F) {
    if (!cam || !cfg || !channels || !F) return fail(RO_EINVAL, "null argument");
    if (k < 1 || k > RO_MAX_LEVELS || m < 1) return fail(RO_EINVAL, "bad k / m");
    if (n_ch < 1) return fail(RO_EINVAL, "need at least one active channel");
    if (n_ch > RO_MAX_CH) return fail(RO_EINVAL, "at most 8 active channels");
    if (cfg->width < 1 || cfg->height < 1) return fail(RO_EINVAL, "empty image");
    memset(F, 0, sizeof(*F));
    F->mode = mode;
    F->n_ch = n_ch;
    F->width = cfg->width;
    F->height = cfg->height;
    // camera.py:35-44
    double fwd[3], right[3], up[3];
    for (int a = 0; a < 3; ++a) fwd[a] = cam->target[a] - cam->position[a];
    const double nf = norm3(fwd);
    for (int a = 0; a < 3; ++a) fwd[a] /= nf;
    cross3(fwd, cam->up, right);
    const double nr = norm3(right);
    for (int a = 0; a < 3; ++a) right[a] /= nr;
    cross3(right, fwd, up);
    for (int a = 0; a < 3; ++a) {
        F->cam_pos[a] = cam->position[a];
        F->cam_fwd[a] = fwd[a];
        F->cam_right[a] = right[a];
        F->cam_up[a] = up[a];
    }
    F->tan_half = std::tan(cam->fov_deg * (M_PI / 180.0) / 2.0);
    F->aspect = (double)cfg->width / (double)cfg->height;
    F->base_step = cfg->base_step;
    F->t0 = cfg->lod_reference_distance;
    F->early_alpha = cfg->early_term_alpha;
    F->eps_h = eps_h;
    F->start_level = cfg->traversal_start_level;
    lod_thresholds(F->lod_threshold);
    int los[RO_MAX_CH], his[RO_MAX_CH];
    for (int i = 0; i < n_ch; ++i) {
        const ro_channel_desc &c = channels[i];
        if (c.slot < 0 || c.slot >= m) return fail(RO_EINVAL, "channel slot out of range");
        if (c.level_lo > c.level_hi) return fail(RO_EINVAL, "level range inverted");
        if (c.npoints < 1 || c.npoints > RO_MAX_TF_POINTS)
            return fail(RO_EINVAL, "transfer function point count outside [1, 16]");
        los[i] = clampi(c.level_lo, 0, k - 1);
        his[i] = clampi(c.level_hi, 0, k - 1);
        ro_channel &ch = F->ch[i];
        ch.slot = c.slot;
        ch.lo = los[i];
        ch.hi = his[i];
        ch.npoints = c.npoints;
        for (int j = 0; j < c.npoints; ++j) {
            ch.tf_x[j] = c.x[j];
            for (int q = 0; q < 4; ++q) ch.tf_rgba[j][q] = c.rgba[j][q];
        }
        const TF tf{c.npoints, c.x, c.rgba};
        double f[256], op[256];
        tf_tables(tf, f, op, ch.empty_below);
        ch.zero_upto = tf_zero_upto(tf);
        tf_seg_start(tf, ch.tf_seg);
    }
    for (int raw = 0; raw < RO_MAX_LEVELS; ++raw) {
        int maxlev = 0;
        for (int i = 0; i < n_ch; ++i) maxlev = std::max(maxlev, clampi(raw, los[i], his[i]));
        const double step = cfg->base_step * (double)(1 << maxlev);
        F->maxlev_tab[raw] = maxlev;
        F->step_tab[raw] = step;
        F->dt_tab[raw] = traversal_depth(step, depth);
    }
    F->n_parts = 1;
    F->part = 0;
    F->tile_rows = 8;
    return RO_OK;
}

// ---- transfer-function queries for host mirrors (no CUDA) ----
static int tf_arg(int32_t n, const double *x, const double *rgba) {
    if (n < 1 || !x || !rgba) return fail(RO_EINVAL, "transfer function needs >= 1 knot");
    return RO_OK;
}
#define RO_TF(n, x, rgba) ro::TF{(n), (x), reinterpret_cast<const double(*)[4]>(rgba)}

extern "C" int ro_tf_evaluate(int32_t n, const double *x, const double *rgba, double v,
                              double *out4) {
    if (int rc = tf_arg(n, x, rgba)) return rc;
    if (!out4) return fail(RO_EINVAL, "null output");
    tf_rgba_at(RO_TF(n, x, rgba), v, out4);
    return RO_OK;
}

extern "C" int ro_tf_first_support(int32_t n, const double *x, const double *rgba, double a,
                                   double *out) {
    if (int rc = tf_arg(n, x, rgba)) return rc;
    if (!out) return fail(RO_EINVAL, "null output");
    *out = tf_first_support(RO_TF(n, x, rgba), a);
    return RO_OK;
}

extern "C" int ro_tf_support_intervals(int32_t n, const double *x, const double *rgba,
                                       double *out, int32_t *n_out) {
    if (int rc = tf_arg(n, x, rgba)) return rc;
    if (!out || !n_out) return fail(RO_EINVAL, "null output");
    *n_out = tf_support_runs(RO_TF(n, x, rgba), out);
    return RO_OK;
}

extern "C" int ro_tf_interval_max_opacity(int32_t n, const double *x, const double *rgba,
                                          double lo, double hi, double *out) {
    if (int rc = tf_arg(n, x, rgba)) return rc;
    if (!out) return fail(RO_EINVAL, "null output");
    const TF tf = RO_TF(n, x, rgba);
    if (hi < lo) std::swap(lo, hi);
    // linear between knots: the maximum sits at an end or at a knot inside
    double best = std::max(tf_alpha_at(tf, lo), tf_alpha_at(tf, hi));
    for (int i = 0; i < n; ++i)
        if (lo < tf.x[i] && tf.x[i] < hi) best = std::max(best, tf.c[i][3]);
    *out = best;
    return RO_OK;
}

extern "C" int ro_tf_tables(int32_t n, const double *x, const double *rgba,
                            double *first_support, double *opacity, uint16_t *empty_below,
                            int32_t *zero_upto) {
    if (int rc = tf_arg(n, x, rgba)) return rc;
    const TF tf = RO_TF(n, x, rgba);
    double f[256], op[256];
    uint16_t eb[256];
    tf_tables(tf, f, op, eb);
    if (first_support) memcpy(first_support, f, sizeof(f));
    if (opacity) memcpy(opacity, op, sizeof(op));
    if (empty_below) memcpy(empty_below, eb, sizeof(eb));
    if (zero_upto) *zero_upto = tf_zero_upto(tf);
    return RO_OK;
}
