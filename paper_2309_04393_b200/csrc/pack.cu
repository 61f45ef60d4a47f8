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
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace ro {
namespace {

struct TF {
    int n;
    const double *x;
    const double (*c)[4];
};

// transfer.py:42-52
void tf_evaluate(const TF &tf, double v, double out[4]) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    if (v < tf.x[0] || v > tf.x[tf.n - 1]) return;
    for (int i = 0; i + 1 < tf.n; ++i) {
        const double x0 = tf.x[i], x1 = tf.x[i + 1];
        if (x0 <= v && v <= x1) {
            const double t = (x1 == x0) ? 0.0 : (v - x0) / (x1 - x0);
            for (int j = 0; j < 4; ++j) out[j] = tf.c[i][j] + (tf.c[i + 1][j] - tf.c[i][j]) * t;
            return;
        }
    }
}

double tf_opacity(const TF &tf, double v) {
    double o[4];
    tf_evaluate(tf, v, o);
    return o[3];
}

struct Interval {
    double s, e;
    bool end_closed;
};

// transfer.py:66-78
std::vector<Interval> support_intervals(const TF &tf) {
    std::vector<Interval> out;
    for (int i = 0; i + 1 < tf.n; ++i) {
        const double x0 = tf.x[i], x1 = tf.x[i + 1];
        if (tf.c[i][3] > 0.0 || tf.c[i + 1][3] > 0.0) {
            const bool end_closed = tf.c[i + 1][3] > 0.0;
            if (!out.empty() && x0 <= out.back().e) {
                out.back().e = x1;
                out.back().end_closed = end_closed;
            } else {
                out.push_back({x0, x1, end_closed});
            }
        }
    }
    return out;
}

// transfer.py:80-87 (inf -> 1e30 as in support_table)
double first_support_at_or_after(const TF &tf, const std::vector<Interval> &iv, double a) {
    if (tf_opacity(tf, a) > 0.0) return a;
    double best = INFINITY;
    for (const Interval &it : iv)
        if (it.e > a || (it.e == a && it.end_closed)) best = std::fmin(best, std::fmax(it.s, a));
    return std::isfinite(best) ? best : 1e30;
}

// transfer.py:115-136
void empty_below(const TF &tf, uint16_t out[256]) {
    const std::vector<Interval> iv = support_intervals(tf);
    double op[256];
    for (int v = 0; v < 256; ++v) op[v] = tf_opacity(tf, (double)v);
    for (int mn = 0; mn < 256; ++mn) {
        const double fv = first_support_at_or_after(tf, iv, (double)mn);
        int e;
        if (fv >= 256.0) {
            e = 256;
        } else if (fv == std::floor(fv)) {
            const int fi = (int)fv;
            e = op[fi] == 0.0 ? fi + 1 : fi;
        } else {
            e = (int)std::ceil(fv);
        }
        out[mn] = (uint16_t)(e < 256 ? e : 256);
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
        empty_below(tf, ch.empty_below);
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
