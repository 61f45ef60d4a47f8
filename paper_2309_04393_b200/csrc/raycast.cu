// raycast.cu -- kernel 1: the per-pixel residency-octree ray caster.
//
// Restates /root/reference/pkg/src/resoctree/kernels.py:209-704
// (raycast_frame) for MODE_RESIDENCY (431-558), MODE_REFERENCE (301-314) and
// the paper's two baseline methods, MODE_PAGETABLE (316-357) and MODE_CLASSIC
// (359-429), with the skip loop (561-635), single-sample compositing (637-694) and the
// skip audit (595-625, 644-655, 707-723).
//
// B200 design:
//  * one thread per pixel, each warp an 8x4 pixel packet so neighbouring
//    rays walk the same octree nodes / bricks (L1-resident words, page-table
//    entries and trilinear taps); 128-thread CTAs;
//  * warp-uniform sample loop: the packet reconverges once per sample;
//  * rays are generated in-kernel from the camera basis (bit-exact with
//    camera.py:32-51, no 50 MB/frame ray upload);
//  * one cursor shared by all channels exactly like the reference, one
//    128-bit load per visited node holding all four channel slots' words;
//    each channel is sampled and composited the moment it resolves (same
//    channel order and arithmetic as the reference's two-pass form), so no
//    per-channel arrays spill to local memory and pollute L1;
//  * division-free addressing: brick sizes are powers of two, so
//    int(p*dim/b) == int(p*dim) >> log2(b) and node coordinates at depth d
//    are the depth-D leaf coordinates shifted right, both bit-exact;
//    u8 -> fp64 conversions use the 2^52 bias trick on the fp64 pipe
//    instead of the (much narrower) conversion pipe;
//  * request recording keeps the reference's first-seen order without a
//    serial buffer: every request event carries key = (pixel << 32 | event
//    index within the pixel) and a fire-and-forget RED.MIN per brick /
//    metadata entry keeps the smallest key (feedback.cu compacts + sorts);
//  * fp64 on the whole decision path, compiled with -fmad=false so every
//    operation rounds like numba's unfused code.
#include "internal.cuh"

#ifndef RO_MINB
#define RO_MINB 4
#endif
#ifndef RO_PERSISTENT
#define RO_PERSISTENT 1
#endif
#ifndef RO_SUBMAX
#define RO_SUBMAX 1
#endif
// RO_DEBUG_CHECKS=1: device-side bounds assertions at every indexed access of
// the ray caster (trap on violation); the GPU suite runs against this build
#ifndef RO_DEBUG_CHECKS
#define RO_DEBUG_CHECKS 0
#endif
#if RO_DEBUG_CHECKS
#define RO_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define RO_ASSERT(c) do { } while (0)
#endif
#ifndef RO_CH_CONST
#define RO_CH_CONST 1
#endif
#if RO_CH_CONST
// warp-uniform per-channel scalars straight from the kernel-parameter bank
#define CH_LO(ci) (F.ch[ci].lo)
#define CH_HI(ci) (F.ch[ci].hi)
#define CH_SLOT(ci) (F.ch[ci].slot)
#else
#define CH_LO(ci) (S.lo[ci])
#define CH_HI(ci) (S.hi[ci])
#define CH_SLOT(ci) (S.slot[ci])
#endif
#ifndef RO_WARPS
#define RO_WARPS 4
#endif
#ifndef RO_TILE_W
#define RO_TILE_W 16
#endif
#ifndef RO_TILE_H
#define RO_TILE_H 8
#endif
#ifndef RO_FAST_DESCENT
#define RO_FAST_DESCENT 1
#endif
#ifndef RO_PREFETCH
#define RO_PREFETCH 0
#endif
// path classes also carry each channel's ZERO nodes: a walk ending on one
// terminates without reading the node's word (1)
#ifndef RO_PATH_ZERO
#define RO_PATH_ZERO 1
#endif
// brick-run histogram (1) or a histogram increment per fetch (0)
#ifndef RO_RUNLEN
#define RO_RUNLEN 0
#endif
// per-channel (slot, lo, hi, zero_upto) as one shared-memory int4 (1) or
// from the kernel-parameter bank (0)
#ifndef RO_CHI
#define RO_CHI 1
#endif
// experiment: the channel's zero_upto kept in a register (from S.chi)
#ifndef RO_ZU_REG
#define RO_ZU_REG 1
#endif
// experiment: 32-bit sub-block table index (slots * sub-blocks < 2^31, checked on the host)
#ifndef RO_SUB32
#define RO_SUB32 1
#endif
// experiment: the channel loop unrolled by two
#ifndef RO_CH_UNROLL2
#define RO_CH_UNROLL2 0
#endif

namespace ro {

namespace {

constexpr int kWarps = RO_WARPS;
constexpr int kBlock = 32 * kWarps;  // default 4 warps on a 16x8 pixel tile
constexpr int kTileW = RO_TILE_W;
constexpr int kTileH = RO_TILE_H;
#ifndef RO_PACK_W
#define RO_PACK_W 8
#endif
constexpr int kPackW = RO_PACK_W, kPackH = 32 / RO_PACK_W;  // warp packet (8x4)
constexpr int kPPT = (kTileW / kPackW) * (kTileH / kPackH);  // packets per tile
static_assert(kTileW % kPackW == 0 && kTileH % kPackH == 0 && kPPT % kWarps == 0,
              "tile shape");
constexpr int kFastDepth = 6;  // longest channel-0 descent handled in parallel
constexpr int kRunBytes = RO_RUNLEN ? 8 : 4;  // per-thread brick-run record
constexpr double kClampHi = 1.0 - 1e-9;
constexpr double kTwo52 = 4503599627370496.0;

struct FrameSmem {
    double tf_x[RO_MAX_CH][RO_MAX_TF_POINTS];
    double tf_rgba[RO_MAX_CH][RO_MAX_TF_POINTS][4];
    // per segment i: fl(x[i+1] - x[i]) and fl(c[i+1] - c[i]) -- the exact
    // intermediate values of the reference's (v - x0) / (x1 - x0) and lerps
    double tf_dx[RO_MAX_CH][RO_MAX_TF_POINTS];
    double tf_drgba[RO_MAX_CH][RO_MAX_TF_POINTS][4];
    // first segment i with x[i+1] >= j, for integer j (search start)
    uint8_t tf_seg[RO_MAX_CH][256];
    uint16_t empty_below[RO_MAX_CH][256];
    int32_t ptoff[RO_MAX_CH][RO_MAX_LEVELS];  // pt_offsets[slot*k + lev]
    int32_t lvl_off[RO_MAX_LEVELS + 1];
    double lod_thr[RO_MAX_LEVELS + 1];
    double step_tab[RO_MAX_LEVELS];
    double dimd[RO_MAX_LEVELS][3];
    int32_t maxlev[RO_MAX_LEVELS];
    int32_t dt_tab[RO_MAX_LEVELS];
    int32_t grids[RO_MAX_LEVELS][3];
    int32_t slot[RO_MAX_CH], lo[RO_MAX_CH], hi[RO_MAX_CH], np[RO_MAX_CH];
    // largest integer value v with opacity(u) == 0 for every u <= v
    int32_t zero_upto[RO_MAX_CH];
    int4 chi[RO_MAX_CH];  // (slot, lo, hi, zero_upto): one LDS.128 per channel visit
    uint32_t nest;        // bit l: dims[l] == 2 dims[l + 1] on every axis
    unsigned long long red[RO_NUM_COUNTERS];
    // frame constants kept out of registers
    double bm1[3];      // brick extent - 1, as fp64 (the reference's B - 1.0)
    double side_d;      // 2^depth
    double inv_t0;      // 1 / t0 (exact when t0 is a power of two)
    int32_t t0_pow2;
    int32_t eps_i;      // (mx - mn) <= eps_h  <=>  (mx - mn) <= eps_i
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
    int32_t *tile_counter;   // persistent-CTA work counter (zeroed per launch)
    const uint8_t *sub_max;  // [S*nsb] dilated 8^3 sub-block maxima (optional)
    int32_t nsb;             // sub-blocks per slot
    const uint8_t *node_fast;    // [num_nodes] k_classify outputs (optional)
    const uint64_t *node_path;
};

__device__ __forceinline__ double lerp(double a, double b, double t) {
    return a + (b - a) * t;
}

// exact non-negative int -> double on the fp64 pipe
__device__ __forceinline__ double i2d(int v) {
    return __hiloint2double(0x43300000, v) - kTwo52;
}

// (int)x for 0 <= x < 2^31 on the fp64 pipe: x + 2^52 rounded toward zero
// is 2^52 + trunc(x) exactly (ulp 1 in [2^52, 2^53)); its low word is the
// integer.  Same value as the F2I.F64.TRUNC conversion, without the
// conversion unit's latency.
__device__ __forceinline__ int d2i_nn(double x) {
    return __double2loint(__dadd_rz(x, kTwo52));
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
__device__ __forceinline__ int lod_raw(double t, double t0, double inv_t0, bool t0_pow2,
                                       const FrameSmem &S) {
    const double ratio = t0_pow2 ? t * inv_t0 : t / t0;  // exact when t0 = 2^k
    if (ratio < 1.0) return 0;
    // ratio >= 1 (or +inf): the unbiased exponent field is ilogb(ratio)
    const int e = ((__double2hiint(ratio) >> 20) & 0x7FF) - 1023;
    if (e >= RO_MAX_LEVELS - 1) return RO_MAX_LEVELS - 1;
    int lev = e;
    if (ratio >= S.lod_thr[lev + 1]) lev += 1;
    else if (lev >= 1 && ratio < S.lod_thr[lev]) lev -= 1;
    return lev;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// kernels.py:119-133
__device__ __forceinline__ void tf_eval(const FrameSmem &S, int ci, double v,
                                        double &r, double &g, double &b,
                                        double &a) {
    r = g = b = a = 0.0;
    const int n = S.np[ci];
    if (n < 2 || v < S.tf_x[ci][0] || v > S.tf_x[ci][n - 1]) return;
    // the reference takes the first segment with x0 <= v <= x1; with strictly
    // increasing knots that is the first i with x[i+1] >= v
    int i = S.tf_seg[ci][d2i_nn(v)];
    while (i < n - 2 && S.tf_x[ci][i + 1] < v) ++i;
    const double dxs = S.tf_dx[ci][i];
    const double t = (dxs == 0.0) ? 0.0 : (v - S.tf_x[ci][i]) / dxs;
    r = S.tf_rgba[ci][i][0] + S.tf_drgba[ci][i][0] * t;
    g = S.tf_rgba[ci][i][1] + S.tf_drgba[ci][i][1] * t;
    b = S.tf_rgba[ci][i][2] + S.tf_drgba[ci][i][2] * t;
    a = S.tf_rgba[ci][i][3] + S.tf_drgba[ci][i][3] * t;
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
// Fire-and-forget (RED.MIN): the lane never waits on the L2 round trip;
// feedback.cu finds the touched entries by scanning the key arrays.
__device__ __forceinline__ void request(unsigned long long *keys, int32_t *, int32_t *,
                             int32_t entry, unsigned long long key) {
    atomicMin(keys + entry, key);
}

// Brick coordinates of one level at the current sample position:
// P = fl(p * dim) (kernels.py:179 numerator), c = int(P / b) = int(P) >> lb.
// per-thread shared-memory arrays addressed by 32-bit shared addresses
// computed once (1) or through generic pointers (0)
#ifndef RO_SMEM_ASM
#define RO_SMEM_ASM 0
#endif
// Experiment: stage the two z-slices of a brick a warp's taps
// need into shared memory with one TMA bulk copy (cp.async.bulk + mbarrier)
// and read the taps from there, instead of eight L1-cached gathers per lane
#ifndef RO_TMA_STAGE
#define RO_TMA_STAGE 0
#endif
#ifndef RO_STATS
#define RO_STATS 0
#endif
#ifndef RO_LOD_INC
#define RO_LOD_INC 1
#endif
// the empty-space skip loop keeps the incremental LOD state too
#ifndef RO_SKIP_LOD_INC
#define RO_SKIP_LOD_INC 1
#endif
#ifndef RO_LP2_LOCAL
#define RO_LP2_LOCAL 0
#endif
#ifndef RO_UNROLL4
#define RO_UNROLL4 0
#endif
#ifndef RO_NEST_DERIVE
#define RO_NEST_DERIVE 0
#endif
#ifndef RO_LP_NOP
#define RO_LP_NOP 0  // 1: taps recompute P = p * dim (3 DMUL, rare) instead of keeping it live
#endif
struct LevelPos {
    int lev;
#if !RO_LP_NOP
    double P[3];
#endif
#if RO_NEST_DERIVE
    int ip[3];  // int(P): coarser exactly-halving levels derive from it by shifts
#endif
    int cb[3];
    int local;  // (cz*gy + cy)*gx + cx
    int sub;    // 4^3 sub-block of int(P) inside the brick (ro_state.sub_max index)
};

__device__ __forceinline__ void level_pos(LevelPos &lp, int lev, double px, double py,
                                          double pz, const FrameSmem &S, int lbx,
                                          int lby, int lbz) {
    lp.lev = lev;
    const double p3[3] = {px, py, pz};
    const int lb3[3] = {lbx, lby, lbz};
    int sb[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double P = p3[a] * S.dimd[lev][a];
#if !RO_LP_NOP
        lp.P[a] = P;
#endif
        const int ip = d2i_nn(P);
#if RO_NEST_DERIVE
        lp.ip[a] = ip;
#endif
        int c = ip >> lb3[a];
        const int g = S.grids[lev][a];
        lp.cb[a] = c > g - 1 ? g - 1 : c;
        // local integer coordinate (>= B only on a clamped edge brick)
        sb[a] = min(ip - (lp.cb[a] << lb3[a]), (1 << lb3[a]) - 1) >> RO_SUB_LOG;
    }
    lp.local = (lp.cb[2] * S.grids[lev][1] + lp.cb[1]) * S.grids[lev][0] + lp.cb[0];
    // (bricks smaller than a sub-block have no sub_max table: lp.sub unused)
    lp.sub = (((sb[2] << max(lby - RO_SUB_LOG, 0)) + sb[1]) << max(lbx - RO_SUB_LOG, 0)) + sb[0];
}

#if RO_NEST_DERIVE
// Position at a coarser level `lev` from a finer one when every level in
// between halves the dims exactly (dims[l] == 2 dims[l+1] on every axis):
// fl(p * dims[l]) = 2^j fl(p * dims[l + j]) exactly (power-of-two scaling
// commutes with rounding), so int(P) at lev is int(P) at src.lev >> j.  The
// fp64 coordinates P themselves are left unset (P[0] = -1): taps_of, the
// only reader, computes them on the rare sample that loads taps.
__device__ __forceinline__ void level_pos_from(LevelPos &lp, int lev, const LevelPos &src,
                                               const FrameSmem &S, int lbx, int lby, int lbz) {
    const int j = lev - src.lev;
    lp.lev = lev;
#if !RO_LP_NOP
    lp.P[0] = -1.0;
#endif
    const int lb3[3] = {lbx, lby, lbz};
    int sb[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int ip = src.ip[a] >> j;
        lp.ip[a] = ip;
        const int c = ip >> lb3[a];
        const int g = S.grids[lev][a];
        lp.cb[a] = c > g - 1 ? g - 1 : c;
        sb[a] = min(ip - (lp.cb[a] << lb3[a]), (1 << lb3[a]) - 1) >> RO_SUB_LOG;
    }
    lp.local = (lp.cb[2] * S.grids[lev][1] + lp.cb[1]) * S.grids[lev][0] + lp.cb[0];
    lp.sub = (((sb[2] << max(lby - RO_SUB_LOG, 0)) + sb[1]) << max(lbx - RO_SUB_LOG, 0)) + sb[0];
}
#endif

#ifndef RO_META_HINT
#define RO_META_HINT 0
#endif
// experiment knob: L1::evict_last on octree-word and page-table loads
__device__ __forceinline__ int ld_meta(const int32_t *p) {
#if RO_META_HINT
    int v;
    asm("ld.global.nc.L1::evict_last.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ uint4 ld_meta4(const uint4 *p) {
#if RO_META_HINT
    uint4 v;
    asm("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

#if RO_SMEM_ASM
__device__ __forceinline__ int lds32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v));
}
#endif

// word of channel slot s (0..3) from a node's four-slot vector: two
// predicated selects, no branch chain
__device__ __forceinline__ uint32_t word_of_slot(const uint4 &wv, int s) {
    const uint32_t lo = (s & 1) ? wv.y : wv.x;
    const uint32_t hi = (s & 1) ? wv.w : wv.z;
    return (s & 2) ? hi : lo;
}

// kernels.py:518-549: nearest resident level in the node's mask, coarser
// first on ties; returns (level, cache slot) or level -1.  The position of
// the chosen level is left in `lp2` (a one-entry cache across channels).
__device__ __forceinline__ int2 substitute(const int32_t *__restrict__ pt, const FrameSmem &S, int ci,
                                int lev, int k, uint32_t mask, double px, double py,
                                double pz, int lbx, int lby, int lbz, LevelPos &lp2,
                                int32_t &e_out, const LevelPos &lp) {
    // Visit the levels present in the mask in the reference's order
    // (distance 1, 2, ...; the coarser one first on a tie) by taking the
    // nearest remaining set bit on either side, instead of scanning every
    // candidate distance.
    uint32_t mk = mask & ((1u << k) - 1u) & ~(1u << lev);
    while (mk) {
        const uint32_t above = mk >> (lev + 1);
        const uint32_t below = mk & ((1u << lev) - 1u);
        const int da = above ? __ffs(above) : 64;
        const int db = below ? lev - (31 - __clz(below)) : 64;
        const int cand = da <= db ? lev + da : lev - db;
        if (lp2.lev != cand) {
#if RO_NEST_DERIVE
            const uint32_t span = ((1u << cand) - 1u) & ~((1u << lev) - 1u);  // levels lev..cand-1
            if (cand > lev && lp.lev == lev && (S.nest & span) == span)
                level_pos_from(lp2, cand, lp, S, lbx, lby, lbz);
            else
#endif
                level_pos(lp2, cand, px, py, pz, S, lbx, lby, lbz);
        }
        RO_ASSERT(cand >= 0 && cand < RO_MAX_LEVELS && lp2.local >= 0);
        const int32_t e2 = S.ptoff[ci][cand] + lp2.local;
        const int pv2 = ld_meta(pt + e2);
        if (pv2 >= 0) {
            e_out = e2;
            return make_int2(cand, pv2);
        }
        mk &= ~(1u << cand);
    }
    return make_int2(-1, -1);
}

// trilinear tap addresses + weights inside one brick (kernels.py:136-174)
struct Taps {
    int o;                // offset of tap (x0, y0, z0) inside the brick
    double tx, ty, tz;
};

// The upper taps are read unclamped at x0+1 / y0+1 / z0+1: the reference
// clamps them to B-1 only when x0 = B-1, and then f = B-1 exactly, so the
// weight is 0 and lerp(a, b, 0) = a + (b - a) * 0 = a for any finite b.  The
// read may touch the next row / slice / brick -- the cache carries one brick
// of tail padding (resoct.h) -- but never changes a result.
__device__ __forceinline__ void taps_of(Taps &tp, const LevelPos &lp, double px, double py,
                                        double pz, int bx, int by, int bz, const FrameSmem &S) {
    const int B[3] = {bx, by, bz};
#if RO_LP_NOP || RO_NEST_DERIVE
    const double p3[3] = {px, py, pz};
#else
    (void)px, (void)py, (void)pz;
#endif
#if RO_NEST_DERIVE && !RO_LP_NOP
    const bool derived = lp.P[0] < 0.0;  // level_pos_from left P unset
#endif
    int i0[3];
    double tw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // lx = P - c*B exactly; fx = lx - 0.5 exactly; clamped to [0, B-1]
#if RO_LP_NOP
        const double P = p3[a] * S.dimd[lp.lev][a];  // the same rounding as level_pos
#elif RO_NEST_DERIVE
        const double P = derived ? p3[a] * S.dimd[lp.lev][a] : lp.P[a];
#else
        const double P = lp.P[a];
#endif
        double f = (P - i2d(lp.cb[a] * B[a])) - 0.5;
        if (f < 0.0) f = 0.0;
        const double bm1 = (double)(B[a] - 1);  // a constant for compile-time bricks
        if (f > bm1) f = bm1;
        const int c0 = d2i_nn(f);
        i0[a] = c0;
        tw[a] = f - i2d(c0);
    }
    tp.o = (i0[2] * by + i0[1]) * bx + i0[0];
    tp.tx = tw[0];
    tp.ty = tw[1];
    tp.tz = tw[2];
}

__device__ __forceinline__ double trilerp(const int v[8], const Taps &tp) {
    const double c00 = lerp(i2d(v[0]), i2d(v[1]), tp.tx);
    const double c10 = lerp(i2d(v[2]), i2d(v[3]), tp.tx);
    const double c01 = lerp(i2d(v[4]), i2d(v[5]), tp.tx);
    const double c11 = lerp(i2d(v[6]), i2d(v[7]), tp.tx);
    return lerp(lerp(c00, c10, tp.ty), lerp(c01, c11, tp.ty), tp.tz);
}

#ifndef RO_TAP_HINT
#define RO_TAP_HINT 0
#endif
// experiment knob: L1 eviction priority of the trilinear tap loads
// (0: plain ld.global.nc; 1: L1::evict_first; 2: L1::no_allocate)
__device__ __forceinline__ uint8_t ld_tap(const uint8_t *p) {
#if RO_TAP_HINT == 1
    unsigned short v;
    asm("ld.global.nc.L1::evict_first.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return (uint8_t)v;
#elif RO_TAP_HINT == 2
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return (uint8_t)v;
#else
    return __ldg(p);
#endif
}

// BX/BY = compile-time brick extent (0: runtime) so the eight tap offsets
// become load immediates off one base address
template <int BX, int BY>
__device__ __forceinline__ void load_taps(int v[8], const uint8_t *__restrict__ p, int bx,
                                          int bxy) {
    const int sx = BX ? BX : bx;
    const int sxy = BX ? BX * BY : bxy;
    v[0] = ld_tap(p);
    v[1] = ld_tap(p + 1);
    v[2] = ld_tap(p + sx);
    v[3] = ld_tap(p + sx + 1);
    v[4] = ld_tap(p + sxy);
    v[5] = ld_tap(p + sxy + 1);
    v[6] = ld_tap(p + sxy + sx);
    v[7] = ld_tap(p + sxy + sx + 1);
}

// audit value from the fully resident reference paging (kernels.py:707-723)
__device__ double ref_value(const ro_frame &F, const FrameSmem &S, int ci, int lev,
                            double qx, double qy, double qz, int bx, int by, int bz,
                            int lbx, int lby, int lbz, int bvox) {
    LevelPos lp;
    level_pos(lp, lev, qx, qy, qz, S, lbx, lby, lbz);
    const int rp = F.ref_pt[S.ptoff[ci][lev] + lp.local];
    if (rp < 0) return -1.0;
    Taps tp;
    taps_of(tp, lp, qx, qy, qz, bx, by, bz, S);
    int v[8];
    load_taps<0, 0>(v, F.ref_cache + (int64_t)rp * bvox + tp.o, bx, bx * by);
    return trilerp(v, tp);
}

// one sampled channel: taps + trilinear + TF; side effects on the usage
// mask / histogram / per-pixel brick switches (kernels.py:660-681)
struct SampleCtx {
    LevelPos lp;   // brick coordinates of the desired level (probe)
    Taps tp;       // tap offsets / weights of tp_lev
    int tp_lev;
    LevelPos lp2;  // the last substitute level (kernels.py:518-549)
};

// Per-frame node classes for the residency walk (kernels.py:444-517).
// A node is "plain" for channel ci when the reference's walk would just step
// through it: valid metadata, not transparent under ci's TF (_is_empty_meta),
// not homogeneous, and some level resident (mask != 0).
//   path[x] byte ci = the plain bits of channel ci along the root -> x path
//     (bit a = the depth-a ancestor, bit depth(x) = x itself) and, with at
//     most 4 channels, byte 4 + ci the same for the ZERO bits (valid and
//     transparent: the walk ends there);
//   fast[x] bit 0 = x is plain for every channel and x and all its ancestors
//     are plain for channel 0 (bit 1: the latter alone).
// One kernel, top-down: CTA b owns the subtree under depth-s node b and
// walks it level by level (a node's classes = its parent's + its own
// words), so every node reads one parent entry instead of its ancestors.
// A sample whose depth-dt node is fast goes straight to the page-table probes
// at dt (channel 0 walks d0..dt through plain nodes, every later channel
// visits only the plain dt node: dt - d0 + n_ch visits, no request events).
// Any other sample reads path[] of its dt node once and every channel steps
// through the plain run of its byte from the cursor, resuming the exact walk
// at the first non-plain node (or probing at dt) -- the reference's visits
// and request events, one 8-byte load instead of a word load per plain node
// (and, up to 4 channels, none for a ZERO terminal).
// path[] needs D <= 7 (8 depths per byte).
__global__ void __launch_bounds__(256) k_classify(const __grid_constant__ ro_frame F,
                                                  const uint32_t *__restrict__ words, int m,
                                                  int D, int s, uint8_t *__restrict__ fast,
                                                  uint64_t *__restrict__ path) {
    __shared__ uint16_t eb[RO_MAX_CH][256];
    __shared__ unsigned long long s_root;  // path class of the subtree root's parent
    __shared__ uint32_t s_chain;           // channel 0 plain along it
    const int n_ch = F.n_ch;
    const int tid = threadIdx.x;
    for (int i = tid; i < n_ch * 256; i += blockDim.x)
        eb[i >> 8][i & 255] = F.ch[i >> 8].empty_below[i & 255];
    __syncthreads();
    const int eps_i = F.eps_h >= 255.0 ? 255 : (F.eps_h < 0.0 ? -1 : (int)F.eps_h);
    const uint32_t all = (1u << n_ch) - 1;
    const bool zbits = n_ch <= 4;
    // bit ci: plain for channel ci; bit 8 + ci: ZERO for channel ci
    auto own_of = [&](int64_t node) -> uint32_t {
        uint32_t r = 0;
        for (int ci = 0; ci < n_ch; ++ci) {
            const uint32_t w = __ldg(words + node * m + F.ch[ci].slot);
            const int mn = (w >> 16) & 0xFF, mx = (int)(w >> 24);
            const bool valid = !(mn == 255 && mx == 0);       // else INVALID: metadata request
            const bool zero = valid && mx < (int)eb[ci][mn];   // K_ZERO
            const bool p = valid && !zero && mx - mn > eps_i &&  // K_CONST
                           (w & 0xFFFFu) != 0;                    // K_MISSU
            r |= ((uint32_t)p << ci) | ((uint32_t)zero << (8 + ci));
        }
        return r;
    };
    // path class of a node at depth d from its parent's and its own bits
    auto compose = [&](uint64_t pp, uint32_t own, int d) -> uint64_t {
        for (int ci = 0; ci < n_ch; ++ci) {
            pp |= (uint64_t)((own >> ci) & 1u) << (8 * ci + d);
            if (zbits) pp |= (uint64_t)((own >> (8 + ci)) & 1u) << (32 + 8 * ci + d);
        }
        return pp;
    };
    const int side_s = 1 << s;
    const int sx = blockIdx.x & (side_s - 1), sy = (blockIdx.x >> s) & (side_s - 1),
              sz = blockIdx.x >> (2 * s);
    if (tid == 0) {  // the root's ancestors (shared with other subtrees: same values)
        uint64_t pc = 0;
        uint32_t ch0 = 1;
        for (int a = 0; a < s; ++a) {
            const int sh = s - a;
            const int64_t node = level_offset(a) +
                                 ((((int64_t)(sz >> sh) << a) + (sy >> sh)) << a) + (sx >> sh);
            const uint32_t o = own_of(node);
            pc = compose(pc, o, a);
            ch0 &= o & 1u;
            fast[node] = (uint8_t)(((o & 0xFFu) == all && ch0) | (ch0 << 1));
            if (path) path[node] = pc;
        }
        s_root = pc;
        s_chain = ch0;
    }
    __syncthreads();
    for (int d = s; d <= D; ++d) {
        const int e = d - s, n = 1 << (3 * e), em = (1 << e) - 1;
        for (int i = tid; i < n; i += blockDim.x) {
            const int gx = (sx << e) + (i & em), gy = (sy << e) + ((i >> e) & em),
                      gz = (sz << e) + (i >> (2 * e));
            const int64_t x = level_offset(d) + ((((int64_t)gz << d) + gy) << d) + gx;
            uint64_t pp;
            uint32_t ch0;
            if (e == 0) {
                pp = s_root;
                ch0 = s_chain;
            } else {  // the parent was written by this CTA one level up
                const int64_t par = level_offset(d - 1) +
                                    ((((int64_t)(gz >> 1) << (d - 1)) + (gy >> 1)) << (d - 1)) +
                                    (gx >> 1);
                ch0 = ((uint32_t)fast[par] >> 1) & 1u;
                pp = path ? path[par] : 0;
            }
            const uint32_t o = own_of(x);
            ch0 &= o & 1u;
            fast[x] = (uint8_t)(((o & 0xFFu) == all && ch0) | (ch0 << 1));
            if (path) path[x] = compose(pp, o, d);
        }
        __syncthreads();  // this level's classes visible to the next level's threads
    }
}

__host__ __device__ constexpr int ilog2c(int v) { return v > 1 ? 1 + ilog2c(v >> 1) : 0; }

// BX / BY / BZ: compile-time brick extent (0: runtime) -- tap offsets, brick
// and sub-block coordinates then use constant shifts and masks
template <int MODE, bool CHECK, int BX, int BY, int BZ>
#ifndef RO_CTAS_PER_SM
#define RO_CTAS_PER_SM (RO_MINB * 4 / kWarps)
#endif
#ifdef RO_MAXNREG  // experiment knob: an explicit register cap instead of a CTA count
__global__ void __maxnreg__(RO_MAXNREG)
#else
__global__ void __launch_bounds__(kBlock, RO_CTAS_PER_SM)
#endif
k_raycast(const __grid_constant__ ro_frame F, const __grid_constant__ RayArgs A) {
    __shared__ FrameSmem S;
#if RO_TMA_STAGE
    // per warp: the staged slab (2 z-slices of a brick, + slack for the
    // weight-0 upper taps that step past it) and its mbarrier
    constexpr int kSlab = 2 * (BX ? BX : 32) * (BY ? BY : 32);
    __shared__ alignas(128) uint8_t stage[kWarps][kSlab + 128];
    __shared__ alignas(8) unsigned long long stage_bar[kWarps];
    uint32_t stage_phase = 0;
    if ((threadIdx.x & 31) == 0) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar[threadIdx.x >> 5]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
#endif
    extern __shared__ int32_t dyn[];  // per-thread channel state
    const int tid = threadIdx.x;
    const int n_ch = F.n_ch;
    const int k = A.L.k;
    const int m = A.L.m;

    // ---- stage frame tables ----
    for (int i = tid; i < n_ch * RO_MAX_TF_POINTS; i += kBlock) {
        const int c = i / RO_MAX_TF_POINTS, p = i % RO_MAX_TF_POINTS;
        S.tf_x[c][p] = F.ch[c].tf_x[p];
        for (int q = 0; q < 4; ++q) S.tf_rgba[c][p][q] = F.ch[c].tf_rgba[p][q];
    }
    for (int i = tid; i < n_ch * RO_MAX_TF_POINTS; i += kBlock) {
        const int c = i / RO_MAX_TF_POINTS, p = i % RO_MAX_TF_POINTS;
        const bool seg = p + 1 < F.ch[c].npoints;
        S.tf_dx[c][p] = seg ? F.ch[c].tf_x[p + 1] - F.ch[c].tf_x[p] : 0.0;
        for (int q = 0; q < 4; ++q)
            S.tf_drgba[c][p][q] = seg ? F.ch[c].tf_rgba[p + 1][q] - F.ch[c].tf_rgba[p][q] : 0.0;
    }
    for (int i = tid; i < n_ch * 256; i += kBlock) {
        const int c = i / 256, j = i % 256;
        S.empty_below[c][j] = F.ch[c].empty_below[j];
        S.tf_seg[c][j] = F.ch[c].tf_seg[j];
    }
    for (int i = tid; i < n_ch * RO_MAX_LEVELS; i += kBlock) {
        const int c = i / RO_MAX_LEVELS, l = i % RO_MAX_LEVELS;
        S.ptoff[c][l] = l < k ? (int32_t)A.L.pt_off[F.ch[c].slot * k + l] : 0;
    }
    if (tid <= RO_MAX_LEVELS) {
        S.lvl_off[tid] = tid <= 10 ? (int32_t)level_offset(tid) : 0;
        S.lod_thr[tid] = F.lod_threshold[tid];
    }
    if (tid < RO_MAX_LEVELS) {
        S.step_tab[tid] = F.step_tab[tid];
        S.maxlev[tid] = F.maxlev_tab[tid];
        S.dt_tab[tid] = F.dt_tab[tid];
        for (int a = 0; a < 3; ++a) {
            S.dimd[tid][a] = (double)A.L.dims[tid][a];
            S.grids[tid][a] = A.L.grids[tid][a];
        }
    }
    if (tid < RO_MAX_CH) {
        S.slot[tid] = F.ch[tid].slot;
        S.lo[tid] = F.ch[tid].lo;
        S.hi[tid] = F.ch[tid].hi;
        S.np[tid] = F.ch[tid].npoints;
        // leading zero-opacity range of the TF (ro_pack_frame)
        S.zero_upto[tid] = F.ch[tid].zero_upto;
        S.chi[tid] = make_int4(F.ch[tid].slot, F.ch[tid].lo, F.ch[tid].hi, F.ch[tid].zero_upto);
    }
    if (tid < RO_NUM_COUNTERS) S.red[tid] = 0;
    if (tid == 0) {
        S.bm1[0] = A.L.bx - 1.0;
        S.bm1[1] = A.L.by - 1.0;
        S.bm1[2] = A.L.bz - 1.0;
        S.side_d = (double)(1 << A.L.depth);
        uint32_t nest = 0;
        for (int l = 0; l + 1 < k; ++l)
            if (A.L.dims[l][0] == 2 * A.L.dims[l + 1][0] &&
                A.L.dims[l][1] == 2 * A.L.dims[l + 1][1] &&
                A.L.dims[l][2] == 2 * A.L.dims[l + 1][2])
                nest |= 1u << l;
        S.nest = nest;
        S.inv_t0 = 1.0 / F.t0;
        S.t0_pow2 = (__double_as_longlong(F.t0) & 0x000FFFFFFFFFFFFFll) == 0;
        S.eps_i = F.eps_h >= 255.0 ? 255 : (F.eps_h < 0.0 ? -1 : (int)F.eps_h);
    }
    // per-thread arrays: [ci*kBlock + tid]
    const int kChStride = n_ch * kBlock;
    // per channel: the current brick run (kernels.py:672-676 prev_brick) as
    // entry | level << 32 | fetch count << 36; the histogram is credited
    // when the run ends, not per fetch
    // (RO_RUNLEN = 0: only the 32-bit entry, 4 bytes per thread and channel)
    unsigned long long *run = reinterpret_cast<unsigned long long *>(dyn);  // n_ch
    int32_t *last_breq = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(dyn) +
                                                     kRunBytes * kChStride);  // n_ch
    int32_t *last_mreq = last_breq + kChStride;       // n_ch
    uint32_t *hist_t = reinterpret_cast<uint32_t *>(last_mreq + kChStride);
    for (int i = 0; i < n_ch * k; ++i) hist_t[i * kBlock + tid] = 0;
#if RO_SMEM_ASM
    // this thread's column of each per-thread array; element i of a
    // channel-indexed array sits at + (i * kBlock) * 4
    const uint32_t s_prev = (uint32_t)__cvta_generic_to_shared(run) + 4u * tid;
    const uint32_t s_breq = (uint32_t)__cvta_generic_to_shared(last_breq) + 4u * tid;
    const uint32_t s_hist = (uint32_t)__cvta_generic_to_shared(hist_t) + 4u * tid;
#endif
    const int lane = tid & 31;
    [[maybe_unused]] const int warp = tid >> 5;
    const int tiles_x = (F.width + kTileW - 1) / kTileW;
    // per-thread work counters (32-bit: a thread's share stays far below 2^32)
    uint32_t c_steps = 0, c_eval = 0, c_skip = 0, c_viol = 0, c_live = 0;
#if RO_STATS
    // instrumentation build only: counters[5..7] = probe misses, tap loads,
    // full TF evaluations
    uint32_t c_s5 = 0, c_s6 = 0, c_s7 = 0;
#define RO_STAT(v) (v) += 1
#else
#define RO_STAT(v) do { } while (0)
#endif

#if RO_PERSISTENT
    // Persistent CTAs: tables are staged once per CTA, then 16x8 pixel tiles
    // are pulled from a global counter in scanline order.
    __shared__ int s_tile;
    const int n_tiles = tiles_x * ((A.local_rows + kTileH - 1) / kTileH);
    while (true) {
    if (tid == 0) s_tile = atomicAdd(A.tile_counter, 1);
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile >= n_tiles) break;
#else
    __syncthreads();  // staged tables visible to every thread
    {
    const int tile = blockIdx.x;
#endif
    for (int wsub = warp; wsub < kPPT; wsub += kWarps) {
    for (int i = 0; i < n_ch; ++i) {
#if RO_RUNLEN
        run[i * kBlock + tid] = 0xFFFFFFFFull;
#else
        reinterpret_cast<int32_t *>(run)[i * kBlock + tid] = -1;
#endif
        last_breq[i * kBlock + tid] = -1;
        last_mreq[i * kBlock + tid] = -1;
    }

    // ---- pixel of this thread: warp = kPackW x kPackH packet ----
    const int x = (tile % tiles_x) * kTileW + (wsub % (kTileW / kPackW)) * kPackW +
                  (lane % kPackW);
    const int ly = (tile / tiles_x) * kTileH + (wsub / (kTileW / kPackW)) * kPackH +
                   lane / kPackW;
    const int tr = F.tile_rows;
    const int gy = ((ly / tr) * F.n_parts + F.part) * tr + (ly % tr);
    const bool active = x < F.width && ly < A.local_rows && gy < F.height;

    const int bx = BX ? BX : A.L.bx, by = BY ? BY : A.L.by, bz = BZ ? BZ : A.L.bz;
    const int lbx = BX ? ilog2c(BX) : __ffs(bx) - 1, lby = BY ? ilog2c(BY) : __ffs(by) - 1,
              lbz = BZ ? ilog2c(BZ) : __ffs(bz) - 1;
    const int bvox = bx * by * bz;
    const int D = A.L.depth;
    const bool vec4 = (m == 4);
    const double t0 = F.t0;
    // (mx - mn) <= eps_h  <=>  (mx - mn) <= floor(eps_h) for integer mx - mn
    const int64_t pix = (int64_t)gy * F.width + x;
    const int64_t lpix = (int64_t)ly * F.width + x;
    const unsigned long long key_hi = (unsigned long long)pix << 32;

    // camera.py:32-51, same operation order as the numpy code
    const double u = (((double)x + 0.5) / (double)F.width * 2.0 - 1.0) *
                     F.tan_half * F.aspect;
    const double v = (1.0 - ((double)gy + 0.5) / (double)F.height * 2.0) * F.tan_half;
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
#if RO_LOD_INC
    // t only grows along the ray, so the raw LOD level only grows: it is
    // recomputed when t / t0 reaches the next level's threshold
    int raw_c = 0;
    double next_thr = -1.0;
#endif
    [[maybe_unused]] int n_probe = 0;  // CHECK: cursor-resolved samples (max_samples)

    // Warp-uniform sample loop: lanes whose ray ended idle until the whole
    // packet is done, so the warp reconverges once per sample.
    bool alive = active && t < tfar && accA < F.early_alpha;
    while (__any_sync(0xffffffffu, alive)) {
        if (alive) {
            double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
            if (px < 0.0) px = 0.0;
            if (py < 0.0) py = 0.0;
            if (pz < 0.0) pz = 0.0;
            if (px > kClampHi) px = kClampHi;
            if (py > kClampHi) py = kClampHi;
            if (pz > kClampHi) pz = kClampHi;

#if RO_LOD_INC
            {
                const double ratio = S.t0_pow2 ? t * S.inv_t0 : t / t0;
                if (ratio >= next_thr) {
                    raw_c = lod_raw(t, t0, S.inv_t0, S.t0_pow2, S);
                    next_thr = S.lod_thr[raw_c + 1];
                }
            }
            const int raw = raw_c;
#else
            const int raw = lod_raw(t, t0, S.inv_t0, S.t0_pow2, S);
#endif
            double step = S.step_tab[raw];
            int jexp = S.maxlev[raw];
            const int dt_ = S.dt_tab[raw];

            SampleCtx sc;
            sc.lp.lev = -1;
            sc.tp_lev = -1;
            sc.lp2.lev = -1;
            // channel contributions, accumulated in the reference's channel
            // order the moment each channel resolves (kernels.py:637-681)
            double sR = 0.0, sG = 0.0, sB = 0.0, trans = 1.0;
            bool any_const = false;
            uint32_t zero_mask = 0;
            bool skippable = false;
            double skip_exit = -1.0;
            int end_depth = prev_depth;

            // usage mask / histogram / per-pixel brick switches of a sampled
            // channel (kernels.py:670-676)
#if RO_ZU_REG
            int zu_cur = 0;  // zero_upto of the channel being sampled (set per channel)
#define RO_ZU(ci) zu_cur
#else
#define RO_ZU(ci) S.zero_upto[ci]
#endif
            auto account = [&](int ci, int lev, int32_t e) {
#if !RO_RUNLEN && RO_SMEM_ASM
                {
                    const uint32_t a_pb = s_prev + ((uint32_t)ci * (kBlock * 4u));
                    if (e != lds32(a_pb)) {
                        sts32(a_pb, e);
                        pixreq += 1;
                        RO_ASSERT(e >= 0 && e < A.L.E);
                        A.required[e] = 1;
                    }
                    RO_ASSERT(lev >= 0 && lev < k && ci < n_ch);
                    const uint32_t a_h = s_hist + ((uint32_t)(ci * k + lev) * (kBlock * 4u));
                    sts32(a_h, lds32(a_h) + 1);
                    return;
                }
#elif !RO_RUNLEN
                int32_t &pb = reinterpret_cast<int32_t *>(run)[ci * kBlock + tid];
                if (e != pb) {
                    pb = e;
                    pixreq += 1;
                    RO_ASSERT(e >= 0 && e < A.L.E);
                    A.required[e] = 1;
                }
                RO_ASSERT(lev >= 0 && lev < k && ci < n_ch);
                hist_t[(ci * k + lev) * kBlock + tid] += 1;
                return;
#endif
                unsigned long long &r = run[ci * kBlock + tid];
                const unsigned long long rv = r;
                if ((uint32_t)rv == (uint32_t)e) {  // same brick: one more fetch
                    r = rv + (1ull << 36);
                    return;
                }
                const uint32_t cnt = (uint32_t)(rv >> 36);
                if (cnt) hist_t[(ci * k + (int)((rv >> 32) & 15)) * kBlock + tid] += cnt;
                RO_ASSERT(lev >= 0 && lev < k && ci < n_ch);
                r = (uint32_t)e | ((unsigned long long)lev << 32) | (1ull << 36);
                pixreq += 1;
                RO_ASSERT(e >= 0 && e < A.L.E);
                A.required[e] = 1;
            };
            // Sub-block skip: the taps with non-zero weight lie within one
            // voxel of int(local coordinate), i.e. inside the dilated 8^3
            // sub-block holding it; if that block's max is in the TF's
            // leading transparent range, so is the trilinear value (a convex
            // combination of those taps) and the channel adds exactly +0.
            auto sub_skip = [&](int ci, int slot_lin, const LevelPos &lp) -> bool {
#if RO_SUBMAX
                if (A.sub_max == nullptr) return false;
                RO_ASSERT(slot_lin >= 0 && slot_lin < A.L.num_slots && lp.sub >= 0 &&
                          lp.sub < A.nsb);
#if RO_SUB32
                return (int)__ldg(A.sub_max + (uint32_t)(slot_lin * A.nsb + lp.sub)) <=
                       RO_ZU(ci);
#else
                return (int)__ldg(A.sub_max + (int64_t)slot_lin * A.nsb + lp.sub) <=
                       RO_ZU(ci);
#endif
#else
                return false;
#endif
            };
            auto finish = [&](int ci, int slot_lin, const Taps &tp) {
                int tv[8];
                RO_ASSERT(slot_lin >= 0 && slot_lin < A.L.num_slots && tp.o >= 0 &&
                          tp.o + (int64_t)bx * by + bx + 1 < 2 * (int64_t)bvox);
                load_taps<BX, BY>(tv, A.cache + (int64_t)slot_lin * bvox + tp.o, bx, bx * by);
                RO_STAT(c_s6);
                // The trilinear value never exceeds the largest tap (every lerp
                // is a rounded convex combination).  If that tap lies in the
                // TF's leading zero-opacity range, r*a, g*a, b*a are +0 and
                // (1 - a) is 1: the channel adds exactly nothing -- skip it.
                const int mt = max(max(max(tv[0], tv[1]), max(tv[2], tv[3])),
                                   max(max(tv[4], tv[5]), max(tv[6], tv[7])));
                if (mt <= RO_ZU(ci)) return;
                RO_STAT(c_s7);
                const double val = trilerp(tv, tp);
                double r, g, b, a;
                tf_eval(S, ci, val, r, g, b, a);
                sR += r * a;
                sG += g * a;
                sB += b * a;
                trans *= (1.0 - a);
            };
            // taps + TF of the desired level (sc.lp holds it)
            auto sample_taps = [&](int ci, int lev, int slot_lin) {
                if (sc.tp_lev != lev) {
                    taps_of(sc.tp, sc.lp, px, py, pz, bx, by, bz, S);
                    sc.tp_lev = lev;
                }
                finish(ci, slot_lin, sc.tp);
            };
            // sample at the desired level (sc.lp already holds it; e = its entry)
            auto sample = [&](int ci, int lev, int slot_lin, int32_t e) {
                account(ci, lev, e);
                if (sub_skip(ci, slot_lin, sc.lp)) return;
                sample_taps(ci, lev, slot_lin);
            };
            // sample at a substitute level (lp2 holds it)
            auto sample2 = [&](int ci, int lev, int slot_lin, int32_t e, const LevelPos &lp2) {
                account(ci, lev, e);
                if (sub_skip(ci, slot_lin, lp2)) return;
                Taps t2;
                taps_of(t2, lp2, px, py, pz, bx, by, bz, S);
                finish(ci, slot_lin, t2);
            };

            // sample channel ci from `slot_lin` at level `lev` (any level)
            auto sample_at = [&](int ci, int lev, int slot_lin) {
                if (sc.lp.lev != lev) level_pos(sc.lp, lev, px, py, pz, S, lbx, lby, lbz);
                sample(ci, lev, slot_lin, S.ptoff[ci][lev] + sc.lp.local);
            };

            if (MODE == RO_MODE_PAGETABLE) {  // kernels.py:316-357
                // desired-level probe per channel; EMPTY entries are skippable
                // up to the exit of their brick box
                bool all_empty = true;
                skip_exit = 1e30;
#pragma unroll 1
                for (int ci = 0; ci < n_ch; ++ci) {
                    const int lev = clampi(raw, CH_LO(ci), CH_HI(ci));
                    if (sc.lp.lev != lev) level_pos(sc.lp, lev, px, py, pz, S, lbx, lby, lbz);
                    const int32_t e = S.ptoff[ci][lev] + sc.lp.local;
                    RO_ASSERT(e >= 0 && e < A.L.E);
                    const int pv = ld_meta(A.pt + e);
                    if (pv >= 0) {
                        all_empty = false;
                        sample(ci, lev, pv, e);
                    } else if (pv == RO_PT_EMPTY) {
                        zero_mask |= 1u << ci;
                        // c*B / float(dim): integer numerator, one IEEE division
                        const double ex = box_exit(
                            ox, oy, oz, dx, dy, dz, i2d(sc.lp.cb[0] * bx) / S.dimd[lev][0],
                            i2d(sc.lp.cb[1] * by) / S.dimd[lev][1],
                            i2d(sc.lp.cb[2] * bz) / S.dimd[lev][2],
                            i2d((sc.lp.cb[0] + 1) * bx) / S.dimd[lev][0],
                            i2d((sc.lp.cb[1] + 1) * by) / S.dimd[lev][1],
                            i2d((sc.lp.cb[2] + 1) * bz) / S.dimd[lev][2]);
                        if (ex < skip_exit) skip_exit = ex;
                    } else {
                        all_empty = false;
                        const unsigned long long key = key_hi | ev++;
                        int32_t &lb = last_breq[ci * kBlock + tid];
                        if (e != lb) {
                            lb = e;
                            request(A.brick_key, nullptr, nullptr, e, key);
                        }
                    }
                }
                skippable = all_empty;
            } else if (MODE == RO_MODE_CLASSIC) {  // kernels.py:359-429
                // per channel, a root-to-target descent of the classic octree
                // (node depth d <-> level cls_depth - d, one brick per node)
                const int CD = F.cls_depth;
                const double cside = (double)(1 << CD);
                const int qx = d2i_nn(px * cside), qy = d2i_nn(py * cside),
                          qz = d2i_nn(pz * cside);
                bool all_empty = true;
                int deep_d = -1, dix = 0, diy = 0, diz = 0;
#pragma unroll 1
                for (int ci = 0; ci < n_ch; ++ci) {
                    const int slot = CH_SLOT(ci);
                    const int lev = clampi(raw, CH_LO(ci), CH_HI(ci));
                    const int d_target = CD - lev > 0 ? CD - lev : 0;
                    int last_slot = -1, last_lev = -1;
                    for (int d = 0;; ++d) {
                        c_steps += 1;
                        const int sh = CD - d;
                        const int ix = qx >> sh, iy = qy >> sh, iz = qz >> sh;
                        const int local = (((iz << d) + iy) << d) + ix;
                        const int nidx = S.lvl_off[d] + local;
                        const int mn = __ldg(F.cls_min + nidx * m + slot);
                        const int mx = __ldg(F.cls_max + nidx * m + slot);
                        if (mx < (int)S.empty_below[ci][mn]) {  // K_ZERO
                            zero_mask |= 1u << ci;
                            if (d > deep_d) { deep_d = d; dix = ix; diy = iy; diz = iz; }
                            break;
                        }
                        const int lev_d = CD - d;
                        const int32_t e = S.ptoff[ci][lev_d] + local;  // grid 2^d per axis
                        A.required[e] = 1;
                        RO_ASSERT(e >= 0 && e < A.L.E);
                    const int pv = ld_meta(A.pt + e);
                        if (pv < 0) {
                            const unsigned long long key = key_hi | ev++;
                            int32_t &lb = last_breq[ci * kBlock + tid];
                            if (e != lb) {
                                lb = e;
                                request(A.brick_key, nullptr, nullptr, e, key);
                            }
                            // descent blocked: deepest resident ancestor
                            if (last_slot >= 0) sample_at(ci, last_lev, last_slot);
                            all_empty = false;
                            break;
                        }
                        last_slot = pv;
                        last_lev = lev_d;
                        if (d == d_target) {
                            sample_at(ci, lev_d, pv);
                            all_empty = false;
                            break;
                        }
                    }
                }
                if (all_empty && deep_d >= 0) {
                    skippable = true;
                    const double s = 1.0 / (double)(1 << deep_d);
                    skip_exit = box_exit(ox, oy, oz, dx, dy, dz, dix * s, diy * s, diz * s,
                                         (dix + 1) * s, (diy + 1) * s, (diz + 1) * s);
                }
            } else if (MODE == RO_MODE_REFERENCE) {  // kernels.py:301-314
#pragma unroll 1
                for (int ci = 0; ci < n_ch; ++ci) {
                    const int lev = clampi(raw, CH_LO(ci), CH_HI(ci));
                    if (sc.lp.lev != lev) level_pos(sc.lp, lev, px, py, pz, S, lbx, lby, lbz);
                    const int32_t e = S.ptoff[ci][lev] + sc.lp.local;
                    const int pv = __ldg(A.pt + e);
                    if (pv >= 0) sample(ci, lev, pv, e);
                }
            } else {
                // kernels.py:431-558 -- one cursor shared by all channels
                const int qx = d2i_nn(px * S.side_d), qy = d2i_nn(py * S.side_d),
                          qz = d2i_nn(pz * S.side_d);
                int d = prev_depth - 1;
                if (d < 0) d = 0;
                if (F.start_level < d) d = F.start_level;
                if (d > dt_) d = dt_;
                bool all_cz = true;
                int cur_node = -1;
                uint4 wv = make_uint4(0, 0, 0, 0);
                const int d0 = d;
                // pre-classified depth-dt node (k_classify): every
                // channel reaches dt through plain nodes and probes there;
                // otherwise its path class drives the walk below
                bool fast = false;
                uint64_t pcls = 0;
                if (A.node_fast != nullptr) {
                    const int sh = D - dt_;
                    const int lx = qx >> sh, lyy = qy >> sh, lz = qz >> sh;
                    const int leaf = S.lvl_off[dt_] + (((lz << dt_) + lyy) << dt_) + lx;
                    RO_ASSERT(leaf >= 0 && leaf < A.L.num_nodes);
                    fast = (__ldg(A.node_fast + leaf) & 1u) != 0;
                    if (fast) {
                        c_steps += dt_ - d0 + n_ch;
                        d = dt_;
                        if (vec4 && leaf != cur_node)
                            wv = ld_meta4(reinterpret_cast<const uint4 *>(A.words) + leaf);
                        cur_node = leaf;
                    } else if (A.node_path != nullptr) {
                        pcls = __ldg(A.node_path + leaf);
                    }
                }
#if RO_FAST_DESCENT
                // Channel 0 walks d0 -> dt through nodes known up front (the
                // ancestors of the sample position).  Load its word at every depth
                // at once and find the first node where it does anything but a
                // plain descent (valid, not empty, not constant, some level
                // resident); the generic loop below resumes exactly there.  Any
                // INVALID ancestor (it would issue a metadata request) stops the
                // fast walk at that node, so requests stay in program order.
                if (!fast && A.node_path == nullptr && dt_ - d0 >= 1 && dt_ - d0 <= kFastDepth) {
                    const int slot0 = CH_SLOT(0);
                    uint32_t pw[kFastDepth];
#pragma unroll
                    for (int i = 0; i < kFastDepth; ++i) {
                        const int dd = d0 + i;
                        pw[i] = 0;
                        if (dd < dt_) {
                            const int sh = D - dd;
                            const int nidx = S.lvl_off[dd] +
                                ((((qz >> sh) << dd) + (qy >> sh)) << dd) + (qx >> sh);
                            RO_ASSERT(nidx >= 0 && nidx < A.L.num_nodes);
                            pw[i] = __ldg(A.words + nidx * m + slot0);
                        }
                    }
                    int stop = dt_ - d0;
#pragma unroll
                    for (int i = kFastDepth - 1; i >= 0; --i) {
                        if (d0 + i < dt_) {
                            const uint32_t w = pw[i];
                            const int mn = (w >> 16) & 0xFF, mx = (w >> 24) & 0xFF;
                            const bool plain = !(mn == 255 && mx == 0) &&
                                               mx >= (int)S.empty_below[0][mn] &&
                                               mx - mn > S.eps_i && (w & 0xFFFFu) != 0;
                            if (!plain) stop = i;
                        }
                    }
                    c_steps += stop;
                    d = d0 + stop;
                }
#endif
                // Fast path, channels 0..3 at channel 0's level: issue their
                // page-table probes, then the sub-block maxima of the hits, as
                // independent loads ahead of the in-order channel loop (pure
                // reads of frame-constant state; every side effect stays in
                // the loop, in the reference's order)
                uint32_t pf_done = 0, pf_hit = 0, pf_skip = 0;
#if RO_PREFETCH
                if (fast) {
                    const int4 c0 = S.chi[0];
                    const int lev0 = clampi(raw, c0.y, c0.z);
                    level_pos(sc.lp, lev0, px, py, pz, S, lbx, lby, lbz);
                    int pv[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        pv[j] = -1;
                        if (j < n_ch) {
                            const int4 cj = S.chi[j];
                            if (clampi(raw, cj.y, cj.z) == lev0) {
                                pf_done |= 1u << j;
                                pv[j] = ld_meta(A.pt + S.ptoff[j][lev0] + sc.lp.local);
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (pv[j] >= 0) {
                            pf_hit |= 1u << j;
#if RO_SUBMAX
                            if (A.sub_max != nullptr &&
                                (int)__ldg(A.sub_max + (int64_t)pv[j] * A.nsb + sc.lp.sub) <=
                                    S.chi[j].w)
                                pf_skip |= 1u << j;
#endif
                        }
                    }
                }
#endif
                // one channel of the sample, in the reference's channel order
                auto channel = [&](const int ci) {
#if RO_CHI
                    const int4 chc = S.chi[ci];
#if RO_ZU_REG
                    zu_cur = chc.w;
#endif
#else
                    const int4 chc = make_int4(CH_SLOT(ci), CH_LO(ci), CH_HI(ci), 0);
#endif
                    const int slot = chc.x;
                    uint32_t mask;
                    if (fast) {
                        mask = (vec4 ? word_of_slot(wv, slot)
                                     : __ldg(A.words + cur_node * m + slot)) & 0xFFFFu;
                    } else {
                    // step through the plain run of ci's path class from the
                    // cursor: those visits neither request nor terminate
                    {
                        int t = d;
                        if (d < dt_) {
                            const uint32_t pm = (uint32_t)(pcls >> (8 * ci)) & 0xFFu;
                            t = d + __ffs(~(pm >> d)) - 1;
                            if (t > dt_) t = dt_;
                        }
#if RO_PATH_ZERO
                        // a ZERO node there: the walk ends on it (K_ZERO)
                        if (n_ch <= 4 && ((pcls >> (32 + 8 * ci + t)) & 1u)) {
                            c_steps += t - d + 1;
                            d = t;
                            zero_mask |= 1u << ci;
                            return;
                        }
#endif
                        c_steps += t - d;
                        d = t;
                    }
                    bool probe = false;
                    while (true) {
                        const int sh = D - d;
                        const int nidx = S.lvl_off[d] +
                            ((((qz >> sh) << d) + (qy >> sh)) << d) + (qx >> sh);
                        c_steps += 1;
                        uint32_t w;
                        if (vec4) {
                            if (nidx != cur_node) {
                                RO_ASSERT(nidx >= 0 && nidx < A.L.num_nodes);
                                wv = ld_meta4(reinterpret_cast<const uint4 *>(A.words) + nidx);
                                cur_node = nidx;
                            }
                            w = word_of_slot(wv, slot);
                        } else {
                            RO_ASSERT(nidx >= 0 && nidx < A.L.num_nodes);
                            w = __ldg(A.words + nidx * m + slot);
                        }
                        const int mn = (w >> 16) & 0xFF, mx = (w >> 24) & 0xFF;
                        mask = w & 0xFFFF;
                        if (mn == 255 && mx == 0) {  // INVALID: metadata request
                            const int32_t mid = nidx * m + slot;
                            const unsigned long long key = key_hi | ev++;
                            int32_t &lm = last_mreq[ci * kBlock + tid];
                            if (mid != lm) {
                                lm = mid;
                                request(A.meta_key, nullptr, nullptr, mid, key);
                            }
                        } else {
                            if (mx < (int)S.empty_below[ci][mn]) {  // K_ZERO
                                zero_mask |= 1u << ci;
                                break;
                            }
                            if (mx - mn <= S.eps_i) {  // K_CONST
                                double r, g, b, a;
                                tf_eval(S, ci, (double)mn, r, g, b, a);
                                sR += r * a;
                                sG += g * a;
                                sB += b * a;
                                trans *= (1.0 - a);
                                any_const = true;
                                break;
                            }
                        }
                        const int lev = clampi(raw, CH_LO(ci), CH_HI(ci));
                        if (mask == 0) {  // K_MISSU: request the desired brick
                            if (sc.lp.lev != lev)
                                level_pos(sc.lp, lev, px, py, pz, S, lbx, lby, lbz);
                            const int32_t gb = S.ptoff[ci][lev] + sc.lp.local;
                            const unsigned long long key = key_hi | ev++;
                            int32_t &lb = last_breq[ci * kBlock + tid];
                            if (gb != lb) {
                                lb = gb;
                                request(A.brick_key, nullptr, nullptr, gb, key);
                            }
                            break;
                        }
                        if (d < dt_) {
                            d += 1;
                            continue;
                        }
                        probe = true;
                        break;
                    }
                    if (!probe) return;
                    }
                    // at traversal depth: probe the desired brick
                    {
                        all_cz = false;
                        const int lev = clampi(raw, chc.y, chc.z);
                        if (sc.lp.lev != lev) level_pos(sc.lp, lev, px, py, pz, S, lbx, lby, lbz);
                        const int32_t e = S.ptoff[ci][lev] + sc.lp.local;
                        RO_ASSERT(e >= 0 && e < A.L.E);
#if RO_TMA_STAGE
                        if (BX == 32 && BY == 32 && !((pf_done >> ci) & 1u) &&
                            __activemask() == 0xffffffffu) {
                            // whole warp here: one group owns the warp's slab
                            const int pv = ld_meta(A.pt + e);
                            bool need = false;
                            if (pv >= 0) {
                                account(ci, lev, e);
                                need = !sub_skip(ci, pv, sc.lp);
                                if (need && sc.tp_lev != lev) {
                                    taps_of(sc.tp, sc.lp, px, py, pz, bx, by, bz, S);
                                    sc.tp_lev = lev;
                                }
                            }
                            const unsigned T = __ballot_sync(0xffffffffu, need);
                            if (T) {
                                const int z0 = need ? sc.tp.o / (bx * by) : -1;
                                const int leader = __ffs(T) - 1;
                                const int lslot = __shfl_sync(0xffffffffu, pv, leader);
                                const int lz0 = __shfl_sync(0xffffffffu, z0, leader);
                                const int w = threadIdx.x >> 5;
                                const uint32_t bar =
                                    (uint32_t)__cvta_generic_to_shared(&stage_bar[w]);
                                const uint32_t dsts = (uint32_t)__cvta_generic_to_shared(stage[w]);
                                if ((threadIdx.x & 31) == leader) {
                                    const uint8_t *srcp = A.cache + (int64_t)lslot * bvox +
                                                          (int64_t)lz0 * (bx * by);
                                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                                    asm volatile(
                                        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                                        ::"r"(bar), "r"(kSlab) : "memory");
                                    asm volatile(
                                        "cp.async.bulk.shared::cluster.global.mbarrier::"
                                        "complete_tx::bytes [%0], [%1], %2, [%3];"
                                        ::"r"(dsts), "l"(srcp), "r"(kSlab), "r"(bar) : "memory");
                                }
                                asm volatile(
                                    "{\n .reg .pred p;\n WAIT%=:\n"
                                    " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                                    " @!p bra WAIT%=;\n}" ::"r"(bar), "r"(stage_phase) : "memory");
                                stage_phase ^= 1u;
                                if (need) {
                                    if (pv == lslot && z0 == lz0) {
                                        const uint8_t *q = stage[w] + (sc.tp.o - lz0 * (bx * by));
                                        int tv[8] = {q[0], q[1], q[bx], q[bx + 1], q[bx * by],
                                                     q[bx * by + 1], q[bx * by + bx],
                                                     q[bx * by + bx + 1]};
                                        RO_STAT(c_s6);
                                        const int mt = max(max(max(tv[0], tv[1]), max(tv[2], tv[3])),
                                                           max(max(tv[4], tv[5]), max(tv[6], tv[7])));
                                        if (mt > S.zero_upto[ci]) {
                                            const double val = trilerp(tv, sc.tp);
                                            double r, g, b, a;
                                            tf_eval(S, ci, val, r, g, b, a);
                                            sR += r * a;
                                            sG += g * a;
                                            sB += b * a;
                                            trans *= (1.0 - a);
                                        }
                                    } else {
                                        finish(ci, pv, sc.tp);
                                    }
                                }
                                __syncwarp();  // every read of the slab before its next fill
                            }
                            if (pv >= 0) return;
                        } else
#endif
                        if ((pf_done >> ci) & 1u) {  // probed ahead
                            if ((pf_hit >> ci) & 1u) {
                                account(ci, lev, e);
                                if (!((pf_skip >> ci) & 1u)) sample_taps(ci, lev, ld_meta(A.pt + e));
                                return;
                            }
                        } else {
                            const int pv = ld_meta(A.pt + e);
                            if (pv >= 0) {
                                sample(ci, lev, pv, e);
                                return;
                            }
                        }
                        {
                            RO_STAT(c_s5);
                            const unsigned long long key = key_hi | ev++;
#if RO_SMEM_ASM
                            const uint32_t a_lb = s_breq + ((uint32_t)ci * (kBlock * 4u));
                            if (e != lds32(a_lb)) {
                                sts32(a_lb, e);
                                request(A.brick_key, nullptr, nullptr, e, key);
                            }
#else
                            int32_t &lb = last_breq[ci * kBlock + tid];
                            if (e != lb) {
                                lb = e;
                                request(A.brick_key, nullptr, nullptr, e, key);
                            }
#endif
                        }
                        // nearest resident level in this node, coarser first
                        int32_t e2 = -1;
#if RO_LP2_LOCAL
                        LevelPos lp2;  // (not cached across channels: fewer live registers)
                        lp2.lev = -1;
#else
                        LevelPos &lp2 = sc.lp2;
#endif
                        const int2 sub = substitute(A.pt, S, ci, lev, k, mask, px, py, pz,
                                                    lbx, lby, lbz, lp2, e2, sc.lp);
                        if (sub.x >= 0) sample2(ci, sub.x, sub.y, e2, lp2);
                    }
                };
#if RO_UNROLL4
                if (fast && n_ch == 4) {
                    // the common case unrolled: every channel-indexed constant,
                    // table and per-thread array offset becomes a constant
#pragma unroll
                    for (int ci = 0; ci < 4; ++ci) channel(ci);
                } else
#endif
                {
#if RO_CH_UNROLL2
#pragma unroll 2
#else
#pragma unroll 1
#endif
                    for (int ci = 0; ci < n_ch; ++ci) channel(ci);
                }
                end_depth = d;
                if (all_cz) {
                    skippable = true;
                    const double s = 1.0 / (double)(1 << d);
                    const int ix = qx >> (D - d), iy = qy >> (D - d), iz = qz >> (D - d);
                    skip_exit = box_exit(ox, oy, oz, dx, dy, dz, ix * s, iy * s, iz * s,
                                         (ix + 1) * s, (iy + 1) * s, (iz + 1) * s);
                }
            }

            if (skippable) {  // kernels.py:561-635 (only ZERO / CONST / MISSU)
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
                        if (CHECK && F.check_skips && zero_mask) {
                            double qx = ox + t * dx, qy = oy + t * dy, qz = oz + t * dz;
                            if (qx < 0.0) qx = 0.0;
                            if (qy < 0.0) qy = 0.0;
                            if (qz < 0.0) qz = 0.0;
                            if (qx > kClampHi) qx = kClampHi;
                            if (qy > kClampHi) qy = kClampHi;
                            if (qz > kClampHi) qz = kClampHi;
                            const int raw2 = lod_raw(t, t0, S.inv_t0, S.t0_pow2, S);
                            for (int ci = 0; ci < n_ch; ++ci) {
                                if (!((zero_mask >> ci) & 1u)) continue;
                                const int lev = clampi(raw2, CH_LO(ci), CH_HI(ci));
                                const double rv = ref_value(F, S, ci, lev, qx, qy, qz, bx, by,
                                                            bz, lbx, lby, lbz, bvox);
                                if (rv >= 0.0) {
                                    double r, g, b, a;
                                    tf_eval(S, ci, rv, r, g, b, a);
                                    if (a > 0.0) c_viol += 1;
                                }
                            }
                        }
                    }
#if RO_LOD_INC && RO_SKIP_LOD_INC
                    // the raw level only grows with t: step / jexp change only
                    // when t / t0 crosses the next level's threshold
                    {
                        const double ratio = S.t0_pow2 ? t * S.inv_t0 : t / t0;
                        if (ratio >= next_thr) {
                            raw_c = lod_raw(t, t0, S.inv_t0, S.t0_pow2, S);
                            next_thr = S.lod_thr[raw_c + 1];
                        }
                        step = S.step_tab[raw_c];
                        jexp = S.maxlev[raw_c];
                    }
#else
                    const int raw2 = lod_raw(t, t0, S.inv_t0, S.t0_pow2, S);
                    step = S.step_tab[raw2];
                    jexp = S.maxlev[raw2];
#endif
                    t += step;
                }
                prev_depth = end_depth;
                if (t == t_before) {
                    if (++stall > D + 2) {  // proven cycle: the reference never returns
                        c_live += 1;
                        alive = false;
                    }
                } else {
                    stall = 0;
                }
            } else {
                stall = 0;
                if (CHECK && F.check_skips && zero_mask) {  // kernels.py:644-655
                    for (int ci = 0; ci < n_ch; ++ci) {
                        if (!((zero_mask >> ci) & 1u)) continue;
                        const int lev = clampi(raw, CH_LO(ci), CH_HI(ci));
                        const double rv = ref_value(F, S, ci, lev, px, py, pz, bx, by, bz, lbx,
                                                    lby, lbz, bvox);
                        if (rv >= 0.0) {
                            double r, g, b, a;
                            tf_eval(S, ci, rv, r, g, b, a);
                            if (a > 0.0) c_viol += 1;
                        }
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
            alive = alive && t < tfar && accA < F.early_alpha;
            if (CHECK && F.max_samples > 0 && ++n_probe >= F.max_samples) alive = false;
        }
    }
    // close every channel's last brick run
    for (int ci = 0; ci < n_ch && RO_RUNLEN; ++ci) {
        const unsigned long long rv = run[ci * kBlock + tid];
        const uint32_t cnt = (uint32_t)(rv >> 36);
        if (cnt) hist_t[(ci * k + (int)((rv >> 32) & 15)) * kBlock + tid] += cnt;
    }
    if (active) {
        const float4 px4 = make_float4(__double2float_rn(accR), __double2float_rn(accG),
                                       __double2float_rn(accB), __double2float_rn(accA));
        const int64_t opix = F.shared_outputs ? pix : lpix;  // full-frame or local rows
        reinterpret_cast<float4 *>(A.image)[opix] = px4;
        A.pix_required[opix] = pixreq;
    }
    }  // packets of the tile
    }  // tile loop

    // parts writing another GPU's buffers (sort-first over peer memory):
    // their stores / atomics are flushed to the owner before the kernel's
    // completion is signalled to any other rank
    if (F.shared_outputs) __threadfence_system();

    // ---- block reductions ----
#if RO_STATS
    unsigned long long vals[8] = {c_steps, c_eval, c_skip, c_viol, c_live, c_s5, c_s6, c_s7};
    constexpr int kNV = 8;
#else
    unsigned long long vals[5] = {c_steps, c_eval, c_skip, c_viol, c_live};
    constexpr int kNV = 5;
#endif
#pragma unroll
    for (int i = 0; i < kNV; ++i) {
        unsigned long long vv = vals[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vv += __shfl_down_sync(0xffffffffu, vv, o);
        if (lane == 0 && vv) atomicAdd(&S.red[i], vv);
    }
    __syncthreads();
    if (tid < kNV && S.red[tid]) atomicAdd(A.counters + tid, S.red[tid]);
    for (int i = tid; i < n_ch * k; i += kBlock) {
        unsigned long long s = 0;
        for (int j = 0; j < kBlock; ++j) s += hist_t[i * kBlock + j];
        if (s) atomicAdd(A.hist + i, s);
    }
}

template <int MODE, bool CHECK, int BX, int BY, int BZ>
cudaError_t launch_b(const ro_frame &F, const RayArgs &A, cudaStream_t s) {
    int n_tiles = ((F.width + kTileW - 1) / kTileW) * ((A.local_rows + kTileH - 1) / kTileH);
    static int sm_count = 0;
    if (sm_count == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    // 4 CTAs of 128 threads stay within the 164 KB shared-memory carveout
    // (more L1) for up to 4 channels x 7 levels
    size_t dyn = (size_t)F.n_ch * kBlock * (kRunBytes + 4 * 2) +
                 (size_t)F.n_ch * A.L.k * kBlock * 4;
#ifdef RO_EXTRA_SMEM
    dyn += RO_EXTRA_SMEM;  // experiment knob: shared-memory / L1 split sensitivity
#endif
    auto kern = k_raycast<MODE, CHECK, BX, BY, BZ>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, dyn);
    if (e != cudaSuccess) return e;
#if RO_PERSISTENT
    int blocks = per_sm * sm_count;
    if (blocks > n_tiles) blocks = n_tiles;
    if (blocks < 1) blocks = 1;
#else
    int blocks = n_tiles;
#endif
    kern<<<blocks, kBlock, dyn, s>>>(F, A);
    return cudaGetLastError();
}

// brick sizes with compile-time tap offsets; anything else uses runtime ones
template <int MODE, bool CHECK>
cudaError_t launch(const ro_frame &F, const RayArgs &A, cudaStream_t s) {
    if (A.L.bx == 32 && A.L.by == 32 && A.L.bz == 32)
        return launch_b<MODE, CHECK, 32, 32, 32>(F, A, s);
    if (A.L.bx == 16 && A.L.by == 16 && A.L.bz == 16)
        return launch_b<MODE, CHECK, 16, 16, 16>(F, A, s);
    return launch_b<MODE, CHECK, 0, 0, 0>(F, A, s);
}

}  // namespace

// Sort-first image assembly: part p's local rows are the row blocks
// b = p, p + n, p + 2n, ... of tile_rows rows (ro_frame.n_parts/part/tile_rows);
// parts [n_parts][part_stride floats] -> full [height][width][4].
__global__ void k_gather_rows(const float4 *__restrict__ parts, int32_t n_parts,
                              int64_t part_stride4, int32_t height, int32_t width,
                              int32_t tile_rows, float4 *__restrict__ full) {
    const int64_t total = (int64_t)height * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t y = (int32_t)(i / width), x = (int32_t)(i - (int64_t)y * width);
        const int32_t b = y / tile_rows, p = b % n_parts;
        const int64_t ly = (int64_t)(b / n_parts) * tile_rows + (y - b * tile_rows);
        full[i] = parts[p * part_stride4 + ly * width + x];
    }
}

int gather_rows(const float *parts, int32_t n_parts, int64_t part_stride, int32_t height,
                int32_t width, int32_t tile_rows, float *full, cudaStream_t s) {
    if (part_stride % 4 || (reinterpret_cast<uintptr_t>(parts) & 15) ||
        (reinterpret_cast<uintptr_t>(full) & 15))
        return fail(RO_EINVAL, "image buffers must be 16-byte aligned RGBA");
    const int64_t total = (int64_t)height * width;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_gather_rows<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const float4 *>(parts),
                                                    n_parts, part_stride / 4, height, width,
                                                    tile_rows, reinterpret_cast<float4 *>(full));
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

// load every ray-caster instantiation of this layout's brick size (CUDA
// loads kernels lazily, at their first launch: a frame-one hitch otherwise)
template <int BX, int BY, int BZ>
int warm_b() {
    const void *kernels[] = {
        (const void *)k_raycast<RO_MODE_RESIDENCY, false, BX, BY, BZ>,
        (const void *)k_raycast<RO_MODE_RESIDENCY, true, BX, BY, BZ>,
        (const void *)k_raycast<RO_MODE_REFERENCE, false, BX, BY, BZ>,
        (const void *)k_raycast<RO_MODE_PAGETABLE, false, BX, BY, BZ>,
        (const void *)k_raycast<RO_MODE_CLASSIC, false, BX, BY, BZ>};
    cudaFuncAttributes fa;
    for (const void *k : kernels) RO_CUDA(cudaFuncGetAttributes(&fa, k));
    return RO_OK;
}

int raycast_warm(ro_ctx *c) {
    cudaFuncAttributes fa;
    RO_CUDA(cudaFuncGetAttributes(&fa, k_classify));
    RO_CUDA(cudaFuncGetAttributes(&fa, k_gather_rows));
    const int *b = c->layout.brick;
    if (b[0] == 32 && b[1] == 32 && b[2] == 32) return warm_b<32, 32, 32>();
    if (b[0] == 16 && b[1] == 16 && b[2] == 16) return warm_b<16, 16, 16>();
    return warm_b<0, 0, 0>();
}

int render(ro_ctx *c, const ro_frame *F, const ro_state *st,
           const ro_outputs *out, cudaStream_t s) {
    if (F->n_ch < 1 || F->n_ch > RO_MAX_CH) return fail(RO_EINVAL, "n_ch outside [1, 8]");
    if (F->width < 1 || F->height < 1) return fail(RO_EINVAL, "empty image");
    if (F->n_parts < 1 || F->part < 0 || F->part >= F->n_parts || F->tile_rows < 1)
        return fail(RO_EINVAL, "bad partition");
    if ((int64_t)F->width * F->height >= (int64_t(1) << 31))
        return fail(RO_EINVAL, "image too large");
    if (!(F->t0 > 0.0) || !(F->base_step > 0.0)) return fail(RO_EINVAL, "t0 / base_step must be > 0");
    if (c->layout.depth > 10) return fail(RO_EINVAL, "ray casting supports octree depth <= 10");
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
    if (F->mode < RO_MODE_RESIDENCY || F->mode > RO_MODE_CLASSIC)
        return fail(RO_EINVAL, "unknown render mode");
    if (F->check_skips && (F->ref_pt == nullptr || F->ref_cache == nullptr))
        return fail(RO_EINVAL, "check_skips needs reference paging");
    if (F->max_samples < 0 || (F->max_samples > 0 && F->mode != RO_MODE_RESIDENCY))
        return fail(RO_EINVAL, "max_samples: >= 0, residency mode only");
    if (F->check_skips && F->mode != RO_MODE_RESIDENCY)
        return fail(RO_EINVAL, "the skip audit runs in residency mode only");
    if (F->mode == RO_MODE_CLASSIC) {
        // render.py:282-295: node depth d owns exactly one brick of level k-1-d
        const int k = c->layout.k;
        if (F->cls_min == nullptr || F->cls_max == nullptr)
            return fail(RO_EINVAL, "classic mode needs classic min / max metadata");
        if (F->cls_depth != k - 1 || k - 1 > 8)
            return fail(RO_EINVAL, "classic octree depth must be k-1 <= 8");
        for (int l = 0; l < k; ++l)
            for (int a = 0; a < 3; ++a)
                if (c->layout.level_grids[l][a] != (1 << (k - 1 - l)))
                    return fail(RO_EINVAL, "classic octree needs power-of-two brick grids");
    }
    if (c->bvox >= (int64_t(1) << 24)) return fail(RO_EINVAL, "brick too large");
    if (F->mode == RO_MODE_RESIDENCY) {
        if (!c->meta_key_ext) {
            int rc = ensure_meta_keys(c);
            if (rc) return rc;
        }
        if (c->layout.m == 4 && (reinterpret_cast<uintptr_t>(st->words) & 15))
            return fail(RO_EINVAL, "octree words must be 16-byte aligned");
    }
    // device views of the two per-pixel outputs (pinned host memory is
    // written through its UVA mapping)
    void *dev_out[2] = {out->image, out->pix_required};
    for (void *&p : dev_out) {
        cudaPointerAttributes pa;
        if (p == nullptr) return fail(RO_EINVAL, "null image / pix_required output");
        if (cudaPointerGetAttributes(&pa, p) != cudaSuccess ||
            pa.type == cudaMemoryTypeUnregistered || pa.devicePointer == nullptr) {
            cudaGetLastError();
            return fail(RO_EINVAL, "image / pix_required must be device or pinned host memory");
        }
        p = pa.devicePointer;
    }
    RayArgs A;
    A.L = c->dl;
    A.words = st->words;
    A.pt = st->pt;
    A.cache = st->cache;
    A.image = static_cast<float *>(dev_out[0]);
    A.required = out->required;
    A.pix_required = static_cast<int32_t *>(dev_out[1]);
    A.hist = reinterpret_cast<unsigned long long *>(out->hist);
    A.counters = reinterpret_cast<unsigned long long *>(out->counters);
    A.brick_key = brick_keys(c);
    A.meta_key = meta_keys(c);
    A.brick_touched = c->brick_touched;
    A.meta_touched = c->meta_touched;
    A.touched_n = c->touched_n;
    A.tile_counter = c->touched_n + 2;
    const bool sub_ok = c->layout.brick[0] >= RO_SUB_E && c->layout.brick[1] >= RO_SUB_E &&
                        c->layout.brick[2] >= RO_SUB_E;
    A.sub_max = sub_ok ? st->sub_max : nullptr;
    A.nsb = sub_ok ? (c->layout.brick[0] >> RO_SUB_LOG) * (c->layout.brick[1] >> RO_SUB_LOG) *
                         (c->layout.brick[2] >> RO_SUB_LOG) : 0;
#if RO_SUB32
    if ((int64_t)A.L.num_slots * A.nsb >= ((int64_t)1 << 31)) A.sub_max = nullptr;
#endif
    A.node_fast = nullptr;
    A.node_path = nullptr;
    A.local_rows = (int32_t)ro_local_rows(F->height, F->n_parts, F->part, F->tile_rows);
    if (!F->shared_outputs) {  // shared outputs are cleared once by their owner
        RO_CUDA(cudaMemsetAsync(out->required, 0, (size_t)c->E, s));
        RO_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(int64_t) * F->n_ch * c->layout.k, s));
        RO_CUDA(cudaMemsetAsync(out->counters, 0, sizeof(int64_t) * RO_NUM_COUNTERS, s));
    }
    // requests of an uncollected previous pass would leak into this frame's
    // lists: reset the context's own key arrays first (caller-owned shared
    // arrays are managed by their owner)
    if (c->keys_dirty && !c->brick_key_ext) {
        RO_CUDA(cudaMemsetAsync(c->brick_key, 0xFF, sizeof(unsigned long long) * c->E, s));
        if (c->meta_key)
            RO_CUDA(cudaMemsetAsync(c->meta_key, 0xFF, sizeof(unsigned long long) * c->n_meta, s));
    }
    c->keys_dirty = true;
    if (A.local_rows == 0) return RO_OK;
    RO_CUDA(cudaMemsetAsync(A.tile_counter, 0, sizeof(int32_t), s));
    if (F->mode == RO_MODE_RESIDENCY && c->node_fast != nullptr && st->words != nullptr) {
        const int D = c->layout.depth, sub = D < 3 ? D : 3;
        k_classify<<<1u << (3 * sub), 256, 0, s>>>(*F, st->words, c->layout.m, D, sub,
                                                   c->node_fast, c->node_path);
        RO_CUDA(cudaGetLastError());
        A.node_fast = c->node_fast;
        A.node_path = c->node_path;
    }
    cudaError_t e;
    if (F->mode == RO_MODE_REFERENCE) {
        e = launch<RO_MODE_REFERENCE, false>(*F, A, s);
    } else if (F->mode == RO_MODE_PAGETABLE) {
        e = launch<RO_MODE_PAGETABLE, false>(*F, A, s);
    } else if (F->mode == RO_MODE_CLASSIC) {
        e = launch<RO_MODE_CLASSIC, false>(*F, A, s);
    } else if (F->check_skips || F->max_samples > 0) {  // audit / probe instantiation
        e = launch<RO_MODE_RESIDENCY, true>(*F, A, s);
    } else {
        e = launch<RO_MODE_RESIDENCY, false>(*F, A, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "k_raycast launch");
    return RO_OK;
}

}  // namespace ro
