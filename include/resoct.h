/*
 * resoct.h -- C ABI of the B200-native residency-octree render path.
 *
 * libresoct.so replaces the reference's numba/numpy hot path behind the
 * reference's Python API.  Every entry point takes plain pointers and sizes
 * (device pointers unless noted), never torch types.  The reference interface
 * each call replaces is cited; all paths are under /root/reference/pkg/src/
 * resoctree/.
 *
 *   ro_render            kernels.py:209-704  raycast_frame (MODE_RESIDENCY /
 *                        MODE_REFERENCE / MODE_PAGETABLE / MODE_CLASSIC,
 *                        check_skips audit), driven by render.py:125-208
 *                        (_run), render.py:236-262 and camera.py:32-51
 *   ro_feedback_collect  render.py:210-215  bricks-first request budget over
 *                        the first-seen request lists of kernels.py:457-517
 *   ro_note_sampled      engine.py:72-81    Engine.note_sampled
 *   ro_apply_bricks      engine.py:85-89    Engine.apply_brick, batched:
 *                        paging.py:187-218 insert_brick (LRU) +
 *                        octree.py:193-246 on_brick_evicted/inserted
 *   ro_evict_bricks      verify.py:110-121  explicit eviction (unmap, release
 *                        slot, octree.on_brick_evicted)
 *   ro_mark_empty        paging.py:228-234  MultiChannelPaging.mark_empty
 *   ro_apply_metadata    engine.py:91-96    Engine.apply_metadata /
 *                        octree.py:263-269 set_node_metadata
 *   ro_write_level_metadata engine.py:138-152 fill_metadata_from_volumes (one
 *                        octree level of one slot from device min/max grids)
 *   ro_swap_channel      engine.py:98-105   Engine.swap_channel =
 *                        paging.py:263-284 + octree.py:271-273
 *   ro_octree_update     octree.py:193-246  on_brick_inserted / on_brick_evicted
 *                        for a list of changed bricks (incremental pass)
 *   ro_rebuild_masks     octree.py:355-395  masks from the resident set
 *                        (ground truth + OR closure), for verification
 *   ro_apply_bricks_lz4  service.py:225-232 fetch + ingest.py:114-117
 *                        decompress_brick + Engine.apply_brick: LZ4 frames
 *                        decoded on the GPU into the cache
 *   ro_lz4_decode        lz4io.py:69-110 decompress (batched, device)
 *   ro_normalize_to_u8 / ro_downsample_box / ro_extract_bricks
 *                        ingest.py:27-95 (device pyramid + bricks)
 *   ro_node_minmax       service.py:102-115 region_min_max / engine.py:186-219
 *                        _box_minmax_grid (one tree level, device volume)
 *   ro_fill_metadata     engine.py:138-152 fill_metadata_from_volumes
 *   ro_pack_frame        render.py:101-122 + camera.py:32-44 + kernels.py:43-66
 *                        + transfer.py:38-120 host packing (for C hosts)
 *   ro_upload_state / ro_download_state
 *                        reference-layout state (paging.py:95-112,
 *                        octree.py:116-118) <-> device state
 *
 * Errors: every call returns 0 on success or a negative RO_E* code; the
 * message is available from ro_last_error() (thread-local).  Asynchronous
 * kernel faults surface at the next synchronising call (ro_sync,
 * ro_feedback_collect, ro_apply_bricks).
 *
 * Threading: single writer per context (paging.py:84-87).  All work of a
 * context is ordered on the caller's stream; ro_apply_bricks additionally
 * uses the context's own upload stream for host->device payload copies.
 */
#ifndef RESOCT_H
#define RESOCT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RO_ABI_VERSION 1
#define RO_MAX_LEVELS 16
#define RO_MAX_PT 256
#define RO_MAX_CH 8
#define RO_MAX_TF_POINTS 16
#define RO_NUM_COUNTERS 8
#define RO_SUB_EDGE 4        /* sub-block edge of ro_state.sub_max */

#define RO_MODE_RESIDENCY 0
#define RO_MODE_REFERENCE 1
#define RO_MODE_PAGETABLE 2  /* page-table-only baseline, kernels.py:316-357 */
#define RO_MODE_CLASSIC 3    /* classic one-node-one-brick octree, kernels.py:359-429 */

/* packed page-table entry: >= 0 cache slot (MAPPED), else: */
#define RO_PT_UNMAPPED (-1)
#define RO_PT_EMPTY (-2)

#define RO_OK 0
#define RO_EINVAL (-1)
#define RO_ECUDA (-2)
#define RO_ENOMEM (-3)
#define RO_ESTATE (-4)

/* Static volume / cache geometry (paging.py:27-112, octree.py:26-39). */
typedef struct ro_layout {
    int32_t m, k, depth;               /* channel slots, levels, octree depth */
    int32_t brick[3];                  /* brick size x, y, z */
    int32_t level_dims[RO_MAX_LEVELS][3];   /* voxels per level, x, y, z */
    int32_t level_grids[RO_MAX_LEVELS][3];  /* bricks per level, x, y, z */
    int64_t pt_offsets[RO_MAX_PT + 1]; /* page-table offsets, m*k+1 used */
    int64_t num_slots;                 /* cache slots S */
} ro_layout;

/* Mutable render state in device memory, owned by the caller. */
typedef struct ro_state {
    uint32_t *words;         /* [N*m] octree words (mask|min<<16|max<<24); may be NULL */
    int32_t *pt;             /* [E]   packed page-table entries */
    uint8_t *cache;          /* [S*bz*by*bx] brick cache, allocated with one more
                                brick of tail padding ((S+1)*bvox bytes): the ray
                                caster may read -- never use -- bytes just past
                                a brick's last tap */
    int64_t *slot_brick;     /* [S]   brick id per slot, -1 free */
    int64_t *slot_last_used; /* [S]   LRU frame stamp */
    int32_t *free_stack;     /* [S]   LIFO free list, top at free_count-1 */
    int32_t *free_count;     /* [1]   device scalar */
    uint8_t *sub_max;        /* [S*nsb] optional (NULL = off), kept by
                                ro_apply_bricks*: for bricks with every side
                                >= 4, nsb = (bx/4)(by/4)(bz/4) sub-blocks of
                                4^3 voxels per slot (RO_SUB_EDGE), each holding
                                the max of its voxels dilated by one on every
                                side (clipped to the brick); lets the ray
                                caster skip the taps of a sample whose
                                neighbourhood is wholly in a transfer
                                function's transparent range (an exact +0
                                contribution) */
} ro_state;

/* One visible channel in importance order (render.py:35-44,101-122). */
typedef struct ro_channel {
    int32_t slot, lo, hi, npoints;
    double tf_x[RO_MAX_TF_POINTS];
    double tf_rgba[RO_MAX_TF_POINTS][4];
    /* interval emptiness (kernels.py:201-206): metadata (mn, mx) is
       transparent iff mx < empty_below[mn] */
    uint16_t empty_below[256];
    /* largest integer scalar v with opacity 0 on [0, v] (-1: none) */
    int32_t zero_upto;
    int32_t _pad;
    /* per integer scalar j: first knot segment i with x[i+1] >= j */
    uint8_t tf_seg[256];
} ro_channel;

/* Per-frame constants, filled on the host. */
typedef struct ro_frame {
    int32_t mode;                 /* RO_MODE_* */
    int32_t n_ch;
    int32_t width, height;        /* full image */
    double cam_pos[3], cam_fwd[3], cam_right[3], cam_up[3];
    double tan_half, aspect;
    double base_step, t0, early_alpha, eps_h;
    int32_t start_level;
    int32_t check_skips;
    /* LOD: raw level L holds iff ratio >= lod_threshold[L] (L = 1..15),
       thresholds found with the same libm log2 the reference calls */
    double lod_threshold[RO_MAX_LEVELS + 1];
    double step_tab[RO_MAX_LEVELS];      /* base_step * 2^maxlev(raw) */
    int32_t maxlev_tab[RO_MAX_LEVELS];   /* max over channels of clamp(raw) */
    int32_t dt_tab[RO_MAX_LEVELS];       /* traversal_depth(step_tab[raw]) */
    /* sort-first partition: rows are cut in blocks of tile_rows; block b is
       rendered by part (b % n_parts).  Outputs are local (compacted rows). */
    int32_t n_parts, part, tile_rows;
    int32_t cls_depth;            /* RO_MODE_CLASSIC: classic octree depth = k-1 */
    const int32_t *ref_pt;        /* audit paging (check_skips), device */
    const uint8_t *ref_cache;
    /* RO_MODE_CLASSIC: per-node min / max u8[n_nodes*m] of the classic octree
       (render.py:271-315 ClassicMetadata.min_arr / max_arr), device */
    const uint8_t *cls_min;
    const uint8_t *cls_max;
    /* sort-first over peer memory: 1 = the outputs are the FULL frame's,
       shared by every part (typically rank 0's buffers, mapped into every
       part's address space by the host -- CUDA IPC memory handles, see
       distributed.PeerFrame): image / pix_required are written at the pixel's global
       row, and ro_render does not clear required / hist / counters (the
       owner clears them once per frame before any part renders). */
    int32_t shared_outputs;
    /* > 0: every ray resolves at most this many samples through the cursor
       (a skippable sample still runs its skip loop) -- the single-sample
       probe behind traverse_sample() (render_units hand traces); residency
       mode only, 0 = unlimited (the product setting) */
    int32_t max_samples;
    ro_channel ch[RO_MAX_CH];
} ro_frame;

/* image and pix_required may be device memory or pinned host memory
   (cudaHostAlloc / cudaHostRegister, UVA-mapped): the ray caster then
   stores the frame straight over PCIe while it runs (zero-copy readback).
   Pageable host memory is rejected. */
typedef struct ro_outputs {
    float *image;          /* [local_rows*width*4] f32 RGBA */
    uint8_t *required;     /* [E] usage mask (zeroed by ro_render) */
    int32_t *pix_required; /* [local_rows*width] */
    int64_t *hist;         /* [n_ch*k] (zeroed by ro_render) */
    int64_t *counters;     /* [RO_NUM_COUNTERS]: steps, evaluated, skipped,
                              violations, livelocks (zeroed by ro_render) */
} ro_outputs;

typedef struct ro_feedback {
    int64_t *brick_keys, *brick_ids; /* [budget] device */
    int64_t *meta_keys, *meta_ids;   /* [budget] device; meta id = node*m+slot */
    int64_t *counts;                 /* [4] HOST (or NULL): unique bricks, unique
                                        metas, bricks emitted, metas emitted */
    int64_t *counts_dev;             /* [4] DEVICE (or NULL): the same counts,
                                        written on the stream */
} ro_feedback;

typedef struct ro_ctx ro_ctx;

int ro_abi_version(void);
const char *ro_last_error(void);

/* ---- host-side frame packing (for C / C++ hosts; no CUDA calls) ---- */
typedef struct ro_camera {          /* camera.py:15-30 */
    double position[3], target[3], up[3];
    double fov_deg;
} ro_camera;

typedef struct ro_render_config {   /* render.py:47-67 RenderConfig */
    int32_t width, height;
    double base_step, lod_reference_distance, early_term_alpha;
    int32_t traversal_start_level, _pad0;
} ro_render_config;

typedef struct ro_channel_desc {    /* render.py:35-44 ChannelSettings */
    int32_t slot, level_lo, level_hi, npoints;
    double x[RO_MAX_TF_POINTS];     /* transfer-function knots (transfer.py:16-36) */
    double rgba[RO_MAX_TF_POINTS][4];
} ro_channel_desc;

/* Fill `frame` for ro_render exactly as the Python mirror does
   (render.py:101-122 channel packing, camera.py:32-44 basis, the LOD /
   step / traversal-depth tables of kernels.py:43-66, the TF emptiness
   tables of transfer.py:38-120).  k / m = levels / channel slots of the
   layout; depth = octree depth in residency mode (0 otherwise); eps_h =
   homogeneity epsilon.  Partition fields default to one part. */
int ro_pack_frame(int32_t k, int32_t m, int32_t depth, int32_t mode,
                  const ro_camera *camera, const ro_render_config *config,
                  const ro_channel_desc *channels, int32_t n_ch, double eps_h,
                  ro_frame *frame);

/* ---- transfer-function queries (host, no CUDA; transfer.py:38-120) ----
   n knots x[n] (strictly increasing), rgba[n][4]; the host mirror
   (transfer.TransferFunction) answers every query through these. */
int ro_tf_evaluate(int32_t n, const double *x, const double *rgba, double v,
                   double *out4);
/* inf{x >= a : opacity(x) > 0}, +inf when none */
int ro_tf_first_support(int32_t n, const double *x, const double *rgba, double a,
                        double *out);
/* maximal opaque intervals as (start, end, end_closed) triples, out[3*(n-1)] */
int ro_tf_support_intervals(int32_t n, const double *x, const double *rgba,
                            double *out, int32_t *n_out);
int ro_tf_interval_max_opacity(int32_t n, const double *x, const double *rgba,
                               double lo, double hi, double *out);
/* per integer scalar: first support (+inf stored as 1e30), opacity, the
   emptiness threshold (ro_channel.empty_below) and zero_upto; any output
   may be NULL */
int ro_tf_tables(int32_t n, const double *x, const double *rgba, double *first_support,
                 double *opacity, uint16_t *empty_below, int32_t *zero_upto);

int ro_create(const ro_layout *layout, ro_ctx **out);
int ro_destroy(ro_ctx *ctx);

/* Pay every one-time cost ahead of the first frame: the request-ordering
   and metadata-key arrays, the scratch and pinned staging of brick batches
   up to max_batch bricks (0: none), and the loading of every kernel the
   frame loop launches (CUDA loads kernels lazily).  Later calls only grow
   buffers that are still too small.  Synchronises the device. */
int ro_reserve(ro_ctx *ctx, int64_t max_batch);

/* Row count this part renders for a (height, n_parts, part, tile_rows). */
int64_t ro_local_rows(int32_t height, int32_t n_parts, int32_t part,
                      int32_t tile_rows);

int ro_render(ro_ctx *ctx, const ro_frame *frame, const ro_state *state,
              const ro_outputs *out, void *stream);

/* Order the frame's first-seen requests and truncate them: with
   bricks_first=1 metas get budget-(bricks emitted) (render.py:210-215),
   otherwise each list is cut to `budget` independently (per-part lists of a
   sort-first frame, merged later).  Everything runs on the device (one
   kernel, no library call).  With fb->counts (host) set the call
   synchronises the stream once at the end to fill it; with only
   fb->counts_dev set it is fully asynchronous. */
int ro_feedback_collect(ro_ctx *ctx, int64_t budget, int32_t bricks_first,
                        const ro_feedback *fb, void *stream);

int ro_note_sampled(ro_ctx *ctx, const ro_state *state,
                    const uint8_t *required, int64_t frame, void *stream);

/* Sort-first request merge: n_parts parts' ordered
   request blocks -- blocks[p] = the 4 x budget ro_feedback arrays
   (brick keys, brick ids, meta keys, meta ids) of part p, counts[p] its
   ro_feedback counts ([2] bricks, [3] metas emitted), all DEVICE -- are
   folded into this context's first-seen key arrays (smallest key per
   entry wins); a following ro_feedback_collect(bricks_first = 1) returns
   exactly the lists of one full-frame pass.  Asynchronous. */
int ro_feedback_merge(ro_ctx *ctx, const int64_t *blocks, const int64_t *counts,
                      int32_t n_parts, int64_t budget, void *stream);

/* Sort-first image assembly: parts [n_parts][part_stride floats] (part p's
   local RGBA rows, ro_frame partition layout) -> full [height][width][4],
   DEVICE buffers, 16-byte aligned.  Asynchronous. */
int ro_gather_rows(const float *parts, int32_t n_parts, int64_t part_stride,
                   int32_t height, int32_t width, int32_t tile_rows, float *full,
                   void *stream);

/* Insert n bricks in order.  ids: HOST array.  payloads: n*brick bytes on the
   host (payload_on_device=0) or device (=1).  Host payloads in page-locked
   memory (cudaHostAlloc / torch pin_memory) are DMA'd straight from the
   caller's buffer on the upload stream, finished before the call returns;
   pageable ones go through the handle's pinned staging buffer.  update_octree=0 for paging-only
   inserts.  slots_out / evicted_out: optional HOST arrays of n.  Synchronises
   the stream. */
int ro_apply_bricks(ro_ctx *ctx, const ro_state *state, const int64_t *ids,
                    int64_t n, const void *payloads, int32_t payload_on_device,
                    int64_t frame, int32_t update_octree, int32_t *slots_out,
                    int64_t *evicted_out, void *stream);

/* ---- brick ingest on the GPU ----
   Bricks travel as standard LZ4 frames (lz4io.py:1-110 over liblz4 1.9.4's
   frame API; ingest.py:114-117 decompress_brick, called by every fetch:
   service.py:71-76, 225-232). */

/* ro_apply_bricks with LZ4-framed payloads: frame i is
   frames[frame_offsets[i] - frame_offsets[0] .. frame_offsets[i+1] - frame_offsets[0]).
   ids / frame_offsets: HOST arrays (n and n+1); frames on the host
   (frames_on_device=0, then indexed from frames + frame_offsets[0]) or the
   device.  Frames are decoded on the device by one warp each straight into
   brick payloads and inserted in order; if any frame is corrupt or does not
   decode to exactly one brick, nothing is inserted and RO_EINVAL names the
   first bad one.  Synchronises the stream. */
int ro_apply_bricks_lz4(ro_ctx *ctx, const ro_state *state, const int64_t *ids,
                        int64_t n, const uint8_t *frames,
                        const int64_t *frame_offsets, int32_t frames_on_device,
                        int64_t frame, int32_t update_octree, int32_t *slots_out,
                        int64_t *evicted_out, void *stream);

/* Batched LZ4 frame decode, all DEVICE arrays: frame i = src[off[i]-off[0] ..
   off[i+1]-off[0]) -> dst + i*dst_stride (at most dst_stride bytes).
   status[i] = 0, or <0: -1 not an LZ4 frame, -2 bad descriptor / header
   checksum, -3 block too large, -4 truncated, -5 corrupt block, -6 size
   differs from expected_size (<0: any size), -7 checksum mismatch, -8
   trailing bytes.  Asynchronous. */
int ro_lz4_decode(ro_ctx *ctx, const uint8_t *src, const int64_t *src_offsets,
                  int64_t n, uint8_t *dst, int64_t dst_stride,
                  int64_t expected_size, int32_t *status, void *stream);

/* ingest.py:27-35 normalize_to_u8 over n device elements of dtype 1 u8,
   2 u16, 3 u32, 4 f32 (min -> 0, max -> 255, round half up). */
int ro_normalize_to_u8(ro_ctx *ctx, const void *src, int32_t dtype, int64_t n,
                       uint8_t *dst, void *stream);
/* ingest.py:38-61 downsample_box of a device level [dz][dy][dx], factors in
   {1, 2}, odd extents edge-replicated: dst [ceil(dz/fz)][ceil(dy/fy)][ceil(dx/fx)]. */
int ro_downsample_box(const uint8_t *src, int32_t dx, int32_t dy, int32_t dz,
                      int32_t fx, int32_t fy, int32_t fz, uint8_t *dst,
                      void *stream);
/* ingest.py:75-95 extract_brick for every brick of a device level, in
   (z, y, x) grid order: dst [gz*gy*gx][bz][by][bx], edge-replicated. */
int ro_extract_bricks(const uint8_t *level, int32_t dx, int32_t dy, int32_t dz,
                      int32_t bx, int32_t by, int32_t bz, uint8_t *dst,
                      void *stream);

/* ---- culling metadata producer on the GPU ---- */

/* Min / max of a device level-0 volume [dz][dy][dx] over every depth-d node
   extent dilated by `pad` voxels (engine.py:109-127 metadata_box; the
   per-request service.py:102-115 region_min_max and the per-level
   engine.py:186-219 _box_minmax_grid compute the same numbers): mins / maxs
   [8^d] in (z, y, x) node order; windows empty on an axis give (0, 0).
   Asynchronous. */
int ro_node_minmax(ro_ctx *ctx, const uint8_t *volume, int32_t dx, int32_t dy,
                   int32_t dz, int32_t d, int32_t pad, uint8_t *mins,
                   uint8_t *maxs, void *stream);
/* engine.py:138-152 fill_metadata_from_volumes for one slot: every tree
   level's min / max written into the octree words (mask bits kept). */
int ro_fill_metadata(ro_ctx *ctx, const ro_state *state, int32_t slot,
                     const uint8_t *volume, int32_t dx, int32_t dy, int32_t dz,
                     int32_t pad, void *stream);

/* octree.py:275-306 compute_node_metadata_from_bricks (min / max part), for
   servers without a metadata endpoint: bricks [n][bz][by][bx] (device) and
   brick-local half-open sub-boxes boxes[n][6] = x0,y0,z0,x1,y1,z1 (device);
   mins / maxs [n] (device; an empty sub-box gives 255 / 0).  Asynchronous. */
int ro_bricks_box_minmax(const uint8_t *bricks, const int32_t *boxes, int64_t n,
                         int32_t bx, int32_t by, int32_t bz, uint8_t *mins,
                         uint8_t *maxs, void *stream);

int ro_evict_bricks(ro_ctx *ctx, const ro_state *state, const int64_t *ids,
                    int64_t n, int32_t update_octree, void *stream);
int ro_mark_empty(ro_ctx *ctx, const ro_state *state, const int64_t *ids,
                  int64_t n, void *stream);

/* HOST arrays of n; later entries win on duplicates. */
int ro_apply_metadata(ro_ctx *ctx, const ro_state *state,
                      const int64_t *node_idx, const int32_t *slot,
                      const int32_t *mn, const int32_t *mx, int64_t n,
                      void *stream);

/* Device grids [side^3] (z, y, x order) of node min/max for octree depth d. */
int ro_write_level_metadata(ro_ctx *ctx, const ro_state *state, int32_t slot,
                            int32_t d, const uint8_t *mins, const uint8_t *maxs,
                            void *stream);

int ro_swap_channel(ro_ctx *ctx, const ro_state *state, int32_t channel_slot,
                    int32_t invalidate_octree, void *stream);

/* ids: HOST array of changed bricks; their leaves are recomputed from the
   current page table, then ancestors re-ORed. */
int ro_octree_update(ro_ctx *ctx, const ro_state *state, const int64_t *ids,
                     int64_t n, void *stream);

int ro_rebuild_masks(ro_ctx *ctx, const ro_state *state, void *stream);

/* Reference-layout state on the HOST (paging.py:95-112 arrays,
   octree.py:116-118 words): pt_status i8[E] (0 UNMAPPED, 1 MAPPED, 2 EMPTY)
   + pt_slot i32[E], words u32[N*m] (may be NULL), cache u8[S*bvox],
   slot_brick / slot_last_used i64[S], the LIFO free list (top last). */
typedef struct ro_host_state {
    const int8_t *pt_status;
    const int32_t *pt_slot;
    const uint32_t *words;
    const uint8_t *cache;
    const int64_t *slot_brick;
    const int64_t *slot_last_used;
    const int32_t *free_list;
    int64_t free_count;
} ro_host_state;

/* Copy a reference-layout host state into the device state (packing the
   page table; sub_max, if present, is rebuilt from the cache).  Synchronises
   the stream. */
int ro_upload_state(ro_ctx *ctx, const ro_host_state *host, const ro_state *state,
                    void *stream);
/* The inverse (host arrays written: pt_status, pt_slot, words, cache,
   slot_brick, slot_last_used, free_list; *free_count_out = free count).
   Synchronises the stream. */
int ro_download_state(ro_ctx *ctx, const ro_state *state, int8_t *pt_status,
                      int32_t *pt_slot, uint32_t *words, uint8_t *cache,
                      int64_t *slot_brick, int64_t *slot_last_used, int32_t *free_list,
                      int64_t *free_count_out, void *stream);

/* ---- sort-first over peer memory ----
   The parts of a frame write straight into one set of buffers: each GPU's
   ray caster stores its pixels into the owner's full-frame image, its usage
   marks / histogram / counters into the owner's, and its first-seen request
   keys into the owner's key arrays with the same RED.MIN atomics a single GPU
   uses -- so the owner's ro_feedback_collect yields exactly the single-GPU
   request lists.  Buffers are shared through CUDA IPC (NVLink / NVSwitch
   peer access), set up by the host (torch's CUDA IPC in distributed.py). */

/* Use caller-owned first-seen key arrays instead of the context's own:
   brick_keys u64[E], meta_keys u64[N*m] (device, every element 0xFF..FF
   between frames; ro_feedback_collect restores that).  The frame's owner
   passes arrays it allocated; every other part passes the owner's arrays
   mapped into its address space (peer memory), so all parts' RED.MIN
   request atomics land in one place.  NULL, NULL returns to the context's
   own arrays.  The context never frees external arrays. */
int ro_set_feedback_buffers(ro_ctx *ctx, unsigned long long *brick_keys,
                            unsigned long long *meta_keys);
/* Let kernels of the current device access `peer_device`'s memory
   (cudaDeviceEnablePeerAccess; already-enabled is not an error). */
int ro_enable_peer_access(int32_t peer_device);

int ro_sync(ro_ctx *ctx, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RESOCT_H */
