// ingest.cu -- brick ingest into the cache on the GPU.
//
//  * LZ4 frame decode.  Bricks travel as standard LZ4 frames
//    (/root/reference/pkg/src/resoctree/lz4io.py:1-110, the system liblz4
//    1.9.4 frame API: LZ4F_compressFrame / LZ4F_decompress), decoded on the
//    host by ingest.py:114-117 (decompress_brick) after every fetch
//    (service.py:71-76, 225-232).  Here the compressed frames are uploaded
//    and decoded by one warp per frame straight into device memory, then
//    inserted by the batched LRU path (ro_apply_bricks_lz4): the PCIe bytes
//    shrink by the compression ratio and no CPU core decompresses.
//    The decoder follows the published LZ4 frame / block format: magic,
//    FLG/BD descriptor with its xxHash32 header checksum, linked or
//    independent blocks up to the declared maximum size, raw (stored) blocks,
//    optional block / content checksums (xxHash32) and content size.
//  * range normalisation to u8 (ingest.py:27-35), 2x box downsampling
//    (ingest.py:38-61) and brick cutting with edge replication
//    (ingest.py:75-95), for building pyramids of device-resident volumes.
//    The reference computes these in fp64; the results are exact small
//    binary fractions, so the integer forms below are bit-identical.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace ro {

int apply_bricks(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                 const void *payloads, int32_t on_device, int64_t frame,
                 int32_t update_octree, int32_t *slots_out, int64_t *evicted_out,
                 cudaStream_t s);

namespace {

constexpr int kLz4Warps = 4;  // warps (frames) per CTA (one-warp decoder)
#ifndef RO_LZ4_PIPE
#define RO_LZ4_PIPE 1
#endif
#ifndef RO_LZ4_MAP
#define RO_LZ4_MAP 1
#endif
#ifndef RO_LZ4_FAST
#define RO_LZ4_FAST 1
#endif
#ifndef RO_DEBUG_CHECKS
#define RO_DEBUG_CHECKS 0
#endif
#if RO_DEBUG_CHECKS  // debug builds: trap on any out-of-range index
#define LZ_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define LZ_ASSERT(c) do { } while (0)
#endif

enum : int32_t {
    LZ4_OK = 0,
    LZ4_E_MAGIC = -1,      // not an LZ4 frame (or a skippable / legacy one)
    LZ4_E_HEADER = -2,     // bad descriptor or header checksum
    LZ4_E_BLOCKSIZE = -3,  // block larger than the declared maximum
    LZ4_E_TRUNCATED = -4,  // input ends inside the frame
    LZ4_E_CORRUPT = -5,    // malformed block (bad offset / overrun)
    LZ4_E_SIZE = -6,       // decoded size differs from the expected one
    LZ4_E_CHECKSUM = -7,   // block or content checksum mismatch
    LZ4_E_TRAILING = -8,   // bytes after the end of the frame
};

__device__ __forceinline__ uint32_t rd32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
           ((uint32_t)p[3] << 24);
}

__device__ __forceinline__ uint32_t rotl32(uint32_t x, int r) {
    return (x << r) | (x >> (32 - r));
}

// xxHash32 (the frame format's checksum), computed identically by every lane
__device__ uint32_t xxh32(const uint8_t *p, int64_t len, uint32_t seed) {
    const uint32_t P1 = 2654435761u, P2 = 2246822519u, P3 = 3266489917u,
                   P4 = 668265263u, P5 = 374761393u;
    int64_t i = 0;
    uint32_t h;
    if (len >= 16) {
        uint32_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        for (; i + 16 <= len; i += 16) {
            v1 = rotl32(v1 + rd32(p + i) * P2, 13) * P1;
            v2 = rotl32(v2 + rd32(p + i + 4) * P2, 13) * P1;
            v3 = rotl32(v3 + rd32(p + i + 8) * P2, 13) * P1;
            v4 = rotl32(v4 + rd32(p + i + 12) * P2, 13) * P1;
        }
        h = rotl32(v1, 1) + rotl32(v2, 7) + rotl32(v3, 12) + rotl32(v4, 18);
    } else {
        h = seed + P5;
    }
    h += (uint32_t)len;
    for (; i + 4 <= len; i += 4) h = rotl32(h + rd32(p + i) * P3, 17) * P4;
    for (; i < len; ++i) h = rotl32(h + p[i] * P5, 11) * P1;
    h ^= h >> 15;
    h *= P2;
    h ^= h >> 13;
    h *= P3;
    h ^= h >> 16;
    return h;
}

// Byte sources of the parser.  GlobalBytes reads the frame where it lies;
// SmemBytes reads a copy in shared memory (4-byte aligned, >= 8 bytes of
// slack) and can fetch an 8-byte window in two word loads, so the common
// sequence (token, short literal run, 2-byte offset) costs one dependent
// load instead of three.
struct GlobalBytes {
    const uint8_t *p;
    static constexpr bool kWindow = false;
    __device__ uint32_t u8(int64_t i) const { return p[i]; }
    __device__ uint64_t win8(int64_t) const { return 0; }
};
struct SmemBytes {
    const uint32_t *w;
    static constexpr bool kWindow = true;
    __device__ uint32_t u8(int64_t i) const { return (w[i >> 2] >> ((i & 3) << 3)) & 0xFFu; }
    __device__ uint64_t win8(int64_t i) const {
        const int64_t q = i >> 2;
        const int r = (int)(i & 3) << 3;
        const uint64_t lo = (uint64_t)w[q] | ((uint64_t)w[q + 1] << 32);
        return r ? (lo >> r) | ((uint64_t)w[q + 2] << (64 - r)) : lo;
    }
};

// The LZ4 frame / block parser, generic over a sink that receives literal
// runs (offset in the frame, length) and matches (offset, length) in stream
// order.  All lanes of the warp parse the same bytes (broadcast loads), so
// control flow stays warp-uniform.  `op` tracks the output position for the
// bounds / offset checks; the sink produces the bytes.
template <class Sink, class Src>
__device__ int32_t lz4_block_parse(const Src &src, int64_t bpos, int64_t bl, Sink &sink,
                                   int64_t &op, int64_t low, int64_t limit) {
    int64_t ip = 0;
    while (true) {
        if (ip >= bl) return LZ4_E_CORRUPT;
        uint64_t win = 0;
        uint32_t token;
        if (Src::kWindow) {
            win = src.win8(bpos + ip);
            token = (uint32_t)win & 0xFFu;
        } else {
            token = src.u8(bpos + ip);
        }
        const int64_t ip0 = ip++;
        int64_t lit = token >> 4;
        if (lit == 15) {
            uint32_t s;
            do {
                if (ip >= bl) return LZ4_E_CORRUPT;
                s = src.u8(bpos + ip++);
                lit += s;
            } while (s == 255);
        }
        if (ip + lit > bl || op + lit > limit) return LZ4_E_CORRUPT;
        const int64_t lit_at = bpos + ip;
        ip += lit;
        if (ip == bl) {  // the last sequence holds literals only
            sink.seq(lit_at, lit, 0, 0, op);
            op += lit;
            return LZ4_OK;
        }
        if (ip + 2 > bl) return LZ4_E_CORRUPT;
        int64_t off;
        if (Src::kWindow && ip + 2 - ip0 <= 8) {
            off = (int64_t)((win >> ((ip - ip0) << 3)) & 0xFFFFu);
        } else {
            off = (int64_t)src.u8(bpos + ip) | ((int64_t)src.u8(bpos + ip + 1) << 8);
        }
        ip += 2;
        int64_t ml = token & 15;
        if (ml == 15) {
            uint32_t s;
            do {
                if (ip >= bl) return LZ4_E_CORRUPT;
                s = src.u8(bpos + ip++);
                ml += s;
            } while (s == 255);
        }
        ml += 4;
        if (off == 0 || off > op + lit - low || op + lit + ml > limit) {
            // report the position the copying decoder would have reached
            op += lit;
            return LZ4_E_CORRUPT;
        }
        sink.seq(lit_at, lit, off, ml, op);
        op += lit + ml;
    }
}

// One frame; the sink receives every byte-producing run in order.  Returns
// the decoded size or an LZ4_E_* code.  `content` (optional) receives the
// position of the content checksum for a sink that checks it later.
template <class Sink, class Src = GlobalBytes>
__device__ int64_t lz4_frame_parse(const uint8_t *__restrict__ src, int64_t len, int64_t cap,
                                   Sink &sink, int64_t *cchk_at, const Src &bytes = Src{}) {
    if (len < 7) return LZ4_E_TRUNCATED;
    if (rd32(src) != 0x184D2204u) return LZ4_E_MAGIC;
    const uint32_t flg = src[4], bd = src[5];
    if ((flg >> 6) != 1 || (flg & 0x02) || (bd & 0x8F)) return LZ4_E_HEADER;
    const int bsid = (bd >> 4) & 7;
    if (bsid < 4) return LZ4_E_HEADER;
    const int64_t bmax = (int64_t)1 << (8 + 2 * bsid);  // 64 KB .. 4 MB
    const bool indep = flg & 0x20, bchk = flg & 0x10, has_size = flg & 0x08,
               cchk = flg & 0x04, has_dict = flg & 0x01;
    int64_t pos = 6;
    int64_t csize = -1;
    if (has_size) {
        if (len < pos + 8) return LZ4_E_TRUNCATED;
        csize = (int64_t)rd32(src + pos) | ((int64_t)rd32(src + pos + 4) << 32);
        pos += 8;
    }
    if (has_dict) pos += 4;
    if (len < pos + 1) return LZ4_E_TRUNCATED;
    if (((xxh32(src + 4, pos - 4, 0) >> 8) & 0xFF) != src[pos]) return LZ4_E_HEADER;
    pos += 1;
    int64_t op = 0;
    while (true) {
        if (pos + 4 > len) return LZ4_E_TRUNCATED;
        const uint32_t bs = rd32(src + pos);
        pos += 4;
        if (bs == 0) break;  // EndMark
        const bool raw = bs >> 31;
        const int64_t bl = bs & 0x7FFFFFFFu;
        if (bl > bmax) return LZ4_E_BLOCKSIZE;
        if (pos + bl + (bchk ? 4 : 0) > len) return LZ4_E_TRUNCATED;
        if (bchk && xxh32(src + pos, bl, 0) != rd32(src + pos + bl)) return LZ4_E_CHECKSUM;
        const int64_t start = op;
        const int64_t limit = min(cap, op + bmax);
        if (raw) {
            if (op + bl > limit) return LZ4_E_SIZE;
            sink.seq(pos, bl, 0, 0, op);
            op += bl;
        } else {
            int32_t rc;
            if (Src::kWindow)
                rc = lz4_block_parse(bytes, pos, bl, sink, op, indep ? start : 0, limit);
            else
                rc = lz4_block_parse(GlobalBytes{src}, pos, bl, sink, op, indep ? start : 0,
                                     limit);
            if (rc != LZ4_OK) return rc == LZ4_E_CORRUPT && op >= limit ? LZ4_E_SIZE : rc;
        }
        pos += bl + (bchk ? 4 : 0);
    }
    if (cchk) {
        if (pos + 4 > len) return LZ4_E_TRUNCATED;
        if (cchk_at) *cchk_at = pos;
        else if (!sink.content_ok(op, rd32(src + pos))) return LZ4_E_CHECKSUM;
        pos += 4;
    }
    if (has_size && op != csize) return LZ4_E_SIZE;
    if (pos != len) return LZ4_E_TRAILING;
    return op;
}

// Sink of the one-warp decoder: lanes copy literal runs from the frame and
// matches from the output.  An overlapping match (offset < length) repeats
// the last `offset` bytes, so output byte j is dst[op - off + j % off]: every
// lane reads only bytes that are already final.
struct CopySink {
    const uint8_t *src;
    uint8_t *dst;
    int lane;
    __device__ void seq(int64_t lit_at, int64_t lit, int64_t off, int64_t ml, int64_t op) {
        for (int64_t i = lane; i < lit; i += 32) dst[op + i] = src[lit_at + i];
        if (!ml) return;  // a literal-only (last) sequence: nothing reads it here
        op += lit;
        __syncwarp();  // literals of this / earlier sequences visible to all lanes
        const int64_t base = op - off;
        if (off >= ml) {
            for (int64_t j = lane; j < ml; j += 32) dst[op + j] = dst[base + j];
        } else {
            for (int64_t j = lane; j < ml; j += 32) dst[op + j] = dst[base + j % off];
        }
        __syncwarp();
    }
    __device__ bool content_ok(int64_t n, uint32_t want) {
        __syncwarp();  // every lane's literal stores visible before hashing
        return xxh32(dst, n, 0) == want;
    }
};

__device__ int64_t lz4_frame_warp(const uint8_t *__restrict__ src, int64_t len, uint8_t *dst,
                                  int64_t cap, int lane) {
    CopySink sink{src, dst, lane};
    return lz4_frame_parse(src, len, cap, sink, nullptr);
}

// ---- two-warp pipelined decode (bricks up to 64 KB) --------------------------
// Warp 0 parses and validates the frame and emits one record per sequence
// into a shared-memory ring; warp 1 consumes the records in order and
// assembles the brick in shared memory (match sources are on-chip), while
// the parser runs ahead.  Producer / consumer synchronise through two
// counters in shared memory (both warps of the same CTA).
struct LzRec {
    int32_t lit_at, lit, off, ml;  // ml < 0: end of stream
};
constexpr int kRing = 256;

// Records are published in groups of kPublish: one fence + head store per
// group instead of per sequence (a noise-floor brick has ~6,700 of them).
constexpr int kPublish = 32;

struct EmitSink {
    LzRec *ring;
    volatile int *head, *tail;
    int h;
    int lane;
    int published = 0;
    int tail_seen = 0;  // last tail read: the ring has room while h - tail_seen < kRing
    __device__ void publish() {
        __threadfence_block();
        __syncwarp();
        if (lane == 0) *head = h;
        published = h;
    }
    __device__ void push(int32_t a, int32_t l, int32_t o, int32_t m) {
        if (h - tail_seen >= kRing) {
            tail_seen = *tail;
            if (h - tail_seen >= kRing) {
                publish();  // the consumer may be waiting for these
                while (h - (tail_seen = *tail) >= kRing) {
                }
            }
        }
        if (lane == 0) ring[h % kRing] = LzRec{a, l, o, m};
        ++h;
        if (m < 0 || h - published >= kPublish) publish();
    }
    __device__ void seq(int64_t lit_at, int64_t lit, int64_t off, int64_t ml, int64_t) {
        push((int32_t)lit_at, (int32_t)lit, (int32_t)off, (int32_t)ml);
    }
    __device__ bool content_ok(int64_t, uint32_t) { return true; }  // checked after copying
};

// The compressed frame itself is first copied into shared memory (when it
// fits in fin_cap bytes): the parse is a serial chain of dependent byte
// reads (token -> literal length -> offset -> match length -> next token),
// so its speed is the load latency, and shared memory answers several
// times sooner than L1 / L2.
__global__ void __launch_bounds__(64)
k_lz4_decode_pipe(int64_t n, const uint8_t *__restrict__ src, const int64_t *__restrict__ off,
                  uint8_t *__restrict__ dst, int64_t stride, int64_t expected,
                  int32_t *__restrict__ status, int32_t *__restrict__ first_bad,
                  int64_t fin_cap) {
    extern __shared__ __align__(16) uint8_t sh[];
    uint8_t *out = sh;
    const int64_t out_bytes = (stride + 15) & ~(int64_t)15;
    LzRec *ring = reinterpret_cast<LzRec *>(sh + out_bytes);
    uint8_t *fin = sh + out_bytes + sizeof(LzRec) * kRing;  // 16-byte aligned
    __shared__ int s_head, s_tail;
    __shared__ long long s_result, s_cchk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const int64_t o0 = off[0];
    const int64_t a = off[i] - o0, b = off[i + 1] - o0;
    const uint8_t *f = src + a;
    const bool staged = b >= a && b - a <= fin_cap;
    if (staged) {
        const int64_t len = b - a;
        for (int64_t j = threadIdx.x; j < len; j += 64) fin[j] = f[j];
        for (int64_t j = len + threadIdx.x; j < len + 16; j += 64) fin[j] = 0;  // window slack
        f = fin;
    }
    if (threadIdx.x == 0) {
        s_head = 0;
        s_tail = 0;
        s_cchk = -1;
    }
    __syncthreads();
    if (warp == 0) {
        EmitSink sink{ring, &s_head, &s_tail, 0, lane};
        int64_t cchk = -1;
        int64_t r;
        if (b < a)
            r = LZ4_E_TRUNCATED;
        else if (staged)
            r = lz4_frame_parse(f, b - a, stride, sink, &cchk,
                                SmemBytes{reinterpret_cast<const uint32_t *>(fin)});
        else
            r = lz4_frame_parse(f, b - a, stride, sink, &cchk);
        sink.push(0, 0, 0, -1);  // end of stream
        if (lane == 0) {
            s_result = r;
            s_cchk = cchk;
        }
    } else {
        int t = 0, avail = 0;
        int64_t op = 0;
        while (true) {
            if (t == avail) {  // every published record consumed: hand back, wait
                if (lane == 0) *(volatile int *)&s_tail = t;
                while ((avail = *(volatile int *)&s_head) == t) {
                }
                __threadfence_block();
            }
            const LzRec r = ring[t % kRing];
            if (r.ml < 0) break;
            for (int64_t q = lane; q < r.lit; q += 32) out[op + q] = f[r.lit_at + q];
            op += r.lit;
            if (r.ml) {
                __syncwarp();
                const int64_t base = op - r.off;
                if (r.off >= r.ml) {
                    for (int64_t j = lane; j < r.ml; j += 32) out[op + j] = out[base + j];
                } else {
                    for (int64_t j = lane; j < r.ml; j += 32) out[op + j] = out[base + j % r.off];
                }
                op += r.ml;
            }
            __syncwarp();
            ++t;
            if (lane == 0 && (t & (kPublish - 1)) == 0) *(volatile int *)&s_tail = t;
        }
    }
    __syncthreads();
    int64_t r = s_result;
    if (r >= 0 && s_cchk >= 0) {   // content checksum over the assembled brick
        const bool ok = xxh32(out, r, 0) == rd32(f + s_cchk);
        if (!ok) r = LZ4_E_CHECKSUM;
    }
    if (r >= 0 && expected >= 0 && r != expected) r = LZ4_E_SIZE;
    if (r >= 0) {
        uint8_t *outp = dst + i * stride;
        if ((((uintptr_t)outp) & 15) == 0) {
            const int64_t n16 = r >> 4;
            for (int64_t j = threadIdx.x; j < n16; j += 64)
                reinterpret_cast<uint4 *>(outp)[j] = reinterpret_cast<const uint4 *>(out)[j];
            for (int64_t j = (n16 << 4) + threadIdx.x; j < r; j += 64) outp[j] = out[j];
        } else {
            for (int64_t j = threadIdx.x; j < r; j += 64) outp[j] = out[j];
        }
    }
    if (threadIdx.x == 0) {
        status[i] = r < 0 ? (int32_t)r : 0;
        if (r < 0 && first_bad) atomicMin(first_bad, (int32_t)i);
    }
}

// ---- one-CTA decode through a source map (bricks up to 32 KB) ---------------
// The pipe decoder executes the sequences strictly in order, one record per
// warp step, behind a parser whose every step is a chain of dependent byte
// reads: a noise-floor brick of ~6,700 sequences takes ~1.8 ms however many
// SMs are idle.  Here the whole CTA decodes one frame and only one dependent
// load per sequence stays serial:
//   A. every byte position p of the block is parsed AS IF a sequence started
//      there (all threads): next[p] = where the following token would be
//      (or "impossible"), next2[p] = next[next[p]], next4[p] likewise;
//   B. one thread follows the chain from position 0 -- one shared-memory
//      load per FOUR sequences -- and marks where each group of four starts;
//   C. all threads re-parse the marked groups, place them with a CTA
//      prefix sum of their lengths, and write a SOURCE per output byte:
//      literal j of the frame (flagged) or output byte op - offset (a match;
//      overlapping matches just point a few bytes back), checking offsets
//      against the output position;
//   D. pointer jumping (map[i] = map[map[i]]) until every byte points at a
//      literal, O(log chain) rounds, then one parallel gather writes the
//      brick.
// Frames of anything but one data block (+ EndMark), any position the
// fast path cannot vouch for, or any malformed sequence re-run the serial
// parser over the whole frame (MapSink, warp 0), which yields the exact
// LZ4_E_* code -- the accept / reject set and the bytes are the serial
// decoder's.
constexpr uint32_t kLitRef = 0x80000000u;
constexpr int kMapThreads = 512;
[[maybe_unused]] constexpr int kMapCap = 32 * 1024;  // output bytes (map entries) per frame
constexpr int64_t kFallback = -100;  // internal: re-run the serial parser

struct MapSink {
    uint32_t *map;
    int lane;
    __device__ void seq(int64_t lit_at, int64_t lit, int64_t off, int64_t ml, int64_t op) {
        const int o = (int)op, la = (int)lit_at, l = (int)lit;
        LZ_ASSERT(o >= 0 && o + l + (int)ml <= kMapCap);
        for (int q = lane; q < l; q += 32) map[o + q] = kLitRef | (uint32_t)(la + q);
        if (!ml) return;
        const int mo = o + l, of = (int)off, m = (int)ml;
        LZ_ASSERT(mo - of >= 0);
        for (int j = lane; j < m; j += 32) map[mo + j] = (uint32_t)(mo + j - of);
    }
    __device__ bool content_ok(int64_t, uint32_t) { return true; }  // checked after the gather
};

// One sequence parsed at block position p (block bytes b[0, bl)).  Returns
// false when no valid sequence can start there.  last = the block ends right
// after its literals.  A non-last sequence ending exactly at bl is invalid
// (the next token read would overrun), as in lz4_block_parse.
__device__ __forceinline__ bool seq_at(const uint8_t *b, int bl, int p, int cap, int &lit_at,
                                       int &lit, int &off, int &ml, int &nx, bool &last) {
    const uint32_t token = b[p];
    int q = p + 1;
    lit = (int)(token >> 4);
    if (lit == 15) {
        uint32_t x;
        do {
            if (q >= bl || lit > cap) return false;
            x = b[q++];
            lit += (int)x;
        } while (x == 255);
    }
    if (lit > cap || q + lit > bl) return false;
    lit_at = q;
    q += lit;
    if (q == bl) {
        last = true;
        off = 0;
        ml = 0;
        nx = bl;
        return true;
    }
    last = false;
    if (q + 2 > bl) return false;
    off = (int)b[q] | ((int)b[q + 1] << 8);
    q += 2;
    ml = (int)(token & 15);
    if (ml == 15) {
        uint32_t x;
        do {
            if (q >= bl || ml > cap) return false;
            x = b[q++];
            ml += (int)x;
        } while (x == 255);
    }
    ml += 4;
    if (lit + ml > cap || q >= bl) return false;
    nx = q;
    return true;
}

// exclusive prefix sum over the CTA (kMapThreads threads); *total = the sum
__device__ __forceinline__ int cta_exclusive_scan(int v, int *scratch, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kMapThreads / 32 ? scratch[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        if (lane < kMapThreads / 32) scratch[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int before = (warp ? scratch[warp - 1] : 0) + x - v;
    *total = scratch[kMapThreads / 32 - 1];
    __syncthreads();  // scratch reusable
    return before;
}

// Phases A-C for one compressed block at frame offset bpos (whole CTA).
// The map region (u32[pcap]) first holds next[] and next2[] (u16 each), nx4
// (u16[pcap], its own region) next4[] whose top bit marks the starts of the
// true chain's groups of four sequences; the map region then receives the
// map.  Returns the output end or kFallback.
__device__ int64_t block_fast(const uint8_t *fin, int bpos, int bl, int op0, int low, int limit,
                              uint32_t *map, uint16_t *nx4, int pcap, int *s_bad, int *scan) {
    const uint8_t *b = fin + bpos;
    const int tid = threadIdx.x;
    const int cap = limit - op0;
    constexpr uint32_t kErr = 0x7FFF, kMark = 0x8000;
    if (bl < 1 || bl >= (int)kErr || bl > pcap || cap > 0xFFFF) return kFallback;
    uint16_t *nx1 = reinterpret_cast<uint16_t *>(map);
    uint16_t *nx2 = nx1 + pcap;
    // A: where the next token would be if a sequence started at p (bl: the
    // block ends after p's literals; kErr: no valid sequence at p), then
    // two and four sequences on (bl / kErr propagate)
    for (int p = tid; p < bl; p += kMapThreads) {
        int la, l, o, m, nx;
        bool last;
        nx1[p] = (uint16_t)(seq_at(b, bl, p, cap, la, l, o, m, nx, last) ? nx : kErr);
    }
    __syncthreads();
    for (int p = tid; p < bl; p += kMapThreads) {
        const uint32_t q = nx1[p];
        nx2[p] = (uint16_t)(q < (uint32_t)bl ? nx1[q] : q);
    }
    __syncthreads();
    for (int p = tid; p < bl; p += kMapThreads) {
        const uint32_t q = nx2[p];
        nx4[p] = (uint16_t)(q < (uint32_t)bl ? nx2[q] : q);
    }
    __syncthreads();
    // B: the true chain from position 0, FOUR sequences per dependent load
    // (next4 < bl implies the three in between are valid); the group starts
    // are marked in next4[]; the last group is checked one step at a time
    if (tid == 0) {
        uint32_t s = 0;
        int bad = 0;
        while (true) {
            const uint32_t a4 = nx4[s];
            nx4[s] = (uint16_t)(a4 | kMark);
            if (a4 >= (uint32_t)bl) {
                uint32_t c = s;
                for (int k = 0; k < 4; ++k) {
                    c = nx1[c];
                    if (c >= (uint32_t)bl) break;
                }
                bad = c != (uint32_t)bl;
                break;
            }
            s = a4;
        }
        *s_bad = bad;
    }
    __syncthreads();
    if (*s_bad) return kFallback;
    // C: output offsets of the marked groups (CTA scan over position chunks),
    // then the sources of every output byte
    constexpr int kChunk = 64;  // bl <= 32 K positions over 512 threads
    const int c0 = tid * kChunk, c1 = min(bl, c0 + kChunk);
    uint64_t marks = 0;
    int sum = 0;
    for (int p = c0; p < c1; ++p) {
        if (nx4[p] & kMark) {
            marks |= 1ull << (p - c0);
            int c = p;
            for (int k = 0; k < 4; ++k) {
                int la, l, of, m, nx;
                bool last;
                seq_at(b, bl, c, cap, la, l, of, m, nx, last);
                sum += l + m;
                if (last) break;
                c = nx;
            }
        }
    }
    int total;
    int o = op0 + cta_exclusive_scan(sum, scan, &total);  // also orders the reads above
    if (total > cap) return kFallback;
    int bad = 0;
    while (marks) {
        int c = c0 + __ffsll((long long)marks) - 1;
        marks &= marks - 1;
        for (int k = 0; k < 4; ++k) {
            int la, l, of, m, nx;
            bool last;
            seq_at(b, bl, c, cap, la, l, of, m, nx, last);
            const uint32_t lsrc = (uint32_t)(bpos + la);
            LZ_ASSERT(o >= 0 && o + l + m <= pcap && la + l <= bl);
            for (int q = 0; q < l; ++q) map[o + q] = kLitRef | (lsrc + q);
            o += l;
            if (last) break;
            if (of == 0 || of > o - low) bad = 1;
            if (bad) {  // the CTA falls back to the serial parser
                marks = 0;
                break;
            }
            for (int q = 0; q < m; ++q) map[o + q] = (uint32_t)(o + q - of);
            o += m;
            c = nx;
        }
    }
    if (__syncthreads_or(bad)) return kFallback;
    return op0 + total;
}

// The frame when it is exactly [header][one block][EndMark][checksums]: all
// threads walk the header (validated as lz4_frame_parse does); the block is
// decoded by block_fast, a raw block mapped directly.
__device__ int64_t frame_fast(const uint8_t *src, int64_t len, int64_t cap, uint32_t *P,
                              uint16_t *nx4, int pcap, int *s_bad, int *scan, int64_t *cchk_at) {
    if (len < 7 || rd32(src) != 0x184D2204u) return kFallback;
    const uint32_t flg = src[4], bd = src[5];
    if ((flg >> 6) != 1 || (flg & 0x02) || (bd & 0x8F)) return kFallback;
    const int bsid = (bd >> 4) & 7;
    if (bsid < 4) return kFallback;
    const int64_t bmax = (int64_t)1 << (8 + 2 * bsid);
    const bool bchk = flg & 0x10, has_size = flg & 0x08, cchk = flg & 0x04,
               has_dict = flg & 0x01;
    int64_t pos = 6, csize = -1;
    if (has_size) {
        if (len < pos + 8) return kFallback;
        csize = (int64_t)rd32(src + pos) | ((int64_t)rd32(src + pos + 4) << 32);
        pos += 8;
    }
    if (has_dict) pos += 4;
    if (len < pos + 1) return kFallback;
    if (((xxh32(src + 4, pos - 4, 0) >> 8) & 0xFF) != src[pos]) return kFallback;
    pos += 1;
    if (pos + 4 > len) return kFallback;
    const uint32_t bs = rd32(src + pos);
    pos += 4;
    int64_t op = 0;
    if (bs != 0) {
        const bool raw = bs >> 31;
        const int64_t bl = bs & 0x7FFFFFFFu;
        if (bl > bmax || pos + bl + (bchk ? 4 : 0) + 4 > len) return kFallback;
        if (bchk && xxh32(src + pos, bl, 0) != rd32(src + pos + bl)) return kFallback;
        const int64_t limit = min(cap, bmax);
        if (raw) {
            if (bl > limit) return kFallback;
            for (int q = threadIdx.x; q < (int)bl; q += kMapThreads)
                P[q] = kLitRef | (uint32_t)(pos + q);
            op = bl;
        } else {
            op = block_fast(src, (int)pos, (int)bl, 0, 0, (int)limit, P, nx4, pcap, s_bad, scan);
            if (op < 0) return kFallback;
        }
        pos += bl + (bchk ? 4 : 0);
        if (rd32(src + pos) != 0) return kFallback;  // a second block: serial path
        pos += 4;
    }
    if (cchk) {
        if (pos + 4 > len) return kFallback;
        *cchk_at = pos;
        pos += 4;
    }
    if (has_size && op != csize) return kFallback;
    if (pos != len) return kFallback;
    return op;
}

__global__ void __launch_bounds__(kMapThreads)
k_lz4_decode_map(int64_t n, const uint8_t *__restrict__ src, const int64_t *__restrict__ off,
                 uint8_t *__restrict__ dst, int64_t stride, int64_t expected,
                 int32_t *__restrict__ status, int32_t *__restrict__ first_bad,
                 int64_t fin_cap, int pcap) {
    extern __shared__ __align__(16) uint8_t sh[];
    uint32_t *map = reinterpret_cast<uint32_t *>(sh);
    uint16_t *nx4 = reinterpret_cast<uint16_t *>(map + pcap);
    uint8_t *fin = reinterpret_cast<uint8_t *>(nx4 + pcap);  // 16-byte aligned
    __shared__ long long s_result, s_cchk;
    __shared__ int s_bad, s_scan[kMapThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const int64_t o0 = off[0];
    const int64_t a = off[i] - o0, b = off[i + 1] - o0;
    const uint8_t *f = src + a;
    const bool staged = b >= a && b - a <= fin_cap;
    if (staged) {
        const int64_t len = b - a;
        for (int64_t j = tid; j < len; j += kMapThreads) fin[j] = f[j];
        for (int64_t j = len + tid; j < len + 16; j += kMapThreads) fin[j] = 0;  // window slack
        f = fin;
    }
    __syncthreads();
    int64_t cchk = -1;
    int64_t r = kFallback;
#if RO_LZ4_FAST
    if (staged) r = frame_fast(f, b - a, stride, map, nx4, pcap, &s_bad, s_scan, &cchk);
#endif
    if (r == kFallback) {
        __syncthreads();
        if (tid < 32) {
            MapSink sink{map, lane};
            int64_t rr;
            cchk = -1;
            if (b < a)
                rr = LZ4_E_TRUNCATED;
            else if (staged)
                rr = lz4_frame_parse(f, b - a, stride, sink, &cchk,
                                     SmemBytes{reinterpret_cast<const uint32_t *>(fin)});
            else
                rr = lz4_frame_parse(f, b - a, stride, sink, &cchk);
            if (lane == 0) {
                s_result = rr;
                s_cchk = cchk;
            }
        }
        __syncthreads();
        r = s_result;
        cchk = s_cchk;
    }
    if (r >= 0 && expected >= 0 && r != expected) r = LZ4_E_SIZE;
    if (r >= 0) {
        const int nr = (int)r;
        // pointer jumping: every entry ends on a literal reference.  An entry
        // read while another thread rewrites it is either value -- both lie
        // on the same chain -- so rounds need no ordering beyond the barrier.
        while (true) {
            int pending = 0;
            for (int q = tid; q < nr; q += kMapThreads) {
                const uint32_t v = map[q];
                if (!(v & kLitRef)) {
                    LZ_ASSERT(v < (uint32_t)q);
                    const uint32_t w = map[v];
                    map[q] = w;
                    pending |= !(w & kLitRef);
                }
            }
            if (!__syncthreads_or(pending)) break;
        }
        uint8_t *outp = dst + i * stride;
        if ((((uintptr_t)outp) & 3) == 0) {
            const int n4 = nr >> 2;
            for (int q = tid; q < n4; q += kMapThreads) {
                const uint4 m4 = reinterpret_cast<const uint4 *>(map)[q];
                const uint32_t v = (uint32_t)f[m4.x & ~kLitRef] |
                                   ((uint32_t)f[m4.y & ~kLitRef] << 8) |
                                   ((uint32_t)f[m4.z & ~kLitRef] << 16) |
                                   ((uint32_t)f[m4.w & ~kLitRef] << 24);
                reinterpret_cast<uint32_t *>(outp)[q] = v;
            }
            for (int q = (n4 << 2) + tid; q < nr; q += kMapThreads) outp[q] = f[map[q] & ~kLitRef];
        } else {
            for (int q = tid; q < nr; q += kMapThreads) outp[q] = f[map[q] & ~kLitRef];
        }
        if (cchk >= 0) {  // content checksum over the written brick
            __syncthreads();
            if (xxh32(outp, r, 0) != rd32(f + cchk)) r = LZ4_E_CHECKSUM;
        }
    }
    if (tid == 0) {
        status[i] = r < 0 ? (int32_t)r : 0;
        if (r < 0 && first_bad) atomicMin(first_bad, (int32_t)i);
    }
}

__global__ void __launch_bounds__(32 * kLz4Warps)
k_lz4_decode(int64_t n, const uint8_t *__restrict__ src, const int64_t *__restrict__ off,
             uint8_t *__restrict__ dst, int64_t stride, int64_t expected,
             int32_t *__restrict__ status, int32_t *__restrict__ first_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * kLz4Warps + (threadIdx.x >> 5);
    if (i >= n) return;
    const int64_t o0 = off[0];
    const int64_t a = off[i] - o0, b = off[i + 1] - o0;
    int64_t r = (b < a) ? LZ4_E_TRUNCATED
                        : lz4_frame_warp(src + a, b - a, dst + i * stride, stride, lane);
    if (r >= 0 && expected >= 0 && r != expected) r = LZ4_E_SIZE;
    if (lane == 0) {
        status[i] = r < 0 ? (int32_t)r : 0;
        if (r < 0 && first_bad) atomicMin(first_bad, (int32_t)i);
    }
}

// ---- normalisation (ingest.py:27-35) ----------------------------------------

template <typename T> struct OrderedKey;
template <> struct OrderedKey<uint8_t> {
    static __device__ uint32_t of(uint8_t v) { return v; }
    static __device__ double val(uint32_t k) { return (double)k; }
};
template <> struct OrderedKey<uint16_t> {
    static __device__ uint32_t of(uint16_t v) { return v; }
    static __device__ double val(uint32_t k) { return (double)k; }
};
template <> struct OrderedKey<uint32_t> {
    static __device__ uint32_t of(uint32_t v) { return v; }
    static __device__ double val(uint32_t k) { return (double)k; }
};
template <> struct OrderedKey<float> {  // total order of finite floats
    static __device__ uint32_t of(float v) {
        const uint32_t u = __float_as_uint(v);
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    }
    static __device__ double val(uint32_t k) {
        const uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
        return (double)__uint_as_float(u);
    }
};

template <typename T>
__global__ void k_minmax(int64_t n, const T *__restrict__ src, uint32_t *__restrict__ mm) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = OrderedKey<T>::of(src[i]);
        lo = min(lo, k);
        hi = max(hi, k);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

template <typename T>
__global__ void k_normalize(int64_t n, const T *__restrict__ src,
                            const uint32_t *__restrict__ mm, uint8_t *__restrict__ dst) {
    const double lo = OrderedKey<T>::val(mm[0]), hi = OrderedKey<T>::val(mm[1]);
    const bool flat = hi == lo;
    const double scale = flat ? 0.0 : 255.0 / (hi - lo);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t out = 0;
        if (!flat) {
            // numpy: floor((data - lo) * (255 / (hi - lo)) + 0.5).clip(0, 255)
            const double v = floor(((double)src[i] - lo) * scale + 0.5);
            out = (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
        }
        dst[i] = out;
    }
}

// ---- 2x box downsampling (ingest.py:38-61) ------------------------------------
// Each averaged axis halves exactly in fp64, so the reference's value is
// sum / 2^f and floor(sum / 2^f + 0.5) == (sum + 2^(f-1)) >> f.
__global__ void k_downsample_box(const uint8_t *__restrict__ src, int dx, int dy, int dz,
                                 int fx, int fy, int fz, int ox, int oy, int oz,
                                 uint8_t *__restrict__ dst) {
    const int64_t total = (int64_t)ox * oy * oz;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % ox), y = (int)((i / ox) % oy), z = (int)(i / ((int64_t)ox * oy));
        int sum = 0;
        for (int c = 0; c < fz; ++c) {
            const int zz = min(z * fz + c, dz - 1);
            for (int b = 0; b < fy; ++b) {
                const int yy = min(y * fy + b, dy - 1);
                for (int a = 0; a < fx; ++a) {
                    const int xx = min(x * fx + a, dx - 1);
                    sum += src[((int64_t)zz * dy + yy) * dx + xx];
                }
            }
        }
        const int f = (fx == 2) + (fy == 2) + (fz == 2);
        dst[i] = (uint8_t)(f ? (sum + (1 << (f - 1))) >> f : sum);
    }
}

// ---- brick cutting with edge replication (ingest.py:75-95) --------------------
// All bricks of one level in (z, y, x) grid order, 16 bytes per thread.
__global__ void k_extract_bricks(const uint8_t *__restrict__ level, int dx, int dy, int dz,
                                 int bx, int by, int bz, int gx, int gy, int64_t n_bricks,
                                 uint8_t *__restrict__ dst) {
    const int64_t bvox = (int64_t)bx * by * bz;
    const int64_t total = n_bricks * bvox;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t br = i / bvox, v = i % bvox;
        const int cx = (int)(br % gx), cy = (int)((br / gx) % gy), cz = (int)(br / ((int64_t)gx * gy));
        const int x = (int)(v % bx), y = (int)((v / bx) % by), z = (int)(v / ((int64_t)bx * by));
        const int xx = min(cx * bx + x, dx - 1), yy = min(cy * by + y, dy - 1),
                  zz = min(cz * bz + z, dz - 1);
        dst[i] = level[((int64_t)zz * dy + yy) * dx + xx];
    }
}

unsigned grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

const char *lz4_reason(int32_t code) {
    switch (code) {
        case LZ4_E_MAGIC: return "not an LZ4 frame";
        case LZ4_E_HEADER: return "bad frame descriptor or header checksum";
        case LZ4_E_BLOCKSIZE: return "block larger than the declared maximum";
        case LZ4_E_TRUNCATED: return "truncated LZ4 frame";
        case LZ4_E_CORRUPT: return "corrupt LZ4 block";
        case LZ4_E_SIZE: return "decompressed size differs from the brick size";
        case LZ4_E_CHECKSUM: return "LZ4 checksum mismatch";
        case LZ4_E_TRAILING: return "trailing bytes after LZ4 frame";
        default: return "LZ4 decode error";
    }
}

}  // namespace

int lz4_decode(ro_ctx *c, const uint8_t *src, const int64_t *off, int64_t n, uint8_t *dst,
               int64_t stride, int64_t expected, int32_t *status, int32_t *first_bad,
               cudaStream_t s) {
    (void)c;
    if (n <= 0) return RO_OK;
#if RO_LZ4_MAP
    // Small batches of bricks up to 32 KB: one CTA per frame
    // (k_lz4_decode_map: parallel parse + serial chain + pointer jumping)
    if (stride <= 32 * 1024) {
        // frames of one block up to 32 KB + framing are staged (any larger
        // one is parsed serially from global memory)
        const int64_t fin_cap = 32 * 1024 + 64;
        const int pcap = 32 * 1024;
        const size_t smem = (sizeof(uint32_t) + sizeof(uint16_t)) * (size_t)pcap +
                            (size_t)fin_cap + 16;
        int dev = 0, optin = 0, sms = 0;
        RO_CUDA(cudaGetDevice(&dev));
        RO_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        RO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (smem + 64 <= (size_t)optin && n <= sms) {
            static size_t attr = 0;
            if (attr < smem) {
                RO_CUDA(cudaFuncSetAttribute(k_lz4_decode_map,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                attr = smem;
            }
            k_lz4_decode_map<<<(unsigned)n, kMapThreads, smem, s>>>(
                n, src, off, dst, stride, expected, status, first_bad, fin_cap, pcap);
            RO_CUDA(cudaGetLastError());
            return RO_OK;
        }
    }
#endif
#if RO_LZ4_PIPE
    // Small batches (one wave of resident CTAs) are latency-bound: the
    // pipelined two-warp decoder finishes a brick sooner.  Larger batches are
    // throughput-bound: the one-warp decoder keeps far more frames in flight
    // (measured: 2.1 vs 2.9 ms per brick; 12 vs 29 GB/s in bulk).
    if (stride <= 64 * 1024) {
        // frames up to max(48 KB, 1.5 x the brick) are parsed from shared memory
        const int64_t fin_cap = std::max<int64_t>(48 * 1024, stride + stride / 2 + 64);
        const size_t smem = (size_t)((stride + 15) & ~(int64_t)15) + sizeof(LzRec) * kRing +
                            (size_t)fin_cap + 16;
        static size_t attr = 0;
        if (attr < smem) {
            RO_CUDA(cudaFuncSetAttribute(k_lz4_decode_pipe,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = smem;
        }
        int per_sm = 0, dev = 0, sms = 0;
        RO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lz4_decode_pipe, 64,
                                                              smem));
        RO_CUDA(cudaGetDevice(&dev));
        RO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (n <= (int64_t)per_sm * sms) {
            k_lz4_decode_pipe<<<(unsigned)n, 64, smem, s>>>(n, src, off, dst, stride, expected,
                                                            status, first_bad, fin_cap);
            RO_CUDA(cudaGetLastError());
            return RO_OK;
        }
    }
#endif
    const int64_t blocks = (n + kLz4Warps - 1) / kLz4Warps;
    k_lz4_decode<<<(unsigned)blocks, 32 * kLz4Warps, 0, s>>>(n, src, off, dst, stride, expected,
                                                            status, first_bad);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

// Upload n LZ4 frames, decode them into brick payloads on the device and
// insert them with the batched LRU (apply_bricks).  Nothing is inserted if a
// frame is corrupt (the reference raises before apply_brick:
// service.py:225-232).
int apply_bricks_lz4(ro_ctx *c, const ro_state *st, const int64_t *ids_h, int64_t n,
                     const uint8_t *frames, const int64_t *off_h, int32_t on_device,
                     int64_t frame, int32_t update_octree, int32_t *slots_out,
                     int64_t *evicted_out, cudaStream_t s) {
    if (n <= 0) return RO_OK;
    if (!ids_h || !frames || !off_h) return fail(RO_EINVAL, "null ids / frames / offsets");
    const int64_t bytes = off_h[n] - off_h[0];
    for (int64_t i = 0; i < n; ++i)
        if (off_h[i + 1] < off_h[i]) return fail(RO_EINVAL, "frame offsets not monotone");
    int rc;
    void *p_frames, *p_off, *p_payload;
    if ((rc = scratch(c, 5, (size_t)bytes + 16, &p_frames))) return rc;
    if ((rc = scratch(c, 6, sizeof(int64_t) * (n + 1) + sizeof(int32_t) * (n + 1) + 64, &p_off)))
        return rc;
    if ((rc = scratch(c, 2, (size_t)c->bvox * n, &p_payload))) return rc;
    int64_t *d_off = (int64_t *)p_off;
    int32_t *d_status = (int32_t *)(d_off + n + 1);
    int32_t *d_first = d_status + n;
    const uint8_t *d_frames;
    if (on_device) {
        d_frames = frames;  // frame i at frames + (off[i] - off[0])
    } else {
        if (c->staging_bytes < (size_t)bytes) {
            if (c->staging) cudaFreeHost(c->staging);
            c->staging = nullptr;
            c->staging_bytes = 0;
            RO_CUDA(cudaMallocHost(&c->staging, (size_t)bytes));
            c->staging_bytes = (size_t)bytes;
        }
        RO_CUDA(cudaEventSynchronize(c->upload_done));  // staging free again
        memcpy(c->staging, frames + off_h[0], (size_t)bytes);
        RO_CUDA(cudaMemcpyAsync(p_frames, c->staging, (size_t)bytes, cudaMemcpyHostToDevice, s));
        RO_CUDA(cudaEventRecord(c->upload_done, s));
        d_frames = (const uint8_t *)p_frames;
    }
    RO_CUDA(cudaMemcpyAsync(d_off, off_h, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    const int32_t big = 0x7FFFFFFF;
    RO_CUDA(cudaMemcpyAsync(d_first, &big, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if ((rc = lz4_decode(c, d_frames, d_off, n, (uint8_t *)p_payload, c->bvox, c->bvox,
                         d_status, d_first, s)))
        return rc;
    int32_t *h = reinterpret_cast<int32_t *>(c->pinned_small);
    RO_CUDA(cudaMemcpyAsync(h + 8, d_first, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RO_CUDA(cudaStreamSynchronize(s));
    if (h[8] != big) {
        int32_t code = 0;
        cudaMemcpy(&code, d_status + h[8], sizeof(int32_t), cudaMemcpyDeviceToHost);
        char msg[160];
        snprintf(msg, sizeof msg, "brick %d of the batch (id %lld): %s", h[8],
                 (long long)ids_h[h[8]], lz4_reason(code));
        return fail(RO_EINVAL, msg);
    }
    return apply_bricks(c, st, ids_h, n, p_payload, 1, frame, update_octree, slots_out,
                        evicted_out, s);
}

int normalize_to_u8(ro_ctx *c, const void *src, int32_t dtype, int64_t n, uint8_t *dst,
                    cudaStream_t s) {
    if (n <= 0) return RO_OK;
    void *p;
    int rc;
    if ((rc = scratch(c, 7, 64, &p))) return rc;
    uint32_t *mm = (uint32_t *)p;
    const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    RO_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s));
    const unsigned g = grid_for(n);
    switch (dtype) {
        case 1:
            k_minmax<<<g, 256, 0, s>>>(n, (const uint8_t *)src, mm);
            k_normalize<<<g, 256, 0, s>>>(n, (const uint8_t *)src, mm, dst);
            break;
        case 2:
            k_minmax<<<g, 256, 0, s>>>(n, (const uint16_t *)src, mm);
            k_normalize<<<g, 256, 0, s>>>(n, (const uint16_t *)src, mm, dst);
            break;
        case 3:
            k_minmax<<<g, 256, 0, s>>>(n, (const uint32_t *)src, mm);
            k_normalize<<<g, 256, 0, s>>>(n, (const uint32_t *)src, mm, dst);
            break;
        case 4:
            k_minmax<<<g, 256, 0, s>>>(n, (const float *)src, mm);
            k_normalize<<<g, 256, 0, s>>>(n, (const float *)src, mm, dst);
            break;
        default:
            return fail(RO_EINVAL, "dtype must be 1 (u8), 2 (u16), 3 (u32) or 4 (f32)");
    }
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int downsample_box(const uint8_t *src, int32_t dx, int32_t dy, int32_t dz, int32_t fx,
                   int32_t fy, int32_t fz, uint8_t *dst, cudaStream_t s) {
    for (int f : {fx, fy, fz})
        if (f != 1 && f != 2) return fail(RO_EINVAL, "downsample factors must be 1 or 2");
    if (dx < 1 || dy < 1 || dz < 1) return fail(RO_EINVAL, "empty level");
    const int ox = (dx + fx - 1) / fx, oy = (dy + fy - 1) / fy, oz = (dz + fz - 1) / fz;
    k_downsample_box<<<grid_for((int64_t)ox * oy * oz), 256, 0, s>>>(src, dx, dy, dz, fx, fy, fz,
                                                                     ox, oy, oz, dst);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

int extract_bricks(const uint8_t *level, int32_t dx, int32_t dy, int32_t dz, int32_t bx,
                   int32_t by, int32_t bz, uint8_t *dst, cudaStream_t s) {
    if (dx < 1 || dy < 1 || dz < 1 || bx < 1 || by < 1 || bz < 1)
        return fail(RO_EINVAL, "empty level or brick");
    const int gx = (dx + bx - 1) / bx, gy = (dy + by - 1) / by, gz = (dz + bz - 1) / bz;
    const int64_t nb = (int64_t)gx * gy * gz;
    k_extract_bricks<<<grid_for(nb * bx * by * bz), 256, 0, s>>>(level, dx, dy, dz, bx, by, bz,
                                                                 gx, gy, nb, dst);
    RO_CUDA(cudaGetLastError());
    return RO_OK;
}

}  // namespace ro
