// topk.cuh -- grid-wide "k smallest keys, in order" for cooperative kernels.
//
// Used where only the first k of a key order survive: the request budget
// (feedback.cu, render.py:210-215) and the LRU victims of a batch
// (residency.cu, paging.py:205-206 argmin over (last_used, slot)).  Instead
// of sorting every candidate, the k-th smallest key is found by a radix
// select (8-bit digits from the top: one histogram pass over the
// candidates per digit, one grid sync each), the <= k survivors are
// gathered, and one CTA sorts them in shared memory.  Keys must be unique.
#pragma once

#include <cooperative_groups.h>

#include <stdint.h>

namespace ro {
namespace topk {

namespace cg = cooperative_groups;

constexpr int kChunk = 8192;  // pairs one CTA sorts in shared memory
constexpr size_t kSortSmem = (size_t)kChunk * (sizeof(unsigned long long) + sizeof(int32_t));
constexpr int kHistWords = 3 * 256;

__device__ __forceinline__ int bit_len64(unsigned long long v) {
    return v ? 64 - __clzll(v) : 0;
}

// Exact need-th smallest key (1-based) among candidates i in [0, n) with
// key_of(i, &q) true and q > lo (when has_lo).  hist: 3 x 256 u32 ring in
// global memory, zero on entry for the steps this call starts at (see
// below); g: ring step counter, identical in every CTA.  Step g accumulates
// into hist[g % 3]; after the grid sync every CTA reads it and CTA 0 clears
// hist[(g + 2) % 3] (nobody reads that one after the sync), so the ring
// stays clean for later calls without extra syncs.
template <typename KeyOf>
__device__ unsigned long long select_kth(cg::grid_group &grid, int64_t n, KeyOf key_of,
                                         bool has_lo, unsigned long long lo, int64_t need,
                                         int top_shift, uint32_t *hist, uint32_t &g,
                                         uint32_t *s_hist) {
    __shared__ uint32_t s_sel[2];
    unsigned long long prefix = 0;
    for (int shift = top_shift; shift >= 0; shift -= 8) {
        uint32_t *H = hist + 256 * (g % 3);
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
        const int hs = shift + 8;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x) {
            unsigned long long q;
            if (!key_of(i, q)) continue;
            if (has_lo && q <= lo) continue;
            if (hs < 64 && (q >> hs) != (prefix >> hs)) continue;
            atomicAdd(&s_hist[(q >> shift) & 255], 1u);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&H[i], s_hist[i]);
        grid.sync();
        // the digit where the running count reaches `need` (one warp per CTA)
        if (threadIdx.x < 32) {
            uint32_t c[8];
            uint32_t run = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = __ldcg(&H[threadIdx.x * 8 + j]);
                run += c[j];
            }
            uint32_t incl = run;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)threadIdx.x >= o) incl += y;
            }
            uint32_t before = incl - run;
            if ((int64_t)before < need && need <= (int64_t)incl) {
                for (int j = 0; j < 8; ++j) {
                    if (need <= (int64_t)(before + c[j])) {
                        s_sel[0] = threadIdx.x * 8 + j;
                        s_sel[1] = before;
                        break;
                    }
                    before += c[j];
                }
            }
        }
        if (blockIdx.x == 0) {
            uint32_t *Hz = hist + 256 * ((g + 2) % 3);
            for (int i = threadIdx.x; i < 256; i += blockDim.x) Hz[i] = 0;
        }
        __syncthreads();
        prefix |= (unsigned long long)s_sel[0] << shift;
        need -= s_sel[1];
        ++g;
        __syncthreads();
    }
    return prefix;
}

// One CTA: ascending bitonic sort of w <= kChunk (key, value) pairs in
// shared memory (smem >= kSortSmem bytes).  Keys ~0 are padding.
__device__ inline void sort_pairs(unsigned long long *sk, int32_t *sv, int w) {
    int np = 1;
    while (np < w) np <<= 1;
    for (int i = w + threadIdx.x; i < np; i += blockDim.x) {
        sk[i] = ~0ull;
        sv[i] = -1;
    }
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < np / 2; i += blockDim.x) {
                const int a = 2 * i - (i & (stride - 1));
                const int b = a + stride;
                const bool up = (a & size) == 0;
                const unsigned long long ka = sk[a], kb = sk[b];
                if ((ka > kb) == up) {
                    sk[a] = kb;
                    sk[b] = ka;
                    const int32_t t = sv[a];
                    sv[a] = sv[b];
                    sv[b] = t;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace topk
}  // namespace ro
