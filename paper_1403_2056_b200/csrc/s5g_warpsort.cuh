// s5g_warpsort.cuh -- one warp finishes one segment of <= 32*ITEMS strings.
//
// The GPU stand-in for the reference's leaves (caching MKQS mkqs.py:196-253,
// LCP insertion sort basecase.py:67-116) once the device-wide S^5 steps have
// cut the input into segments of at most 256 strings.  Lane l holds slots
// l*ITEMS .. l*ITEMS+ITEMS-1 in registers: (word, group<<8 | tag).  A round is
// a bitonic network over (group, word, tag) -- in-lane stages for distances
// below ITEMS, shuffle stages above -- followed by word-parallel LCPs at
// every word change (XOR/clz), terminator-equal runs finalised, and runs of
// equal non-terminated words re-keyed one word deeper as the next round's
// groups.  A group id is the slot its run starts at, so finished slots
// (group = own slot) never move.  No shared-memory barriers: the latency of
// the re-keying gathers is hidden by the other warps of the SM.
#pragma once
#include "s5g_kernels.cuh"

namespace s5g {

constexpr int WS_NT = 256;  // 8 warps per CTA, one segment per warp

template <int ITEMS>
struct WarpLists {
    static constexpr int CAP = 32 * ITEMS;
};

__device__ __forceinline__ bool ws_less(uint64_t ka, uint32_t ma, uint64_t kb, uint32_t mb) {
    const uint32_t ga = ma >> 8 & 0xff, gb = mb >> 8 & 0xff;
    if (ga != gb) return ga < gb;
    if (ka != kb) return ka < kb;
    return (ma & 0xff) < (mb & 0xff);
}

template <int ITEMS>
__device__ __forceinline__ void ws_bitonic(uint64_t (&key)[ITEMS], uint32_t (&meta)[ITEMS],
                                           int lane) {
    constexpr int P = 32 * ITEMS;
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < ITEMS) {
#pragma unroll
                for (int e = 0; e < ITEMS; e++) {
                    const int f = e ^ j;
                    if (f > e) {
                        const int i = lane * ITEMS + e;
                        const bool up = (i & k) == 0;
                        if (ws_less(key[f], meta[f], key[e], meta[e]) == up) {
                            uint64_t tk = key[e]; key[e] = key[f]; key[f] = tk;
                            uint32_t tm = meta[e]; meta[e] = meta[f]; meta[f] = tm;
                        }
                    }
                }
            } else {
                const int lx = j / ITEMS;
#pragma unroll
                for (int e = 0; e < ITEMS; e++) {
                    const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lx);
                    const uint32_t om = __shfl_xor_sync(0xffffffffu, meta[e], lx);
                    const int i = lane * ITEMS + e;
                    const bool up = (i & k) == 0;
                    const bool lower = (i & j) == 0;  // this slot keeps the smaller if up
                    const bool other_less = ws_less(ok, om, key[e], meta[e]);
                    if (other_less == (lower == up)) {
                        key[e] = ok;
                        meta[e] = om;
                    }
                }
            }
        }
    }
}

template <int ITEMS>
__global__ void __launch_bounds__(WS_NT) k_warp_sort(
    const SegDev* __restrict__ segs, int64_t nsegs, const int64_t* __restrict__ hA,
    const uint64_t* __restrict__ kA, const int64_t* __restrict__ hB,
    const uint64_t* __restrict__ kB, const uint8_t* __restrict__ arena, int64_t alen,
    int64_t* __restrict__ out_h, int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    constexpr int CAP = 32 * ITEMS;
    __shared__ int64_t s_h[WS_NT / 32][CAP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (WS_NT / 32) + w;
    if (gw >= nsegs) return;  // whole warp
    const SegDev sg = segs[gw];
    const int m = sg.n;
    const int64_t lo = sg.lo;
    const int64_t* sh = (sg.flags & SEG_IN_B) ? hB : hA;
    const uint64_t* sk = (sg.flags & SEG_IN_B) ? kB : kA;
    const bool valid = sg.flags & SEG_KEYS_VALID;
    int64_t* wh = s_h[w];
    int64_t depth = sg.depth;
    unsigned fetches = 0;
    uint64_t key[ITEMS];
    uint32_t meta[ITEMS];  // bit 16 active | group << 8 | tag
    // coalesced handle loads into the warp's staging area
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = e * 32 + lane;
        if (i < m) wh[i] = sh[lo + i];
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = lane * ITEMS + e;
        if (i < m) {
            key[e] = valid ? sk[lo + i] : load_key(arena, alen, wh[i], depth);
            meta[e] = (1u << 16) | (0u << 8) | (uint32_t)i;
        } else {
            key[e] = ~0ull;
            meta[e] = ((uint32_t)i << 8) | (uint32_t)i;  // own group, stays last
        }
    }
    if (!valid) fetches += min(ITEMS, max(0, m - lane * ITEMS));
    for (;;) {
        ws_bitonic<ITEMS>(key, meta, lane);
        // predecessor / successor slots
        const uint64_t prev_last = __shfl_up_sync(0xffffffffu, key[ITEMS - 1], 1);
        bool brk[ITEMS];
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = lane * ITEMS + e;
            const bool act = meta[e] >> 16 & 1;
            const int grp = meta[e] >> 8 & 0xff;
            brk[e] = true;
            if (act && i != grp) {
                const uint64_t pk = e ? key[e - 1] : prev_last;
                if (pk != key[e]) {
                    if (lcps) lcps[lo + i] = depth + (__clzll(pk ^ key[e]) >> 3);
                } else {
                    brk[e] = false;
                    const int tpv = term_pos(key[e]);
                    if (lcps && tpv < WORD) lcps[lo + i] = depth + tpv;
                }
            }
        }
        // next slot's break flag (first item of the next lane)
        const bool next_brk0 = __shfl_down_sync(0xffffffffu, brk[0], 1);
        const bool next_act0 = __shfl_down_sync(0xffffffffu, meta[0] >> 16 & 1u, 1);
        bool keep[ITEMS];
        bool any = false;
        uint32_t run = 0;  // 1 + start slot of the latest kept run start in this lane
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = lane * ITEMS + e;
            const bool act = meta[e] >> 16 & 1;
            bool nb, na;
            if (e + 1 < ITEMS) {
                nb = brk[e + 1];
                na = meta[e + 1] >> 16 & 1;
            } else {
                nb = next_brk0;
                na = next_act0 && lane < 31;
            }
            keep[e] = act && term_pos(key[e]) == WORD && (!brk[e] || (na && !nb));
            any |= keep[e];
            if (keep[e] && brk[e]) run = i + 1;
        }
        if (!__any_sync(0xffffffffu, any) || depth > alen) break;  // alen: corrupt-input guard
        // inclusive max-scan of run starts across lanes
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = max(incl, y);
        }
        uint32_t cur = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) cur = 0;
        depth += WORD;
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = lane * ITEMS + e;
            if (keep[e] && brk[e]) cur = i + 1;
            const uint32_t tag = meta[e] & 0xff;
            if (keep[e]) {
                meta[e] = (1u << 16) | ((cur - 1) << 8) | tag;
            } else {
                meta[e] = ((uint32_t)i << 8) | tag;  // finished: own group, inactive
            }
        }
#pragma unroll
        for (int e = 0; e < ITEMS; e++)
            if (meta[e] >> 16 & 1) {
                key[e] = load_key(arena, alen, wh[meta[e] & 0xff], depth);
                fetches++;
            }
    }
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = lane * ITEMS + e;
        if (i < m) out_h[lo + i] = wh[meta[e] & 0xff];
    }
    fetches = __reduce_add_sync(0xffffffffu, fetches);
    if (lane == 0) {
        if (fetches) atomicAdd(&ctr->seg_fetches, (unsigned long long)fetches);
        atomicAdd(&ctr->small_elems, (unsigned long long)m);
    }
}

}  // namespace s5g

namespace s5g {

// ---------------------------------------------------------------------------
// CTA form: W warps x 256 slots (8 per lane) finish one segment of up to
// 256*W strings.  Distances below 256 run in registers / shuffles exactly as
// in k_warp_sort; distances >= 256 cross warps through shared memory.
// meta = active << 22 | group << 11 | tag (11-bit slots).

__device__ __forceinline__ bool cs_less(uint64_t ka, uint32_t ma, uint64_t kb, uint32_t mb) {
    const uint32_t ga = ma >> 11 & 0x7ff, gb = mb >> 11 & 0x7ff;
    if (ga != gb) return ga < gb;
    if (ka != kb) return ka < kb;
    return (ma & 0x7ff) < (mb & 0x7ff);
}

template <int W>
struct CtaSortSmem {
    int64_t h[256 * W];
    uint64_t xk[256 * W];
    uint32_t xm[256 * W];
    uint64_t last_key[W];
    uint32_t first_brk[W], first_act[W], wmax[W];
};

template <int W>
__global__ void __launch_bounds__(32 * W) k_cta_sort(
    const SegDev* __restrict__ segs, int64_t nsegs, const int64_t* __restrict__ hA,
    const uint64_t* __restrict__ kA, const int64_t* __restrict__ hB,
    const uint64_t* __restrict__ kB, const uint8_t* __restrict__ arena, int64_t alen,
    int64_t* __restrict__ out_h, int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    constexpr int ITEMS = 8, P = 256 * W, NT = 32 * W;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    CtaSortSmem<W>& S = *reinterpret_cast<CtaSortSmem<W>*>(smem_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const SegDev sg = segs[blockIdx.x];
    const int m = sg.n;
    const int64_t lo = sg.lo;
    const int64_t* sh = (sg.flags & SEG_IN_B) ? hB : hA;
    const uint64_t* sk = (sg.flags & SEG_IN_B) ? kB : kA;
    const bool valid = sg.flags & SEG_KEYS_VALID;
    int64_t depth = sg.depth;
    unsigned fetches = 0;
    for (int i = threadIdx.x; i < m; i += NT) S.h[i] = sh[lo + i];
    __syncthreads();
    uint64_t key[ITEMS];
    uint32_t meta[ITEMS];
    const int base = threadIdx.x * ITEMS;  // first slot of this thread
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = base + e;
        if (i < m) {
            key[e] = valid ? sk[lo + i] : load_key(arena, alen, S.h[i], depth);
            meta[e] = (1u << 22) | (uint32_t)i;
        } else {
            key[e] = ~0ull;
            meta[e] = ((uint32_t)i << 11) | (uint32_t)i;
        }
    }
    if (!valid) fetches += min(ITEMS, max(0, m - base));
    for (;;) {
        // ---- bitonic network over (group, word, tag) ----------------------
#pragma unroll 1
        for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j < ITEMS) {
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
#pragma unroll
                        for (int jj = 1; jj < ITEMS; jj <<= 1) {
                            if (jj != j) continue;
                            const int f = e ^ jj;
                            if (f > e) {
                                const bool up = ((base + e) & k) == 0;
                                if (cs_less(key[f], meta[f], key[e], meta[e]) == up) {
                                    uint64_t tk = key[e]; key[e] = key[f]; key[f] = tk;
                                    uint32_t tm = meta[e]; meta[e] = meta[f]; meta[f] = tm;
                                }
                            }
                        }
                    }
                } else if (j < 256) {
                    const int lx = j / ITEMS;
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lx);
                        const uint32_t om = __shfl_xor_sync(0xffffffffu, meta[e], lx);
                        const int i = base + e;
                        const bool up = (i & k) == 0, lower = (i & j) == 0;
                        if (cs_less(ok, om, key[e], meta[e]) == (lower == up)) {
                            key[e] = ok;
                            meta[e] = om;
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        S.xk[base + e] = key[e];
                        S.xm[base + e] = meta[e];
                    }
                    __syncthreads();
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        const int i = base + e;
                        const uint64_t ok = S.xk[i ^ j];
                        const uint32_t om = S.xm[i ^ j];
                        const bool up = (i & k) == 0, lower = (i & j) == 0;
                        if (cs_less(ok, om, key[e], meta[e]) == (lower == up)) {
                            key[e] = ok;
                            meta[e] = om;
                        }
                    }
                    __syncthreads();
                }
            }
        }
        // ---- LCPs at word changes, run breaks -------------------------------
        uint64_t prev_last = __shfl_up_sync(0xffffffffu, key[ITEMS - 1], 1);
        if (lane == 31) S.last_key[w] = key[ITEMS - 1];
        __syncthreads();
        if (lane == 0 && w > 0) prev_last = S.last_key[w - 1];
        bool brk[ITEMS];
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            const bool act = meta[e] >> 22 & 1;
            const int grp = meta[e] >> 11 & 0x7ff;
            brk[e] = true;
            if (act && i != grp) {
                const uint64_t pk = e ? key[e - 1] : prev_last;
                if (pk != key[e]) {
                    if (lcps) lcps[lo + i] = depth + (__clzll(pk ^ key[e]) >> 3);
                } else {
                    brk[e] = false;
                    const int tpv = term_pos(key[e]);
                    if (lcps && tpv < WORD) lcps[lo + i] = depth + tpv;
                }
            }
        }
        bool next_brk0 = __shfl_down_sync(0xffffffffu, brk[0], 1);
        bool next_act0 = __shfl_down_sync(0xffffffffu, meta[0] >> 22 & 1u, 1);
        if (lane == 0) {
            S.first_brk[w] = brk[0];
            S.first_act[w] = meta[0] >> 22 & 1u;
        }
        __syncthreads();
        if (lane == 31) {
            next_brk0 = w + 1 < W ? S.first_brk[w + 1] : true;
            next_act0 = w + 1 < W ? S.first_act[w + 1] : false;
        }
        bool keep[ITEMS];
        bool any = false;
        uint32_t run = 0;
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            const bool act = meta[e] >> 22 & 1;
            bool nb, na;
            if (e + 1 < ITEMS) {
                nb = brk[e + 1];
                na = meta[e + 1] >> 22 & 1;
            } else {
                nb = next_brk0;
                na = next_act0;
            }
            keep[e] = act && term_pos(key[e]) == WORD && (!brk[e] || (na && !nb));
            any |= keep[e];
            if (keep[e] && brk[e]) run = i + 1;
        }
        if (!__syncthreads_or(any) || depth > alen) break;  // alen: corrupt-input guard
        // run starts: max-scan over the CTA
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = max(incl, y);
        }
        if (lane == 31) S.wmax[w] = incl;
        __syncthreads();
        uint32_t cur = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) cur = 0;
        for (int v = 0; v < w; v++) cur = max(cur, S.wmax[v]);
        depth += WORD;
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            if (keep[e] && brk[e]) cur = i + 1;
            const uint32_t tag = meta[e] & 0x7ff;
            meta[e] = keep[e] ? ((1u << 22) | ((cur - 1) << 11) | tag) : (((uint32_t)i << 11) | tag);
        }
#pragma unroll
        for (int e = 0; e < ITEMS; e++)
            if (meta[e] >> 22 & 1) {
                key[e] = load_key(arena, alen, S.h[meta[e] & 0x7ff], depth);
                fetches++;
            }
        __syncthreads();  // S.wmax / S.last_key reuse
    }
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = base + e;
        if (i < m) out_h[lo + i] = S.h[meta[e] & 0x7ff];
    }
    fetches = __reduce_add_sync(0xffffffffu, fetches);
    if (lane == 0 && fetches) atomicAdd(&ctr->seg_fetches, (unsigned long long)fetches);
    if (threadIdx.x == 0) atomicAdd(&ctr->small_elems, (unsigned long long)m);
}

}  // namespace s5g
