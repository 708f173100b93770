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
    int64_t h[256 * W];           // handle by tag
    uint64_t xk[256 * W];
    uint32_t xm[256 * W];
    uint16_t ord[256 * W];        // tag at slot (group mode)
    uint16_t gs[128 * W], ge[128 * W];  // group mode: first / last slot of each run
    uint64_t last_key[W];
    uint32_t first_brk[W], first_act[W], wmax[W], wcnt[W];
};

// Bitonic network on one warp's 32*IT slots, comparator cs_less.
template <int IT>
__device__ __forceinline__ void cs_bitonic(uint64_t (&key)[IT], uint32_t (&meta)[IT], int lane) {
    constexpr int P = 32 * IT;
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < IT) {
#pragma unroll
                for (int e = 0; e < IT; e++) {
                    const int f = e ^ j;
                    if (f > e) {
                        const bool up = ((lane * IT + e) & k) == 0;
                        if (cs_less(key[f], meta[f], key[e], meta[e]) == up) {
                            uint64_t tk = key[e]; key[e] = key[f]; key[f] = tk;
                            uint32_t tm = meta[e]; meta[e] = meta[f]; meta[f] = tm;
                        }
                    }
                }
            } else {
                const int lx = j / IT;
#pragma unroll
                for (int e = 0; e < IT; e++) {
                    const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lx);
                    const uint32_t om = __shfl_xor_sync(0xffffffffu, meta[e], lx);
                    const int i = lane * IT + e;
                    const bool up = (i & k) == 0, lower = (i & j) == 0;
                    if (cs_less(ok, om, key[e], meta[e]) == (lower == up)) {
                        key[e] = ok;
                        meta[e] = om;
                    }
                }
            }
        }
    }
}

// One warp finishes one run of gn <= 32*IT strings (slots g0.. of the
// segment) that share `depth` characters: re-key one word deeper, sort,
// LCPs, recurse on equal runs -- all in registers.  Writes the final tag
// order back to ord[g0 .. g0+gn).
template <int IT>
__device__ void cs_finish_group(const int64_t* __restrict__ hbt, uint16_t* __restrict__ ord,
                                int g0, int gn, int64_t depth, const uint8_t* __restrict__ arena,
                                int64_t alen, int64_t* __restrict__ lcp_seg, unsigned& fetches,
                                int lane) {
    uint64_t key[IT];
    uint32_t meta[IT];
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int i = lane * IT + e;
        if (i < gn) {
            const uint32_t tag = ord[g0 + i];
            key[e] = load_key(arena, alen, hbt[tag], depth);
            meta[e] = (1u << 22) | tag;
            fetches++;
        } else {
            key[e] = ~0ull;
            meta[e] = (uint32_t)i << 11;
        }
    }
    for (;;) {
        cs_bitonic<IT>(key, meta, lane);
        const uint64_t prev_last = __shfl_up_sync(0xffffffffu, key[IT - 1], 1);
        bool brk[IT];
#pragma unroll
        for (int e = 0; e < IT; e++) {
            const int i = lane * IT + e;
            const bool act = meta[e] >> 22 & 1;
            brk[e] = true;
            if (act && i != (int)(meta[e] >> 11 & 0x7ff)) {
                const uint64_t pk = e ? key[e - 1] : prev_last;
                if (pk != key[e]) {
                    if (lcp_seg) lcp_seg[g0 + i] = depth + (__clzll(pk ^ key[e]) >> 3);
                } else {
                    brk[e] = false;
                    const int tpv = term_pos(key[e]);
                    if (lcp_seg && tpv < WORD) lcp_seg[g0 + i] = depth + tpv;
                }
            }
        }
        const bool next_brk0 = __shfl_down_sync(0xffffffffu, brk[0], 1);
        const bool next_act0 = __shfl_down_sync(0xffffffffu, meta[0] >> 22 & 1u, 1);
        bool keep[IT];
        bool any = false;
        uint32_t run = 0;
#pragma unroll
        for (int e = 0; e < IT; e++) {
            const int i = lane * IT + e;
            const bool act = meta[e] >> 22 & 1;
            bool nb, na;
            if (e + 1 < IT) {
                nb = brk[e + 1];
                na = meta[e + 1] >> 22 & 1;
            } else {
                nb = next_brk0;
                na = next_act0 && lane < 31;
            }
            keep[e] = act && term_pos(key[e]) == WORD && (!brk[e] || (na && !nb));
            any |= keep[e];
            if (keep[e] && brk[e]) run = i + 1;
        }
        if (!__any_sync(0xffffffffu, any) || depth > alen) break;  // alen: corrupt-input guard
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
        for (int e = 0; e < IT; e++) {
            const int i = lane * IT + e;
            if (keep[e] && brk[e]) cur = i + 1;
            const uint32_t tag = meta[e] & 0x7ff;
            meta[e] = keep[e] ? ((1u << 22) | ((cur - 1) << 11) | tag) : (((uint32_t)i << 11) | tag);
        }
#pragma unroll
        for (int e = 0; e < IT; e++)
            if (meta[e] >> 22 & 1) {
                key[e] = load_key(arena, alen, hbt[meta[e] & 0x7ff], depth);
                fetches++;
            }
    }
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int i = lane * IT + e;
        if (i < gn) ord[g0 + i] = (uint16_t)(meta[e] & 0x7ff);
    }
}

template <int W>
__global__ void __launch_bounds__(32 * W, 24 / W) k_cta_sort(
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
    int64_t* lcp_seg = lcps ? lcps + lo : nullptr;
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
    bool group_mode = false;
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
                    if (lcp_seg) lcp_seg[i] = depth + (__clzll(pk ^ key[e]) >> 3);
                } else {
                    brk[e] = false;
                    const int tpv = term_pos(key[e]);
                    if (lcp_seg && tpv < WORD) lcp_seg[i] = depth + tpv;
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
        bool keep[ITEMS], kend[ITEMS];
        bool any = false;
        uint32_t run = 0, nstart = 0, nend = 0;
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
            kend[e] = keep[e] && (!na || nb);  // last slot of a kept run
            any |= keep[e];
            if (keep[e] && brk[e]) { run = i + 1; nstart++; }
            nend += kend[e];
        }
        if (!__syncthreads_or(any) || depth > alen) break;  // alen: corrupt-input guard
        // run starts: max-scan over the CTA (next round's group ids)
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
        // longest kept run decides: CTA round again, or one warp per run
        uint32_t longest = 0, c2 = cur;
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            if (keep[e] && brk[e]) c2 = i + 1;
            if (kend[e]) longest = max(longest, (uint32_t)i + 2 - c2);
        }
        longest = __reduce_max_sync(0xffffffffu, longest);
        if (lane == 0) S.wcnt[w] = longest;
        __syncthreads();
        uint32_t lmax = 0;
        for (int v = 0; v < W; v++) lmax = max(lmax, S.wcnt[v]);
        if (W == 8 && lmax <= 256) {
            // ---- group mode: write the slot order, list the kept runs --------
#pragma unroll
            for (int e = 0; e < ITEMS; e++) S.ord[base + e] = (uint16_t)(meta[e] & 0x7ff);
            // starts and ends are counted separately: a run may span threads
            const uint32_t mine = nstart | (nend << 16);
            const uint32_t ns = __reduce_add_sync(0xffffffffu, mine);
            uint32_t pre = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += y;
            }
            pre -= mine;
            __syncthreads();
            if (lane == 0) S.wcnt[w] = ns;
            __syncthreads();
            uint32_t off = 0, tot2 = 0;
            for (int v = 0; v < W; v++) {
                if (v < w) off += S.wcnt[v];
                tot2 += S.wcnt[v];
            }
            const uint32_t ngroups = tot2 & 0xffff;
            uint32_t gi = (off + pre) & 0xffff, ge_i = (off + pre) >> 16;
#pragma unroll
            for (int e = 0; e < ITEMS; e++) {
                const int i = base + e;
                if (keep[e] && brk[e]) S.gs[gi++] = (uint16_t)i;
                if (kend[e]) S.ge[ge_i++] = (uint16_t)i;
            }
            if (threadIdx.x == 0) S.wcnt[0] = ngroups;
            __syncthreads();
            group_mode = true;
            break;
        }
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
        __syncthreads();  // S.wmax / S.last_key / S.wcnt reuse
    }
    if (!group_mode) {
#pragma unroll
        for (int e = 0; e < ITEMS; e++) S.ord[base + e] = (uint16_t)(meta[e] & 0x7ff);
    } else {
        // one warp per remaining run, each finished entirely in registers
        const uint32_t ngroups = S.wcnt[0];
        for (uint32_t g = w; g < ngroups; g += W) {
            const int g0 = S.gs[g], gn = S.ge[g] - g0 + 1;
            if (gn <= 32)
                cs_finish_group<1>(S.h, S.ord, g0, gn, depth + WORD, arena, alen, lcp_seg, fetches, lane);
            else if (gn <= 64)
                cs_finish_group<2>(S.h, S.ord, g0, gn, depth + WORD, arena, alen, lcp_seg, fetches, lane);
            else if (gn <= 128)
                cs_finish_group<4>(S.h, S.ord, g0, gn, depth + WORD, arena, alen, lcp_seg, fetches, lane);
            else
                cs_finish_group<8>(S.h, S.ord, g0, gn, depth + WORD, arena, alen, lcp_seg, fetches, lane);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += NT) out_h[lo + i] = S.h[S.ord[i]];
    fetches = __reduce_add_sync(0xffffffffu, fetches);
    if (lane == 0 && fetches) atomicAdd(&ctr->seg_fetches, (unsigned long long)fetches);
    if (threadIdx.x == 0) atomicAdd(&ctr->small_elems, (unsigned long long)m);
}

}  // namespace s5g
