// s5g_warpsort.cuh -- register-resident finishers for segments of <= 2048
// strings: the GPU stand-in for the reference's leaves (caching MKQS
// mkqs.py:196-253, LCP insertion sort basecase.py:67-116).
//
// A round sorts the active slots by (group, 8-byte word at the round's depth,
// tag) with a bitonic network held in registers (in-lane stages below 8 /
// IT, shuffle stages below 256, shared-memory stages above), then writes the
// LCPs at every word change from XOR/clz (shared_chars, strset.py:194-206),
// finalises terminator-equal runs, and re-keys runs of equal non-terminated
// words one word deeper as the next round's groups.  A group id is the slot
// its run starts at, so finished slots (group = own slot) never move, and
// the tag (position in the segment) keeps ties in input order: stable.
//
// Compare-exchange cost is the bottleneck (ncu: ~45% of the instructions in
// a 3-way comparator), so whenever the varying bits of the round's words fit,
// a slot is ONE u64: group | PEXT(word, varying-bit mask) | tag, compared and
// moved as a single value; the words stay in shared memory by tag.  The
// PEXT is a six-step register compress network (pext_key).
#pragma once
#include "s5g_kernels.cuh"

namespace s5g {

__device__ unsigned long long g_fin_ctr[12];  // s5g_finisher_counters

// meta = active << 22 | group << 11 | tag   (11-bit slots and tags)
__device__ __forceinline__ bool cs_less(uint64_t ka, uint32_t ma, uint64_t kb, uint32_t mb) {
    const uint32_t ga = ma >> 11 & 0x7ff, gb = mb >> 11 & 0x7ff;
    if (ga != gb) return ga < gb;
    if (ka != kb) return ka < kb;
    return (ma & 0x7ff) < (mb & 0x7ff);
}

struct Pext {
    uint64_t V;      // varying-bit mask
    uint64_t mv[6];  // bits moved right by 2^i in step i of the compress network
    int cb;          // popcount(V)
};

__device__ uint8_t g_pext8[256 * 256];  // [mask * 256 + byte] = pext(byte, mask)

// Byte-wise PEXT through a 256x256 table (L1): cheap to set up, so the warp
// finisher's many small rounds use it (a few strings per lane and round).
struct PextLut {
    uint64_t V;   // varying-bit mask
    uint64_t SH;  // 6-bit shift of byte b's extracted bits at 6b
    int cb;       // popcount(V)
};

__device__ __forceinline__ PextLut pext_lut_setup(uint64_t V) {
    PextLut p;
    p.V = V;
    p.cb = __popcll(V);
    uint64_t sh = 0;
    int acc = 0;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        sh |= (uint64_t)acc << (6 * b);
        acc += __popc((uint32_t)(V >> (8 * b)) & 255u);
    }
    p.SH = sh;
    return p;
}

__device__ __forceinline__ uint64_t pext_lut_key(uint64_t x, const PextLut& p) {
    uint64_t c = 0;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const uint32_t m = (uint32_t)(p.V >> (8 * b)) & 255u;
        if (m)
            c |= (uint64_t)__ldg(&g_pext8[m * 256 + ((uint32_t)(x >> (8 * b)) & 255u)])
                 << ((p.SH >> (6 * b)) & 63);
    }
    return c;
}

// Bit-extract (PEXT) under a mask uniform over the caller, as the
// compress network of Hacker's Delight 7-4: the mask's six move sets are
// derived once per round (~170 instructions), after which an extract is 6
// register-only steps.  The CTA rounds pack up to 2048 words per round with
// it (through the table, ~12 instructions and an L1 load per byte, packing
// was a fifth of the CTA finishers' instructions).  Order-preserving: the
// kept bits keep their significance order, exactly as pext_lut_key.
__device__ __forceinline__ Pext pext_setup(uint64_t V) {
    Pext p;
    p.V = V;
    p.cb = __popcll(V);
    uint64_t m = V, mk = ~m << 1;
#pragma unroll
    for (int i = 0; i < 6; i++) {
        uint64_t mp = mk ^ (mk << 1);  // parallel suffix of the zeros to the right
        mp ^= mp << 2;
        mp ^= mp << 4;
        mp ^= mp << 8;
        mp ^= mp << 16;
        mp ^= mp << 32;
        const uint64_t mv = mp & m;
        p.mv[i] = mv;
        m = (m ^ mv) | (mv >> (1 << i));
        mk &= ~mp;
    }
    return p;
}

__device__ __forceinline__ uint64_t pext_key(uint64_t x, const Pext& p) {
    x &= p.V;
#pragma unroll
    for (int i = 0; i < 6; i++) {
        const uint64_t t = x & p.mv[i];
        x = (x ^ t) | (t >> (1 << i));
    }
    return x;
}

// Words at `depth` of the active slots, from the work records while `depth`
// is inside their cache (cd: depth of w[0], cnv: valid words), else every
// active record is refilled with its next three words (one gather round trip
// for up to three rounds; duplicate-heavy runs advance a word per round).
// cd / cnv / depth are uniform over the caller (one warp, or the CTA when
// CTA), and each tag is in one slot, so the record writes never conflict.
// The refill walks the slots (tags staged in `scratch[0 .. nslots)`) in one
// rolled loop: inlined per register slot, the gather code would double the
// finishers' instruction footprint.
template <int N, bool CTA>
__device__ __forceinline__ void rekey(uint64_t (&key)[N], const uint32_t (&meta)[N],
                                      Rec* __restrict__ segrec, const int64_t* __restrict__ hbt,
                                      int64_t& cd, int& cnv, int64_t depth,
                                      const uint8_t* __restrict__ arena, int64_t alen,
                                      unsigned& fetches, uint64_t* __restrict__ scratch,
                                      int slot0, int nslots, int tid, int nthreads) {
    const int64_t off = depth - cd;
    if ((off & 7) == 0 && (off >> 3) < cnv) {
        const int r = (int)(off >> 3);
#pragma unroll
        for (int e = 0; e < N; e++)
            if (meta[e] >> 22 & 1) key[e] = segrec[meta[e] & 0x7ff].w[r];
        return;
    }
#pragma unroll
    for (int e = 0; e < N; e++)
        if (slot0 + e < nslots) scratch[slot0 + e] = (meta[e] >> 22 & 1) ? (meta[e] & 0x7ff) : ~0ull;
    if (CTA) __syncthreads(); else __syncwarp();
    for (int q = tid; q < nslots; q += nthreads) {
        const uint64_t t = scratch[q];
        if (t != ~0ull) {
            S5G_CHECK(t < 2048u);  // an 11-bit tag of the segment
            uint64_t w3[3];
            load_words3(arena, alen, hbt[t], depth, w3);
            segrec[t].w[0] = w3[0];
            segrec[t].w[1] = w3[1];
            segrec[t].w[2] = w3[2];
            fetches += 3;
        }
    }
    if (CTA) __syncthreads(); else __syncwarp();
#pragma unroll
    for (int e = 0; e < N; e++)
        if (meta[e] >> 22 & 1) key[e] = segrec[meta[e] & 0x7ff].w[0];
    cd = depth;
    cnv = NCACHE;
}

__device__ __forceinline__ void cex_u64(uint64_t& a, uint64_t& b, bool up) {
    const bool sw = (b < a) == up;
    const uint64_t x = a, y = b;
    a = sw ? y : x;
    b = sw ? x : y;
}

// ---------------------------------------------------------------------------
// warp-level networks over 32*IT slots (slot = lane*IT + e)

// In-lane stage at compile-time distance J < IT (direction varies with e
// while k < IT).  The stage loops below are NOT unrolled over (k, j): the
// finishers inline several of these networks, and fully unrolled they
// overflow the instruction cache (ncu: "no instruction" was the top stall).
template <int J, int IT>
__device__ __forceinline__ void warp_inlane_u64(uint64_t (&c)[IT], int i0, int k) {
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int f = e ^ J;
        if (f > e) cex_u64(c[e], c[f], ((i0 + e) & k) == 0);
    }
}

template <int J, int IT>
__device__ __forceinline__ void warp_inlane_u(uint64_t (&c)[IT], bool up) {
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int f = e ^ J;
        if (f > e) cex_u64(c[e], c[f], up);
    }
}

template <int IT>
__device__ __forceinline__ void warp_bitonic_u64(uint64_t (&c)[IT], int lane) {
    constexpr int P = 32 * IT;
    const int i0 = lane * IT;
    // k < IT (only when IT = 4, 8): directions vary inside the thread
    if constexpr (IT >= 4) {
        warp_inlane_u64<1, IT>(c, i0, 2);
        warp_inlane_u64<2, IT>(c, i0, 4);
        warp_inlane_u64<1, IT>(c, i0, 4);
    } else if constexpr (IT == 2) {
        warp_inlane_u64<1, IT>(c, i0, 2);
    }
    if constexpr (IT >= 8) {
        warp_inlane_u64<4, IT>(c, i0, 8);
        warp_inlane_u64<2, IT>(c, i0, 8);
        warp_inlane_u64<1, IT>(c, i0, 8);
    }
#pragma unroll 1
    for (int k = 2 * IT; k <= P; k <<= 1) {
        const bool upk = (i0 & k) == 0;
        // partner in another lane; direction uniform over e
#pragma unroll 1
        for (int j = k >> 1; j >= IT; j >>= 1) {
            const int lx = j / IT;
            const bool keep_min = ((i0 & j) == 0) == upk;
#pragma unroll
            for (int e = 0; e < IT; e++) {
                const uint64_t o = __shfl_xor_sync(0xffffffffu, c[e], lx);
                c[e] = ((o < c[e]) == keep_min) ? o : c[e];
            }
        }
        if constexpr (IT >= 8) warp_inlane_u<4, IT>(c, upk);
        if constexpr (IT >= 4) warp_inlane_u<2, IT>(c, upk);
        if constexpr (IT >= 2) warp_inlane_u<1, IT>(c, upk);
    }
}

template <int IT>
__device__ __forceinline__ void warp_bitonic_generic(uint64_t (&key)[IT], uint32_t (&meta)[IT],
                                                     int lane) {
    constexpr int P = 32 * IT;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < IT) {
#pragma unroll
                for (int e = 0; e < IT; e++) {
#pragma unroll
                    for (int jj = 1; jj < IT; jj <<= 1) {
                        if (jj != j) continue;
                        const int f = e ^ jj;
                        if (f > e) {
                            const bool up = ((lane * IT + e) & k) == 0;
                            if (cs_less(key[f], meta[f], key[e], meta[e]) == up) {
                                uint64_t tk = key[e]; key[e] = key[f]; key[f] = tk;
                                uint32_t tm = meta[e]; meta[e] = meta[f]; meta[f] = tm;
                            }
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

__device__ __forceinline__ uint64_t warp_or64(uint64_t x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ uint64_t warp_and64(uint64_t x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x &= __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// First stop of two raw little-endian 8-byte windows of strings equal so
// far: the lowest byte where they differ or where `ra` holds its terminator
// (bytes past the arena read 0), or 8 if none.  Raw words: no byte swap or
// terminator masking on the long equal stretches of deep-LCP pairs (they
// were a third of the C4 finishers' instructions as load_key).
__device__ __forceinline__ int raw_stop(uint64_t ra, uint64_t rb) {
    const uint64_t x = (ra ^ rb) | zero_bytes(ra);
    return x ? (__ffsll((long long)x) - 1) >> 3 : WORD;
}

// LCP of the strings at a and b, known equal before depth d, capped at cap:
// the warp compares 32 words (256 characters) per step.
__device__ __forceinline__ int64_t warp_lcp_from(const uint8_t* __restrict__ arena, int64_t alen,
                                                 int64_t a, int64_t b, int64_t d, int64_t cap,
                                                 unsigned& fetches, int lane) {
    for (; d < cap; d += 32 * WORD) {
        const uint64_t ra = load_word_le(arena, alen, a + d + WORD * lane);
        const uint64_t rb = load_word_le(arena, alen, b + d + WORD * lane);
        fetches += 2;
        const int p = raw_stop(ra, rb);
        const uint32_t m = __ballot_sync(0xffffffffu, p < WORD);
        if (m) {
            const int f = __ffs(m) - 1;
            const int64_t l = d + WORD * lane + p;
            return min(cap, __shfl_sync(0xffffffffu, l, f));
        }
    }
    return cap;
}

// The kept slots form ONE run (group): all its strings share `depth`
// characters; return their common prefix length (>= depth) so the next
// round starts where they first differ (suffixes of texts with long copied
// blocks otherwise advance one word per round).  lcp(s0, s1) is found by the
// whole warp (256 characters per step); the other members, one per lane,
// are checked against s0 only up to that bound.  Runs of more than 32
// strings keep the word-per-round path.
template <int IT>
__device__ __forceinline__ int64_t run_common_prefix(const uint32_t (&meta)[IT],
                                                     const int64_t* __restrict__ hbt, int64_t depth,
                                                     const uint8_t* __restrict__ arena,
                                                     int64_t alen, unsigned& fetches,
                                                     uint64_t* __restrict__ xs, int lane) {
    uint32_t mine = 0;
#pragma unroll
    for (int e = 0; e < IT; e++) mine += meta[e] >> 22 & 1;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t r = __shfl_sync(0xffffffffu, incl, 31);
    if (r < 2 || r > 32) return depth;
    uint32_t k = incl - mine;  // member rank of my first active slot (slot order)
#pragma unroll
    for (int e = 0; e < IT; e++)
        if (meta[e] >> 22 & 1) xs[k++] = (uint64_t)hbt[meta[e] & 0x7ff];
    __syncwarp();
    const int64_t h0 = (int64_t)xs[0], h1 = (int64_t)xs[1];
    const int64_t hm = lane < (int)r ? (int64_t)xs[lane] : 0;
    __syncwarp();
    int64_t c = warp_lcp_from(arena, alen, h0, h1, depth, INT64_MAX, fetches, lane);
    if (c > depth && r > 2) {
        int64_t my = c;
        if (lane >= 2 && lane < (int)r) {
            for (int64_t d = depth; d < my; d += WORD) {
                const int p = raw_stop(load_word_le(arena, alen, h0 + d), load_word_le(arena, alen, hm + d));
                fetches += 2;
                if (p < WORD) {
                    my = min(my, d + p);
                    break;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) my = min(my, __shfl_xor_sync(0xffffffffu, my, o));
        c = my;
    }
    return c;
}

constexpr int SMALL_RUN = 8;  // runs finished by direct comparisons
#ifndef FSR_ROUNDS
#define FSR_ROUNDS 4             // ... once tied for this many warp rounds (tuned on C3 / C4)
#endif

// Order two strings sharing d characters: (a <= b, their LCP); a warp-wide
// 256-character compare per step on raw words (raw_stop).
__device__ __forceinline__ bool warp_le(const uint8_t* __restrict__ arena, int64_t alen,
                                       int64_t a, int64_t b, int64_t d, int64_t* l,
                                       unsigned& fetches, int lane) {
    for (;; d += 32 * WORD) {
        const uint64_t ra = load_word_le(arena, alen, a + d + WORD * lane);
        const uint64_t rb = load_word_le(arena, alen, b + d + WORD * lane);
        fetches += 2;
        const int p = raw_stop(ra, rb);
        const uint32_t m = __ballot_sync(0xffffffffu, p < WORD);
        if (m) {
            const int f = __ffs(m) - 1;
            const int64_t lf = d + WORD * lane + p;
            // at the stop byte: a's terminator with b equal (equal strings),
            // or the first differing byte (a terminator is the smallest byte)
            const uint32_t ca = p < WORD ? (uint32_t)(ra >> (8 * p)) & 255u : 0u;
            const uint32_t cb = p < WORD ? (uint32_t)(rb >> (8 * p)) & 255u : 0u;
            const int le = ca <= cb;
            *l = __shfl_sync(0xffffffffu, lf, f);
            return __shfl_sync(0xffffffffu, le, f);
        }
    }
}

// After a round: every kept run (slots tied on all characters before
// `depth`) of 2..SMALL_RUN strings is sorted by direct warp-wide string
// comparisons (stable insertion sort: ties keep tag order), its interior LCPs
// written, and its slots retired (keep = false).  Returns whether any run was
// finished.  xs (slot-indexed, gn entries) is scratch.
template <int IT>
__device__ bool finish_small_runs(bool (&keep)[IT], const bool (&brk)[IT], uint32_t (&meta)[IT],
                                  const int64_t* __restrict__ hbt, int64_t depth,
                                  const uint8_t* __restrict__ arena, int64_t alen,
                                  uint64_t* __restrict__ xs, int gn,
                                  int64_t* __restrict__ lcp_run, unsigned& fetches, int lane) {
    // run starts and ends among the kept slots, in slot order
    bool small_any = false;
    uint32_t starts[IT];
#pragma unroll
    for (int e = 0; e < IT; e++) starts[e] = __ballot_sync(0xffffffffu, keep[e] && brk[e]);
    // stage (handle << 11 | tag) of every kept slot
#pragma unroll
    for (int e = 0; e < IT; e++)
        if (keep[e]) xs[lane * IT + e] = ((uint64_t)hbt[meta[e] & 0x7ff] << 11) | (meta[e] & 0x7ff);
    __syncwarp();
    // walk the runs in slot order (run start slot s = lane' * IT + e')
    uint32_t done_mask[IT];
#pragma unroll
    for (int e = 0; e < IT; e++) done_mask[e] = 0;
    for (int L = 0; L < 32; L++) {
#pragma unroll
        for (int e = 0; e < IT; e++) {
            if (!(starts[e] >> L & 1)) continue;
            const int s = L * IT + e;
            // run length: kept slots from s while no new start / not past keep
            int z = 1;
            while (s + z < gn && z <= SMALL_RUN) {
                const int q = s + z, ql = q / IT, qe = q % IT;
                bool kq = false, bq = false;
#pragma unroll
                for (int f = 0; f < IT; f++)
                    if (f == qe) {
                        kq = __shfl_sync(0xffffffffu, keep[f], ql);
                        bq = __shfl_sync(0xffffffffu, brk[f], ql);
                    }
                if (!kq || bq) break;
                z++;
            }
            if (z > SMALL_RUN || z < 2) continue;
            small_any = true;
            // stable insertion sort of xs[s .. s+z) by string content; an
            // element that stays put keeps the LCP its one comparison found
            int64_t lk[SMALL_RUN];
            bool moved = false;
            for (int k = 1; k < z; k++) {
                const uint64_t x = xs[s + k];
                int j = k - 1;
                int64_t l = 0;
                while (j >= 0 && !warp_le(arena, alen, (int64_t)(xs[s + j] >> 11), (int64_t)(x >> 11),
                                          depth, &l, fetches, lane)) {
                    __syncwarp();
                    if (lane == 0) xs[s + j + 1] = xs[s + j];
                    __syncwarp();
                    j--;
                }
                moved |= j != k - 1;
                lk[k] = l;
                __syncwarp();
                if (lane == 0) xs[s + j + 1] = x;
                __syncwarp();
            }
            for (int k = 1; k < z; k++) {
                int64_t l = lk[k];
                if (moved)
                    warp_le(arena, alen, (int64_t)(xs[s + k - 1] >> 11), (int64_t)(xs[s + k] >> 11),
                            depth, &l, fetches, lane);
                if (lane == 0 && lcp_run) lcp_run[s + k] = l;
            }
            // retire the run's slots (lane l' owns slots l'*IT .. l'*IT+IT-1)
            for (int k = 0; k < z; k++) {
                const int q = s + k;
                if (lane == q / IT) {
#pragma unroll
                    for (int f = 0; f < IT; f++)
                        if (f == q % IT) done_mask[f] = 1;
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < IT; e++)
        if (done_mask[e]) {
            const int i = lane * IT + e;
            keep[e] = false;
            meta[e] = ((uint32_t)i << 11) | (uint32_t)(xs[i] & 0x7ff);  // finished, new tag
        }
    return __any_sync(0xffffffffu, small_any);
}

// One warp finishes one run of gn <= 32*IT strings that occupy slots
// g0 .. g0+gn-1 of the segment and share `depth` characters.  On entry the
// words at `depth` are in key[] (slot order = ord[g0 + i]) when have_keys,
// else they are fetched.  Writes LCPs (absolute depths) for the run's
// interior and the final tag order back to ord[g0 ..].
template <int IT>
__device__ void warp_finish(const int64_t* __restrict__ hbt, uint16_t* __restrict__ ord,
                            uint64_t* __restrict__ kb, uint64_t* __restrict__ xs,
                            Rec* __restrict__ segrec, int64_t cd,
                            int cnv, int g0, int gn, int64_t depth, uint64_t (&key)[IT],
                            const uint8_t* __restrict__ arena, int64_t alen,
                            int64_t* __restrict__ lcp_seg, unsigned& fetches, int lane,
                            bool have_keys = false) {
    // have_keys: key[] already holds the words at depth of slots lane*IT+e
    // (k_warp_sort's one-load prologue)
    uint32_t meta[IT];
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int i = lane * IT + e;
        if (!have_keys || i >= gn) key[e] = ~0ull;
        meta[e] = i < gn ? (1u << 22) | ord[g0 + i] : (uint32_t)i << 11;
    }
    if (!have_keys)
        rekey<IT, false>(key, meta, segrec, hbt, cd, cnv, depth, arena, alen, fetches, xs + g0,
                         lane * IT, gn, lane, 32);
    int wrounds = 0;
    for (;;) {
        // ---- sort the active slots by (group, word, tag) ------------------
        uint64_t o = 0, a = ~0ull;
#pragma unroll
        for (int e = 0; e < IT; e++)
            if (meta[e] >> 22 & 1) { o |= key[e]; a &= key[e]; }
        const PextLut px = pext_lut_setup(warp_or64(o) ^ warp_and64(a));
        if (px.cb == 0) {
            // all active words equal: the slots are already in (group, tag)
            // order (duplicate-heavy inputs spend most rounds here)
        } else if (px.cb <= 45) {
            // words by tag (kb) and by slot (xs, packed in one rolled loop)
#pragma unroll
            for (int e = 0; e < IT; e++) {
                const int i = lane * IT + e;
                if (meta[e] >> 22 & 1) kb[meta[e] & 0x7ff] = key[e];
                if (i < gn) xs[g0 + i] = key[e];
            }
            __syncwarp();
            for (int q = lane; q < gn; q += 32) xs[g0 + q] = pext_lut_key(xs[g0 + q], px);
            __syncwarp();
            uint64_t c[IT];
#pragma unroll
            for (int e = 0; e < IT; e++) {
                const uint32_t tag = meta[e] & 0x7ff;
                if (meta[e] >> 22 & 1)
                    c[e] = ((uint64_t)(meta[e] >> 11 & 0xff) << 56) | (xs[g0 + lane * IT + e] << 11) | tag;
                else
                    c[e] = ((uint64_t)(lane * IT + e) << 56) | tag;
            }
            __syncwarp();
            warp_bitonic_u64<IT>(c, lane);
#pragma unroll
            for (int e = 0; e < IT; e++) {
                const uint32_t tag = (uint32_t)c[e] & 0x7ff;
                if (meta[e] >> 22 & 1) key[e] = kb[tag];
                meta[e] = (meta[e] & ~0x7ffu) | tag;
            }
            __syncwarp();
        } else {
            warp_bitonic_generic<IT>(key, meta, lane);
        }
        // ---- LCPs at word changes, run breaks -----------------------------
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
        }
        if (!__any_sync(0xffffffffu, any) || depth > alen) break;  // alen: corrupt-input guard
        // runs still tied after FSR_ROUNDS + 1 words: finish the small ones directly
        // (pairs of suffixes inside copied blocks share kilobytes)
        if (wrounds >= FSR_ROUNDS && finish_small_runs<IT>(keep, brk, meta, hbt, depth + WORD, arena, alen,
                                                  xs + g0, gn, lcp_seg ? lcp_seg + g0 : nullptr,
                                                  fetches, lane)) {
            any = false;
#pragma unroll
            for (int e = 0; e < IT; e++) any |= keep[e];
            if (!__any_sync(0xffffffffu, any)) break;
        }
#pragma unroll
        for (int e = 0; e < IT; e++)
            if (keep[e] && brk[e]) run = lane * IT + e + 1;
        uint32_t incl = run;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o2);
            if (lane >= o2) incl = max(incl, y);
        }
        uint32_t cur = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) cur = 0;
        depth += WORD;
        uint32_t nstarts = 0;
#pragma unroll
        for (int e = 0; e < IT; e++) {
            const int i = lane * IT + e;
            if (keep[e] && brk[e]) {
                cur = i + 1;
                nstarts++;
            }
            const uint32_t tag = meta[e] & 0x7ff;
            meta[e] = keep[e] ? ((1u << 22) | ((cur - 1) << 11) | tag) : (((uint32_t)i << 11) | tag);
        }
        // a single run still tied after three words: jump to its common prefix
        if (++wrounds >= 3 && __reduce_add_sync(0xffffffffu, nstarts) == 1)
            depth = run_common_prefix<IT>(meta, hbt, depth, arena, alen, fetches, xs + g0, lane);
        rekey<IT, false>(key, meta, segrec, hbt, cd, cnv, depth, arena, alen, fetches, xs + g0,
                     lane * IT, gn, lane, 32);
    }
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int i = lane * IT + e;
        if (i < gn) ord[g0 + i] = (uint16_t)(meta[e] & 0x7ff);
    }
}

// ---------------------------------------------------------------------------
// k_warp_sort: one warp per segment of <= 32*ITEMS strings

// one segment per warp; 8 warps per CTA (4 for 256-string segments, whose
// per-warp staging would exceed the 48 KB of static shared memory)
__host__ __device__ constexpr int ws_nt(int items) { return items >= 8 ? 128 : 256; }
// 4 CTAs per SM: caps k_warp_sort<8> at 128 registers (it took 167, 3 CTAs)
constexpr int WS_MINB = 4;
#ifndef GROUP_MODE_MIN_W
#define GROUP_MODE_MIN_W 8
#endif

template <int ITEMS>
__global__ void __launch_bounds__(ws_nt(ITEMS), WS_MINB) k_warp_sort(
    const SegDev* __restrict__ segs, int64_t nsegs, Rec* __restrict__ recA,
    Rec* __restrict__ recB, const uint8_t* __restrict__ arena, int64_t alen,
    int64_t* __restrict__ out_h, int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    constexpr int CAP = 32 * ITEMS, WS_NT = ws_nt(ITEMS);
    __shared__ int64_t s_h[WS_NT / 32][CAP];
    __shared__ uint64_t s_k[WS_NT / 32][CAP];
    __shared__ uint16_t s_o[WS_NT / 32][CAP];
    __shared__ uint64_t s_x[WS_NT / 32][CAP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (WS_NT / 32) + w;
    if (gw >= nsegs) return;  // whole warp
    const SegDev sg = segs[gw];
    const int m = sg.n;
    const int64_t lo = sg.lo;
    Rec* segrec = ((sg.flags & SEG_IN_B) ? recB : recA) + lo;
    const int nv = sg.flags & SEG_NV_MASK;
    int64_t* wh = s_h[w];
    uint16_t* wo = s_o[w];
    unsigned fetches = 0;
    // one 32-byte load per string: its handle and, when cached, the word at
    // the segment's depth (slot = tag = lane * ITEMS + e)
    uint64_t key[ITEMS];
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = lane * ITEMS + e;
        if (i < m) {
            const Rec r = segrec[i];
            wh[i] = r.h;
            wo[i] = (uint16_t)i;
            key[e] = r.w[0];
        }
    }
    __syncwarp();
    warp_finish<ITEMS>(wh, wo, s_k[w], s_x[w], segrec, sg.depth, nv, 0, m, sg.depth, key, arena, alen,
                       lcps ? lcps + lo : nullptr, fetches, lane, nv >= 1);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = e * 32 + lane;
        if (i < m) {
            S5G_CHECK(wo[i] < m);
            out_h[lo + i] = wh[wo[i]];
        }
    }
    fetches = __reduce_add_sync(0xffffffffu, fetches);
    if (lane == 0) {
        if (fetches) atomicAdd(&ctr->seg_fetches, (unsigned long long)fetches);
        atomicAdd(&ctr->small_elems, (unsigned long long)m);
    }
}

// ---------------------------------------------------------------------------
// k_cta_sort: W warps x 256 slots (8 per lane) finish one segment of up to
// 256*W strings.  The first round(s) run CTA-wide; once every remaining run
// has <= 256 strings, each run goes to one warp (warp_finish).

template <int W>
struct CtaSortSmem {
    int64_t h[256 * W];           // handle by tag
    uint64_t kb[256 * W];         // word by tag (composite rounds, warp runs)
    uint64_t xk[256 * W];         // cross-warp exchange
    union {
        // the two-word first round keeps the second word by tag here; the
        // generic exchange, the slot order and the run list come later
        uint64_t kb1[256 * W];
        struct {
            uint32_t xm[256 * W];
            uint16_t ord[256 * W];        // tag at slot
            uint16_t gs[128 * W], ge[128 * W];  // first / last slot of each remaining run
        };
    };
    uint64_t red[4 * W];
    uint64_t last_key[W], last_key1[W];
    uint32_t first_brk[W], first_act[W], wmax[W], wcnt[W];
    Pext px[2];  // the round's bit-extract plans (read in the packing loop)
};

// In-lane stage at distance J < 8.  The direction bit (slot & k) is the same
// for all 8 slots of a thread once k >= 8; below that it varies with e.
template <int J, typename T>
__device__ __forceinline__ void cta_inlane(T (&c)[8], int base, int k) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
        const int f = e ^ J;
        if (f > e) {
            const bool up = ((base + e) & k) == 0;
            const bool sw = (c[f] < c[e]) == up;
            const T x = c[e], y = c[f];
            c[e] = sw ? y : x;
            c[f] = sw ? x : y;
        }
    }
}

// In-lane stage at distance J < 8 once k >= 8: one direction for all 8
// slots of the thread (base is a multiple of 8).
template <int J, typename T>
__device__ __forceinline__ void cta_inlane_u(T (&c)[8], bool up) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
        const int f = e ^ J;
        if (f > e) {
            const bool sw = (c[f] < c[e]) == up;
            const T x = c[e], y = c[f];
            c[e] = sw ? y : x;
            c[f] = sw ? x : y;
        }
    }
}

template <int W, typename T>
__device__ void cta_bitonic(T (&c)[8], int base, T* xch) {
    constexpr int P = 256 * W, NT = 32 * W;
    // k = 2, 4: directions vary inside the thread
    cta_inlane<1>(c, base, 2);
    cta_inlane<2>(c, base, 4);
    cta_inlane<1>(c, base, 4);
#pragma unroll 1
    for (int k = 8; k <= P; k <<= 1) {
        const bool upk = (base & k) == 0;
        // distances >= 8: partner slot differs in a lane/warp bit, and the
        // keep-the-smaller decision is uniform across the thread's slots
#pragma unroll 1
        for (int j = k >> 1; j >= 8; j >>= 1) {
            const bool keep_min = ((base & j) == 0) == upk;
            if (j < 256) {
                const int lx = j / 8;
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const T o = __shfl_xor_sync(0xffffffffu, c[e], lx);
                    c[e] = ((o < c[e]) == keep_min) ? o : c[e];
                }
            } else {
                // [e][thread] layout: conflict-free; partner = thread ^ (j / 8)
                const int pt = threadIdx.x ^ (j / 8);
#pragma unroll
                for (int e = 0; e < 8; e++) xch[e * NT + threadIdx.x] = c[e];
                __syncthreads();
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const T o = xch[e * NT + pt];
                    c[e] = ((o < c[e]) == keep_min) ? o : c[e];
                }
                __syncthreads();
            }
        }
        cta_inlane_u<4>(c, upk);
        cta_inlane_u<2>(c, upk);
        cta_inlane_u<1>(c, upk);
    }
}

template <int W>
__device__ void cta_bitonic_generic(uint64_t (&key)[8], uint32_t (&meta)[8], int base,
                                    CtaSortSmem<W>& S) {
    constexpr int P = 256 * W;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < 8) {
#pragma unroll
                for (int e = 0; e < 8; e++) {
#pragma unroll
                    for (int jj = 1; jj < 8; jj <<= 1) {
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
                const int lx = j / 8;
#pragma unroll
                for (int e = 0; e < 8; e++) {
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
                constexpr int NT = 32 * W;
                const int pt = threadIdx.x ^ (j / 8);
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    S.xk[e * NT + threadIdx.x] = key[e];
                    S.xm[e * NT + threadIdx.x] = meta[e];
                }
                __syncthreads();
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const int i = base + e;
                    const uint64_t ok = S.xk[e * NT + pt];
                    const uint32_t om = S.xm[e * NT + pt];
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
}

#ifndef CTA_SORT_WARPS_PER_SM
#define CTA_SORT_WARPS_PER_SM 24  // 80 registers per thread
#endif
template <int W>
__global__ void __launch_bounds__(32 * W, CTA_SORT_WARPS_PER_SM / W) k_cta_sort(
    const SegDev* __restrict__ segs, int64_t nsegs, Rec* __restrict__ recA,
    Rec* __restrict__ recB, const uint8_t* __restrict__ arena, int64_t alen,
    int64_t* __restrict__ out_h, int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    constexpr int ITEMS = 8, NT = 32 * W;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    CtaSortSmem<W>& S = *reinterpret_cast<CtaSortSmem<W>*>(smem_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const SegDev sg = segs[blockIdx.x];
    const int m = sg.n;
    const int64_t lo = sg.lo;
    Rec* segrec = ((sg.flags & SEG_IN_B) ? recB : recA) + lo;
    const int nv = sg.flags & SEG_NV_MASK;
    const int64_t d0 = sg.depth;
    int64_t* lcp_seg = lcps ? lcps + lo : nullptr;
    int64_t depth = sg.depth;
    unsigned fetches = 0;
    uint64_t key[ITEMS];
    uint32_t meta[ITEMS];
    const int base = threadIdx.x * ITEMS;  // first slot of this thread
    int64_t cd = d0;  // record cache: words from depth cd, cnv of them valid
    int cnv = nv;
#pragma unroll
    for (int e = 0; e < ITEMS; e++) {
        const int i = base + e;
        key[e] = ~0ull;
        meta[e] = i < m ? (1u << 22) | (uint32_t)i : ((uint32_t)i << 11) | (uint32_t)i;
    }
    if (nv >= 1) {
        // one 32-byte load per string brings its handle, the word at the
        // segment's depth and the next one (the first round's two-word
        // window) -- instead of three dependent rounds of loads
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            if (i < m) {
                const Rec r = segrec[i];
                S.h[i] = r.h;
                key[e] = r.w[0];
                if (nv >= 2) S.kb1[i] = r.w[1];
            }
        }
        __syncthreads();
    } else {
        for (int i = threadIdx.x; i < m; i += NT) S.h[i] = segrec[i].h;
        __syncthreads();
        rekey<ITEMS, true>(key, meta, segrec, S.h, cd, cnv, depth, arena, alen, fetches, S.xk, base,
                           256 * W, threadIdx.x, NT);
    }
    bool group_mode = false, first_round = true, used_two = false;
    int rounds = 0;
    uint64_t k1[ITEMS];  // second word of the slot in a two-word round
    for (;;) {
        // ---- sort by (group, word, tag): packed u32/u64 when the bits fit --
        bool two = false;  // this round sorts by the words at depth and depth + 8
        int jb = 0;        // ... the leading jb characters of the second one
        {
            // the first round may take the record's second cached word along
            // when both words' varying bits fit one u64 beside the tag: one
            // round instead of two for low-entropy keys (DNA: 4 bits/char)
            const bool try_two = first_round && cnv >= 2;  // (first round: depth == cd)
            uint64_t o = 0, a = ~0ull, o1 = 0, a1 = ~0ull;
#pragma unroll
            for (int e = 0; e < ITEMS; e++) {
                k1[e] = 0;
                if (meta[e] >> 22 & 1) {
                    o |= key[e];
                    a &= key[e];
                    if (try_two) {
                        k1[e] = nv >= 2 ? S.kb1[base + e] : segrec[base + e].w[1];
                        o1 |= k1[e];
                        a1 &= k1[e];
                    }
                }
            }
            o = warp_or64(o);
            a = warp_and64(a);
            if (try_two) {
                o1 = warp_or64(o1);
                a1 = warp_and64(a1);
            }
            if (lane == 0) { S.red[w] = o; S.red[W + w] = a; S.red[2 * W + w] = o1; S.red[3 * W + w] = a1; }
            __syncthreads();
            o = 0;
            a = ~0ull;
            o1 = 0;
            a1 = ~0ull;
#pragma unroll
            for (int v = 0; v < W; v++) {
                o |= S.red[v];
                a &= S.red[W + v];
                o1 |= S.red[2 * W + v];
                a1 &= S.red[3 * W + v];
            }
            const int cb0 = __popcll(o ^ a);  // word0 bits (the plans: thread 0, below)
            if (try_two) {
                // as many leading characters of word1 as fit beside word0's
                // varying bits in 53 bits; u32 single-word rounds are cheaper
                // when ties after word0 are unlikely (m^2 <= 2^cb0)
                const uint64_t V1 = o1 ^ a1;
                int bits = cb0;
                while (jb < WORD && bits + __popc((uint32_t)(V1 >> (56 - 8 * jb)) & 255u) <= 53)
                    bits += __popc((uint32_t)(V1 >> (56 - 8 * jb)) & 255u), jb++;
                const bool u32_ok = cb0 <= 21 && (uint64_t)m * (uint64_t)m <= (1ull << cb0);
                two = jb > 0 && !u32_ok;
                if (!two) jb = 0;
                const uint64_t keep1 = jb == WORD ? ~0ull : ~(~0ull >> (8 * jb));
#pragma unroll
                for (int e = 0; e < ITEMS; e++) k1[e] &= keep1;  // window of jb chars (0: none)
                o1 &= keep1;
                a1 &= keep1;
            }
            const int mode = two ? 0 : (first_round && cb0 <= 21) ? 1 : (cb0 <= 42) ? 2 : 3;
            if (cb0 == 0 && (!two || (o1 ^ a1) == 0)) {
                // every active slot has the same window: already in (group,
                // tag) order, nothing to sort
            } else if (mode != 3) {
                // stage the words by tag (kb, kb1) and by slot (xk), pack the
                // varying bits of every slot in one rolled loop, build the
                // sort values: two-word (word0 bits | word1 bits | tag), u32
                // (word bits | tag) on the first round, else (group | bits | tag)
                if (threadIdx.x == 0) {
                    S.px[0] = pext_setup(o ^ a);
                    S.px[1] = pext_setup(o1 ^ a1);
                }
#pragma unroll
                for (int e = 0; e < ITEMS; e++) {
                    const uint32_t tag = meta[e] & 0x7ff;
                    if (meta[e] >> 22 & 1) {
                        S.kb[tag] = key[e];
                        if (two) S.kb1[tag] = k1[e];  // tag == slot in the first round
                    }
                    S.xk[base + e] = key[e];
                }
                __syncthreads();
                const int lim = first_round ? m : 256 * W;
                const Pext p0 = S.px[0], p1 = S.px[1];
                for (int q = threadIdx.x; q < lim; q += NT) {
                    uint64_t v = pext_key(S.xk[q], p0);
                    if (two) v = (v << p1.cb) | pext_key(S.kb1[q], p1);
                    S.xk[q] = v;
                }
                __syncthreads();
                if (mode == 1) {
                    uint32_t c[ITEMS];
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        const uint32_t tag = meta[e] & 0x7ff;
                        c[e] = (meta[e] >> 22 & 1) ? (((uint32_t)S.xk[base + e] << 11) | tag) : 0xffffffffu;
                    }
                    __syncthreads();  // xk becomes the exchange buffer
                    cta_bitonic<W, uint32_t>(c, base, reinterpret_cast<uint32_t*>(S.xk));
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        if (meta[e] >> 22 & 1) {
                            const uint32_t tag = c[e] & 0x7ff;
                            key[e] = S.kb[tag];
                            meta[e] = (meta[e] & ~0x7ffu) | tag;
                        }
                    }
                } else {
                    uint64_t c[ITEMS];
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        const uint32_t tag = meta[e] & 0x7ff;
                        if (mode == 0)
                            c[e] = (meta[e] >> 22 & 1) ? ((S.xk[base + e] << 11) | tag) : ~0ull;
                        else
                            c[e] = (meta[e] >> 22 & 1)
                                       ? (((uint64_t)(meta[e] >> 11 & 0x7ff) << 53) | (S.xk[base + e] << 11) | tag)
                                       : (((uint64_t)(base + e) << 53) | tag);
                    }
                    __syncthreads();  // xk becomes the exchange buffer
                    cta_bitonic<W, uint64_t>(c, base, S.xk);
#pragma unroll
                    for (int e = 0; e < ITEMS; e++) {
                        const uint32_t tag = (uint32_t)c[e] & 0x7ff;
                        if (meta[e] >> 22 & 1) {
                            key[e] = S.kb[tag];
                            if (two) k1[e] = S.kb1[tag];
                        }
                        if (mode == 0) {
                            if (meta[e] >> 22 & 1) meta[e] = (meta[e] & ~0x7ffu) | tag;
                        } else {
                            meta[e] = (meta[e] & ~0x7ffu) | tag;
                        }
                    }
                }
            } else {
                cta_bitonic_generic<W>(key, meta, base, S);
            }
        }
        rounds++;
        used_two |= two;
        // ---- LCPs at word changes, run breaks -------------------------------
        // (a two-word round compares (word, word1); a string whose first word
        // holds its terminator has word1 = 0, so pair equality is string
        // equality within the 16-character window)
        const int step = WORD + jb;
        uint64_t prev_last = __shfl_up_sync(0xffffffffu, key[ITEMS - 1], 1);
        uint64_t prev_last1 = __shfl_up_sync(0xffffffffu, k1[ITEMS - 1], 1);
        if (lane == 31) {
            S.last_key[w] = key[ITEMS - 1];
            S.last_key1[w] = k1[ITEMS - 1];
        }
        __syncthreads();
        if (lane == 0 && w > 0) {
            prev_last = S.last_key[w - 1];
            prev_last1 = S.last_key1[w - 1];
        }
        bool brk[ITEMS];
        int tw[ITEMS];  // terminator position in the round's window (step if none)
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            const bool act = meta[e] >> 22 & 1;
            const int grp = meta[e] >> 11 & 0x7ff;
            brk[e] = true;
            tw[e] = term_pos(key[e]);
            // masked word1: a zero byte at jb marks the window end (tw == step)
            if (two && tw[e] == WORD) tw[e] = WORD + min(term_pos(k1[e]), jb);
            if (act && i != grp) {
                const uint64_t pk = e ? key[e - 1] : prev_last;
                const uint64_t pk1 = e ? k1[e - 1] : prev_last1;
                if (pk != key[e]) {
                    if (lcp_seg) lcp_seg[i] = depth + (__clzll(pk ^ key[e]) >> 3);
                } else if (pk1 != k1[e]) {  // two-word round only
                    if (lcp_seg) lcp_seg[i] = depth + WORD + (__clzll(pk1 ^ k1[e]) >> 3);
                } else {
                    brk[e] = false;
                    if (lcp_seg && tw[e] < step) lcp_seg[i] = depth + tw[e];
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
            keep[e] = act && tw[e] == step && (!brk[e] || (na && !nb));
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
        // longest kept run decides: another CTA round, or one warp per run
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
        if (lmax <= (W >= GROUP_MODE_MIN_W ? 256u : 64u)) {
            // ---- group mode: slot order + list of the kept runs -------------
#pragma unroll
            for (int e = 0; e < ITEMS; e++) S.ord[base + e] = (uint16_t)(meta[e] & 0x7ff);
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
            uint32_t gi = (off + pre) & 0xffff, ge_i = (off + pre) >> 16;
#pragma unroll
            for (int e = 0; e < ITEMS; e++) {
                const int i = base + e;
                if (keep[e] && brk[e]) S.gs[gi++] = (uint16_t)i;
                if (kend[e]) S.ge[ge_i++] = (uint16_t)i;
            }
            __syncthreads();
            if (threadIdx.x == 0) S.wcnt[0] = tot2 & 0xffff;
            __syncthreads();
            group_mode = true;
            depth += step;
            break;
        }
        depth += step;
        first_round = false;
#pragma unroll
        for (int e = 0; e < ITEMS; e++) {
            const int i = base + e;
            if (keep[e] && brk[e]) cur = i + 1;
            const uint32_t tag = meta[e] & 0x7ff;
            meta[e] = keep[e] ? ((1u << 22) | ((cur - 1) << 11) | tag) : (((uint32_t)i << 11) | tag);
        }
        rekey<ITEMS, true>(key, meta, segrec, S.h, cd, cnv, depth, arena, alen, fetches, S.xk, base,
                       256 * W, threadIdx.x, NT);
        __syncthreads();  // S.wmax / S.last_key / S.wcnt / S.red reuse
    }
    if (!group_mode) {
#pragma unroll
        for (int e = 0; e < ITEMS; e++) S.ord[base + e] = (uint16_t)(meta[e] & 0x7ff);
    } else {
        // one warp per remaining run, each finished entirely in registers
        const uint32_t ngroups = S.wcnt[0];
        for (uint32_t g = w; g < ngroups; g += W) {
            const int g0 = S.gs[g], gn = S.ge[g] - g0 + 1;
            const int64_t d = depth;
            if (gn <= 32) {
                uint64_t r1[1];
                warp_finish<1>(S.h, S.ord, S.kb, S.xk, segrec, cd, cnv, g0, gn, d, r1, arena, alen, lcp_seg, fetches, lane);
            } else if (gn <= 64) {
                uint64_t r2[2];
                warp_finish<2>(S.h, S.ord, S.kb, S.xk, segrec, cd, cnv, g0, gn, d, r2, arena, alen, lcp_seg, fetches, lane);
            } else if constexpr (W >= GROUP_MODE_MIN_W) {
                // (smaller CTAs enter group mode only with runs <= 64)
                if (gn <= 128) {
                    uint64_t r4[4];
                    warp_finish<4>(S.h, S.ord, S.kb, S.xk, segrec, cd, cnv, g0, gn, d, r4, arena, alen, lcp_seg, fetches, lane);
                } else {
                    uint64_t r8[8];
                    warp_finish<8>(S.h, S.ord, S.kb, S.xk, segrec, cd, cnv, g0, gn, d, r8, arena, alen, lcp_seg, fetches, lane);
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += NT) {
        S5G_CHECK(S.ord[i] < m);
        out_h[lo + i] = S.h[S.ord[i]];
    }
    fetches = __reduce_add_sync(0xffffffffu, fetches);
    if (lane == 0 && fetches) atomicAdd(&ctr->seg_fetches, (unsigned long long)fetches);
    if (threadIdx.x == 0) {
        atomicAdd(&ctr->small_elems, (unsigned long long)m);
        unsigned long long* fc = g_fin_ctr + 4 * (W == 2 ? 0 : W == 4 ? 1 : 2);
        atomicAdd(fc + 0, 1ull);
        atomicAdd(fc + 1, (unsigned long long)rounds);
        atomicAdd(fc + 2, used_two ? 1ull : 0ull);
        atomicAdd(fc + 3, group_mode ? 1ull : 0ull);
    }
}

}  // namespace s5g
