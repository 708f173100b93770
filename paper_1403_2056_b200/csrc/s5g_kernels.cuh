// s5g_kernels.cuh -- sm_100a kernels of the S^5 string sorter.
//
// Pipeline of one device-wide S^5 step over a batch of "large" segments
// (the GPU form of s5_step, ssss.py:281-297, and of the fully parallel step
// _ParallelS5Run._phased_step, parallel.py:359-398):
//   k_sample_tree  draw_sample + select_splitters (ssss.py:76-146), 1 CTA/step
//   k_classify     classify_keys + per-tile bincount (ssss.py:149-181, 292)
//   k_scan_cols    tile-minor prefix per bucket      (parallel.py:379-385)
//   k_scan_buckets bucket-major exclusive scan, children, boundary records
//   k_scatter      stable scatter (argsort(kind=stable) + gather, ssss.py:295)
// Segments of up to MED_MAX strings take a whole step in one CTA
// (k_step_cta); segments of up to SMALL_MAX strings are finished by the
// register finishers k_warp_sort / k_cta_sort (s5g_warpsort.cuh): the GPU
// stand-in for the MKQS / insertion leaves (mkqs.py:196-253,
// basecase.py:67-116) -- repeated stable sorts on 8-byte keys with depth
// advancing by a word.
#pragma once
#include "s5g_device.cuh"

namespace s5g {

constexpr int TILE = 32768;     // elements per classify / scatter CTA
constexpr int MIN_TILE = 8192;  // ... at least, for a root step spread over all SMs
constexpr int CLS_NT = 512;
constexpr int SC_NT = 512;
constexpr int SC_ITEMS = 4;
constexpr int SC_SUB = SC_NT * SC_ITEMS;  // 4096-element stable sub-tiles
constexpr int SC_RB = 7;                  // radix bits per ranking pass
constexpr int SC_R = 1 << SC_RB;
constexpr uint16_t BID_SENTINEL = 0x3FFF; // > any bucket id (max 16382)
constexpr int SAMPLE_NT = 1024;

// Work record of one string: its handle and the next three words from the
// segment's depth (the paper's character cache, widened to one 32-byte
// sector: scatters write whole sectors, and the finishers find the next two
// words without a gather).  Words past the terminator are 0.
struct __align__(32) Rec {
    int64_t h;
    uint64_t w[3];
};
constexpr int NCACHE = 3;

// SegDev.flags: number of valid cached words (0..3) | data in buffer B
enum : int32_t { SEG_NV_MASK = 3, SEG_IN_B = 4 };

struct StepDev {
    int64_t lo, n, depth;
    int32_t v, levels, nb, nvalid;   // nvalid: cached words valid at depth (0 = refill)
    int64_t tile0;
    int32_t ntiles, sblk0;  // sblk0: first 1024-bucket block of k_scan_buckets
    int64_t cnt_off;   // first entry in the tile x bucket count matrix
    int64_t bk_off;    // first entry in tot / bstart
    int64_t tree_off;  // first entry in tree / inorder / tpos / eqb (even)
    int64_t cblk0;     // first 32-column block of k_scan_cols
    int32_t count;     // sample size (>= v)
    int32_t tile;      // strings per classify / scatter CTA (<= TILE)
};

struct SegDev {
    int64_t lo, depth;
    int32_t n, flags;
};

// small segments are finished in registers in seven size classes: one warp
// for <= 32, 64, 128, 256 strings (1, 2, 4, 8 slots per lane), 2, 4 or 8
// warps of 256 slots for <= 512, 1024, 2048
constexpr int NCLS = 7;
constexpr int SMALL_MAX = 2048;
#ifndef SEG_TARGET_CFG
#define SEG_TARGET_CFG 1024
#endif
constexpr int SEG_TARGET = SEG_TARGET_CFG;   // device-wide steps aim at buckets of this size

struct Counters {
    unsigned long long n_large, n_bound, fetches, seg_fetches, small_elems;
    unsigned long long n_cls[NCLS];
    unsigned long long cls_elems[NCLS];
};

struct ClassLists {
    int64_t off[NCLS];
};

// tree_capacity (ssss.py:67-73)
__host__ __device__ inline int64_t tree_capacity(int64_t n, int64_t v) {
    int64_t limit = v < (n / 2 > 1 ? n / 2 : 1) ? v : (n / 2 > 1 ? n / 2 : 1);
    int d = 0;
    while ((1LL << (d + 1)) - 1 <= limit) d++;
    const int64_t t = (1LL << d) - 1;
    return t > 1 ? t : 1;
}

// Splitters for a GPU step: v+1 range buckets of about SEG_TARGET strings
// each (the reference's tree_capacity caps it; v and the sample size never
// change the output, only the bucket sizes).
__host__ __device__ inline int64_t gpu_tree_capacity(int64_t n, int64_t vcap) {
    int64_t want = 1;
    while (want < VMAX && (want + 1) * SEG_TARGET < n) want = 2 * want + 1;
    const int64_t t = tree_capacity(n, vcap);
    return want < t ? want : t;
}

__host__ __device__ inline int levels_of(int64_t v) {
    int l = 0;
    while ((1LL << l) < v + 1) l++;
    return l;
}

// oversampling: the reference's alpha = 2 for big trees, up to 16 for small
// ones (tighter buckets, same output)
__host__ __device__ inline int sample_count(int64_t v) {
    int a = (int)(1024 / (v + 1));
    a = a < 16 ? a : 16;
    a = a > OVERSAMPLE ? a : OVERSAMPLE;
    return a * (int)(v + 1) - 1;
}

// segments a single CTA takes through a whole S^5 step (k_step_cta)
#ifndef MED_MAX_CFG
#define MED_MAX_CFG 32768
#endif
constexpr int MED_MAX = MED_MAX_CFG;
#ifndef MED_VMAX_CFG
#define MED_VMAX_CFG 31
#endif
#ifndef MED_FREE_V
#define MED_FREE_V 1  // 0: splitter counts 2^L - 1 only, 4-fold oversampling (the earlier plan)
#endif
#ifndef MED_TARGET_CFG
#define MED_TARGET_CFG (MED_FREE_V ? 745 : 1024)
#endif
constexpr int MED_VMAX = MED_VMAX_CFG;  // <= 2*MED_VMAX+1 <= 255 buckets (uint8 ids)
constexpr int MED_NB = 2 * MED_VMAX + 1;
constexpr int MED_TARGET = MED_TARGET_CFG;  // strings per bucket a fused step aims at
static_assert(MED_NB <= 255, "k_step_cta keeps bucket ids in uint8");

// Splitters of a fused single-CTA step: buckets of about MED_TARGET strings,
// so its children mostly go straight to the warp finishers (a coarser split
// sent C5's 4096-string segments through another CTA-wide sort level).
__host__ __device__ inline int64_t med_tree_capacity(int64_t n, int64_t vcap) {
    int64_t want = 1;
    while (want < MED_VMAX && (want + 1) * MED_TARGET < n) want = 2 * want + 1;
    const int64_t t = tree_capacity(n, vcap);
    return want < t ? want : t;
}
__host__ __device__ inline int med_sample_count(int64_t v) {
    const int a = sample_count(v);
    const int cap = 4 * (int)(v + 1) - 1;
    return a < cap ? a : cap;
}

// Why: a fused step's children should FIT a finisher class, not straddle
// one.  With 2^L - 1 splitters and 4-fold oversampling C5's 4096-string
// segments split into 4 pieces of 1024 +- 50 %: half of them overflowed the
// 1024-slot class into the 2048-slot one at ~60 % fill.  Six pieces of
// 683 +- 25 % (MED_TARGET 745, 16-fold oversampling) nearly all fit it:
// C5 36.5 -> 35.9 ms, C4 7.20 -> 7.05 ms, C2 / C3 unchanged.  Measured
// alternatives: target 820 / 32-fold 35.9 (C2 +0.6 %), 820 / 64-fold 36.6,
// 380 / 32-fold 36.1 (C3 +7 %, C4 +4 %), 640 / 16 36.0 (C3 +6 %), 900 / 16
// 36.0, 745 / 8 36.1, 1024 / 16 36.6.
// Fused steps with a free number of splitters (MED_FREE_V): `veff` real
// splitters -- buckets of about MED_TARGET strings, not rounded to 2^L - 1 --
// in the complete tree of v = 2^L - 1 >= veff nodes, its last v - veff
// splitters the sample's ~0 padding (empty buckets at the top end).  With
// a-fold oversampling the sample has a (veff + 1) - 1 keys and select_tree is
// given a (v + 1) - 1: its equidistant picks at k a - 1 land on real keys for
// k <= veff and in the padding above.
#ifndef MED_OVERSAMPLE
#define MED_OVERSAMPLE 16
#endif
struct MedPlan { int v, veff, count, countp; };
__host__ __device__ inline MedPlan med_plan(int64_t n, int64_t vcap) {
    MedPlan p;
#if MED_FREE_V
    int64_t want = (n + MED_TARGET - 1) / MED_TARGET - 1;
    want = want < 1 ? 1 : want > MED_VMAX ? MED_VMAX : want;
    const int64_t t = tree_capacity(n, vcap);
    p.veff = (int)(want < t ? want : t);
    p.v = 1;
    while (p.v < p.veff) p.v = 2 * p.v + 1;
    int a = MED_OVERSAMPLE;
    while (a > 2 && a * (p.v + 1) > 16 * (MED_VMAX + 1)) a >>= 1;  // StepCtaSmem::s
    p.count = a * (p.veff + 1) - 1;
    p.countp = a * (p.v + 1) - 1;
#else
    p.v = p.veff = (int)med_tree_capacity(n, vcap);
    p.count = p.countp = med_sample_count(p.v);
#endif
    return p;
}

__host__ __device__ inline int size_class(int64_t n) {
    return n <= 32 ? 0 : n <= 64 ? 1 : n <= 128 ? 2 : n <= 256 ? 3 : n <= 512 ? 4 : n <= 1024 ? 5 : 6;
}

// ---------------------------------------------------------------------------
// shared-memory sorts

template <int NT>
__device__ void bitonic_u64(uint64_t* s, int P) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P / 2; i += NT) {
                int lo = 2 * i - (i & (j - 1)), hi = lo + j;
                bool up = (lo & k) == 0;
                uint64_t a = s[lo], b = s[hi];
                if ((a > b) == up) { s[lo] = b; s[hi] = a; }
            }
            __syncthreads();
        }
}

// Register bitonic of P = NT*IT keys (slot = threadIdx.x*IT + e): in-lane
// stages below IT, shuffles below 32*IT, shared memory above.
template <int J, int IT>
__device__ __forceinline__ void rb_inlane(uint64_t (&c)[IT], int base, int k) {
#pragma unroll
    for (int e = 0; e < IT; e++) {
        const int f = e ^ J;
        if (f > e) {
            const bool up = ((base + e) & k) == 0;
            const bool sw = (c[f] < c[e]) == up;
            const uint64_t x = c[e], y = c[f];
            c[e] = sw ? y : x;
            c[f] = sw ? x : y;
        }
    }
}

template <int IT>
__device__ void reg_bitonic_keys(uint64_t (&c)[IT], int P, uint64_t* xch, bool cta) {
    const int base = threadIdx.x * IT;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < IT) {
                if (j == 1) rb_inlane<1, IT>(c, base, k);
                else if (j == 2) rb_inlane<2, IT>(c, base, k);
                else if (j == 4) rb_inlane<4, IT>(c, base, k);
                else if (j == 8) rb_inlane<8, IT>(c, base, k);
            } else {
                const bool keep_min = ((base & j) == 0) == ((base & k) == 0);
                if (j < 32 * IT) {
                    const int lx = j / IT;
#pragma unroll
                    for (int e = 0; e < IT; e++) {
                        const uint64_t o = __shfl_xor_sync(0xffffffffu, c[e], lx);
                        c[e] = ((o < c[e]) == keep_min) ? o : c[e];
                    }
                } else {
                    // exchange through shared memory in [e][thread] layout: a
                    // warp touches 32 consecutive words per access (no bank
                    // conflicts); partner slot = same e, thread ^ (j / IT)
                    const int nt = cta ? (int)blockDim.x : 32;
                    const int pt = threadIdx.x ^ (j / IT);
#pragma unroll
                    for (int e = 0; e < IT; e++) xch[e * nt + threadIdx.x] = c[e];
                    if (cta) __syncthreads(); else __syncwarp();
#pragma unroll
                    for (int e = 0; e < IT; e++) {
                        const uint64_t o = xch[e * nt + pt];
                        c[e] = ((o < c[e]) == keep_min) ? o : c[e];
                    }
                    if (cta) __syncthreads(); else __syncwarp();
                }
            }
        }
    }
}

// Sort a full top-level sample s[0..16*NT) in place: 16 keys per thread in
// registers; distances < 512 never touch shared memory.
template <int NT>
__device__ void sort_sample16(uint64_t* s) {
    constexpr int IT = 16;
    uint64_t c[IT];
#pragma unroll
    for (int e = 0; e < IT; e++) c[e] = s[threadIdx.x * IT + e];
    __syncthreads();
    reg_bitonic_keys<IT>(c, NT * IT, s, true);
#pragma unroll
    for (int e = 0; e < IT; e++) s[threadIdx.x * IT + e] = c[e];
    __syncthreads();
}

// Sort (meta.group, key, meta.tag) lexicographically; meta = group<<16 | tag.
template <int NT>
__device__ void bitonic_pairs(uint64_t* key, uint32_t* meta, int P) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P / 2; i += NT) {
                int lo = 2 * i - (i & (j - 1)), hi = lo + j;
                bool up = (lo & k) == 0;
                uint64_t a = key[lo], b = key[hi];
                uint32_t ma = meta[lo], mb = meta[hi];
                bool gt = (ma >> 16) != (mb >> 16) ? (ma >> 16) > (mb >> 16)
                          : a != b               ? a > b
                                                 : (ma & 0xffff) > (mb & 0xffff);
                if (gt == up) {
                    key[lo] = b; key[hi] = a;
                    meta[lo] = mb; meta[hi] = ma;
                }
            }
            __syncthreads();
        }
}

// One stable LSD counting pass over SC_SUB (key, val) uint16 pairs by the
// SC_RB-bit digit at `shift`.  Warp w owns elements [w*128, w*128+128),
// item j / lane l is element w*128 + j*32 + l, so (digit, warp, item, lane)
// order is input order: stability comes from warp-minor digit offsets plus
// match_any ranks inside each warp.
template <int ITEMS = SC_ITEMS>
__device__ void rank_pass(const uint16_t* kin, const uint16_t* vin, uint16_t* kout,
                          uint16_t* vout, int shift, uint16_t* cnt, uint32_t* wsum) {
    constexpr int NW = SC_NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* cnt32 = reinterpret_cast<uint32_t*>(cnt);
    for (int i = threadIdx.x; i < SC_R * NW / 2; i += SC_NT) cnt32[i] = 0;
    __syncthreads();
    uint16_t kk[ITEMS], vv[ITEMS];
    uint32_t loc[ITEMS], dg[ITEMS];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        int e = w * (32 * ITEMS) + j * 32 + lane;
        kk[j] = kin[e];
        vv[j] = vin[e];
        uint32_t d = (kk[j] >> shift) & (SC_R - 1);
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t base = cnt[d * NW + w];
        __syncwarp();
        if (lane == __ffs(peers) - 1) cnt[d * NW + w] = (uint16_t)(base + __popc(peers));
        __syncwarp();
        loc[j] = base + __popc(peers & lt);
        dg[j] = d;
    }
    __syncthreads();
    // exclusive scan over (digit-major, warp-minor): SC_R*NW = 4096 entries
    {
        constexpr int PER = SC_R * NW / SC_NT;
        uint32_t v[PER], s = 0;
#pragma unroll
        for (int i = 0; i < PER; i++) { v[i] = cnt[threadIdx.x * PER + i]; s += v[i]; }
        uint32_t run = block_excl_sum<SC_NT>(s, wsum, nullptr);
#pragma unroll
        for (int i = 0; i < PER; i++) { cnt[threadIdx.x * PER + i] = (uint16_t)run; run += v[i]; }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        uint32_t pos = cnt[dg[j] * NW + w] + loc[j];
        kout[pos] = kk[j];
        vout[pos] = vv[j];
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// splitter selection, ssss.py:85-146, level-synchronous.
// The reference recursion fill(slot_lo, slot_hi, a, b) runs here one tree
// level at a time: node state (a, b, parent-sample-index) lives in shared
// memory; the "skip samples equal to the pick" loops become lower/upper
// bound searches.  tree[node] equals inorder[mid_slot(node)], so both are
// written from the node's own pick.

__device__ __forceinline__ int lower_bound_u64(const uint64_t* s, int a, int b, uint64_t x) {
    while (a < b) {
        int m = (a + b) >> 1;
        if (s[m] < x) a = m + 1; else b = m;
    }
    return a;
}
__device__ __forceinline__ int upper_bound_u64(const uint64_t* s, int a, int b, uint64_t x) {
    while (a < b) {
        int m = (a + b) >> 1;
        if (s[m] <= x) a = m + 1; else b = m;
    }
    return a;
}
// Equal-run bounds around a pick m (s[m] == x, s sorted), galloping out of
// m: O(log run) probes, one probe when x is not duplicated (a full binary
// search over the node's range was 14 bank-conflicted probes at the top).
__device__ __forceinline__ int run_lo(const uint64_t* s, int a, int m, uint64_t x) {
    int hi = m, k = 1;  // s[hi] >= x
    for (;;) {
        const int p = m - k;
        if (p < a) return lower_bound_u64(s, a, hi, x);
        if (s[p] < x) return lower_bound_u64(s, p + 1, hi, x);
        hi = p;
        k <<= 1;
    }
}
__device__ __forceinline__ int run_hi(const uint64_t* s, int m, int b, uint64_t x) {
    int lo = m + 1, k = 1;  // first index > x lies in [lo, b]
    for (;;) {
        const int p = m + k;
        if (p >= b) return upper_bound_u64(s, lo, b, x);
        if (s[p] > x) return upper_bound_u64(s, lo, p, x);
        lo = p + 1;
        k <<= 1;
    }
}

template <int NT>
__device__ void select_tree(const uint64_t* s, int count, int v, int L, int16_t* sa, int16_t* sb,
                            int16_t* sp, uint64_t* tree, uint64_t* inorder, uint8_t* tpos,
                            uint16_t* eqb) {
    if (threadIdx.x == 0) {
        sa[1] = 0;
        sb[1] = (int16_t)count;
        sp[1] = (int16_t)(count / 2);
    }
    __syncthreads();
    for (int l = 0; l < L; l++) {
        const int first = 1 << l;
        for (int p = threadIdx.x; p < first; p += NT) {
            int node = first + p;
            int a = sa[node], b = sb[node], par = sp[node];
            uint64_t val;
            int la, lb, ra, rb, cp;
            if (a >= b) {  // exhausted by duplicate skipping: reuse the parent pick
                val = s[par];
                la = lb = ra = rb = 0;
                cp = par;
            } else {
                int m = (a + b) >> 1;
                val = s[m];
                la = a;
                lb = run_lo(s, a, m, val);
                ra = run_hi(s, m, b, val);
                rb = b;
                cp = m;
            }
            tree[node] = val;
            int slot = p * (1 << (L - l)) + (1 << (L - l - 1)) - 1;
            inorder[slot] = val;
            if (l + 1 < L) {
                sa[2 * node] = (int16_t)la; sb[2 * node] = (int16_t)lb; sp[2 * node] = (int16_t)cp;
                sa[2 * node + 1] = (int16_t)ra; sb[2 * node + 1] = (int16_t)rb;
                sp[2 * node + 1] = (int16_t)cp;
            }
        }
        __syncthreads();
    }
    // term_pos / eq_final per in-order slot, and the equality bucket each
    // node maps to: 2*eq_leftmost[node_to_inorder[node]] + 1 (ssss.py:137-143).
    // `inorder` may be global memory: it is scanned from a copy in the (now
    // dead) sample's shared memory -- binary searches into it in place were
    // 8 x 13 dependent L2 round trips per thread (0.04 ms of the root step).
    uint64_t* ino = const_cast<uint64_t*>(s);  // count >= v
    for (int i = threadIdx.x; i < v; i += NT) ino[i] = inorder[i];
    __syncthreads();
    // eq_leftmost of every in-order slot = start of its run of equal
    // splitters: a block max-scan of run starts (chunks of consecutive slots
    // per thread), kept in sa; a node's slot is its level-order position
    // mapped through the complete tree's in-order numbering
    {
        const int per = (v + NT - 1) / NT, i0 = threadIdx.x * per, i1 = min(v, i0 + per);
        uint32_t mx = 0;
        for (int i = i0; i < i1; i++) {
            tpos[i] = (uint8_t)term_pos(ino[i]);
            if (i == 0 || ino[i] != ino[i - 1]) mx = i + 1;
        }
        __shared__ uint32_t wsum[32];
        uint32_t run = block_excl_max<NT>(mx, wsum);
        for (int i = i0; i < i1; i++) {
            if (i == 0 || ino[i] != ino[i - 1]) run = i + 1;
            sa[i] = (int16_t)(run - 1);
        }
    }
    __syncthreads();
    for (int node = 1 + threadIdx.x; node <= v; node += NT) {
        const int l = 31 - __clz(node), p = node - (1 << l);
        const int slot = p * (1 << (L - l)) + (1 << (L - l - 1)) - 1;
        eqb[node] = (uint16_t)(2 * sa[slot] + 1);
    }
    if (threadIdx.x == 0) { tree[0] = 0; eqb[0] = 0; }
}

}  // namespace s5g
