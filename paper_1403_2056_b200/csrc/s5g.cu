// s5g.cu -- kernels, host driver and C ABI of the B200 S^5 sorter.
//
// Host driver = the GPU form of s5_sort_items (ssss.py:310-358) /
// _ParallelS5Run.execute (parallel.py:400-445): rounds of batched
// device-wide S^5 steps over "large" segments, then one launch that finishes
// every small segment in a CTA, then the boundary-LCP fix-up.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <omp.h>

#include <algorithm>
#include <atomic>
#include <sys/mman.h>

#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "s5g.h"
#include "s5g_kernels.cuh"
#include "s5g_warpsort.cuh"
#include "s5g_merge.cuh"

namespace s5g {

// ---------------------------------------------------------------------------
// kernels

__device__ __forceinline__ uint64_t exact_key(const uint8_t* arena, int64_t alen, int64_t h,
                                              int64_t d) {
    for (int64_t p = h; p < h + d; p++)
        if (p >= alen || arena[p] == 0) return 0;
    return load_key(arena, alen, h, d);
}

__global__ void k_extract_keys(const uint8_t* __restrict__ arena, int64_t alen,
                               const int64_t* __restrict__ handles, int64_t n, int64_t depth,
                               uint64_t* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = exact_key(arena, alen, handles[i], depth);
}

// Copy handles into the work records and cache each string's first three words.
__global__ void k_init(const uint8_t* __restrict__ arena, int64_t alen,
                       const int64_t* __restrict__ handles, int64_t n, int64_t depth,
                       Rec* __restrict__ recA) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        Rec r;
        r.h = handles[i];
        load_words3(arena, alen, r.h, depth, r.w);
        recA[i] = r;
    }
}

template <int NT, bool BIG>
__global__ void __launch_bounds__(NT) k_sample_tree(
    const StepDev* __restrict__ steps, const uint8_t* __restrict__ arena, int64_t alen,
    const Rec* __restrict__ recX, uint64_t seed, uint64_t* __restrict__ tree_g, uint64_t* __restrict__ inorder_g, uint8_t* __restrict__ tpos_g,
    uint16_t* __restrict__ eqb_g, const int64_t* __restrict__ hroot) {
    extern __shared__ __align__(16) uint8_t smem[];
    const StepDev sd = steps[blockIdx.x];
    const int v = sd.v, count = sd.count;
    int P = 1;
    while (P < count) P <<= 1;
    uint64_t* s = reinterpret_cast<uint64_t*>(smem);
    int16_t* sa = reinterpret_cast<int16_t*>(s + P);
    int16_t* sb = sa + (v + 1);
    int16_t* sp = sb + (v + 1);
    // draw_sample (ssss.py:76-82): uniform positions from a counter-based
    // stream keyed by (seed, lo, hi, depth) -- the tuple the reference seeds
    // default_rng with; the picks never influence the output.
    const uint64_t key0 = splitmix64(seed ^ splitmix64(sd.lo ^ splitmix64(sd.n ^ splitmix64(sd.depth))));
    for (int j = threadIdx.x; j < P; j += NT) {
        uint64_t x = ~0ull;
        if (j < count) {
            const int64_t idx = sample_pos(key0, j, count, sd.n);
            if (hroot) {  // the root step, sampled from the input while k_init runs
                x = load_key(arena, alen, hroot[sd.lo + idx], sd.depth);
            } else {
                const Rec* r = recX + sd.lo + idx;
                x = sd.nvalid ? r->w[0] : load_key(arena, alen, r->h, sd.depth);
            }
        }
        s[j] = x;
    }
    __syncthreads();
    if (BIG && P == 16 * NT)
        sort_sample16<NT>(s);  // top-level samples (16 per thread): registers + shuffles
    else
        bitonic_u64<NT>(s, P);  // smaller samples: shared-memory network
    select_tree<NT>(s, count, v, sd.levels, sa, sb, sp, tree_g + sd.tree_off,
                           inorder_g + sd.tree_off, tpos_g + sd.tree_off, eqb_g + sd.tree_off);
}

// Root sample on a thread-block cluster: the 16384-key root sample is sorted
// by 8 CTAs (2048 keys each, register bitonic), then merged by rank -- each
// key's position = its index in its own run + the number of keys of every
// other run ordered before it (equal keys of lower-ranked CTAs first, so the
// ranks are a permutation).  Every CTA first copies all 8 runs out of
// distributed shared memory with coalesced 16-byte loads (random remote
// loads in the binary searches were DSMEM-request bound: 0.11 ms), searches
// locally, then stores its keys into CTA 0's shared memory at their ranks;
// CTA 0 selects the splitter tree.  One CTA did the whole 16384-key sort in
// 0.19 ms on the critical path of the root step; the cluster draws the same
// sample, so the tree is identical.
constexpr int SCL = 8, SCL_IT = 2, SCL_RUN = SAMPLE_NT * SCL_IT;  // 8 x 2048 keys

__global__ void __cluster_dims__(SCL, 1, 1) __launch_bounds__(SAMPLE_NT) k_sample_root(
    const StepDev* __restrict__ steps, const uint8_t* __restrict__ arena, int64_t alen,
    const int64_t* __restrict__ hroot, uint64_t seed, uint64_t* __restrict__ tree_g,
    uint64_t* __restrict__ inorder_g, uint8_t* __restrict__ tpos_g, uint16_t* __restrict__ eqb_g) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t smem[];
    const StepDev sd = steps[0];
    const int v = sd.v, count = sd.count;
    constexpr int P = SCL * SCL_RUN;
    uint64_t* run = reinterpret_cast<uint64_t*>(smem);  // this CTA's sorted keys
    uint64_t* all = run + SCL_RUN;  // copies of all runs; then (CTA 0) the merged sample
    int16_t* sa = reinterpret_cast<int16_t*>(all + P);
    int16_t* sb = sa + (v + 1);
    int16_t* sp = sb + (v + 1);
    const int r = (int)cluster.block_rank();
    const uint64_t key0 = splitmix64(seed ^ splitmix64(sd.lo ^ splitmix64(sd.n ^ splitmix64(sd.depth))));
    uint64_t c[SCL_IT];
    int64_t hv[SCL_IT];
#pragma unroll
    for (int e = 0; e < SCL_IT; e++) {  // same sample positions as k_sample_tree
        const int j = r * SCL_RUN + threadIdx.x * SCL_IT + e;
        hv[e] = j < count ? hroot[sd.lo + sample_pos(key0, j, count, sd.n)] : -1;
    }
#pragma unroll
    for (int e = 0; e < SCL_IT; e++) c[e] = hv[e] >= 0 ? load_key(arena, alen, hv[e], sd.depth) : ~0ull;
    reg_bitonic_keys<SCL_IT>(c, SCL_RUN, run, true);
#pragma unroll
    for (int e = 0; e < SCL_IT; e++) run[threadIdx.x * SCL_IT + e] = c[e];
    cluster.sync();  // every run sorted and visible cluster-wide
    {
        constexpr int V4 = SCL_RUN / 2;  // uint4 per run
        uint4* dst = reinterpret_cast<uint4*>(all);
#pragma unroll
        for (int q = 0; q < SCL; q++) {
            const uint4* src = reinterpret_cast<const uint4*>(cluster.map_shared_rank(run, q));
            for (int i = threadIdx.x; i < V4; i += SAMPLE_NT) dst[q * V4 + i] = src[i];
        }
    }
    __syncthreads();
    int pos[SCL_IT];
#pragma unroll
    for (int e = 0; e < SCL_IT; e++) {
        const uint64_t x = c[e];
        int lo[SCL];
#pragma unroll
        for (int q = 0; q < SCL; q++) lo[q] = 0;
        // branch-free binary searches, the runs interleaved; runs of lower
        // rank count keys <= x, higher rank keys < x (own run: skipped)
#pragma unroll 1
        for (int half = SCL_RUN / 2; half > 0; half >>= 1) {
#pragma unroll
            for (int q = 0; q < SCL; q++) {
                const uint64_t y = all[q * SCL_RUN + lo[q] + half - 1];
                const bool before = q < r ? y <= x : y < x;
                lo[q] += before ? half : 0;
            }
        }
        int p = threadIdx.x * SCL_IT + e;
#pragma unroll
        for (int q = 0; q < SCL; q++) {
            if (q == r) continue;
            const uint64_t y = all[q * SCL_RUN + lo[q]];
            p += lo[q] + ((lo[q] == SCL_RUN - 1) && (q < r ? y <= x : y < x));
        }
        pos[e] = p;
    }
    cluster.sync();  // all searches done: CTA 0's copy region can take the merge
    uint64_t* s0 = cluster.map_shared_rank(all, 0);
#pragma unroll
    for (int e = 0; e < SCL_IT; e++) s0[pos[e]] = c[e];
    cluster.sync();  // CTA 0 holds the merged sample
    if (r != 0) return;
    select_tree<SAMPLE_NT>(all, count, v, sd.levels, sa, sb, sp, tree_g + sd.tree_off,
                           inorder_g + sd.tree_off, tpos_g + sd.tree_off, eqb_g + sd.tree_off);
}

// Test entry: select_splitters on a given sorted sample.
__global__ void __launch_bounds__(SAMPLE_NT) k_select_only(const uint64_t* sample, int count, int cap,
                                                           int v, int L, uint64_t* tree, uint64_t* inorder,
                                                           uint8_t* tpos, uint16_t* eqb) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* s = reinterpret_cast<uint64_t*>(smem);
    int16_t* sa = reinterpret_cast<int16_t*>(s + cap);
    int16_t* sb = sa + (v + 1);
    int16_t* sp = sb + (v + 1);
    for (int j = threadIdx.x; j < count; j += SAMPLE_NT) s[j] = sample[j];
    __syncthreads();
    select_tree<SAMPLE_NT>(s, count, v, L, sa, sb, sp, tree, inorder, tpos, eqb);
}

// classify_keys (ssss.py:149-181).  Unroll: branch-free descent, tracking
// the last splitter the key went left at (= inorder[leaf], the smallest
// splitter >= key) for the single equality test.  Equal: early exit on a hit.
template <int VARIANT>
__device__ __forceinline__ uint32_t classify_one(uint64_t key, const uint64_t* tree,
                                                 const uint16_t* eqb, int v, int L) {
    int idx = 1;
    if (VARIANT == S5G_VARIANT_UNROLL) {
        uint64_t succ = 0;
        for (int l = 0; l < L; l++) {
            uint64_t t = tree[idx];
            bool r = key > t;
            succ = r ? succ : t;
            idx = 2 * idx + r;
        }
        int leaf = idx - (v + 1);
        return 2 * leaf + ((leaf < v) && key == succ);
    } else {
        for (int l = 0; l < L; l++) {
            uint64_t t = tree[idx];
            if (key == t) return eqb[idx];
            idx = 2 * idx + (key > t);
        }
        return 2 * (idx - (v + 1));
    }
}

template <int VARIANT>
__global__ void __launch_bounds__(CLS_NT) k_classify(
    const StepDev* __restrict__ steps, const int32_t* __restrict__ tile_step,
    const uint8_t* __restrict__ arena, int64_t alen, Rec* __restrict__ recX,
    uint16_t* __restrict__ bid, uint32_t* __restrict__ cnt,
    const uint64_t* __restrict__ tree_g, const uint16_t* __restrict__ eqb_g,
    Counters* __restrict__ ctr, const int64_t* __restrict__ hroot) {
    // hroot != null: the root step builds the work records itself from the
    // input handles (k_init fused in: one pass over the input instead of a
    // record write + re-read)
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ unsigned fetched;
    // tree (level order) | per-tile histogram as packed u16 pairs (a tile has
    // < 65536 strings) | eq-bucket table (equal variant only)
    uint64_t* tree = reinterpret_cast<uint64_t*>(smem);                  // VMAX+1
    uint32_t* hist = reinterpret_cast<uint32_t*>(tree + VMAX + 1);        // (NBMAX+1)/2
    uint16_t* eqb = reinterpret_cast<uint16_t*>(hist + (NBMAX + 1) / 2);  // VMAX+1
    const int t = blockIdx.x;
    const StepDev sd = steps[tile_step[t]];
    const int ti = t - (int)sd.tile0;
    const int64_t beg = sd.lo + (int64_t)ti * sd.tile;
    const int64_t end = min(beg + sd.tile, sd.lo + sd.n);
    const int v = sd.v, L = sd.levels, nb = sd.nb;
    const uint32_t tree_bytes = (uint32_t)(v + 1) * 8u;
    if (threadIdx.x == 0) {
        fetched = 0;
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&bar, tree_bytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(tree_g + sd.tree_off);
        for (uint32_t off = 0; off < tree_bytes; off += 32768u)
            bulk_g2s(reinterpret_cast<uint8_t*>(tree) + off, src + off,
                     min(32768u, tree_bytes - off), &bar);
    }
    for (int b = threadIdx.x; b < (nb + 1) / 2; b += CLS_NT) hist[b] = 0;
    if (VARIANT == S5G_VARIANT_EQUAL)
        for (int i = threadIdx.x; i <= v; i += CLS_NT) eqb[i] = eqb_g[sd.tree_off + i];
    __syncthreads();
    mbar_wait(&bar, 0);
    const int lane = threadIdx.x & 31;
    unsigned my_fetch = 0;
    constexpr int U = 6;  // keys in flight per thread (8: 0.47 ms, 6: 0.45 ms for the C2 root)
    for (int64_t base = beg; base < end; base += (int64_t)CLS_NT * U) {
        uint64_t key[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t i = base + u * CLS_NT + threadIdx.x;
            ok[u] = i < end;
            key[u] = 0;
            if (ok[u]) {
                if (hroot) {
                    Rec r;
                    r.h = hroot[i];
                    load_words3(arena, alen, r.h, sd.depth, r.w);
                    recX[i] = r;
                    key[u] = r.w[0];
                } else if (sd.nvalid) {
                    key[u] = recX[i].w[0];
                } else {  // refill the record's three cached words
                    uint64_t wv[3];
                    load_words3(arena, alen, recX[i].h, sd.depth, wv);
                    recX[i].w[0] = wv[0];
                    recX[i].w[1] = wv[1];
                    recX[i].w[2] = wv[2];
                    key[u] = wv[0];
                    my_fetch += 3;
                }
            }
        }
        uint32_t b[U];
#pragma unroll
        for (int u = 0; u < U; u++) b[u] = classify_one<VARIANT>(key[u], tree, eqb, v, L);
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t i = base + u * CLS_NT + threadIdx.x;
            uint32_t mask = __ballot_sync(0xffffffffu, ok[u]);
            if (ok[u]) {
                S5G_CHECK(b[u] < (uint32_t)nb);
                bid[i] = (uint16_t)b[u];
                uint32_t peers = __match_any_sync(mask, b[u]);
                if (lane == __ffs(peers) - 1)
                    atomicAdd(&hist[b[u] >> 1], (uint32_t)__popc(peers) << (16 * (b[u] & 1)));
            }
        }
    }
    if (my_fetch) atomicAdd(&fetched, my_fetch);
    __syncthreads();
    uint32_t* row = cnt + sd.cnt_off + (int64_t)ti * nb;
    for (int b = threadIdx.x; b < nb; b += CLS_NT) row[b] = (hist[b >> 1] >> (16 * (b & 1))) & 0xffffu;
    if (threadIdx.x == 0 && fetched) atomicAdd(&ctr->fetches, (unsigned long long)fetched);
}

// Test entry: classify given keys against a given tree.
template <int VARIANT>
__global__ void k_classify_only(const uint64_t* __restrict__ keys, int64_t n,
                                const uint64_t* __restrict__ tree_g,
                                const uint16_t* __restrict__ eqb_g, int v, int L,
                                uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* tree = reinterpret_cast<uint64_t*>(smem);
    uint16_t* eqb = reinterpret_cast<uint16_t*>(tree + v + 1);
    for (int i = threadIdx.x; i <= v; i += blockDim.x) {
        tree[i] = tree_g[i];
        eqb[i] = eqb_g ? eqb_g[i] : 0;
    }
    __syncthreads();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint16_t)classify_one<VARIANT>(keys[i], tree, eqb, v, L);
}

// Tile-minor running prefix per bucket column; bucket totals.  One CTA per
// 32 bucket columns: lane = column (coalesced 128 B rows), warp = a chunk of
// tiles; chunk sums are scanned in shared memory, then applied.  A chunk is
// walked in blocks of SCAN_REG tiles whose column loads are issued together
// (one at a time they were a serial chain of round trips: 0.085 ms at C2's
// 592 tiles).
constexpr int SCAN_REG = 16, SCAN_KEEP = 24;

__global__ void __launch_bounds__(1024) k_scan_cols(const StepDev* __restrict__ steps,
                                                    const int32_t* __restrict__ cblk_step,
                                                    uint32_t* __restrict__ cnt,
                                                    uint32_t* __restrict__ tot) {
    __shared__ uint32_t part[32][33];
    const int si = cblk_step[blockIdx.x];
    const StepDev sd = steps[si];
    const int bl = threadIdx.x & 31, c = threadIdx.x >> 5;
    const int b = (blockIdx.x - (int)sd.cblk0) * 32 + bl;
    const int per = (sd.ntiles + 31) / 32;
    const int t0 = c * per, t1 = min(sd.ntiles, t0 + per);
    uint32_t* col = cnt + sd.cnt_off + b;
    uint32_t s = 0;
    // chunks of up to SCAN_KEEP tiles (C2: 592 tiles -> 19) stay in registers
    // between the two passes: one round of loads in all
    const bool keep = per <= SCAN_KEEP;
    uint32_t kv[SCAN_KEEP];
    if (b < sd.nb && keep) {
#pragma unroll
        for (int k = 0; k < SCAN_KEEP; k++) kv[k] = t0 + k < t1 ? col[(int64_t)(t0 + k) * sd.nb] : 0u;
#pragma unroll
        for (int k = 0; k < SCAN_KEEP; k++) s += kv[k];
    } else if (b < sd.nb)
        for (int tb = t0; tb < t1; tb += SCAN_REG) {
            uint32_t v[SCAN_REG];
#pragma unroll
            for (int k = 0; k < SCAN_REG; k++) v[k] = tb + k < t1 ? col[(int64_t)(tb + k) * sd.nb] : 0u;
#pragma unroll
            for (int k = 0; k < SCAN_REG; k++) s += v[k];
        }
    part[c][bl] = s;
    __syncthreads();
    if (c == 0) {
        uint32_t run = 0;
        for (int i = 0; i < 32; i++) {
            uint32_t x = part[i][bl];
            part[i][bl] = run;
            run += x;
        }
        if (b < sd.nb) tot[sd.bk_off + b] = run;
    }
    __syncthreads();
    if (b < sd.nb && keep) {
        uint32_t run = part[c][bl];
#pragma unroll
        for (int k = 0; k < SCAN_KEEP; k++)
            if (t0 + k < t1) {
                col[(int64_t)(t0 + k) * sd.nb] = run;
                run += kv[k];
            }
    } else if (b < sd.nb) {
        uint32_t run = part[c][bl];
        for (int tb = t0; tb < t1; tb += SCAN_REG) {
            uint32_t v[SCAN_REG];
#pragma unroll
            for (int k = 0; k < SCAN_REG; k++) v[k] = tb + k < t1 ? col[(int64_t)(tb + k) * sd.nb] : 0u;
#pragma unroll
            for (int k = 0; k < SCAN_REG; k++)
                if (tb + k < t1) {
                    col[(int64_t)(tb + k) * sd.nb] = run;
                    run += v[k];
                }
        }
    }
}

// Append `item` to a device list at *counter, one atomic per warp and list
// (a top-level step emits ~16K children; per-thread atomics on the same
// counters serialised).  Every lane of the warp must call it.
template <typename T>
__device__ __forceinline__ void warp_append(bool want, const T& item, T* list,
                                            unsigned long long* counter) {
    const uint32_t m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (want) list[base + __popc(m & lanemask_lt())] = item;
}

// Bucket-major exclusive scan (bounds), child segments, boundary records:
// one CTA per 1024 buckets of a step; its offset is the sum of the step's
// earlier bucket totals (read from L2), so the top step's 16K buckets take
// 16 CTAs instead of one CTA's sequential chunks.
__global__ void __launch_bounds__(1024) k_scan_buckets(
    const StepDev* __restrict__ steps, const int32_t* __restrict__ sblk_step,
    const uint32_t* __restrict__ tot,
    uint32_t* __restrict__ bstart, const uint8_t* __restrict__ tpos_g, int dst_in_b,
    int64_t small_max, SegDev* __restrict__ large_out, SegDev* __restrict__ small_out,
    ClassLists cls,
    int64_t* __restrict__ blist, int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    __shared__ uint32_t wsum[32];
    __shared__ unsigned long long cls_el[NCLS];
    const StepDev sd = steps[sblk_step[blockIdx.x]];
    const int nb = sd.nb;
    constexpr int NT = 1024;
    const int nv = sd.nvalid ? sd.nvalid : NCACHE;  // classify refilled
    if (threadIdx.x < NCLS) cls_el[threadIdx.x] = 0;
    const int base = (blockIdx.x - sd.sblk0) * NT;
    uint32_t carry = 0;
    {
        uint32_t part = 0;
        for (int b = threadIdx.x; b < base; b += NT) part += tot[sd.bk_off + b];
        block_excl_sum<NT>(part, wsum, &carry);  // total of the earlier buckets
    }
    {
        const int b = base + threadIdx.x;
        const uint32_t size = b < nb ? tot[sd.bk_off + b] : 0;
        uint32_t total;
        const uint32_t run = carry + block_excl_sum<NT>(size, wsum, &total);
        bool bound = false, child = false;
        SegDev c{};
        int ci = -1;
        if (b < nb) {
            bstart[sd.bk_off + b] = run;
            if (size) {
                bound = lcps && run > 0;  // boundary to the previous non-empty bucket
                if (bound) lcps[sd.lo + run] = sd.depth;  // resolved by k_boundary
                const bool odd = b & 1;
                const int tp = odd ? tpos_g[sd.tree_off + (b >> 1)] : WORD;
                child = !(size == 1 || (odd && tp < WORD));
                if (child) {
                    c.lo = sd.lo + run;
                    c.depth = sd.depth + (odd ? WORD : 0);
                    c.n = (int32_t)size;
                    c.flags = (odd ? nv - 1 : nv) | (dst_in_b ? SEG_IN_B : 0);
                    ci = (int64_t)size <= small_max ? size_class(size) : -1;
                }
            }
        }
        warp_append<int64_t>(bound, sd.lo + run, blist, &ctr->n_bound);
        warp_append<SegDev>(child && ci < 0, c, large_out, &ctr->n_large);
#pragma unroll 1
        for (int k = 0; k < NCLS; k++) {
            warp_append<SegDev>(child && ci == k, c, small_out + cls.off[k], &ctr->n_cls[k]);
            const uint32_t el = __reduce_add_sync(0xffffffffu, (child && ci == k) ? size : 0u);
            if ((threadIdx.x & 31) == 0 && el) atomicAdd(&cls_el[k], (unsigned long long)el);
        }
    }
    __syncthreads();
    if (threadIdx.x < NCLS && cls_el[threadIdx.x])
        atomicAdd(&ctr->cls_elems[threadIdx.x], cls_el[threadIdx.x]);
}

// Stable scatter of (handle, key) into bucket order.  Singleton and
// terminator-covering equality buckets are final: their handles go straight
// to the output and the equality bucket's interior LCPs are written
// (ssss.py:345-357).
//
// Stability without a local sort: the tile is cut into 128-string chunks
// taken by the CTA's warps round-robin, and the chunks update the per-bucket
// running offsets (shared memory) strictly in chunk order -- a turn passed
// from warp to warp on named barriers.  Inside a chunk, __match_any_sync gives every
// string its rank among the earlier same-bucket strings of its 32-string
// round.  Everything else (record loads for the next chunk, the ranks, the
// 32-byte record writes) runs outside the turn, so the chain costs one
// shared read-modify-write per distinct bucket of a round.
#ifndef SCX_IT_CFG
#define SCX_IT_CFG 4
#endif
constexpr int SCX_IT = SCX_IT_CFG;                             // rounds of 32 per chunk
constexpr int SCX_CHUNK = 32 * SCX_IT;                // strings per warp turn
constexpr int SCX_SUB = SCX_CHUNK * (SC_NT / 32);     // 2048 strings per CTA pass
static_assert(SC_NT / 32 == 16, "named-barrier turn chain assumes 16 warps");

// Turn hand-off between consecutive warps on hardware named barriers: warp
// w waits on barrier w (bar.sync, 64 threads) until warp w-1 arrives there
// (bar.arrive, which does not block and orders the arriving warp's shared
// stores before the waiting warp's loads).  Barrier 0 doubles as the 15 -> 0
// hand-off, so no __syncthreads may follow the chained loop.
__device__ __forceinline__ void turn_wait(int w) {
    asm volatile("bar.sync %0, 64;" ::"r"(w) : "memory");
}
__device__ __forceinline__ void turn_pass(int w) {
    asm volatile("bar.arrive %0, 64;" ::"r"((w + 1) & (SC_NT / 32 - 1)) : "memory");
}

// L2 policy of the scatter: the records are read once (streaming loads,
// evict-first) and written to 16 383 slowly advancing bucket frontiers; the
// stores carry an evict_last policy so the partially written 128-byte lines
// of the frontiers outlive the streamed input in the L2 and reach DRAM as
// whole lines more often (C5 root scatter 6.60 -> 6.09 ms, C2 2.31 -> 2.28 ms
// per sort).  A record is ONE 32-byte store: split into two 16-byte stores
// the same policy took 11.4 ms (partial sectors are read-modified-written).
#ifndef SC_HINTS
#define SC_HINTS 2  // 0: plain, 1: streaming loads, 2: + evict_last stores
#endif
__device__ __forceinline__ Rec sc_load_rec(const Rec* p) {
#if SC_HINTS >= 1
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p);
    const ulonglong2 a = __ldcs(q), b = __ldcs(q + 1);
    Rec r;
    r.h = (int64_t)a.x;
    r.w[0] = a.y;
    r.w[1] = b.x;
    r.w[2] = b.y;
    return r;
#else
    return *p;
#endif
}
__device__ __forceinline__ void sc_store_rec(Rec* p, const Rec& r, uint64_t pol) {
#if SC_HINTS >= 2
    asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "l"((uint64_t)r.h), "l"(r.w[0]), "l"(r.w[1]), "l"(r.w[2]), "l"(pol) : "memory");
#else
    *p = r;
#endif
}

__global__ void __launch_bounds__(SC_NT, 2) k_scatter(
    const StepDev* __restrict__ steps, const int32_t* __restrict__ tile_step,
    const Rec* __restrict__ recX, const uint16_t* __restrict__ bid,
    const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ tot,
    const uint32_t* __restrict__ bstart, const uint8_t* __restrict__ tpos_g,
    Rec* __restrict__ recY, int64_t* __restrict__ out_h, int64_t* __restrict__ lcps) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* run_off = reinterpret_cast<uint32_t*>(smem);  // NBMAX+1
    // per-bucket facts for the write phase, so no write waits on a dependent
    // global load: bit 7 = singleton, bits 0-3 = terminator position of an
    // equality bucket's splitter (WORD for range buckets / no terminator)
    uint8_t* bfact = reinterpret_cast<uint8_t*>(run_off + NBMAX + 1);  // NBMAX+1
    const int t = blockIdx.x;
    const StepDev sd = steps[tile_step[t]];
    const int ti = t - (int)sd.tile0;
    const int64_t beg = sd.lo + (int64_t)ti * sd.tile;
    const int64_t end = min(beg + sd.tile, sd.lo + sd.n);
    const int nb = sd.nb;
    const uint32_t* row = cnt + sd.cnt_off + (int64_t)ti * nb;
    const uint8_t* tp = tpos_g + sd.tree_off;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    uint64_t pol = 0;
#if SC_HINTS >= 2
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    for (int b = threadIdx.x; b < nb; b += SC_NT) {
        run_off[b] = bstart[sd.bk_off + b] + row[b];
        const uint32_t tpv = (b & 1) ? tp[b >> 1] : WORD;
        bfact[b] = (uint8_t)(tpv | (tot[sd.bk_off + b] == 1 ? 0x80u : 0u));
    }
    // bucket ids run one chunk ahead: the turn never waits on a load
    uint32_t nbid[SCX_IT];
#pragma unroll
    for (int j = 0; j < SCX_IT; j++) {
        const int64_t e = beg + (int64_t)w * SCX_CHUNK + j * 32 + lane;
        nbid[j] = e < end ? bid[e] : BID_SENTINEL;
    }
    __syncthreads();
    for (int64_t c0 = beg + (int64_t)w * SCX_CHUNK, tn = w; c0 < end;
         c0 += SCX_SUB, tn += SC_NT / 32) {
        Rec rec[SCX_IT];
        uint32_t myb[SCX_IT], peers[SCX_IT];
#pragma unroll
        for (int j = 0; j < SCX_IT; j++) {
            const int64_t e = c0 + j * 32 + lane;
            myb[j] = nbid[j];
            if (e < end) rec[j] = sc_load_rec(recX + e);
            const int64_t en = e + SCX_SUB;
            nbid[j] = en < end ? bid[en] : BID_SENTINEL;
        }
#pragma unroll
        for (int j = 0; j < SCX_IT; j++) peers[j] = __match_any_sync(0xffffffffu, myb[j]);
        // ---- this warp's turn: chunks update the running offsets in order
        if (tn) turn_wait(w);
        uint32_t rel[SCX_IT];
#pragma unroll
        for (int j = 0; j < SCX_IT; j++) {
            const int leader = __ffs(peers[j]) - 1;
            uint32_t base = 0;
            if (lane == leader && myb[j] != BID_SENTINEL) {
                base = run_off[myb[j]];
                run_off[myb[j]] = base + __popc(peers[j]);
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            rel[j] = base + __popc(peers[j] & lt);
            __syncwarp();
        }
        turn_pass(w);
        // ---- writes (whole 32-byte sectors) -------------------------------
#pragma unroll
        for (int j = 0; j < SCX_IT; j++) {
            const uint32_t b = myb[j];
            if (b == BID_SENTINEL) continue;
            S5G_CHECK(rel[j] < (uint32_t)sd.n && b < (uint32_t)nb);
            const int64_t pos = sd.lo + rel[j];
            const uint32_t f = bfact[b];
            const bool odd = b & 1;
            const int tpv = f & 0xf;
            if ((f & 0x80) || tpv < WORD) {
                out_h[pos] = rec[j].h;
                if (lcps && !(f & 0x80) && rel[j] != bstart[sd.bk_off + b]) lcps[pos] = sd.depth + tpv;
            } else if (odd) {
                // equality bucket: continues one word deeper -> shift the cache
                Rec o;
                o.h = rec[j].h;
                o.w[0] = rec[j].w[1];
                o.w[1] = rec[j].w[2];
                o.w[2] = 0;
                sc_store_rec(recY + pos, o, pol);
            } else {
                sc_store_rec(recY + pos, rec[j], pol);
            }
        }
    }
}

// A whole S^5 step of one segment of at most MED_MAX strings in one CTA
// (sample + select_splitters + classify + counts + stable scatter +
// children), so the many small steps of later rounds cost one launch
// instead of five and never round-trip their counts through global memory.
// Bucket ids (<= 63 buckets) are kept in shared memory by the count pass,
// so the scatter's turn chain never waits on a record load.  Same outputs as
// the device-wide step (ssss.py:281-358).
#ifndef STEP_NT_CFG
#define STEP_NT_CFG 256  // 4 CTAs per SM: more independent CTAs fill the step's barrier stalls (C5 37.6 -> 36.4 ms, C2 2.28 -> 2.23; 512: 2 CTAs, 1024: 41.8 ms)
#endif
constexpr int STEP_NT = STEP_NT_CFG;                  // threads of a fused single-CTA step
constexpr int STEP_MINB = 1024 / STEP_NT;             // resident CTAs per SM (32 warps)
#ifndef STEP_SC_IT
#define STEP_SC_IT 2
#endif
#ifndef STEP_STACK
#define STEP_STACK 64  // children a fused step keeps for itself (depth-first)
#endif
struct StepCtaSmem {
    uint64_t s[16 * (MED_VMAX + 1)];       // sorted sample
    uint64_t tree[MED_VMAX + 1], inorder[MED_VMAX + 1];
    uint32_t hist[MED_NB + 1], bst[MED_NB + 1], run_off[MED_NB + 1];
    uint32_t woff[STEP_NT / 32][MED_NB + 1];  // per-warp running offsets of the scatter
    uint8_t bids[MED_MAX];  // bucket of every string (<= 63 buckets), from the count pass
    uint16_t eqb[MED_VMAX + 1];
    int16_t sa[MED_VMAX + 1], sb[MED_VMAX + 1], sp[MED_VMAX + 1];
    uint8_t tpos[MED_VMAX + 1];
    uint32_t wsum[32];
};

template <int VARIANT>
__global__ void __launch_bounds__(STEP_NT, STEP_MINB) k_step_cta(
    const SegDev* __restrict__ segs, Rec* __restrict__ recA, Rec* __restrict__ recB,
    const uint8_t* __restrict__ arena, int64_t alen, uint64_t seed, int64_t vcap,
    int64_t small_max, SegDev* __restrict__ large_out, SegDev* __restrict__ small_out,
    ClassLists cls, int64_t* __restrict__ blist, int64_t* __restrict__ out_h,
    int64_t* __restrict__ lcps, Counters* __restrict__ ctr) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    StepCtaSmem& S = *reinterpret_cast<StepCtaSmem*>(smem_raw);
    SegDev sg = segs[blockIdx.x];
    if (sg.n > MED_MAX) return;  // device-wide path
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned my_fetch = 0;
    __shared__ uint64_t s_red[2][STEP_NT / 32][NCACHE];
    __shared__ int s_flag;
    // Depth-first: children too big for the finishers are pushed on a
    // CTA-local stack and stepped by this CTA right away, while their records
    // (just written by this CTA) are still in the L2 -- instead of a round
    // trip through the next round's launch and HBM.
    __shared__ SegDev s_stk[STEP_STACK];
    __shared__ int s_top;
    if (threadIdx.x == 0) s_top = 0;
    __syncthreads();
    for (;;) {
    const int n = sg.n;
    const int64_t lo = sg.lo;
    int64_t depth = sg.depth;
    const bool in_b = sg.flags & SEG_IN_B;
    Rec* X = (in_b ? recB : recA) + lo;
    Rec* Y = (in_b ? recA : recB) + lo;
    int nvalid = sg.flags & SEG_NV_MASK;
    const MedPlan mp = med_plan(n, vcap);
    const int v = mp.v, L = levels_of(v), nb = 2 * v + 1;
    const int count = mp.count;  // real sample keys; the rest of [0, P) is ~0 padding
    int P = 1;
    while (P < mp.countp) P <<= 1;
    // cached words consumed in place: X[i].w[wo] is the word at `depth`,
    // nvalid words from wo on are valid
    int wo = 0;
    for (;;) {
        // ---- refill the cached words when the segment ran out of them ----
        if (!nvalid) {
            for (int i = threadIdx.x; i < n; i += STEP_NT) {
                uint64_t wv[3];
                load_words3(arena, alen, X[i].h, depth, wv);
                X[i].w[0] = wv[0];
                X[i].w[1] = wv[1];
                X[i].w[2] = wv[2];
                my_fetch += 3;
            }
            nvalid = NCACHE;
            wo = 0;
            __syncthreads();  // the CTA's own record writes are visible after this
        }
        // ---- draw_sample (ssss.py:76-82) ----------------------------------
        const uint64_t key0 = splitmix64(seed ^ splitmix64(lo ^ splitmix64((uint64_t)n ^ splitmix64(depth))));
        uint64_t so = 0, sa = ~0ull;
        for (int j = threadIdx.x; j < P; j += STEP_NT) {
            uint64_t x = ~0ull;
            if (j < count) {
                x = X[splitmix64(key0 + j) % (uint64_t)n].w[wo];
                so |= x;
                sa &= x;
            }
            S.s[j] = x;
        }
        for (int b = threadIdx.x; b <= MED_NB; b += STEP_NT) S.hist[b] = 0;
        // ---- a constant sample: are the leading cached words equal over
        // the whole segment?  Then no step is needed -- the stable scatter
        // would be the identity and the only child the segment itself a word
        // deeper -- so the depth advances in place, up to all cached words
        // at once (duplicate-heavy and shared-prefix segments: C5's 16-
        // character vocabulary words)
        so = warp_or64(so);
        sa = warp_and64(sa);
        if (lane == 0) {
            s_red[0][warp][0] = so;
            s_red[1][warp][0] = sa;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t o = 0, x = ~0ull;
            for (int q = 0; q < STEP_NT / 32; q++) {
                o |= s_red[0][q][0];
                x &= s_red[1][q][0];
            }
            s_flag = o == x && term_pos(o) == WORD;
        }
        __syncthreads();
        if (s_flag) {
            uint64_t wor[NCACHE], wand[NCACHE];
#pragma unroll
            for (int k = 0; k < NCACHE; k++) {
                wor[k] = 0;
                wand[k] = ~0ull;
            }
            for (int i = threadIdx.x; i < n; i += STEP_NT) {
                const Rec r = X[i];
#pragma unroll
                for (int k = 0; k < NCACHE; k++) {
                    wor[k] |= r.w[k];
                    wand[k] &= r.w[k];
                }
            }
#pragma unroll
            for (int k = 0; k < NCACHE; k++) {
                wor[k] = warp_or64(wor[k]);
                wand[k] = warp_and64(wand[k]);
                if (lane == 0) {
                    s_red[0][warp][k] = wor[k];
                    s_red[1][warp][k] = wand[k];
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int k0 = 0;  // leading cached words equal everywhere, no terminator
                for (int k = wo; k < wo + nvalid; k++) {
                    uint64_t o = 0, x = ~0ull;
                    for (int q = 0; q < STEP_NT / 32; q++) {
                        o |= s_red[0][q][k];
                        x &= s_red[1][q][k];
                    }
                    if (o != x || term_pos(o) < WORD) break;
                    k0++;
                }
                s_flag = k0;
            }
            __syncthreads();
            const int k0 = s_flag;
            __syncthreads();
            if (k0 && depth <= alen) {
                depth += (int64_t)WORD * k0;
                wo += k0;
                nvalid -= k0;
                continue;
            }
        }
        // ---- select_splitters (ssss.py:85-146) ------------------------------
        bitonic_u64<STEP_NT>(S.s, P);
        select_tree<STEP_NT>(S.s, mp.countp, v, L, S.sa, S.sb, S.sp, S.tree, S.inorder, S.tpos, S.eqb);
        __syncthreads();
        // ---- classify + bucket counts (ssss.py:149-181, 292) -------------
        constexpr int CU = 4;  // keys in flight per thread
        for (int base = 0; base < n; base += STEP_NT * CU) {
            uint64_t key[CU];
#pragma unroll
            for (int u = 0; u < CU; u++) {
                const int i = base + u * STEP_NT + threadIdx.x;
                key[u] = i < n ? X[i].w[wo] : 0;
            }
#pragma unroll
            for (int u = 0; u < CU; u++) {
                const int i = base + u * STEP_NT + threadIdx.x;
                const bool ok = i < n;
                const uint32_t b = ok ? classify_one<VARIANT>(key[u], S.tree, S.eqb, v, L) : 0;
                const uint32_t mask = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    S.bids[i] = (uint8_t)b;
                    const uint32_t peers = __match_any_sync(mask, b);
                    if (lane == __ffs(peers) - 1) atomicAdd(&S.hist[b], (uint32_t)__popc(peers));
                }
            }
        }
        __syncthreads();
        break;
    }
    // ---- bucket starts, children, boundary records (one warp) -----------
    if (threadIdx.x < 32) {
        constexpr int BPL = (MED_NB + 31) / 32;  // buckets per lane
        uint32_t sz[BPL], run = 0, mine = 0;
#pragma unroll
        for (int k = 0; k < BPL; k++) {
            const int b = lane * BPL + k;
            sz[k] = b < nb ? S.hist[b] : 0;
            mine += sz[k];
        }
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        run = incl - mine;
        const int nv = nvalid ? nvalid : NCACHE;
#pragma unroll
        for (int k = 0; k < BPL; k++) {
            const int b = lane * BPL + k;
            if (b < nb) {
                S.bst[b] = run;
                S.run_off[b] = run;
                const uint32_t size = sz[k];
                if (size) {
                    if (lcps && run > 0) {
                        lcps[lo + run] = depth;  // resolved by k_boundary
                        blist[atomicAdd(&ctr->n_bound, 1ull)] = lo + run;
                    }
                    const bool odd = b & 1;
                    const int tp = odd ? S.tpos[b >> 1] : WORD;
                    if (!(size == 1 || (odd && tp < WORD))) {
                        SegDev c;
                        c.lo = lo + run;
                        c.depth = depth + (odd ? WORD : 0);
                        c.n = (int32_t)size;
                        c.flags = (odd ? nv - 1 : nv) | (in_b ? 0 : SEG_IN_B);
                        if ((int64_t)size <= small_max) {
                            const int ci = size_class(size);
                            small_out[cls.off[ci] + atomicAdd(&ctr->n_cls[ci], 1ull)] = c;
                            atomicAdd(&ctr->cls_elems[ci], (unsigned long long)size);
                        } else {
                            // a child of a fused step fits one (<= MED_MAX):
                            // this CTA steps it next while it is L2-hot
                            const int slot = atomicAdd(&s_top, 1);
                            if (slot < STEP_STACK)
                                s_stk[slot] = c;
                            else
                                large_out[atomicAdd(&ctr->n_large, 1ull)] = c;
                        }
                    }
                }
                run += sz[k];
            }
        }
    }
    __syncthreads();
    // ---- stable scatter without a turn chain: warp w owns the contiguous
    // range [w*per, (w+1)*per) of the segment; per-warp bucket counts (from
    // the ids in shared memory) scanned bucket-major / warp-minor give every
    // warp its own running offsets, so warps never wait on each other
    {
        constexpr int NW = STEP_NT / 32;
        const int w = threadIdx.x >> 5;
        const uint32_t lt = lanemask_lt();
        const int per = (n + NW - 1) / NW;
        const int r0 = min(n, w * per), r1 = min(n, r0 + per);
        for (int b = lane; b < nb; b += 32) S.woff[w][b] = 0;
        __syncwarp();
        for (int e0 = r0; e0 < r1; e0 += 32) {
            const int e = e0 + lane;
            const bool ok = e < r1;
            const uint32_t m = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const uint32_t b = S.bids[e];
                const uint32_t peers = __match_any_sync(m, b);
                if (lane == __ffs(peers) - 1) S.woff[w][b] += __popc(peers);
            }
            __syncwarp();
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += STEP_NT) {
            uint32_t run = S.bst[b];
#pragma unroll
            for (int q = 0; q < NW; q++) {
                const uint32_t t = S.woff[q][b];
                S.woff[q][b] = run;
                run += t;
            }
        }
        __syncthreads();
        constexpr int IT = STEP_SC_IT;  // rounds of 32 whose loads are issued together
        for (int e0 = r0; e0 < r1; e0 += 32 * IT) {
            Rec rec[IT];
            uint32_t myb[IT], rel[IT];
#pragma unroll
            for (int j = 0; j < IT; j++) {
                const int e = e0 + j * 32 + lane;
                myb[j] = BID_SENTINEL;
                if (e < r1) {
                    rec[j] = X[e];
                    myb[j] = S.bids[e];
                }
            }
#pragma unroll
            for (int j = 0; j < IT; j++) {
                const uint32_t peers = __match_any_sync(0xffffffffu, myb[j]);
                const int leader = __ffs(peers) - 1;
                uint32_t base = 0;
                if (lane == leader && myb[j] != BID_SENTINEL) {
                    base = S.woff[w][myb[j]];
                    S.woff[w][myb[j]] = base + __popc(peers);
                }
                base = __shfl_sync(0xffffffffu, base, leader);
                rel[j] = base + __popc(peers & lt);
                __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < IT; j++) {
                const uint32_t b = myb[j];
                if (b == BID_SENTINEL) continue;
                S5G_CHECK(rel[j] < (uint32_t)n && b < (uint32_t)nb);
                const uint32_t size = S.hist[b];
                const bool odd = b & 1;
                const int tpv = odd ? S.tpos[b >> 1] : WORD;
                if (size == 1 || (odd && tpv < WORD)) {
                    out_h[lo + rel[j]] = rec[j].h;
                    if (lcps && size > 1 && rel[j] != S.bst[b]) lcps[lo + rel[j]] = depth + tpv;
                } else {
                    // the child's cached words start one further for an
                    // equality bucket, after the wo words consumed in place
                    const int sh = wo + (odd ? 1 : 0);
                    Rec o;
                    o.h = rec[j].h;
#pragma unroll
                    for (int k = 0; k < NCACHE; k++) {
                        uint64_t x = 0;
#pragma unroll
                        for (int q = 0; q < NCACHE; q++)
                            if (q == k + sh) x = rec[j].w[q];
                        o.w[k] = x;
                    }
                    Y[rel[j]] = o;
                }
            }
        }
    }
    // ---- next segment of this CTA: the most recently pushed child ----------
    __syncthreads();  // the scatter's writes and the children pushes are done
    const int top = min(s_top, STEP_STACK);
    if (top == 0) break;
    sg = s_stk[top - 1];
    __syncthreads();
    if (threadIdx.x == 0) s_top = top - 1;
    __syncthreads();
    }
    my_fetch = __reduce_add_sync(0xffffffffu, my_fetch);
    if (lane == 0 && my_fetch) atomicAdd(&ctr->fetches, (unsigned long long)my_fetch);
}

// LCP at a bucket boundary of a device-wide step at depth d: both strings
// share d characters and their d-words differ (ssss.py:242-263).
__global__ void k_boundary(const int64_t* __restrict__ blist, int64_t nbound,
                           const int64_t* __restrict__ out_h, int64_t* __restrict__ lcps,
                           const uint8_t* __restrict__ arena, int64_t alen) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nbound) return;
    int64_t p = blist[i];
    int64_t d = lcps[p];
    uint64_t a = load_key(arena, alen, out_h[p - 1], d);
    uint64_t b = load_key(arena, alen, out_h[p], d);
    lcps[p] = d + shared_chars(a, b);
}

__global__ void k_dchar(const uint8_t* __restrict__ arena, const int64_t* __restrict__ h,
                        const int64_t* __restrict__ lcps, int64_t n, uint8_t* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        int64_t l = lcps[i];
        out[i] = arena[h[i] + (l < 0 ? 0 : l)];
    }
}

// Multi-GPU partition: destination rank of every string =
// number of splitters (s_j, g_j) ordered before (string, global index),
// comparing full strings against the splitter byte strings, ties by global
// input index.  Splitters live in one device blob (sp_off[j]..sp_off[j+1]).
__device__ __forceinline__ int cmp_string_splitter(const uint8_t* __restrict__ arena, int64_t alen,
                                                   int64_t h, const uint8_t* __restrict__ sp,
                                                   int64_t sp_len) {
    for (int64_t i = 0;; i++) {
        const int c = (h + i) < alen ? arena[h + i] : 0;
        const int d = i < sp_len ? sp[i] : 0;
        if (c != d) return c < d ? -1 : 1;
        if (c == 0) return 0;
    }
}

__global__ void k_partition(const uint8_t* __restrict__ arena, int64_t alen,
                            const int64_t* __restrict__ handles, int64_t n, int64_t base_index,
                            const int64_t* __restrict__ str_gidx,
                            const uint8_t* __restrict__ sp_blob, const int64_t* __restrict__ sp_off,
                            const int64_t* __restrict__ sp_gidx, int nsp,
                            int32_t* __restrict__ out_rank) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t h = handles[i], g = str_gidx ? str_gidx[i] : base_index + i;
    int lo = 0, hi = nsp;  // first splitter greater than (string, g)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        int c = cmp_string_splitter(arena, alen, h, sp_blob + sp_off[mid], sp_off[mid + 1] - sp_off[mid]);
        if (c == 0) c = g < sp_gidx[mid] ? -1 : (g > sp_gidx[mid] ? 1 : 0);
        if (c < 0) hi = mid; else lo = mid + 1;
    }
    out_rank[i] = lo;
}

// String lengths (terminator scan, word at a time).
__global__ void k_lengths(const uint8_t* __restrict__ arena, int64_t alen,
                          const int64_t* __restrict__ handles, int64_t n, int64_t* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t h = handles[i];
    int64_t len = 0;
    for (;;) {
        const uint64_t be = bswap64(load_word_le(arena, alen, h + len));
        const uint64_t z = zero_bytes(be);
        if (z) { len += __clzll(z) >> 3; break; }
        len += WORD;
    }
    out[i] = len;
}

// Pack strings (terminator included) to dst[dst_off[i] ..]: the send buffer
// of the multi-GPU exchange.
// Eight lanes per string (its bytes and terminator, arena[h .. h+L]): the
// source is read as aligned words with funnel shifts (load_word_le), the
// destination written as aligned 8-byte words -- the eight lanes of a string
// write 64 contiguous bytes per round -- with byte stores only at the two
// edges a string shares with its neighbours (one lane per edge byte).  (One
// thread per string walked its ~15 words alone: 1 TB/s on C5's strings; a
// warp per string with byte stores was a chain of dependent round trips.)
constexpr int PACK_G = 8;
#ifndef PACK_S_CFG
#define PACK_S_CFG 2
#endif
#ifndef PLAN_MINB
#define PLAN_MINB 8  // k_plan_sizes: 2 strings, <= 32 registers: 2.66 ms on 2^25 C5 strings (4 strings at 47 registers: 2.71)
#endif
constexpr int PACK_S = PACK_S_CFG;  // strings per lane group: their loads are issued together
#ifndef PACK_SP_CFG
#define PACK_SP_CFG 2
#endif
#ifndef PACK_MINB
#define PACK_MINB 6
#endif
constexpr int PACK_SP = PACK_SP_CFG;  // ... in k_pack: 2 strings and <= 42 registers (6 CTAs per SM) --
// 2.66 ms on 2^25 C5 strings against 3.27 with 4 strings at 64 registers, 2.86 with 1 string at 32
__global__ void __launch_bounds__(256, PACK_MINB) k_pack(const uint8_t* __restrict__ arena, int64_t alen,
                       const int64_t* __restrict__ handles, const int64_t* __restrict__ lens,
                       const int64_t* __restrict__ dst_off, int64_t n, uint8_t* __restrict__ dst) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t grp = t / PACK_G;
    const int sub = (int)(t % PACK_G);
    int64_t h[PACK_SP], o[PACK_SP], e[PACK_SP], a[PACK_SP], z[PACK_SP];
#pragma unroll
    for (int u = 0; u < PACK_SP; u++) {
        const int64_t i = grp * PACK_SP + u;
        h[u] = o[u] = e[u] = 0;  // (an empty copy)
        if (i < n) {
            h[u] = handles[i];
            o[u] = dst_off[i];
            // lens == NULL: sizes from the exclusive offsets (s5g_pack_plan's)
            e[u] = lens ? o[u] + lens[i] + 1 : dst_off[i + 1];  // with the terminator
        }
    }
#pragma unroll
    for (int u = 0; u < PACK_SP; u++) {
        a[u] = min((o[u] + 7) & ~int64_t(7), e[u]);
        z[u] = max(e[u] & ~int64_t(7), a[u]);
    }
    // the word at dst offset q of string u: its bytes, then zeros
    auto word_at = [&](int u, int64_t q) -> uint64_t {
        uint64_t w = load_word_le(arena, alen, h[u] + (q - o[u]));
        const int64_t left = e[u] - 1 - q;  // string bytes left at q (the rest is 0)
        if (left < 8) w &= left > 0 ? (~0ull >> (64 - 8 * left)) : 0ull;
        return w;
    };
    auto byte_at = [&](int u, int64_t q) -> uint8_t {
        const int64_t sp = h[u] + (q - o[u]);
        return q < e[u] - 1 && sp < alen ? arena[sp] : 0;
    };
    // two rounds of 64 bytes per string with all the group's loads in flight
#pragma unroll
    for (int r = 0; r < 2; r++) {
        uint64_t w[PACK_SP];
#pragma unroll
        for (int u = 0; u < PACK_SP; u++) {
            const int64_t q = a[u] + 8 * (sub + PACK_G * r);
            w[u] = q < z[u] ? word_at(u, q) : 0;
        }
#pragma unroll
        for (int u = 0; u < PACK_SP; u++) {
            const int64_t q = a[u] + 8 * (sub + PACK_G * r);
            if (q < z[u]) *reinterpret_cast<uint64_t*>(dst + q) = w[u];
        }
    }
#pragma unroll
    for (int u = 0; u < PACK_SP; u++) {
        for (int64_t q = a[u] + 8 * (sub + PACK_G * 2); q < z[u]; q += 8 * PACK_G)
            *reinterpret_cast<uint64_t*>(dst + q) = word_at(u, q);
        if (o[u] + sub < a[u]) dst[o[u] + sub] = byte_at(u, o[u] + sub);  // < 8 head bytes
        if (z[u] + sub < e[u]) dst[z[u] + sub] = byte_at(u, z[u] + sub);  // < 8 tail bytes
    }
}

// ---------------------------------------------------------------------------
// input side: load_delimited (strset.py:113-134) on the device.  Pass 1 remaps
// the delimiter to 0 (flagging embedded zeros) and counts terminators per
// chunk; a single CTA scans the chunk counts; pass 2 writes the string starts.
constexpr int LD_NT = 256, LD_CHUNK = LD_NT * 64;

// Each thread owns 64 contiguous bytes of a 16 KB chunk, read and written as
// four 16-byte vectors (the byte-at-a-time version ran at ~250 GB/s); the
// zero bytes of a word are found with zero_bytes (exact, no carries).
// data is 16-byte aligned and readable (and writable) for round_up(len, 16)
// bytes: the arena pads past len (S5G_ARENA_PAD).
__device__ __forceinline__ uint64_t ld_zero_mask(uint64_t w, int64_t base, int64_t len) {
    uint64_t z = zero_bytes(w);  // bit 7 of every zero byte
    if (base + 8 > len) {        // bytes past the end do not count
        const int keep = base >= len ? 0 : (int)(len - base);
        z &= keep ? (~0ull >> (64 - 8 * keep)) : 0ull;
    }
    return z;
}

__global__ void k_ld_count(uint8_t* __restrict__ data, int64_t len, int delim,
                           uint32_t* __restrict__ chunk_cnt, int* __restrict__ bad) {
    __shared__ uint32_t wsum[32];
    const int64_t t0 = (int64_t)blockIdx.x * LD_CHUNK + (int64_t)threadIdx.x * 64;
    uint32_t cntv = 0;
    const uint64_t dpat = (uint64_t)(uint8_t)delim * ONES;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t o = t0 + 16 * q;
        if (o >= len) break;
        uint4* p = reinterpret_cast<uint4*>(data + o);
        uint4 v = *p;
        uint64_t w[2] = {(uint64_t)v.x | (uint64_t)v.y << 32, (uint64_t)v.z | (uint64_t)v.w << 32};
        bool changed = false;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int64_t base = o + 8 * h;
            if (delim != 0) {
                if (ld_zero_mask(w[h], base, len)) *bad = 1;  // byte 0 is reserved as terminator
                const uint64_t m = ld_zero_mask(w[h] ^ dpat, base, len);  // delimiter bytes
                if (m) {
                    w[h] &= ~((m >> 7) * 0xffull);  // remap them to 0
                    changed = true;
                }
            }
            cntv += __popcll(ld_zero_mask(w[h], base, len));
        }
        if (changed)
            *p = make_uint4((uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32));
    }
    uint32_t total;
    block_excl_sum<LD_NT>(cntv, wsum, &total);
    if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = total;
}

__global__ void k_ld_scan(uint32_t* __restrict__ chunk_cnt, int64_t nchunks, int64_t* __restrict__ n_out) {
    __shared__ uint32_t wsum[32];
    constexpr int NT = 1024;
    const int64_t per = (nchunks + NT - 1) / NT;
    const int64_t b0 = threadIdx.x * per, b1 = min(b0 + per, nchunks);
    uint64_t s = 0;
    for (int64_t i = b0; i < b1; i++) s += chunk_cnt[i];
    uint32_t total;
    uint32_t run = block_excl_sum<NT>((uint32_t)s, wsum, &total);
    for (int64_t i = b0; i < b1; i++) {
        const uint32_t v = chunk_cnt[i];
        chunk_cnt[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) *n_out = total;
}

// string k starts right after terminator k-1 (string 0 at offset 0)
// rank64 (optional): terminators before each 64-byte block, i.e. the index of
// the first string starting after the block's first byte -- the rank
// directory s5g_rank_positions reads.
__global__ void k_ld_write(const uint8_t* __restrict__ data, int64_t len,
                           const uint32_t* __restrict__ chunk_off, int64_t* __restrict__ handles,
                           uint32_t* __restrict__ rank64) {
    __shared__ uint32_t wsum[32];
    const int64_t t0 = (int64_t)blockIdx.x * LD_CHUNK + (int64_t)threadIdx.x * 64;
    uint64_t z[8];  // zero-byte masks of the thread's 64 bytes, in order
    uint32_t cntv = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t o = t0 + 16 * q;
        z[2 * q] = z[2 * q + 1] = 0;
        if (o < len) {
            const uint4 v = *reinterpret_cast<const uint4*>(data + o);
            z[2 * q] = ld_zero_mask((uint64_t)v.x | (uint64_t)v.y << 32, o, len);
            z[2 * q + 1] = ld_zero_mask((uint64_t)v.z | (uint64_t)v.w << 32, o + 8, len);
        }
        cntv += __popcll(z[2 * q]) + __popcll(z[2 * q + 1]);
    }
    uint32_t k = chunk_off[blockIdx.x] + block_excl_sum<LD_NT>(cntv, wsum, nullptr);
    if (rank64 && t0 < len) rank64[t0 >> 6] = k;
    if (blockIdx.x == 0 && threadIdx.x == 0) handles[0] = 0;
#pragma unroll
    for (int j = 0; j < 8; j++)
        for (uint64_t m = z[j]; m; m &= m - 1) {
            const int64_t i = t0 + 8 * j + (__ffsll((long long)m) - 1) / 8;
            handles[k + 1] = i + 1;  // start of the next string (dropped if past the end)
            k++;
        }
}

// ---- exchange plumbing of the multi-GPU paths --------------------------
// Stable grouping of strings by destination rank (the per-rank counts and
// the order of the all-to-all send buffer): per 2048-string chunk a
// histogram, a destination-major / chunk-minor exclusive scan, then one
// stable 7-bit ranking pass per chunk writes every string's position.
constexpr int GD_SUB = SC_SUB;  // 2048 strings per chunk (SC_NT threads x SC_ITEMS)

__global__ void __launch_bounds__(SC_NT) k_gd_hist(const int32_t* __restrict__ dest, int64_t n,
                                                   int G, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[128];
    const int64_t nch = (n + GD_SUB - 1) / GD_SUB;
    for (int g = threadIdx.x; g < G; g += SC_NT) h[g] = 0;
    __syncthreads();
    const int64_t c0 = (int64_t)blockIdx.x * GD_SUB;
    for (int64_t i = c0 + threadIdx.x; i < min(c0 + GD_SUB, n); i += SC_NT) atomicAdd(&h[dest[i]], 1u);
    __syncthreads();
    for (int g = threadIdx.x; g < G; g += SC_NT) hist[(int64_t)g * nch + blockIdx.x] = h[g];
}

__global__ void __launch_bounds__(1024) k_gd_scan(uint32_t* __restrict__ hist, int64_t len,
                                                  int64_t nch, int G, int64_t n,
                                                  int64_t* __restrict__ counts) {
    __shared__ uint32_t wsum[32];
    constexpr int NT = 1024;
    const int64_t per = (len + NT - 1) / NT;
    const int64_t b0 = threadIdx.x * per, b1 = min(b0 + per, len);
    uint32_t s = 0;
    for (int64_t i = b0; i < b1; i++) s += hist[i];
    uint32_t run = block_excl_sum<NT>(s, wsum, nullptr);
    for (int64_t i = b0; i < b1; i++) {
        const uint32_t v = hist[i];
        hist[i] = run;
        run += v;
    }
    __syncthreads();
    // per-destination totals from the scanned offsets
    for (int g = threadIdx.x; g < G; g += NT) {
        const int64_t lo = (int64_t)g * nch, hi = lo + nch;
        counts[g] = (hi < len ? (int64_t)hist[hi] : n) - (int64_t)hist[lo];
    }
}

__global__ void __launch_bounds__(SC_NT) k_gd_write(const int32_t* __restrict__ dest, int64_t n,
                                                    const uint32_t* __restrict__ off,
                                                    int64_t* __restrict__ order) {
    __shared__ uint32_t wsum[32];
    __shared__ uint16_t rcnt[SC_R * (SC_NT / 32)];
    __shared__ uint16_t kA[GD_SUB], vA[GD_SUB], kB[GD_SUB], vB[GD_SUB];
    const int64_t nch = (n + GD_SUB - 1) / GD_SUB;
    const int64_t c0 = (int64_t)blockIdx.x * GD_SUB;
    const int m = (int)min((int64_t)GD_SUB, n - c0);
    for (int e = threadIdx.x; e < GD_SUB; e += SC_NT) {
        kA[e] = e < m ? (uint16_t)dest[c0 + e] : (uint16_t)BID_SENTINEL;
        vA[e] = (uint16_t)e;
    }
    __syncthreads();
    rank_pass(kA, vA, kB, vB, 0, rcnt, wsum);
    // run starts in the ranked chunk: q - start = rank among equal dests
    const int q0 = threadIdx.x * SC_ITEMS;
    uint32_t st[SC_ITEMS], mx = 0;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; i++) {
        const int q = q0 + i;
        if (q < m && (q == 0 || kB[q - 1] != kB[q])) mx = q + 1;
        st[i] = mx;
    }
    const uint32_t before = block_excl_max<SC_NT>(mx, wsum);
#pragma unroll
    for (int i = 0; i < SC_ITEMS; i++) {
        const int q = q0 + i;
        if (q >= m) break;
        const uint32_t start = (st[i] ? st[i] : before) - 1;
        const int g = kB[q];
        order[off[(int64_t)g * nch + blockIdx.x] + (q - start)] = c0 + vB[q];
    }
}

// Input position of every sorted handle, for unique handles below map_len:
// map[handle] = position, then a gather (no search, no sort).
__global__ void k_pos_scatter(const int64_t* __restrict__ handles, int64_t n,
                              int32_t* __restrict__ map) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) map[handles[i]] = (int32_t)i;
}
__global__ void k_pos_gather(const int64_t* __restrict__ query, int64_t m,
                             const int32_t* __restrict__ map, int64_t* __restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < m) out[j] = map[query[j]];
}

__global__ void k_iota_i32(int32_t* __restrict__ out, int64_t n) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < n) out[j] = (int32_t)j;
}
// in_handles strictly ascending (the string starts of a received arena): the
// input position of a sorted handle is its rank -- a binary search whose top
// levels stay in the L2 -- instead of two radix sorts of (handle, index).
__global__ void k_pos_ascending(const int64_t* __restrict__ h, int64_t n, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i + 1 < n && h[i] >= h[i + 1]) *bad = 1;
}
// Four queries per thread, branch-free (every query walks the same
// ceil(log2(n + 1)) levels): four independent loads in flight per thread --
// with one query per thread the search was a chain of ~25 dependent loads.
constexpr int POS_Q = 4;
__global__ void k_pos_search(const int64_t* __restrict__ in_h, const int64_t* __restrict__ out_h,
                             int64_t n, int64_t top, int64_t* __restrict__ out_pos) {
    const int64_t j0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q[POS_Q], pos[POS_Q];
#pragma unroll
    for (int u = 0; u < POS_Q; u++) {
        const int64_t j = j0 + u * stride;
        q[u] = j < n ? out_h[j] : 0;
        pos[u] = 0;  // elements below q[u] found so far
    }
    for (int64_t step = top; step > 0; step >>= 1) {
#pragma unroll
        for (int u = 0; u < POS_Q; u++) {
            const int64_t p = pos[u] + step;
            if (p <= n && __ldg(in_h + p - 1) < q[u]) pos[u] = p;
        }
    }
#pragma unroll
    for (int u = 0; u < POS_Q; u++) {
        const int64_t j = j0 + u * stride;
        if (j < n) {
            S5G_CHECK(pos[u] < n && in_h[pos[u]] == q[u]);
            out_pos[j] = pos[u];
        }
    }
}
// Index of the string starting at each query handle of an arena loaded by
// s5g_load_delimited_rank: the terminators before the handle's 64-byte block
// (rank64) plus those in the block before the handle -- one directory entry
// and at most eight aligned words per query, all loads independent (the
// binary search over the starts walked ~25 dependent levels).
__global__ void k_rank_positions(const uint8_t* __restrict__ arena, int64_t alen,
                                 const uint32_t* __restrict__ rank64,
                                 const int64_t* __restrict__ query, int64_t m,
                                 int64_t* __restrict__ out_pos) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t h = query[j];
    S5G_CHECK(h >= 0 && h < alen);
    const int64_t b0 = h & ~int64_t(63);
    uint32_t r = rank64[h >> 6];
    const int full = (int)((h - b0) >> 3), rest = (int)(h & 7);
    uint64_t w[8];
#pragma unroll
    for (int q = 0; q < 8; q++)
        w[q] = q <= full ? __ldg(reinterpret_cast<const unsigned long long*>(arena + b0 + 8 * q)) : ~0ull;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        uint64_t z = zero_bytes(w[q]);
        if (q == full) z &= rest ? (~0ull >> (64 - 8 * rest)) : 0ull;  // bytes before h only
        if (q <= full) r += __popcll(z);
    }
    out_pos[j] = r;
}
__global__ void k_pos_match(const int32_t* __restrict__ in_pos, const int32_t* __restrict__ out_idx,
                            int64_t n, int64_t* __restrict__ out_pos) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out_pos[out_idx[k]] = in_pos[k];
}
// exchange plan: handle and size (with terminator) of the k-th string in
// send order.  Eight lanes per string look at eight consecutive aligned words
// per round and vote for the first terminator (one thread per string walked
// its words alone, a chain of dependent loads per string).
__global__ void __launch_bounds__(256, PLAN_MINB) k_plan_sizes(const uint8_t* __restrict__ arena, int64_t alen,
                             const int64_t* __restrict__ handles, const int64_t* __restrict__ order,
                             int64_t n, int64_t* __restrict__ out_h, int64_t* __restrict__ size) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t grp = t / PACK_G;
    const int sub = (int)(t % PACK_G), lane = threadIdx.x & 31, g0 = lane & ~(PACK_G - 1);
    // PACK_S strings per lane group: handles, then the first 128 bytes of
    // each, are fetched with all loads in flight
    int64_t h[PACK_S];
    uint64_t w0[PACK_S], w1[PACK_S];
#pragma unroll
    for (int u = 0; u < PACK_S; u++) {
        const int64_t k = grp * PACK_S + u;
        h[u] = k < n ? handles[order[k]] : -1;
    }
#pragma unroll
    for (int u = 0; u < PACK_S; u++) {
        const int64_t a = (h[u] & ~int64_t(7)) + 8 * sub;  // this lane's aligned word
        w0[u] = h[u] >= 0 ? ld8_guard(arena, alen, a) : 0;  // (0 at or past alen: ends the string)
        w1[u] = h[u] >= 0 ? ld8_guard(arena, alen, a + 8 * PACK_G) : 0;
    }
#pragma unroll
    for (int u = 0; u < PACK_S; u++) {
        const int64_t k = grp * PACK_S + u;
        const bool live = h[u] >= 0;
        int64_t a = (h[u] & ~int64_t(7)) + 8 * sub;
        bool done = !live;
        int64_t e = alen;
        for (int r = 0;; r++) {
            uint64_t z = 0;
            if (!done) {
                uint64_t w = r == 0 ? w0[u] : r == 1 ? w1[u] : ld8_guard(arena, alen, a);
                if (a < h[u]) w |= ~0ull >> (64 - 8 * (h[u] - a));  // bytes before the string
                z = zero_bytes(w);
            }
            const unsigned vote = (__ballot_sync(0xffffffffu, z != 0) >> g0) & ((1u << PACK_G) - 1);
            const int first = vote ? __ffs(vote) - 1 : 0;
            const uint64_t zf = __shfl_sync(0xffffffffu, z, g0 + first);
            if (!done && vote) {
                e = (a - 8 * sub) + 8 * first + ((__ffsll((long long)zf) - 1) >> 3);
                done = true;
            }
            a += 8 * PACK_G;
            if (__all_sync(0xffffffffu, done)) break;
        }
        if (live && sub == 0) {
            out_h[k] = h[u];
            size[k] = min(e, alen) - h[u] + 1;
        }
    }
}
// bytes per destination from the exclusive offsets (off[n] = total)
__global__ void k_plan_dest(const int64_t* __restrict__ off, int64_t n,
                            const int64_t* __restrict__ counts, int32_t G,
                            int64_t* __restrict__ dest_bytes) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t a = 0;
    for (int g = 0; g < G; g++) {
        const int64_t b = a + counts[g];
        dest_bytes[g] = off[b] - off[a];
        a = b;
    }
}

__global__ void k_minmax_i64(const int64_t* __restrict__ x, int64_t n, int64_t* __restrict__ mm) {
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = x[i];
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(reinterpret_cast<long long*>(mm), (long long)lo);
        atomicMax(reinterpret_cast<long long*>(mm) + 1, (long long)hi);
    }
}

__global__ void k_gather_i64(const int64_t* __restrict__ src, const int64_t* __restrict__ idx,
                             int64_t m, int64_t* __restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < m) out[j] = src[idx[j]];
}

// dist_stats (strset.py:290-309) from an exact LCP array: since every LCP is
// at most the length of both its strings, D_i = max(h_i, h_{i+1}) + 1 with
// h_0 = h_n = 0, and L = sum of lcps[1:].
__global__ void k_dist_stats(const int64_t* __restrict__ lcps, int64_t n,
                             unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sD[32], sL[32];
    unsigned long long d = 0, l = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t hi = i > 0 ? lcps[i] : 0, hn = i + 1 < n ? lcps[i + 1] : 0;
        d += (unsigned long long)(max(hi, hn) + 1);
        l += (unsigned long long)hi;
    }
    for (int o = 16; o; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        l += __shfl_xor_sync(0xffffffffu, l, o);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sD[w] = d; sL[w] = l; }
    __syncthreads();
    if (threadIdx.x == 0) {
        d = l = 0;
        for (int v = 0; v < (int)(blockDim.x / 32); v++) { d += sD[v]; l += sL[v]; }
        atomicAdd(&out[0], d);
        atomicAdd(&out[1], l);
    }
}

__global__ void k_single(const int64_t* __restrict__ handles, int64_t* __restrict__ out_h) {
    out_h[0] = handles[0];
}

// ---------------------------------------------------------------------------
// host side

static thread_local std::string g_err;
static std::atomic<size_t> g_l2_fetch{32};  // s5g_set_l2_fetch_granularity
static thread_local int g_sms = 148;        // multiprocessors of the current device
// Threading contract (s5g.h): sorts on one device are serialised by its
// mutex (they share the device's side streams, events and staging buffers);
// sorts on different devices run concurrently.
constexpr int MAX_DEV = 64;
static std::mutex g_dev_mu[MAX_DEV];
static std::mutex g_prof_mu;  // profile table + timeline

// ---- live per-kernel timing (CUDA events on the launching stream) --------
enum KernelId { K_INIT, K_SAMPLE, K_CLASSIFY, K_SCAN_COLS, K_SCAN_BUCKETS, K_SCATTER, K_SEG_WARP,
                K_SEG_WARP2, K_SEG_WARP4, K_SEG_WARP8, K_SEG_CTA2, K_SEG_CTA4, K_SEG_CTA8,
                K_BOUNDARY, K_DCHAR, K_STEP_CTA, K_COUNT };
static const char* kKernelNames[K_COUNT] = {"k_init", "k_sample_tree", "k_classify",
                                            "k_scan_cols", "k_scan_buckets", "k_scatter",
                                            "k_warp_sort<1>", "k_warp_sort<2>",
                                            "k_warp_sort<4>", "k_warp_sort<8>", "k_cta_sort<2>",
                                            "k_cta_sort<4>", "k_cta_sort<8>", "k_boundary",
                                            "k_dchar", "k_step_cta"};
struct ProfEntry {
    long long launches = 0, units = 0, bytes = 0;
    double ms = 0;
};
static bool g_prof = false;
// profile level 2: every kernel of a sort on the caller's stream (no side
// streams), so each launch's event time is its own and the per-kernel sums
// add up to the step -- the live counterpart of ncu's serialized launch list
static bool g_prof_serial = false;
static ProfEntry g_prof_tab[K_COUNT];
// timeline of the last profiled sort: (kernel id, stream, start ms, end ms)
// relative to an event recorded on the launching stream when the sort began
struct TimelineEntry {
    int kid, stream;
    float t0, t1;
};
static std::vector<TimelineEntry> g_timeline;
static cudaEvent_t g_tl_base = nullptr;
static std::atomic<unsigned long long> g_launches{0};

struct Profiler {
    cudaStream_t st;
    int sid;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    std::vector<long long> units, bytes;
    explicit Profiler(cudaStream_t s, int id = 0) : st(s), sid(id) {}
    static std::vector<cudaEvent_t>& pool() {
        static thread_local std::vector<cudaEvent_t> p;
        return p;
    }
    static cudaEvent_t take() {
        auto& p = pool();
        if (p.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = p.back();
        p.pop_back();
        return e;
    }
    int begin() {
        g_launches++;
        if (!g_prof) return -1;
        cudaEvent_t a = take(), b = take();
        cudaEventRecord(a, st);
        ev.push_back({-1, {a, b}});
        units.push_back(0);
        bytes.push_back(0);
        return (int)ev.size() - 1;
    }
    void end(int slot, int kid, long long u, long long by) {
        if (slot < 0) return;
        ev[slot].first = kid;
        units[slot] = u;
        bytes[slot] = by;
        cudaEventRecord(ev[slot].second.second, st);
    }
    void set_bytes(int kid, long long by) {
        for (size_t i = 0; i < ev.size(); i++)
            if (ev[i].first == kid) bytes[i] = by;
    }
    // call after the stream is synchronized
    void flush() {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (size_t i = 0; i < ev.size(); i++) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[i].second.first, ev[i].second.second);
            if (ev[i].first >= 0 && g_tl_base) {
                float t0 = 0, t1 = 0;
                cudaEventElapsedTime(&t0, g_tl_base, ev[i].second.first);
                cudaEventElapsedTime(&t1, g_tl_base, ev[i].second.second);
                g_timeline.push_back({ev[i].first, sid, t0, t1});
            }
            if (ev[i].first >= 0) {
                g_prof_tab[ev[i].first].launches++;
                g_prof_tab[ev[i].first].ms += ms;
                g_prof_tab[ev[i].first].units += units[i];
                g_prof_tab[ev[i].first].bytes += bytes[i];
            }
            pool().push_back(ev[i].second.first);
            pool().push_back(ev[i].second.second);
        }
        ev.clear();
        units.clear();
        bytes.clear();
    }
    ~Profiler() { flush(); }
};
// Algorithmic bytes per launch: what the kernel must read and write at
// minimum, not what it happens to move.
#define SPROF(p, kid, units_, bytes_, launch)      \
    do {                                           \
        int slot_ = (p).begin();                   \
        launch;                                    \
        (p).end(slot_, kid, (units_), (bytes_));   \
    } while (0)
#define PROF(kid, units_, bytes_, launch)          \
    do {                                           \
        int slot_ = prof.begin();                  \
        launch;                                    \
        prof.end(slot_, kid, (units_), (bytes_));  \
    } while (0)

static int g_sms_of() { return g_sms; }

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(S5G_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)


static int64_t small_max_of(int64_t t_medium) {
    // segments of size <= small_max finish in one CTA; the reference
    // switches to its leaves below t_medium (ssss.py:326)
    return std::min<int64_t>(SMALL_MAX, std::max<int64_t>(1, t_medium - 1));
}

#ifndef WIDE_TILE
// strings per classify / scatter CTA of a big full-width step.  The tile x
// bucket count matrix (and its column scan) shrinks with the tile, the
// scatter's time does not depend on it (C5 root: 6.6 / 6.5 / 6.6 / 6.8 ms at
// 65280 / 32768 / 16384 / 8192, column scan 0.30 / 0.72 / 1.50 / 3.02 ms).
// k_classify packs a tile's bucket counts as u16: a tile stays below 65536.
#define WIDE_TILE 65280
#endif
static_assert(WIDE_TILE < 65536, "k_classify's per-tile bucket counts are u16");

struct Workspace {
    Rec *recA, *recB;
    uint16_t* bid;
    uint32_t* cnt;
    uint32_t *tot, *bstart;
    uint64_t *tree, *inorder;
    uint8_t* tpos;
    uint16_t* eqb;
    StepDev* steps;
    StepDev* root_step;
    int32_t* tile_step;
    SegDev* large[2];
    SegDev* small;   // NCLS lists; class c holds cls_cap[c] entries at cls_off[c]
    int64_t* blist;
    Counters* ctr;
    int64_t steps_cap, tiles_cap, cnt_cap, bk_cap, tree_cap;
    int64_t cls_cap[NCLS], cls_off[NCLS];
};

static size_t carve(Workspace* w, uint8_t* base, int64_t n, int64_t t_medium) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> uint8_t* {
        off = (off + 255) & ~size_t(255);
        uint8_t* p = base ? base + off : nullptr;
        off += bytes;
        return p;
    };
    const int64_t nn = std::max<int64_t>(n, 1);
    const int64_t large_min = small_max_of(t_medium) + 1;
    w->steps_cap = nn / large_min + 2;
    // big steps round their tile count up to whole waves: <= 2x the tiles
    // the smallest tile of a step over more than 2 x g_sms tiles (a small root's
    // MIN_TILE tiles are bounded by the 2 * NBMAX term of cnt_cap)
    const int64_t ctile = std::min<int64_t>(TILE, WIDE_TILE);
    w->tiles_cap = 2 * (nn / ctile) + w->steps_cap + 1 + (nn + 2 * w->steps_cap) / 32 +
                   (nn + 2 * w->steps_cap) / 1024 + 2 * w->steps_cap + 2;
    w->cnt_cap = nn * (2 * (int64_t)NBMAX / ctile + 2) + w->steps_cap * 2 +
                 2 * (int64_t)NBMAX;  // a small root's MIN_TILE tiles: <= (n / MIN_TILE + 1) * NBMAX
    w->bk_cap = nn + 2 * w->steps_cap;
    w->tree_cap = nn / 2 + 4 * w->steps_cap + 2;
    {
        // a class-c segment has more than lower[c] strings
        static const int64_t lower[NCLS] = {1, 32, 64, 128, 256, 512, 1024};
        int64_t off = 0;
        for (int c = 0; c < NCLS; c++) {
            w->cls_cap[c] = nn / (lower[c] + 1) + 2;
            w->cls_off[c] = off;
            off += w->cls_cap[c];
        }
    }
    w->recA = (Rec*)take(sizeof(Rec) * nn);
    w->recB = (Rec*)take(sizeof(Rec) * nn);
    w->bid = (uint16_t*)take(2 * nn);
    w->cnt = (uint32_t*)take(4 * w->cnt_cap);
    w->tot = (uint32_t*)take(4 * w->bk_cap);
    w->bstart = (uint32_t*)take(4 * w->bk_cap);
    w->tree = (uint64_t*)take(8 * w->tree_cap);
    w->inorder = (uint64_t*)take(8 * w->tree_cap);
    w->tpos = (uint8_t*)take(w->tree_cap);
    w->eqb = (uint16_t*)take(2 * w->tree_cap);
    w->steps = (StepDev*)take(sizeof(StepDev) * w->steps_cap);
    w->root_step = (StepDev*)take(sizeof(StepDev));
    w->tile_step = (int32_t*)take(4 * w->tiles_cap);
    w->large[0] = (SegDev*)take(sizeof(SegDev) * w->steps_cap);
    w->large[1] = (SegDev*)take(sizeof(SegDev) * w->steps_cap);
    w->small = (SegDev*)take(sizeof(SegDev) * (w->cls_off[NCLS - 1] + w->cls_cap[NCLS - 1]));
    w->blist = (int64_t*)take(8 * nn);
    w->ctr = (Counters*)take(sizeof(Counters));
    return off + 256;
}


// samples of at least this many keys sort with 1024 threads per step
// (C1's root: 2048 keys on 256 threads were 0.05 ms of its 0.37 ms sort)
constexpr int SAMPLE_WIDE_P = 2048;
static size_t smem_sample(int P, int v) { return (size_t)P * 8 + (size_t)3 * (v + 1) * 2 + 16; }
static constexpr size_t SMEM_SAMPLE_ROOT =
    (size_t)SCL_RUN * 8 + (size_t)SCL * SCL_RUN * 8 + (size_t)3 * (VMAX + 1) * 2 + 16;
static constexpr size_t SMEM_CLS_UNROLL = (size_t)(VMAX + 1) * 8 + (size_t)(NBMAX + 1) / 2 * 4;
static constexpr size_t SMEM_CLS = SMEM_CLS_UNROLL + (size_t)(VMAX + 1) * 2;
static constexpr size_t SMEM_SC = (size_t)(NBMAX + 1) * 5;
// A single full-width step over many tiles (the root) scatters with ONE CTA
// per SM (this much shared memory prevents a second): half the tiles in
// flight halve every bucket's write frontier, so more of a bucket's 128-byte
// lines are completed in the L2 before they are written back (C5 root
// scatter 7.3 -> 6.5 ms, C2 0.48 -> 0.41 ms); batched later steps keep two
// CTAs per SM (one is slower there: 1.6 -> 2.4 ms).
#ifndef SC_WIDE_PAD
#define SC_WIDE_PAD 40000
#endif
static constexpr size_t SMEM_SC_WIDE = SMEM_SC + SC_WIDE_PAD;

static int set_smem_attrs() {
    // per device: kernel attributes + the byte-PEXT table of the finishers
    static unsigned long long done_mask = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    if (dev < 64 && (done_mask >> dev & 1ull)) return 0;
    {
        static uint8_t lut[256 * 256];
        for (int m = 0; m < 256; m++)
            for (int x = 0; x < 256; x++) {
                int r = 0, k = 0;
                for (int b = 0; b < 8; b++)
                    if (m >> b & 1) r |= ((x >> b) & 1) << k++;
                lut[m * 256 + x] = (uint8_t)r;
            }
        CK(cudaMemcpyToSymbol(g_pext8, lut, sizeof(lut)));
    }
    CK(cudaFuncSetAttribute(k_sample_root, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)SMEM_SAMPLE_ROOT));
    CK(cudaFuncSetAttribute(k_sample_tree<SAMPLE_NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem_sample(2 * (VMAX + 1), VMAX)));
    CK(cudaFuncSetAttribute(k_sample_tree<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem_sample(2 * (VMAX + 1), VMAX)));
    CK(cudaFuncSetAttribute(k_sample_tree<SAMPLE_NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem_sample(2 * (VMAX + 1), VMAX)));
    CK(cudaFuncSetAttribute(k_select_only, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem_sample(2 * (VMAX + 1), VMAX)));
    CK(cudaFuncSetAttribute(k_classify<S5G_VARIANT_UNROLL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_CLS_UNROLL));
    CK(cudaFuncSetAttribute(k_classify<S5G_VARIANT_EQUAL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_CLS));
    CK(cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_SC_WIDE));
    CK(cudaFuncSetAttribute(k_step_cta<S5G_VARIANT_UNROLL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(StepCtaSmem)));
    CK(cudaFuncSetAttribute(k_step_cta<S5G_VARIANT_EQUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(StepCtaSmem)));
    CK(cudaFuncSetAttribute(k_cta_sort<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(CtaSortSmem<2>)));
    CK(cudaFuncSetAttribute(k_cta_sort<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(CtaSortSmem<4>)));
    CK(cudaFuncSetAttribute(k_cta_sort<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(CtaSortSmem<8>)));

    if (dev < 64) done_mask |= 1ull << dev;
    return 0;
}

static inline unsigned blocks_for(int64_t n, int nt) { return (unsigned)((n + nt - 1) / nt); }

// Random 8-byte gathers from the arena and scattered 8-byte stores: ask the
// L2 for 32-byte (sector) fetches instead of whole lines while we sort, and
// put the caller's setting back afterwards.
struct L2Granularity {
    size_t saved = 0;
    bool ok = false;
    explicit L2Granularity(size_t bytes) {
        ok = cudaDeviceGetLimit(&saved, cudaLimitMaxL2FetchGranularity) == cudaSuccess &&
             cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, bytes) == cudaSuccess;
        cudaGetLastError();
    }
    ~L2Granularity() {
        if (ok) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, saved);
        cudaGetLastError();
    }
};

// Pinned host staging for the per-round descriptor uploads and counter /
// segment-list downloads (async copies, one sync per round).
struct Staging {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            cap = std::max(bytes, cap * 2);
            if (cudaMallocHost(&p, cap) != cudaSuccess) {
                p = nullptr;
                cap = 0;
            }
        }
        return p;
    }
};
static Staging g_stage_up[MAX_DEV], g_stage_down[MAX_DEV];

static int sort_impl_body(const s5g_sort_args* a, int dev_id);

static int sort_impl(const s5g_sort_args* a) {
    // argument errors are reported without touching the device
    if (a->n < 0 || a->arena_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (a->variant != S5G_VARIANT_UNROLL && a->variant != S5G_VARIANT_EQUAL)
        return fail(S5G_E_VARIANT, "unknown classify variant");
    if (a->n > INT32_MAX) return fail(S5G_E_INVALID, "n exceeds 2^31-1");
    if (a->n == 0) return 0;
    int dev_id = 0;
    CK(cudaGetDevice(&dev_id));
    if (dev_id >= MAX_DEV) return fail(S5G_E_INVALID, "device id >= 64");
    std::lock_guard<std::mutex> lk(g_dev_mu[dev_id]);
    L2Granularity l2g(g_l2_fetch);
    return sort_impl_body(a, dev_id);
}

static int sort_impl_body(const s5g_sort_args* a, int dev_id) {
    const int64_t n = a->n;
    cudaStream_t st = (cudaStream_t)a->stream;
    if (n < 0 || a->arena_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (a->variant != S5G_VARIANT_UNROLL && a->variant != S5G_VARIANT_EQUAL)
        return fail(S5G_E_VARIANT, "unknown classify variant");
    if (n > INT32_MAX) return fail(S5G_E_INVALID, "n exceeds 2^31-1");
    if (n == 0) return 0;
    if (!a->arena || !a->handles || !a->out_handles)
        return fail(S5G_E_INVALID, "null buffer");
    if (a->out_dchar && !a->out_lcps) return fail(S5G_E_INVALID, "dchar needs lcps");
    if (int rc = set_smem_attrs()) return rc;
    const int64_t t_medium = a->t_medium > 0 ? a->t_medium : (1 << 20);
    const int64_t vcap = std::max<int64_t>(1, std::min<int64_t>(a->v > 0 ? a->v : VMAX, VMAX));
    int64_t* lcps = a->out_lcps;
    if (a->stats) a->stats->scratch_words += n;
    if (n == 1) {
        g_launches++;
        k_single<<<1, 1, 0, st>>>(a->handles, a->out_handles);
        if (lcps) CK(cudaMemsetAsync(lcps, 0xff, 8, st));
        if (a->out_dchar) {
            g_launches++;
            k_dchar<<<1, 32, 0, st>>>(a->arena, a->out_handles, lcps, 1, a->out_dchar);
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        return 0;
    }
    // side stream (per device, created once): finishers of earlier rounds run
    // there concurrently with the next round's device-wide step
    // and a high-priority stream for the root step's sample, drawn from the
    // input while k_init copies it (its one CTA is scheduled first)
    static cudaStream_t s_st2[MAX_DEV], s_hi[MAX_DEV], s_pool[MAX_DEV][3];
    static cudaEvent_t s_fork[MAX_DEV], s_join[MAX_DEV], s_samp[MAX_DEV], s_pfork[MAX_DEV],
        s_pjoin[MAX_DEV][3];
    if (!s_st2[dev_id]) {  // created under the device's mutex
        int lo_prio = 0, hi_prio = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        CK(cudaStreamCreateWithFlags(&s_st2[dev_id], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&s_hi[dev_id], cudaStreamNonBlocking, hi_prio));
        CK(cudaEventCreateWithFlags(&s_fork[dev_id], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s_join[dev_id], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s_samp[dev_id], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s_pfork[dev_id], cudaEventDisableTiming));
        for (int q = 0; q < 3; q++) {
            CK(cudaStreamCreateWithFlags(&s_pool[dev_id][q], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&s_pjoin[dev_id][q], cudaEventDisableTiming));
        }
    }
    if (g_prof) {
        if (!g_tl_base) CK(cudaEventCreate(&g_tl_base));
        g_timeline.clear();
        CK(cudaEventRecord(g_tl_base, st));
    }
    Profiler prof(st);
    Workspace w;
    size_t need = carve(&w, nullptr, n, t_medium);
    if (!a->workspace || a->workspace_bytes < need)
        return fail(S5G_E_WORKSPACE, "workspace too small: need " + std::to_string(need));
    carve(&w, (uint8_t*)a->workspace, n, t_medium);
    const int64_t small_max = small_max_of(t_medium);
    ClassLists cls_lists;
    for (int c = 0; c < NCLS; c++) cls_lists.off[c] = w.cls_off[c];

    Counters hc{};
    cudaStream_t st2 = s_st2[dev_id], st_hi = s_hi[dev_id];
    cudaEvent_t ev_fork = s_fork[dev_id], ev_join = s_join[dev_id], ev_samp = s_samp[dev_id];
    Profiler prof2(st2, 1), prof_hi(st_hi, 2);
    // finisher size classes run side by side (their launch tails overlap):
    // warp classes on pool 0, k_cta_sort<2> / <4> on pools 1 / 2, <8> on the
    // caller's finisher stream
    Profiler prof_pool[3] = {Profiler(s_pool[dev_id][0], 3), Profiler(s_pool[dev_id][1], 3),
                             Profiler(s_pool[dev_id][2], 3)};
    bool fin_side_used = false;
    const bool serial = g_prof_serial;
    unsigned long long fin_done[NCLS] = {0}, fin_done_el[NCLS] = {0};
    // launch the finishers for list entries [fin_done[c], hc.n_cls[c])
    auto launch_finishers = [&](cudaStream_t fs_main, Profiler& fp_main) -> cudaError_t {
        cudaError_t e0 = cudaEventRecord(s_pfork[dev_id], fs_main);
        if (e0 != cudaSuccess) return e0;
        bool used[3] = {false, false, false};
        // the warp classes share pool 0: the largest first, so the short
        // launches fill the tail instead of delaying it
        static const int order[NCLS] = {3, 2, 1, 0, 4, 5, 6};
        for (int oi = 0; oi < NCLS; oi++) {
            const int c = order[oi];
            const int q = c < 4 ? 0 : c - 3;  // pool stream of this class (3 = main)
            const bool on_pool = q < 3 && !serial;
            cudaStream_t fs = on_pool ? s_pool[dev_id][q] : fs_main;
            Profiler& fp = on_pool ? prof_pool[q] : fp_main;
            const long long cnt_c = (long long)(hc.n_cls[c] - fin_done[c]);
            const long long el_c = (long long)(hc.cls_elems[c] - fin_done_el[c]);
            if ((long long)hc.n_cls[c] > w.cls_cap[c]) return cudaErrorMemoryAllocation;
            if (cnt_c <= 0) continue;
            const int wnt = ws_nt(c == 0 ? 1 : c == 1 ? 2 : c == 2 ? 4 : 8);
            const unsigned grid = blocks_for(cnt_c, wnt / 32);
            const SegDev* lst = w.small + w.cls_off[c] + fin_done[c];
            if (on_pool && !used[q]) {
                used[q] = true;
                cudaError_t ew = cudaStreamWaitEvent(fs, s_pfork[dev_id], 0);
                if (ew != cudaSuccess) return ew;
            }
            switch (c) {
                case 0: SPROF(fp, K_SEG_WARP + 0, el_c, 32LL * el_c, (k_warp_sort<1><<<grid, wnt, 0, fs>>>(
                            lst, cnt_c, w.recA, w.recB, a->arena, a->arena_len, a->out_handles, lcps, w.ctr))); break;
                case 1: SPROF(fp, K_SEG_WARP + 1, el_c, 32LL * el_c, (k_warp_sort<2><<<grid, wnt, 0, fs>>>(
                            lst, cnt_c, w.recA, w.recB, a->arena, a->arena_len, a->out_handles, lcps, w.ctr))); break;
                case 2: SPROF(fp, K_SEG_WARP + 2, el_c, 32LL * el_c, (k_warp_sort<4><<<grid, wnt, 0, fs>>>(
                            lst, cnt_c, w.recA, w.recB, a->arena, a->arena_len, a->out_handles, lcps, w.ctr))); break;
                case 3: SPROF(fp, K_SEG_WARP + 3, el_c, 32LL * el_c, (k_warp_sort<8><<<grid, wnt, 0, fs>>>(
                            lst, cnt_c, w.recA, w.recB, a->arena, a->arena_len, a->out_handles, lcps, w.ctr))); break;
                case 4: SPROF(fp, K_SEG_CTA2, el_c, 32LL * el_c, (k_cta_sort<2><<<(unsigned)cnt_c, 64,
                            sizeof(CtaSortSmem<2>), fs>>>(lst, cnt_c, w.recA, w.recB, a->arena,
                            a->arena_len, a->out_handles, lcps, w.ctr))); break;
                case 5: SPROF(fp, K_SEG_CTA4, el_c, 32LL * el_c, (k_cta_sort<4><<<(unsigned)cnt_c, 128,
                            sizeof(CtaSortSmem<4>), fs>>>(lst, cnt_c, w.recA, w.recB, a->arena,
                            a->arena_len, a->out_handles, lcps, w.ctr))); break;
                default: SPROF(fp, K_SEG_CTA8, el_c, 32LL * el_c, (k_cta_sort<8><<<(unsigned)cnt_c, 256,
                            sizeof(CtaSortSmem<8>), fs>>>(lst, cnt_c, w.recA, w.recB, a->arena,
                            a->arena_len, a->out_handles, lcps, w.ctr))); break;
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            fin_done[c] = hc.n_cls[c];
            fin_done_el[c] = hc.cls_elems[c];
        }
        for (int q = 0; q < 3; q++)
            if (used[q]) {
                cudaError_t ej = cudaEventRecord(s_pjoin[dev_id][q], s_pool[dev_id][q]);
                if (ej == cudaSuccess) ej = cudaStreamWaitEvent(fs_main, s_pjoin[dev_id][q], 0);
                if (ej != cudaSuccess) return ej;
            }
        return cudaSuccess;
    };
    CK(cudaMemsetAsync(w.ctr, 0, sizeof(Counters), st));
    // segments of <= MED_MAX strings take their step in one CTA (k_step_cta);
    // the step hook wants every step's bounds, so it keeps the device-wide path
    const bool fused = !a->step_cb;
    // root step sampled early (device-wide root only): same StepDev fields
    // the round loop plans for it (lo, n, depth, v, count, levels, tree_off 0)
    const bool early_root = n > small_max && !(fused && n <= MED_MAX);
    if (early_root) {
        StepDev d{};
        d.lo = 0;
        d.n = n;
        d.depth = a->depth;
        d.v = (int32_t)gpu_tree_capacity(n, vcap);
        d.count = sample_count(d.v);
        d.levels = levels_of(d.v);
        d.nb = 2 * d.v + 1;
        d.nvalid = NCACHE;
        CK(cudaEventRecord(ev_fork, st));  // the caller's stream order (handles ready)
        CK(cudaStreamWaitEvent(st_hi, ev_fork, 0));
        CK(cudaMemcpyAsync(w.root_step, &d, sizeof(StepDev), cudaMemcpyHostToDevice, st_hi));
        int P = 1;
        while (P < d.count) P <<= 1;
        const long long sb = (long long)d.count * 16 + 27LL * d.v;
        if (P == SCL * SCL_RUN)
            SPROF(prof_hi, K_SAMPLE, 1, sb,
                  (k_sample_root<<<SCL, SAMPLE_NT, SMEM_SAMPLE_ROOT, st_hi>>>(
                      w.root_step, a->arena, a->arena_len, a->handles, a->seed, w.tree,
                      w.inorder, w.tpos, w.eqb)));
        else if (P >= SAMPLE_WIDE_P)  // one CTA: the widest that fits the sample
            SPROF(prof_hi, K_SAMPLE, 1, sb,
                  (k_sample_tree<SAMPLE_NT, false><<<1, SAMPLE_NT, smem_sample(P, d.v), st_hi>>>(
                      w.root_step, a->arena, a->arena_len, w.recA, a->seed, w.tree, w.inorder,
                      w.tpos, w.eqb, a->handles)));
        else
            SPROF(prof_hi, K_SAMPLE, 1, sb,
                  (k_sample_tree<256, false><<<1, 256, smem_sample(P, d.v), st_hi>>>(
                      w.root_step, a->arena, a->arena_len, w.recA, a->seed, w.tree, w.inorder,
                      w.tpos, w.eqb, a->handles)));
        CK(cudaGetLastError());
        CK(cudaEventRecord(ev_samp, st_hi));
    }
    if (!early_root) {  // else the root's k_classify builds the records
        PROF(K_INIT, n, 56LL * n, (k_init<<<blocks_for(n, 256), 256, 0, st>>>(a->arena, a->arena_len,
                                                                     a->handles, n, a->depth,
                                                                     w.recA)));
        CK(cudaGetLastError());
    }
    hc.fetches = 0;
    int64_t n_jobs = 0;
    std::vector<SegDev> large;
    SegDev root{0, a->depth, (int32_t)n, NCACHE};

    if (n <= small_max) {
        const int cls = size_class(n);
        CK(cudaMemcpyAsync(w.small + w.cls_off[cls], &root, sizeof(SegDev),
                           cudaMemcpyHostToDevice, st));
        hc.n_cls[cls] = 1;
        hc.cls_elems[cls] = n;
        CK(cudaMemcpyAsync(&w.ctr->n_cls[cls], &hc.n_cls[cls], 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(&w.ctr->cls_elems[cls], &hc.cls_elems[cls], 8, cudaMemcpyHostToDevice, st));
    } else {
        large.push_back(root);
        // the round's device list is w.large[round & 1] (k_step_cta reads it)
        if (fused && n <= MED_MAX)
            CK(cudaMemcpyAsync(w.large[0], &root, sizeof(SegDev), cudaMemcpyHostToDevice, st));
    }
    int in_b = 0;  // data of this round's segments lives in buffer B
    int round = 0;
    std::vector<StepDev> steps;
    std::vector<int32_t> tile_step, cblk_step, sblk_step;
    std::vector<uint32_t> h_tot, h_bstart;
    std::vector<uint64_t> h_inorder;
    std::vector<int64_t> h_bounds;
    bool side_pending = false;
    auto launch_side = [&]() -> int {
        if (!side_pending) return 0;
        side_pending = false;
        if (serial) {
            CK(launch_finishers(st, prof));
            return 0;
        }
        CK(cudaStreamWaitEvent(st2, ev_fork, 0));
        CK(launch_finishers(st2, prof2));
        fin_side_used = true;
        return 0;
    };
    while (!large.empty()) {
        // ---- medium segments: a whole step per CTA ------------------------
        int64_t n_med = 0, med_elems = 0;
        if (fused)
            for (const auto& sgm : large)
                if (sgm.n <= MED_MAX) {
                    n_med++;
                    med_elems += sgm.n;
                }
        if (n_med) {
            n_jobs += n_med;
            if (a->variant == S5G_VARIANT_UNROLL)
                PROF(K_STEP_CTA, med_elems, 66LL * med_elems,
                     (k_step_cta<S5G_VARIANT_UNROLL><<<(unsigned)large.size(), STEP_NT, sizeof(StepCtaSmem), st>>>(
                         w.large[round & 1], w.recA, w.recB, a->arena, a->arena_len, a->seed, vcap,
                         small_max, w.large[(round + 1) & 1], w.small, cls_lists, w.blist,
                         a->out_handles, lcps, w.ctr)));
            else
                PROF(K_STEP_CTA, med_elems, 66LL * med_elems,
                     (k_step_cta<S5G_VARIANT_EQUAL><<<(unsigned)large.size(), STEP_NT, sizeof(StepCtaSmem), st>>>(
                         w.large[round & 1], w.recA, w.recB, a->arena, a->arena_len, a->seed, vcap,
                         small_max, w.large[(round + 1) & 1], w.small, cls_lists, w.blist,
                         a->out_handles, lcps, w.ctr)));
            CK(cudaGetLastError());
        }
        if (int rc = launch_side()) return rc;
        // ---- plan the round's device-wide steps (host) --------------------
        steps.clear();
        tile_step.clear();
        int64_t cnt_off = 0, bk_off = 0, tree_off = 0, tile0 = 0;
        size_t i0 = 0;
        // a round may be split into batches when it exceeds the capacities
        int batch = 0;
        while (i0 < large.size()) {
            steps.clear();
            tile_step.clear();
            cnt_off = bk_off = tree_off = tile0 = 0;
            size_t i = i0;
            for (; i < large.size(); i++) {
                const SegDev& s = large[i];
                if (fused && s.n <= MED_MAX) continue;  // k_step_cta did it
                StepDev d{};
                d.lo = s.lo;
                d.n = s.n;
                d.depth = s.depth;
                d.v = (int32_t)gpu_tree_capacity(s.n, vcap);
                d.count = sample_count(d.v);
                d.levels = levels_of(d.v);
                d.nb = 2 * d.v + 1;
                d.nvalid = s.flags & SEG_NV_MASK;
                d.ntiles = (int32_t)((s.n + TILE - 1) / TILE);
                if (d.nb >= NBMAX && s.n >= (int64_t)WIDE_TILE * 4 * g_sms)
                    // a full-width (16 383-bucket) step over many strings: tiles
                    // of WIDE_TILE, so a tile holds ~WIDE_TILE / 16 383 strings
                    // per bucket and the ~2 x g_sms tiles in flight keep each
                    // bucket's write frontier (all buckets: ~16 383 x 2 g_sms x
                    // WIDE_TILE / 16 383 records) inside the L2 -- a bucket's
                    // 128-byte lines are completed there instead of leaving as
                    // scattered 32-byte sector writes
                    d.ntiles = (int32_t)((s.n + WIDE_TILE - 1) / WIDE_TILE);
                if (round == 0 && d.ntiles < 2 * g_sms)
                    // a small root (C1: 10^6 strings = 31 tiles) would run on a
                    // fifth of the SMs: spread it over up to two CTAs per SM
                    d.ntiles = (int32_t)std::max<int64_t>(
                        d.ntiles, std::min<int64_t>(2 * g_sms, (s.n + MIN_TILE - 1) / MIN_TILE));
                if (d.ntiles >= g_sms) {
                    // big steps: a whole number of waves of 2 CTAs per SM
                    const int wave = 2 * g_sms;
                    d.ntiles = (d.ntiles + wave - 1) / wave * wave;
                }
                d.tile = (int32_t)((s.n + d.ntiles - 1) / d.ntiles);
                d.ntiles = (int32_t)((s.n + d.tile - 1) / d.tile);
                int64_t need_cnt = (int64_t)d.ntiles * d.nb;
                if ((int64_t)steps.size() + 1 > w.steps_cap ||
                    tile0 + d.ntiles + (bk_off + d.nb) / 32 + (bk_off + d.nb) / 1024 +
                            2 * ((int64_t)steps.size() + 1) > w.tiles_cap ||
                    cnt_off + need_cnt > w.cnt_cap || bk_off + d.nb > w.bk_cap ||
                    tree_off + d.v + 2 > w.tree_cap) {
                    if (steps.empty()) return fail(S5G_E_WORKSPACE, "step exceeds capacity");
                    break;
                }
                d.tile0 = tile0;
                d.cnt_off = cnt_off;
                d.bk_off = bk_off;
                d.tree_off = tree_off;
                for (int t = 0; t < d.ntiles; t++) tile_step.push_back((int32_t)steps.size());
                tile0 += d.ntiles;
                cnt_off += need_cnt;
                bk_off += d.nb;
                tree_off += (d.v + 1 + 1) & ~int64_t(1);
                steps.push_back(d);
            }
            i0 = i;
            const int nsteps = (int)steps.size();
            if (!nsteps) break;
            cblk_step.clear();
            sblk_step.clear();
            for (int si = 0; si < nsteps; si++) {
                steps[si].cblk0 = (int64_t)cblk_step.size();
                for (int b = 0; b < steps[si].nb; b += 32) cblk_step.push_back(si);
                steps[si].sblk0 = (int32_t)sblk_step.size();
                for (int b = 0; b < steps[si].nb; b += 1024) sblk_step.push_back(si);
            }
            n_jobs += nsteps;
            {
                // the first batch of a round follows the round's stream sync;
                // later batches must wait for the previous batch's upload
                // before the staging buffer is rewritten (or reallocated)
                if (batch++) CK(cudaStreamSynchronize(st));
                const size_t b1 = sizeof(StepDev) * nsteps, b2 = 4 * tile_step.size(),
                             b3 = 4 * cblk_step.size(), b4 = 4 * sblk_step.size();
                uint8_t* up = (uint8_t*)g_stage_up[dev_id].get(b1 + b2 + b3 + b4);
                if (!up) return fail(S5G_E_CUDA, "cudaMallocHost failed");
                memcpy(up, steps.data(), b1);
                memcpy(up + b1, tile_step.data(), b2);
                memcpy(up + b1 + b2, cblk_step.data(), b3);
                memcpy(up + b1 + b2 + b3, sblk_step.data(), b4);
                CK(cudaMemcpyAsync(w.steps, up, b1, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(w.tile_step, up + b1, b2 + b3 + b4, cudaMemcpyHostToDevice, st));
            }
            Rec* recX = in_b ? w.recB : w.recA;
            Rec* recY = in_b ? w.recA : w.recB;
            int maxv = 1;
            long long sample_bytes = 0;
            int maxP = 1;
            for (auto& d : steps) {
                maxv = std::max(maxv, d.v);
                while (maxP < d.count) maxP <<= 1;
                sample_bytes += (long long)d.count * (d.nvalid ? 8 : 16) + 27LL * d.v;
            }
            static const bool trace = getenv("S5G_TRACE") != nullptr;
            if (trace) {
                int64_t nmax = 0, tot = 0;
                int nv0 = 0;
                for (auto& d : steps) {
                    nmax = std::max<int64_t>(nmax, d.n);
                    tot += d.n;
                    nv0 += d.nvalid == 0;
                }
                fprintf(stderr, "[s5g] round %d: %d device-wide steps (%lld strings, largest %lld, %d refill), "
                                "maxP %d maxv %d, %lld fused segments (%lld strings)\n",
                        round, nsteps, (long long)tot, (long long)nmax, nv0, maxP, maxv,
                        (long long)n_med, (long long)med_elems);
            }
            if (round == 0 && early_root) {
                CK(cudaStreamWaitEvent(st, ev_samp, 0));  // root tree drawn on st_hi
            } else if (maxP == 16 * SAMPLE_NT)
                PROF(K_SAMPLE, nsteps, sample_bytes,
                     (k_sample_tree<SAMPLE_NT, true><<<nsteps, SAMPLE_NT, smem_sample(maxP, maxv), st>>>(
                         w.steps, a->arena, a->arena_len, recX, a->seed, w.tree, w.inorder, w.tpos,
                         w.eqb, nullptr)));
            else if (maxP >= SAMPLE_WIDE_P)
                PROF(K_SAMPLE, nsteps, sample_bytes,
                     (k_sample_tree<SAMPLE_NT, false><<<nsteps, SAMPLE_NT, smem_sample(maxP, maxv), st>>>(
                         w.steps, a->arena, a->arena_len, recX, a->seed, w.tree, w.inorder, w.tpos,
                         w.eqb, nullptr)));
            else
                PROF(K_SAMPLE, nsteps, sample_bytes,
                     (k_sample_tree<256, false><<<nsteps, 256, smem_sample(maxP, maxv), st>>>(
                         w.steps, a->arena, a->arena_len, recX, a->seed, w.tree, w.inorder, w.tpos,
                         w.eqb, nullptr)));
            CK(cudaGetLastError());
            const unsigned ntiles = (unsigned)tile0;
            const int64_t* root_h = (round == 0 && early_root) ? a->handles : nullptr;
            int64_t round_elems = 0, cls_bytes = 0;
            for (auto& d : steps) {
                round_elems += d.n;
                cls_bytes += (root_h ? 74LL : d.nvalid ? 10LL : 66LL) * d.n;  // root: h, 3 words, record, id
            }
            if (a->variant == S5G_VARIANT_UNROLL)
                PROF(K_CLASSIFY, round_elems, cls_bytes,
                     (k_classify<S5G_VARIANT_UNROLL><<<ntiles, CLS_NT, SMEM_CLS_UNROLL, st>>>(
                         w.steps, w.tile_step, a->arena, a->arena_len, recX, w.bid, w.cnt,
                         w.tree, w.eqb, w.ctr, root_h)));
            else
                PROF(K_CLASSIFY, round_elems, cls_bytes,
                     (k_classify<S5G_VARIANT_EQUAL><<<ntiles, CLS_NT, SMEM_CLS, st>>>(
                         w.steps, w.tile_step, a->arena, a->arena_len, recX, w.bid, w.cnt,
                         w.tree, w.eqb, w.ctr, root_h)));
            CK(cudaGetLastError());
            PROF(K_SCAN_COLS, cnt_off, 8LL * cnt_off + 4LL * bk_off,
                 (k_scan_cols<<<(unsigned)cblk_step.size(), 1024, 0, st>>>(
                     w.steps, w.tile_step + tile0, w.cnt, w.tot)));
            CK(cudaGetLastError());
            PROF(K_SCAN_BUCKETS, bk_off, 8LL * bk_off,
                 (k_scan_buckets<<<(unsigned)sblk_step.size(), 1024, 0, st>>>(
                     w.steps, w.tile_step + tile0 + cblk_step.size(), w.tot, w.bstart, w.tpos, !in_b,
                                                         small_max, w.large[(round + 1) & 1],
                                                         w.small, cls_lists, w.blist, lcps,
                                                         w.ctr)));
            CK(cudaGetLastError());
            PROF(K_SCATTER, round_elems, 66LL * round_elems,
                 (k_scatter<<<ntiles, SC_NT,
                              nsteps == 1 && steps[0].nb >= NBMAX && ntiles >= 4u * g_sms ? SMEM_SC_WIDE : SMEM_SC,
                              st>>>(w.steps, w.tile_step, recX, w.bid,
                                                           w.cnt, w.tot, w.bstart, w.tpos, recY,
                                                           a->out_handles, lcps)));
            CK(cudaGetLastError());
            if (a->step_cb) {
                h_tot.resize(bk_off);
                h_bstart.resize(bk_off);
                h_inorder.resize(tree_off);
                CK(cudaMemcpyAsync(h_tot.data(), w.tot, 4 * bk_off, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(h_bstart.data(), w.bstart, 4 * bk_off, cudaMemcpyDeviceToHost,
                                   st));
                CK(cudaMemcpyAsync(h_inorder.data(), w.inorder, 8 * tree_off,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (auto& d : steps) {
                    h_bounds.resize(d.nb + 1);
                    for (int b = 0; b < d.nb; b++) h_bounds[b] = h_bstart[d.bk_off + b];
                    h_bounds[d.nb] = d.n;
                    a->step_cb(a->step_ctx, d.lo, d.lo + d.n, d.depth, d.v, h_bounds.data(),
                               h_inorder.data() + d.tree_off);
                }
            }
        }
        // ---- next round's large segments ---------------------------------
        {
            // counters + a speculative prefix of the next round's list in one sync
            const int64_t spec = std::min<int64_t>(w.steps_cap, 4096);
            uint8_t* down = (uint8_t*)g_stage_down[dev_id].get(sizeof(Counters) + sizeof(SegDev) * spec);
            if (!down) return fail(S5G_E_CUDA, "cudaMallocHost failed");
            SegDev* dl = reinterpret_cast<SegDev*>(down + sizeof(Counters));
            CK(cudaMemcpyAsync(down, w.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(dl, w.large[(round + 1) & 1], sizeof(SegDev) * spec,
                               cudaMemcpyDeviceToHost, st));
            CK(cudaMemsetAsync(&w.ctr->n_large, 0, 8, st));
            CK(cudaStreamSynchronize(st));
            memcpy(&hc, down, sizeof(Counters));
            large.resize(hc.n_large);
            const int64_t have = std::min<int64_t>((int64_t)hc.n_large, spec);
            if (have) memcpy(large.data(), dl, sizeof(SegDev) * have);
            if ((int64_t)hc.n_large > spec) {
                CK(cudaMemcpyAsync(large.data() + spec, w.large[(round + 1) & 1] + spec,
                                   sizeof(SegDev) * (hc.n_large - spec), cudaMemcpyDeviceToHost,
                                   st));
                CK(cudaStreamSynchronize(st));
            }
        }
        if (hc.n_large) {
            // this round's small segments: finish them on the side stream while
            // the next round runs (disjoint positions; the host already synced).
            // Launched after the next round's first kernel is queued.
            CK(cudaEventRecord(ev_fork, st));
            side_pending = true;
        }
        in_b ^= 1;
        round++;
        if (round > a->arena_len / WORD + 64) return fail(S5G_E_INVALID, "no progress: corrupt input");
    }
    // finishers for whatever the last round produced (earlier rounds' small
    // segments were launched on the side stream while later rounds ran)
    CK(launch_finishers(st, prof));
    if (fin_side_used) {
        CK(cudaEventRecord(ev_join, st2));
        CK(cudaStreamWaitEvent(st, ev_join, 0));
    }
    long long n_small = 0;
    for (int c = 0; c < NCLS; c++) n_small += (long long)hc.n_cls[c];
    if (lcps) {
        if (hc.n_bound)
            PROF(K_BOUNDARY, (long long)hc.n_bound, 56LL * (long long)hc.n_bound,
                 (k_boundary<<<blocks_for(hc.n_bound, 256), 256, 0, st>>>(
                     w.blist, (int64_t)hc.n_bound, a->out_handles, lcps, a->arena,
                     a->arena_len)));
        CK(cudaMemsetAsync(lcps, 0xff, 8, st));
        if (a->out_dchar)
            PROF(K_DCHAR, n, 17LL * n,
                 (k_dchar<<<blocks_for(n, 256), 256, 0, st>>>(a->arena, a->out_handles, lcps, n,
                                                              a->out_dchar)));
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(&hc, w.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // register finishers: record (32 B) in per string, handle + lcp (16 B) out;
    // modelled as 32 B/string in the launches above
    if (a->stats) {
        // the initial cache fill (k_init / the root classify: 3 words per
        // string) + every refill and direct comparison counted on the device
        a->stats->word_fetches += NCACHE * n + (int64_t)hc.fetches + (int64_t)hc.seg_fetches;
        a->stats->jobs_enqueued += n_jobs + n_small;
        a->stats->jobs_executed += n_jobs + n_small;
    }
    return 0;
}

// ---- host-buffer entry (s5g_sort_host) ----------------------------------
// Device buffers come from a library-owned memory pool (never the device's
// default pool, whose attributes belong to the caller / PyTorch): it keeps
// its memory between calls, s5g_release_cached_memory() trims it.  Host
// buffers that are page-locked (cudaHostAlloc / cudaHostRegister) are copied
// directly; pageable ones go through a ring of pinned staging chunks, filled
// and drained by all host threads (OpenMP) while the DMA of the previous
// chunk runs, so a pageable `bytes` buffer moves at close to the PCIe rate.
struct HostCtx {
    static constexpr int NSLOT = 4;
    static constexpr size_t CHUNK = size_t(64) << 20;
    std::mutex mu;
    cudaMemPool_t pool = nullptr;
    cudaStream_t st = nullptr;
    uint8_t* slot[NSLOT] = {};
    cudaEvent_t ev[NSLOT] = {};
    int init(int dev) {
        if (pool) return 0;
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        CK(cudaMemPoolCreate(&pool, &props));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        return 0;
    }
    cudaError_t ring() {
        if (slot[0]) return cudaSuccess;
        for (int k = 0; k < NSLOT; k++) {
            cudaError_t e = cudaHostAlloc((void**)&slot[k], CHUNK, cudaHostAllocPortable);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    static bool pinned(const void* p) {
        cudaPointerAttributes at{};
        const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess;
        cudaGetLastError();
        return ok && at.type == cudaMemoryTypeHost;
    }
    // first-touch every page of a pageable host buffer (all host threads)
    static void prefault(void* p, size_t bytes) {
        if (!p || !bytes || pinned(p)) return;
        {
            // transparent huge pages for the 2 MB-aligned interior (THP in
            // "madvise" mode): 512x fewer faults
            const uintptr_t a = ((uintptr_t)p + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
            const uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)((2u << 20) - 1);
            if (e > a) madvise((void*)a, e - a, MADV_HUGEPAGE);
        }
        volatile uint8_t* b = (volatile uint8_t*)p;
        const int64_t pages = (int64_t)((bytes + 4095) >> 12);
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < pages; q++) b[q << 12] = 0;
    }
    static void par_copy(void* dst, const void* src, size_t bytes) {
        const int64_t parts = (int64_t)std::min<size_t>(64, (bytes + (1 << 20) - 1) >> 20);
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < parts; q++) {
            const size_t lo = bytes * q / parts, hi = bytes * (q + 1) / parts;
            memcpy((uint8_t*)dst + lo, (const uint8_t*)src + lo, hi - lo);
        }
    }
    cudaError_t h2d(void* dst, const void* src, size_t bytes) {
        if (!bytes) return cudaSuccess;
        if (pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        cudaError_t e = ring();
        for (size_t off = 0, c = 0; e == cudaSuccess && off < bytes; off += CHUNK, c++) {
            const int k = (int)(c % NSLOT);
            const size_t len = std::min(CHUNK, bytes - off);
            // the slot's previous DMA (this call's or an earlier copy's) must
            // be done before the host overwrites it (a never-recorded event
            // counts as complete)
            e = cudaEventSynchronize(ev[k]);
            if (e != cudaSuccess) break;
            par_copy(slot[k], (const uint8_t*)src + off, len);
            e = cudaMemcpyAsync((uint8_t*)dst + off, slot[k], len, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaEventRecord(ev[k], st);
        }
        return e;
    }
    cudaError_t d2h(void* dst, const void* src, size_t bytes) {
        if (!bytes) return cudaSuccess;
        if (pinned(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
        cudaError_t e = ring();
        const size_t nc = (bytes + CHUNK - 1) / CHUNK;
        // DMA chunk c into slot c % NSLOT; drain chunk c - NSLOT + 1 meanwhile
        for (size_t c = 0; e == cudaSuccess && c < nc + NSLOT - 1; c++) {
            if (c < nc) {
                const int k = (int)(c % NSLOT);
                const size_t off = c * CHUNK, len = std::min(CHUNK, bytes - off);
                e = cudaMemcpyAsync(slot[k], (const uint8_t*)src + off, len, cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaEventRecord(ev[k], st);
            }
            if (e == cudaSuccess && c + 1 >= NSLOT) {
                const size_t d = c + 1 - NSLOT;
                const int k = (int)(d % NSLOT);
                const size_t off = d * CHUNK, len = std::min(CHUNK, bytes - off);
                e = cudaEventSynchronize(ev[k]);
                if (e == cudaSuccess) par_copy((uint8_t*)dst + off, slot[k], len);
            }
        }
        return e;
    }
};
static HostCtx g_host[MAX_DEV];


}  // namespace s5g

// ---------------------------------------------------------------------------
// C ABI

using namespace s5g;

extern "C" {

int s5g_version(void) { return S5G_VERSION; }

void s5g_profile_enable(int on) {
    g_prof = on != 0;
    g_prof_serial = on == 2;
}

void s5g_profile_reset(void) {
    for (auto& e : g_prof_tab) e = ProfEntry();
}

int s5g_profile_read(s5g_kernel_profile* out, int max_entries) {
    int k = 0;
    for (int i = 0; i < K_COUNT && k < max_entries; i++, k++) {
        std::snprintf(out[k].name, sizeof(out[k].name), "%s", kKernelNames[i]);
        out[k].launches = g_prof_tab[i].launches;
        out[k].units = g_prof_tab[i].units;
        out[k].ms = g_prof_tab[i].ms;
        out[k].bytes = g_prof_tab[i].bytes;
    }
    return k;
}

int s5g_profile_timeline(int* kid, int* stream, float* t0, float* t1, int max_entries) {
    int k = 0;
    for (const auto& e : g_timeline) {
        if (k >= max_entries) break;
        kid[k] = e.kid;
        stream[k] = e.stream;
        t0[k] = e.t0;
        t1[k] = e.t1;
        k++;
    }
    return (int)g_timeline.size();
}

unsigned long long s5g_launch_count(void) { return g_launches; }

void s5g_set_l2_fetch_granularity(int bytes) { g_l2_fetch = bytes > 0 ? (size_t)bytes : 32; }

int s5g_finisher_counters(unsigned long long* out, int n, int reset) {
    unsigned long long h[12];
    CK(cudaMemcpyFromSymbol(h, g_fin_ctr, sizeof(h)));
    for (int i = 0; i < n && i < 12; i++) out[i] = h[i];
    if (reset) {
        std::memset(h, 0, sizeof(h));
        CK(cudaMemcpyToSymbol(g_fin_ctr, h, sizeof(h)));
    }
    return 0;
}

const char* s5g_last_error(void) { return g_err.c_str(); }

size_t s5g_workspace_bytes(int64_t n, int64_t t_medium) {
    Workspace w;
    return carve(&w, nullptr, n, t_medium > 0 ? t_medium : (1 << 20));
}

int s5g_sort(const s5g_sort_args* args) {
    if (!args) return fail(S5G_E_INVALID, "null args");
    return sort_impl(args);
}

int s5g_sort_host(const uint8_t* arena, int64_t arena_len, const int64_t* handles, int64_t n,
                  int64_t depth, int64_t* out_handles, int64_t* out_lcps, uint8_t* out_dchar,
                  int32_t variant, int32_t v, uint64_t seed, int64_t t_medium, s5g_stats* stats) {
    if (n < 0 || arena_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (variant != S5G_VARIANT_UNROLL && variant != S5G_VARIANT_EQUAL)
        return fail(S5G_E_VARIANT, "unknown classify variant");
    if (n == 0) return 0;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev >= MAX_DEV) return fail(S5G_E_INVALID, "device id >= 64");
    HostCtx& hx = g_host[dev];
    // one host-buffer sort per device at a time: the staging ring is shared
    // (the sort itself takes the device mutex inside)
    std::lock_guard<std::mutex> lk(hx.mu);
    if (int rc = hx.init(dev)) return rc;
    cudaStream_t st = hx.st;
    const int64_t tm = t_medium > 0 ? t_medium : (1 << 20);
    size_t ws = s5g_workspace_bytes(n, tm);
    size_t alen_pad = ((size_t)arena_len + S5G_ARENA_PAD + 15) & ~size_t(15);
    uint8_t *d_arena = nullptr, *d_ws = nullptr, *d_dchar = nullptr;
    int64_t *d_h = nullptr, *d_out = nullptr, *d_lcp = nullptr;
    int rc = 0;
    auto cleanup = [&]() {
        cudaFreeAsync(d_arena, st); cudaFreeAsync(d_ws, st); cudaFreeAsync(d_h, st);
        cudaFreeAsync(d_out, st); cudaFreeAsync(d_lcp, st); cudaFreeAsync(d_dchar, st);
        cudaStreamSynchronize(st);
    };
#define CKH(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            rc = fail(S5G_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
            cleanup();                                                                   \
            return rc;                                                                   \
        }                                                                                \
    } while (0)
    CKH(cudaMallocFromPoolAsync((void**)&d_arena, alen_pad, hx.pool, st));
    CKH(cudaMallocFromPoolAsync((void**)&d_ws, ws, hx.pool, st));
    CKH(cudaMallocFromPoolAsync((void**)&d_h, 8 * n, hx.pool, st));
    CKH(cudaMallocFromPoolAsync((void**)&d_out, 8 * n, hx.pool, st));
    if (out_lcps || out_dchar) CKH(cudaMallocFromPoolAsync((void**)&d_lcp, 8 * n, hx.pool, st));
    if (out_dchar) CKH(cudaMallocFromPoolAsync((void**)&d_dchar, n, hx.pool, st));
    CKH(cudaMemsetAsync(d_arena + arena_len, 0, alen_pad - arena_len, st));
    // S5G_HOST_TIMING=1: phase times of this call on stderr (tuning aid)
    static const bool timing = getenv("S5G_HOST_TIMING") != nullptr;
    auto now = []() { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    auto t0 = now();
    CKH(hx.h2d(d_h, handles, 8 * n));
    CKH(hx.h2d(d_arena, arena, arena_len));
    auto t1 = now();
    // handles must lie in the arena (the reference's "handle outside the
    // buffer" / "not zero-terminated" checks, strset.py:64-78, done here on
    // the device: one pass over the uploaded handles instead of two numpy
    // passes over the host array)
    int64_t* d_mm = nullptr;
    CKH(cudaMallocFromPoolAsync((void**)&d_mm, 16, hx.pool, st));
    {
        const int64_t init[2] = {INT64_MAX, INT64_MIN};
        CKH(cudaMemcpyAsync(d_mm, init, 16, cudaMemcpyHostToDevice, st));
        g_launches++;
        k_minmax_i64<<<std::min<int64_t>(2 * g_sms_of(), blocks_for(n, 256)), 256, 0, st>>>(d_h, n, d_mm);
        CKH(cudaGetLastError());
    }
    // fresh pageable output arrays fault in page by page on first write
    // (~0.6 s for C5's 4.3 GB on one thread, after the sort): fault them in
    // now, as huge pages where the kernel allows, on all host threads, while
    // the input DMA runs (page-locking them in place instead was slower:
    // cudaHostRegister / Unregister of 4.3 GB cost ~0.6 s)
    HostCtx::prefault(out_handles, 8 * (size_t)n);
    HostCtx::prefault(out_lcps, 8 * (size_t)n);
    HostCtx::prefault(out_dchar, (size_t)n);
    int64_t mm[2];
    CKH(cudaMemcpyAsync(mm, d_mm, 16, cudaMemcpyDeviceToHost, st));
    CKH(cudaFreeAsync(d_mm, st));
    CKH(cudaStreamSynchronize(st));  // the input is on the device; mm is valid
    if (mm[0] < 0 || mm[1] >= arena_len) {
        cleanup();
        return fail(S5G_E_INVALID, "handle outside the buffer");
    }
    s5g_sort_args a{};
    a.arena = d_arena; a.arena_len = arena_len; a.handles = d_h; a.n = n; a.depth = depth;
    a.out_handles = d_out; a.out_lcps = d_lcp; a.out_dchar = d_dchar;
    a.workspace = d_ws; a.workspace_bytes = ws; a.stream = st;
    a.variant = variant; a.v = v; a.seed = seed; a.t_medium = tm; a.stats = stats;
    auto t2 = now();
    rc = sort_impl(&a);
    if (rc) { std::string keep = g_err; cleanup(); g_err = keep; return rc; }
    auto t3 = now();
    CKH(hx.d2h(out_handles, d_out, 8 * n));
    if (out_lcps) CKH(hx.d2h(out_lcps, d_lcp, 8 * n));
    if (out_dchar) CKH(hx.d2h(out_dchar, d_dchar, n));
    CKH(cudaStreamSynchronize(st));
    auto t4 = now();
    if (timing)
        fprintf(stderr, "s5g_sort_host: issue H2D %.1f ms, prefault + H2D wait %.1f ms, sort %.1f ms, "
                        "D2H %.1f ms (input %s)\n", ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4),
                HostCtx::pinned(arena) ? "pinned" : "pageable");
    cleanup();
#undef CKH
    return 0;
}

void s5g_release_cached_memory(void) {
    for (int d = 0; d < MAX_DEV; d++) {
        std::lock_guard<std::mutex> lk(g_host[d].mu);
        if (g_host[d].pool) cudaMemPoolTrimTo(g_host[d].pool, 0);
    }
}

// ---- one host process, G devices (parallel_s5's p, parallel.py:468-492) ----
// The reference forks p workers over one shared set; here p devices each
// take one part of a sample-sort partition: G-1 string splitters (sampled
// prefixes, ties broken by input position) cut the input into G ranges of
// the output order; every device receives the whole arena, classifies all
// strings against the splitters (s5g_partition, redundantly -- it costs a
// few string compares per string), keeps its own range in input order
// (s5g_group_by_dest is stable) and sorts it; the parts land at their output
// offsets, and the host fixes the LCP at every part boundary -- the
// _boundary_lcps of parallel.py:447-455.
static int64_t host_lcp(const uint8_t* a, int64_t alen, int64_t x, int64_t y) {
    int64_t l = 0;
    while (x + l < alen && y + l < alen && a[x + l] == a[y + l] && a[x + l] != 0) l++;
    return l;
}

static int multi_part(int dev, int k, int G, const s5g_multi_args* m, const std::vector<uint8_t>& sp,
                      const std::vector<int64_t>& sp_off, const std::vector<int64_t>& sp_g,
                      std::vector<int64_t>& counts_out, s5g_stats* st_out) {
    CK(cudaSetDevice(dev));
    HostCtx& hx = g_host[dev];
    std::lock_guard<std::mutex> lk(hx.mu);
    if (int rc = hx.init(dev)) return rc;
    cudaStream_t st = hx.st;
    const int64_t n = m->n, alen = m->arena_len;
    const size_t alen_pad = ((size_t)alen + S5G_ARENA_PAD + 15) & ~size_t(15);
    std::vector<void*> bufs;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 16), hx.pool, st) != cudaSuccess) return nullptr;
        bufs.push_back(p);
        return p;
    };
    struct Free {
        std::vector<void*>& b;
        cudaStream_t s;
        ~Free() {
            for (void* p : b) cudaFreeAsync(p, s);
            cudaStreamSynchronize(s);
        }
    } fr{bufs, st};
    const int nsp = G - 1;
    uint8_t* d_arena = (uint8_t*)alloc(alen_pad);
    int64_t* d_all = (int64_t*)alloc(8 * n);
    int32_t* d_dest = (int32_t*)alloc(4 * n);
    int64_t* d_order = (int64_t*)alloc(8 * n);
    int64_t* d_cnt = (int64_t*)alloc(8 * G);
    const size_t gws = s5g_group_workspace_bytes(n, G);
    void* d_gws = alloc(gws);
    uint8_t* d_sp = (uint8_t*)alloc(sp.size());
    int64_t* d_spo = (int64_t*)alloc(8 * sp_off.size());
    int64_t* d_spg = (int64_t*)alloc(8 * std::max<size_t>(1, sp_g.size()));
    if (!d_arena || !d_all || !d_dest || !d_order || !d_cnt || !d_gws || !d_sp || !d_spo || !d_spg)
        return fail(S5G_E_CUDA, "device allocation failed");
    CK(cudaMemsetAsync(d_arena + alen, 0, alen_pad - alen, st));
    CK(hx.h2d(d_arena, m->arena, alen));
    CK(hx.h2d(d_all, m->handles, 8 * n));
    if (!sp.empty()) CK(cudaMemcpyAsync(d_sp, sp.data(), sp.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_spo, sp_off.data(), 8 * sp_off.size(), cudaMemcpyHostToDevice, st));
    if (!sp_g.empty()) CK(cudaMemcpyAsync(d_spg, sp_g.data(), 8 * sp_g.size(), cudaMemcpyHostToDevice, st));
    if (int rc = s5g_partition(d_arena, alen, d_all, n, 0, nullptr, d_sp, d_spo, d_spg, nsp, d_dest, st))
        return rc;
    if (int rc = s5g_group_by_dest(d_dest, n, G, d_order, d_cnt, d_gws, gws, st)) return rc;
    std::vector<int64_t> cnt(G);
    CK(cudaMemcpyAsync(cnt.data(), d_cnt, 8 * G, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t off = 0;
    for (int q = 0; q < k; q++) off += cnt[q];
    const int64_t mk = cnt[k];
    counts_out = cnt;
    if (mk == 0) return 0;
    int64_t* d_part = (int64_t*)alloc(8 * mk);
    int64_t* d_oh = (int64_t*)alloc(8 * mk);
    int64_t* d_ol = m->out_lcps || m->out_dchar ? (int64_t*)alloc(8 * mk) : nullptr;
    const int64_t tm = m->t_medium > 0 ? m->t_medium : (1 << 20);
    const size_t ws = s5g_workspace_bytes(mk, tm);
    void* d_ws = alloc(ws);
    if (!d_part || !d_oh || !d_ws || ((m->out_lcps || m->out_dchar) && !d_ol))
        return fail(S5G_E_CUDA, "device allocation failed");
    g_launches++;
    k_gather_i64<<<blocks_for(mk, 256), 256, 0, st>>>(d_all, d_order + off, mk, d_part);
    CK(cudaGetLastError());
    s5g_sort_args a{};
    a.arena = d_arena; a.arena_len = alen; a.handles = d_part; a.n = mk; a.depth = m->depth;
    a.out_handles = d_oh; a.out_lcps = d_ol; a.out_dchar = nullptr;
    a.workspace = d_ws; a.workspace_bytes = ws; a.stream = st;
    a.variant = m->variant; a.v = m->v; a.seed = m->seed; a.t_medium = tm; a.stats = st_out;
    if (int rc = sort_impl(&a)) return rc;
    CK(hx.d2h(m->out_handles + off, d_oh, 8 * mk));
    if (m->out_lcps) CK(hx.d2h(m->out_lcps + off, d_ol, 8 * mk));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_sort_multi(const s5g_multi_args* m) {
    if (!m) return fail(S5G_E_INVALID, "null args");
    if (m->n < 0 || m->arena_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (m->variant != S5G_VARIANT_UNROLL && m->variant != S5G_VARIANT_EQUAL)
        return fail(S5G_E_VARIANT, "unknown classify variant");
    if (m->num_devices < 1 || !m->device_ids) return fail(S5G_E_INVALID, "num_devices must be >= 1");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int k = 0; k < m->num_devices; k++)
        if (m->device_ids[k] < 0 || m->device_ids[k] >= ndev || m->device_ids[k] >= MAX_DEV)
            return fail(S5G_E_INVALID, "device id " + std::to_string(m->device_ids[k]) +
                                           " is not one of the " + std::to_string(ndev) +
                                           " visible CUDA devices");
    const int64_t n = m->n;
    if (n == 0) return 0;
    const int G = m->num_devices;
    if (G == 1) {
        int prev = 0;
        CK(cudaGetDevice(&prev));
        CK(cudaSetDevice(m->device_ids[0]));
        const int rc = s5g_sort_host(m->arena, m->arena_len, m->handles, n, m->depth, m->out_handles,
                                     m->out_lcps, m->out_dchar, m->variant, m->v, m->seed,
                                     m->t_medium, m->stats);
        cudaSetDevice(prev);
        return rc;
    }
    // G-1 splitters: sampled string prefixes (<= SPLIT_MAX bytes) with their
    // input positions, sorted, equally spaced (dist.pick_splitters)
    constexpr int SPLIT_MAX = 64;
    const int64_t S = std::min<int64_t>(n, 1024LL * G);
    const uint8_t* A = m->arena;
    std::vector<std::pair<std::string, int64_t>> smp(S);
    for (int64_t j = 0; j < S; j++) {
        const int64_t pos = S == n ? j : (int64_t)(splitmix64(m->seed ^ splitmix64((uint64_t)j + 0x51ull)) % (uint64_t)n);
        const int64_t h = m->handles[pos];
        if (h < 0 || h >= m->arena_len) return fail(S5G_E_INVALID, "handle outside the buffer");
        int64_t L = 0;
        while (L < SPLIT_MAX && h + L < m->arena_len && A[h + L]) L++;
        smp[j] = {std::string((const char*)A + h, (size_t)L), pos};
    }
    std::sort(smp.begin(), smp.end(), [](const auto& x, const auto& y) {
        const int c = std::memcmp(x.first.data(), y.first.data(), std::min(x.first.size(), y.first.size()));
        if (c) return c < 0;
        if (x.first.size() != y.first.size()) return x.first.size() < y.first.size();
        return x.second < y.second;
    });
    std::vector<uint8_t> sp;
    std::vector<int64_t> sp_off{0}, sp_g;
    for (int k = 1; k < G; k++) {
        const auto& pk = smp[(size_t)(k * S / G)];
        sp.insert(sp.end(), pk.first.begin(), pk.first.end());
        sp_off.push_back((int64_t)sp.size());
        sp_g.push_back(pk.second);
    }
    std::vector<int> rcs(G, 0);
    std::vector<std::string> errs(G);
    std::vector<std::vector<int64_t>> counts(G);
    std::vector<s5g_stats> sts(G);
    std::vector<std::thread> th;
    for (int k = 0; k < G; k++) {
        sts[k] = s5g_stats{};
        th.emplace_back([&, k]() {
            rcs[k] = multi_part(m->device_ids[k], k, G, m, sp, sp_off, sp_g, counts[k], &sts[k]);
            if (rcs[k]) errs[k] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (int k = 0; k < G; k++)
        if (rcs[k]) return fail(rcs[k], "device " + std::to_string(m->device_ids[k]) + ": " + errs[k]);
    // boundary LCPs between consecutive non-empty parts; lcps[0] = -1
    const std::vector<int64_t>& cnt = counts[0];
    if (m->out_lcps) {
        int64_t off = 0, prev_last = -1;
        for (int k = 0; k < G; k++) {
            if (cnt[k]) {
                if (prev_last >= 0)
                    m->out_lcps[off] = host_lcp(A, m->arena_len, m->out_handles[prev_last], m->out_handles[off]);
                prev_last = off + cnt[k] - 1;
            }
            off += cnt[k];
        }
        m->out_lcps[0] = -1;
        if (m->out_dchar) {
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; i++) {
                const int64_t l = m->out_lcps[i];
                m->out_dchar[i] = A[m->out_handles[i] + (l < 0 ? 0 : l)];
            }
        }
    }
    if (m->stats)
        for (int k = 0; k < G; k++) {
            m->stats->char_cmps += sts[k].char_cmps;
            m->stats->word_fetches += sts[k].word_fetches;
            m->stats->scratch_words += sts[k].scratch_words;
            m->stats->jobs_enqueued += sts[k].jobs_enqueued;
            m->stats->jobs_executed += sts[k].jobs_executed;
        }
    return 0;
}

int s5g_extract_keys(const uint8_t* arena, int64_t arena_len, const int64_t* handles, int64_t n,
                     int64_t depth, uint64_t* out_keys, void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_extract_keys<<<blocks_for(n, 256), 256, 0, st>>>(arena, arena_len, handles, n, depth,
                                                       out_keys);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_select_splitters(const uint64_t* sample, int64_t count, int64_t v, uint64_t* tree,
                         uint64_t* inorder, uint8_t* term_pos, uint16_t* eq_bucket, void* stream) {
    if (v < 1 || v > VMAX || ((v + 1) & v) != 0 || count < 1 || count > 2 * (VMAX + 1))
        return fail(S5G_E_INVALID, "v must be 2^d-1 <= 8191 and 1 <= count <= 16384");
    if (int rc = set_smem_attrs()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t cap = std::max(count, v);  // select_tree reuses the sample region (>= v words)
    size_t smem = (size_t)cap * 8 + (size_t)3 * (v + 1) * 2 + 16;
    g_launches++;
    k_select_only<<<1, SAMPLE_NT, smem, st>>>(sample, (int)count, (int)cap, (int)v, levels_of(v), tree,
                                              inorder, term_pos, eq_bucket);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_classify(const uint64_t* keys, int64_t n, const uint64_t* tree, const uint16_t* eq_bucket,
                 int64_t v, int32_t variant, uint16_t* out_bucket, void* stream) {
    if (variant != S5G_VARIANT_UNROLL && variant != S5G_VARIANT_EQUAL)
        return fail(S5G_E_VARIANT, "unknown classify variant");
    if (v < 1 || v > VMAX || ((v + 1) & v) != 0) return fail(S5G_E_INVALID, "bad v");
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    size_t smem = (size_t)(v + 1) * 10;
    if (smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(k_classify_only<S5G_VARIANT_UNROLL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_classify_only<S5G_VARIANT_EQUAL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    g_launches++;
    if (variant == S5G_VARIANT_UNROLL)
        k_classify_only<S5G_VARIANT_UNROLL><<<blocks_for(n, 256), 256, smem, st>>>(
            keys, n, tree, eq_bucket, (int)v, levels_of(v), out_bucket);
    else
        k_classify_only<S5G_VARIANT_EQUAL><<<blocks_for(n, 256), 256, smem, st>>>(
            keys, n, tree, eq_bucket, (int)v, levels_of(v), out_bucket);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_partition(const uint8_t* arena, int64_t arena_len, const int64_t* handles, int64_t n,
                  int64_t base_index, const int64_t* string_gidx, const uint8_t* splitters,
                  const int64_t* splitter_off, const int64_t* splitter_gidx, int32_t nsplitters,
                  int32_t* out_rank, void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    if (nsplitters < 0) return fail(S5G_E_INVALID, "negative splitter count");
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_partition<<<blocks_for(n, 256), 256, 0, st>>>(arena, arena_len, handles, n, base_index,
                                                    string_gidx, splitters, splitter_off, splitter_gidx,
                                                    nsplitters, out_rank);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_lengths(const uint8_t* arena, int64_t arena_len, const int64_t* handles, int64_t n,
                int64_t* out_len, void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_lengths<<<blocks_for(n, 256), 256, 0, st>>>(arena, arena_len, handles, n, out_len);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_pack(const uint8_t* arena, int64_t arena_len, const int64_t* handles,
             const int64_t* lengths, const int64_t* dst_off, int64_t n, uint8_t* dst,
             void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_pack<<<blocks_for((n + PACK_SP - 1) / PACK_SP * PACK_G, 256), 256, 0, st>>>(arena, arena_len, handles, lengths, dst_off, n,
                                                dst);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_load_delimited(uint8_t* data, int64_t len, int32_t delimiter, int64_t* out_handles,
                       int64_t* out_n, void* workspace, size_t workspace_bytes, void* stream) {
    return s5g_load_delimited_n(data, len, delimiter, out_handles, len + 1, out_n, workspace,
                                workspace_bytes, stream);
}

int s5g_load_delimited_n(uint8_t* data, int64_t len, int32_t delimiter, int64_t* out_handles,
                         int64_t capacity, int64_t* out_n, void* workspace,
                         size_t workspace_bytes, void* stream) {
    return s5g_load_delimited_rank(data, len, delimiter, out_handles, capacity, out_n, nullptr,
                                   workspace, workspace_bytes, stream);
}

int s5g_load_delimited_rank(uint8_t* data, int64_t len, int32_t delimiter, int64_t* out_handles,
                            int64_t capacity, int64_t* out_n, uint32_t* out_rank64,
                            void* workspace, size_t workspace_bytes, void* stream) {
    if (len < 0 || delimiter < 0 || delimiter > 255) return fail(S5G_E_INVALID, "delimiter must be a byte value");
    if (capacity < 0) return fail(S5G_E_INVALID, "negative capacity");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nchunks = (len + LD_CHUNK - 1) / LD_CHUNK;
    if (workspace_bytes < (size_t)nchunks * 4 + 16) return fail(S5G_E_WORKSPACE, "workspace too small");
    int* bad = (int*)workspace;
    int64_t* d_n = (int64_t*)((uint8_t*)workspace + 8);
    uint32_t* chunk = (uint32_t*)((uint8_t*)workspace + 16);
    CK(cudaMemsetAsync(workspace, 0, 16, st));
    if (len == 0) {
        *out_n = 0;
        return 0;
    }
    g_launches += 3;
    k_ld_count<<<(unsigned)nchunks, LD_NT, 0, st>>>(data, len, delimiter, chunk, bad);
    k_ld_scan<<<1, 1024, 0, st>>>(chunk, nchunks, d_n);
    CK(cudaGetLastError());
    int hbad = 0;
    int64_t hn = 0;
    CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hn, d_n, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // the count, before any start is written
    if (hbad) return fail(S5G_E_INVALID, "input contains byte 0, which is reserved as terminator");
    // (k_ld_write stores a start after every terminator: count + 1 entries)
    if (hn + 1 > capacity) return fail(S5G_E_INVALID, "more strings than out_handles has room for");
    k_ld_write<<<(unsigned)nchunks, LD_NT, 0, st>>>(data, len, chunk, out_handles, out_rank64);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    *out_n = hn;
    return 0;
}

size_t s5g_group_workspace_bytes(int64_t n, int32_t G) {
    const int64_t nch = (std::max<int64_t>(n, 1) + GD_SUB - 1) / GD_SUB;
    return (size_t)(4 * nch * std::max(G, 1)) + 64;
}

int s5g_group_by_dest(const int32_t* dest, int64_t n, int32_t G, int64_t* out_order,
                      int64_t* out_counts, void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0 || G < 1 || G > 127) return fail(S5G_E_INVALID, "need n >= 0 and 1 <= G <= 127");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        CK(cudaMemsetAsync(out_counts, 0, 8 * (size_t)G, st));
        CK(cudaStreamSynchronize(st));
        return 0;
    }
    if (workspace_bytes < s5g_group_workspace_bytes(n, G)) return fail(S5G_E_WORKSPACE, "workspace too small");
    const int64_t nch = (n + GD_SUB - 1) / GD_SUB;
    uint32_t* hist = (uint32_t*)workspace;
    g_launches += 3;
    k_gd_hist<<<(unsigned)nch, SC_NT, 0, st>>>(dest, n, G, hist);
    k_gd_scan<<<1, 1024, 0, st>>>(hist, nch * G, nch, G, n, out_counts);
    k_gd_write<<<(unsigned)nch, SC_NT, 0, st>>>(dest, n, hist, out_order);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_positions(const int64_t* handles, int64_t n, const int64_t* query, int64_t m,
                  int32_t* map, int64_t map_len, int64_t* out_pos, void* stream) {
    if (n < 0 || m < 0 || map_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (n > INT32_MAX) return fail(S5G_E_INVALID, "n exceeds 2^31-1");
    cudaStream_t st = (cudaStream_t)stream;
    g_launches += 2;
    if (n) k_pos_scatter<<<blocks_for(n, 256), 256, 0, st>>>(handles, n, map);
    if (m) k_pos_gather<<<blocks_for(m, 256), 256, 0, st>>>(query, m, map, out_pos);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

static int bits_for(int64_t x) {
    int b = 1;
    while (b < 63 && (x >> b)) b++;
    return b;
}

size_t s5g_input_positions_workspace_bytes(int64_t n) {
    const int64_t nn = std::max<int64_t>(n, 1);
    size_t t1 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (const int64_t*)nullptr, (int64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::min<int64_t>(nn, INT32_MAX));
    return 2 * 8 * (size_t)nn + 3 * 4 * (size_t)nn + t1 + 4 * 256;
}

int s5g_input_positions(const int64_t* in_handles, const int64_t* out_handles, int64_t n,
                        int64_t max_handle, int64_t* out_pos, void* workspace,
                        size_t workspace_bytes, void* stream) {
    if (n < 0) return fail(S5G_E_INVALID, "negative n");
    if (n > INT32_MAX) return fail(S5G_E_INVALID, "n exceeds 2^31-1");
    if (n == 0) return 0;
    if (workspace_bytes < s5g_input_positions_workspace_bytes(n))
        return fail(S5G_E_WORKSPACE, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t* w = (uint8_t*)workspace;
    auto take = [&](size_t b) { uint8_t* p = w; w += (b + 255) & ~size_t(255); return p; };
    int64_t* k_in = (int64_t*)take(8 * n);
    int64_t* k_out = (int64_t*)take(8 * n);
    int32_t* iota = (int32_t*)take(4 * n);
    int32_t* v_in = (int32_t*)take(4 * n);
    int32_t* v_out = (int32_t*)take(4 * n);
    {
        // strictly ascending input handles (a received arena's string starts):
        // rank by binary search
        int* bad = (int*)iota;
        int hbad = 0;
        CK(cudaMemsetAsync(bad, 0, 4, st));
        g_launches++;
        k_pos_ascending<<<blocks_for(n, 256), 256, 0, st>>>(in_handles, n, bad);
        CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!hbad) {
            g_launches++;
            int64_t top = 1;
            while (top * 2 <= n) top *= 2;
            k_pos_search<<<blocks_for((n + POS_Q - 1) / POS_Q, 256), 256, 0, st>>>(in_handles, out_handles, n,
                                                                                 top, out_pos);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
            return 0;
        }
    }
    size_t tb = 0;
    const int end_bit = bits_for(std::max<int64_t>(max_handle, 1));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, in_handles, k_in, iota, v_in, (int)n, 0, end_bit, st));
    void* tmp = take(tb);
    g_launches += 6;
    k_iota_i32<<<blocks_for(n, 256), 256, 0, st>>>(iota, n);
    // stable sorts by handle: the k-th occurrence of a handle in input order
    // and the k-th in output order are the same string (equal handles are
    // equal strings, kept in input order by the stable sort)
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, in_handles, k_in, iota, v_in, (int)n, 0, end_bit, st));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, out_handles, k_out, iota, v_out, (int)n, 0, end_bit, st));
    k_pos_match<<<blocks_for(n, 256), 256, 0, st>>>(v_in, v_out, n, out_pos);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_rank_positions(const uint8_t* arena, int64_t arena_len, const uint32_t* rank64,
                       const int64_t* query, int64_t m, int64_t* out_pos, void* stream) {
    if (m < 0 || arena_len < 0) return fail(S5G_E_INVALID, "negative size");
    if (m == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_rank_positions<<<blocks_for(m, 256), 256, 0, st>>>(arena, arena_len, rank64, query, m, out_pos);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_gather_i64(const int64_t* src, const int64_t* idx, int64_t n, int64_t* out, void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_gather_i64<<<blocks_for(n, 256), 256, 0, st>>>(src, idx, n, out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

size_t s5g_pack_plan_workspace_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr,
                                  std::max<int64_t>(n, 1) + 1);
    return 8 * (size_t)(std::max<int64_t>(n, 1) + 1) + t + 256;
}

int s5g_pack_plan(const uint8_t* arena, int64_t arena_len, const int64_t* handles,
                  const int64_t* order, int64_t n, const int64_t* counts, int32_t G,
                  int64_t* out_handles, int64_t* out_off, int64_t* out_dest_bytes,
                  void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0 || G < 1) return fail(S5G_E_INVALID, "bad size");
    if (workspace_bytes < s5g_pack_plan_workspace_bytes(n)) return fail(S5G_E_WORKSPACE, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* size = (int64_t*)workspace;
    void* tmp = (uint8_t*)workspace + ((8 * (size_t)(std::max<int64_t>(n, 1) + 1) + 255) & ~size_t(255));
    size_t tb = workspace_bytes - ((8 * (size_t)(std::max<int64_t>(n, 1) + 1) + 255) & ~size_t(255));
    g_launches += 3;
    CK(cudaMemsetAsync(size + n, 0, 8, st));
    if (n) k_plan_sizes<<<blocks_for((n + PACK_S - 1) / PACK_S * PACK_G, 256), 256, 0, st>>>(arena, arena_len, handles, order, n, out_handles, size);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, size, out_off, n + 1, st));
    k_plan_dest<<<1, 32, 0, st>>>(out_off, n, counts, G, out_dest_bytes);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

int s5g_dist_stats(const int64_t* lcps, int64_t n, int64_t* out_D, int64_t* out_L, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        *out_D = *out_L = 0;
        return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    }
    unsigned long long* d_out = nullptr;
    CK(cudaMallocAsync((void**)&d_out, 16, st));
    CK(cudaMemsetAsync(d_out, 0, 16, st));
    g_launches++;
    k_dist_stats<<<(unsigned)std::min<int64_t>(blocks_for(n, 256), 4 * 148), 256, 0, st>>>(lcps, n, d_out);
    CK(cudaGetLastError());
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, d_out, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d_out, st));
    CK(cudaStreamSynchronize(st));
    *out_D = (int64_t)h[0];
    *out_L = (int64_t)h[1];
    return 0;
}

static int64_t merge_ncand_cap(int64_t n, int32_t k) { return n / MERGE_M + k + 1; }

size_t s5g_merge_workspace_bytes(int64_t n, int32_t k) {
    const int64_t nc = merge_ncand_cap(std::max<int64_t>(n, 0), std::max(k, 1));
    const int64_t nch = n / MC_CHUNK + 2;
    return (size_t)(nc * (int64_t)std::max(k, 1) * 8 + nc * 8 + std::max<int64_t>(n, 1) * 4 +
                    nc * 4 + nch * 4) + 64 + 5 * 256;
}

int s5g_kway_merge(const uint8_t* arena, int64_t arena_len, int32_t k, const int64_t* run_offsets,
                   const int64_t* handles, const int64_t* lcps, const uint8_t* dchar,
                   int64_t shared, int64_t* out_handles, int64_t* out_lcps, void* workspace,
                   size_t workspace_bytes, void* stream, s5g_stats* stats) {
    if (k < 1 || k > MERGE_KMAX) return fail(S5G_E_INVALID, "k must be in 1..16");
    if (!run_offsets) return fail(S5G_E_INVALID, "null run_offsets");
    if (shared < 0) return fail(S5G_E_INVALID, "negative shared prefix");
    MergeRuns R{};
    R.k = k;
    int64_t ncand = 0;
    for (int j = 0; j <= k; j++) {
        R.off[j] = run_offsets[j] - run_offsets[0];
        if (j && R.off[j] < R.off[j - 1]) return fail(S5G_E_INVALID, "run offsets decrease");
    }
    for (int j = 0; j < k; j++) {
        R.coff[j] = ncand;
        ncand += (R.off[j + 1] - R.off[j] + MERGE_M - 1) / MERGE_M;
    }
    R.coff[k] = ncand;
    const int64_t n = R.off[k];
    if (n == 0) return 0;
    if (n > INT32_MAX) return fail(S5G_E_INVALID, "n exceeds 2^31-1");
    if (!arena || !handles || !lcps || !out_handles || !out_lcps) return fail(S5G_E_INVALID, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    handles += run_offsets[0];
    lcps += run_offsets[0];
    if (dchar) dchar += run_offsets[0];
    if (workspace_bytes < s5g_merge_workspace_bytes(n, k) || !workspace)
        return fail(S5G_E_WORKSPACE, "workspace too small");
    size_t off = 0;
    auto take = [&](size_t bytes) -> uint8_t* {
        off = (off + 255) & ~size_t(255);
        uint8_t* p = (uint8_t*)workspace + off;
        off += bytes;
        return p;
    };
    int64_t* cut = (int64_t*)take(8 * ncand * k);
    int64_t* cand_out = (int64_t*)take(8 * ncand);
    int32_t* cand_at = (int32_t*)take(4 * n);
    int32_t* order = (int32_t*)take(4 * ncand);
    const int64_t nch = (n + MC_CHUNK - 1) / MC_CHUNK;
    uint32_t* chunk = (uint32_t*)take(4 * nch);
    int64_t* d_n = (int64_t*)take(8);
    unsigned long long* words = (unsigned long long*)take(8);
    CK(cudaMemsetAsync(words, 0, 8, st));
    if (k == 1) {
        CK(cudaMemcpyAsync(out_handles, handles, 8 * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(out_lcps, lcps, 8 * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(out_lcps, &shared, 8, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        return 0;
    }
    CK(cudaMemsetAsync(cand_at, 0xff, 4 * n, st));
    g_launches += 6;
    k_merge_cands<<<blocks_for(ncand, 128), 128, 0, st>>>(arena, arena_len, handles, R, ncand,
                                                          shared, cut, cand_out, cand_at, words);
    k_mc_count<<<(unsigned)nch, MC_NT, 0, st>>>(cand_at, n, chunk);
    k_ld_scan<<<1, 1024, 0, st>>>(chunk, nch, d_n);
    k_mc_write<<<(unsigned)nch, MC_NT, 0, st>>>(cand_at, n, chunk, order);
    k_merge_jobs<<<blocks_for(ncand, 128), 128, 0, st>>>(arena, arena_len, handles, lcps, dchar, R,
                                                         order, ncand, shared, cut, cand_out,
                                                         out_handles, out_lcps, words);
    k_merge_fix<<<blocks_for(ncand, 256), 256, 0, st>>>(arena, arena_len, order, ncand, cand_out,
                                                         shared, out_handles, out_lcps, words);
    CK(cudaGetLastError());
    unsigned long long hw = 0;
    CK(cudaMemcpyAsync(&hw, words, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (stats) stats->word_fetches += (int64_t)hw;
    return 0;
}

int s5g_fill_dchar(const uint8_t* arena, const int64_t* handles, const int64_t* lcps, int64_t n,
                   uint8_t* out_dchar, void* stream) {
    if (n <= 0) return n < 0 ? fail(S5G_E_INVALID, "negative n") : 0;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches++;
    k_dchar<<<blocks_for(n, 256), 256, 0, st>>>(arena, handles, lcps, n, out_dchar);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
