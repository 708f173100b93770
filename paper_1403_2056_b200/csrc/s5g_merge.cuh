// s5g_merge.cuh -- K-way LCP merge of sorted runs on the GPU: the merge
// phase of partitioned_merge_sort (parallel.py:885-994) and kway_lcp_merge /
// LoserTree / lcp_compare(_cached) (lcpmerge.py:57-140, 250-424).
//
// The reference splits one merge into independent jobs (split_merge_jobs,
// lcpmerge.py:427-486) that its workers run as tournament merges.  Here the
// jobs come from candidates -- every MERGE_M-th string of every run: an
// LCP-bounded binary search puts each candidate into every other run (ties
// go to the earlier run, so the merge is stable), the candidate's output
// position is the sum of those cut positions, and consecutive candidates in
// output order delimit a job of about MERGE_M strings.  One thread runs one
// job as an LCP loser tree; players carry (handle, lcp to the last output,
// cached distinguishing character), unequal LCPs decide without reading
// characters, equal LCPs compare 8-byte words from the LCP on.  The first
// LCP of every job is recomputed against the previous job's last string
// (the reference's boundary recompute, parallel.py:989-991).
#pragma once
#include "s5g_kernels.cuh"

namespace s5g {

constexpr int MERGE_KMAX = 16;
constexpr int MERGE_M = 64;   // candidate stride in every run
constexpr int MC_NT = 256, MC_PER = 16, MC_CHUNK = MC_NT * MC_PER;  // compaction

struct MergeRuns {
    int k;
    int64_t off[MERGE_KMAX + 1];   // run j: [off[j], off[j+1]) of the concatenated arrays
    int64_t coff[MERGE_KMAX + 1];  // candidates of run j: [coff[j], coff[j+1])
};

// Compare the strings at a and b, known equal before depth d: <0, 0, >0,
// their LCP in *l (lcp, strset.py:209-217, a word at a time) and the two
// characters at that position (0 past a terminator).
__device__ __forceinline__ int str_cmp_chars(const uint8_t* __restrict__ arena, int64_t alen,
                                             int64_t a, int64_t b, int64_t d, int64_t* l,
                                             unsigned& words, uint32_t& ca, uint32_t& cb) {
    for (;;) {
        const uint64_t wa = load_key(arena, alen, a, d), wb = load_key(arena, alen, b, d);
        words += 2;
        if (wa != wb) {
            const int k = __clzll(wa ^ wb) >> 3;
            *l = d + k;
            ca = (uint32_t)(wa >> (56 - 8 * k)) & 255u;
            cb = (uint32_t)(wb >> (56 - 8 * k)) & 255u;
            return wa < wb ? -1 : 1;
        }
        const int tp = term_pos(wa);
        if (tp < WORD) {
            *l = d + tp;
            ca = cb = 0;
            return 0;
        }
        d += WORD;
    }
}

__device__ __forceinline__ int str_cmp_from(const uint8_t* __restrict__ arena, int64_t alen,
                                            int64_t a, int64_t b, int64_t d, int64_t* l,
                                            unsigned& words) {
    uint32_t ca, cb;
    return str_cmp_chars(arena, alen, a, b, d, l, words, ca, cb);
}

// Cut positions of candidate c in every run (number of strings of run j that
// precede c in the stable merged order) and its output position.
__global__ void k_merge_cands(const uint8_t* __restrict__ arena, int64_t alen,
                              const int64_t* __restrict__ handles, MergeRuns R, int64_t ncand,
                              int64_t shared, int64_t* __restrict__ cut,
                              int64_t* __restrict__ cand_out, int32_t* __restrict__ cand_at,
                              unsigned long long* __restrict__ words_ctr) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncand) return;
    int kc = 0;
    while (kc + 1 < R.k && R.coff[kc + 1] <= c) kc++;
    const int64_t i = (c - R.coff[kc]) * MERGE_M;
    const int64_t hc = handles[R.off[kc] + i];
    unsigned words = 0;
    int64_t outp = 0;
    for (int j = 0; j < R.k; j++) {
        int64_t p = i;
        if (j != kc) {
            const int64_t* run = handles + R.off[j];
            int64_t lo = 0, hi = R.off[j + 1] - R.off[j];
            int64_t llo = shared, lhi = shared;  // lcp(c, run[lo-1]), lcp(c, run[hi])
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                int64_t l;
                const int r = str_cmp_from(arena, alen, run[mid], hc, min(llo, lhi), &l, words);
                if (r < 0 || (r == 0 && j < kc)) {  // run[mid] precedes c
                    lo = mid + 1;
                    llo = l;
                } else {
                    hi = mid;
                    lhi = l;
                }
            }
            p = lo;
        }
        cut[c * R.k + j] = p;
        outp += p;
    }
    cand_out[c] = outp;
    cand_at[outp] = (int32_t)c;
    if (words) atomicAdd(words_ctr, (unsigned long long)words);
}

// Compaction of cand_at (>= 0 entries) into output order: count, scan, write.
__global__ void k_mc_count(const int32_t* __restrict__ cand_at, int64_t n,
                           uint32_t* __restrict__ chunk_cnt) {
    __shared__ uint32_t wsum[32];
    const int64_t t0 = (int64_t)blockIdx.x * MC_CHUNK + (int64_t)threadIdx.x * MC_PER;
    uint32_t cnt = 0;
    for (int64_t i = t0; i < min(t0 + MC_PER, n); i++) cnt += cand_at[i] >= 0;
    uint32_t total;
    block_excl_sum<MC_NT>(cnt, wsum, &total);
    if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = total;
}

__global__ void k_mc_write(const int32_t* __restrict__ cand_at, int64_t n,
                           const uint32_t* __restrict__ chunk_off, int32_t* __restrict__ order) {
    __shared__ uint32_t wsum[32];
    const int64_t t0 = (int64_t)blockIdx.x * MC_CHUNK + (int64_t)threadIdx.x * MC_PER;
    uint32_t cnt = 0;
    for (int64_t i = t0; i < min(t0 + MC_PER, n); i++) cnt += cand_at[i] >= 0;
    uint32_t k = chunk_off[blockIdx.x] + block_excl_sum<MC_NT>(cnt, wsum, nullptr);
    for (int64_t i = t0; i < min(t0 + MC_PER, n); i++)
        if (cand_at[i] >= 0) order[k++] = cand_at[i];
}

// lcp_compare / lcp_compare_cached (lcpmerge.py:57-140) for players a < b
// (indices), both trailing the last output with LCPs ha, hb.  Returns the
// winner; the loser's LCP becomes lcp(a, b) and its cached character the one
// at that position.  Ties go to a (the earlier stream): stable.
struct Player {
    int64_t s;   // handle, -1 = exhausted
    int64_t h;   // lcp to the last output
    uint32_t c;  // character at h (cached mode)
};

__device__ __forceinline__ int lcp_game(Player* P, int a, int b, bool cached,
                                        const uint8_t* __restrict__ arena, int64_t alen,
                                        unsigned& words) {
    Player& A = P[a];
    Player& B = P[b];
    if (A.s < 0) {
        A.h = 0;
        return b;
    }
    if (B.s < 0) {
        B.h = 0;
        return a;
    }
    if (A.h != B.h) {
        if (A.h < B.h) return b;  // b shares more with the last output: smaller
        return a;
    }
    // equal LCPs: characters from h on
    const int64_t h = A.h;
    if (cached && (A.c != B.c || A.c == 0)) {
        // decided by the cached characters: the loser keeps (h, its char)
        return A.c <= B.c ? a : b;
    }
    int64_t l;
    uint32_t ca, cb;
    const int r = str_cmp_chars(arena, alen, A.s, B.s, cached ? h + 1 : h, &l, words, ca, cb);
    Player& L = r <= 0 ? B : A;
    L.h = l;
    L.c = r <= 0 ? cb : ca;  // the loser's character at the new LCP
    return r <= 0 ? a : b;
}

// One merge job per thread: a loser tree over the K runs' subranges.
__global__ void k_merge_jobs(const uint8_t* __restrict__ arena, int64_t alen,
                             const int64_t* __restrict__ handles, const int64_t* __restrict__ lcps,
                             const uint8_t* __restrict__ dchar, MergeRuns R,
                             const int32_t* __restrict__ order, int64_t ncand, int64_t shared,
                             const int64_t* __restrict__ cut, const int64_t* __restrict__ cand_out,
                             int64_t* __restrict__ out_h, int64_t* __restrict__ out_l,
                             unsigned long long* __restrict__ words_ctr) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ncand) return;
    const int K = R.k;
    int KP = 1;
    while (KP < K) KP <<= 1;
    const int64_t c = order[t], c2 = t + 1 < ncand ? order[t + 1] : -1;
    const bool cached = dchar != nullptr;
    Player P[MERGE_KMAX];
    int64_t cur[MERGE_KMAX], lim[MERGE_KMAX];
    int node[MERGE_KMAX];
    unsigned words = 0;
    for (int j = 0; j < KP; j++) {
        P[j].s = -1;
        P[j].h = 0;
        P[j].c = 0;
        cur[j] = lim[j] = 0;
        if (j < K) {
            cur[j] = R.off[j] + cut[c * K + j];
            lim[j] = R.off[j] + (c2 >= 0 ? cut[c2 * K + j] : R.off[j + 1] - R.off[j]);
            if (cur[j] < lim[j]) {
                P[j].s = handles[cur[j]];
                P[j].h = shared;
                if (cached) P[j].c = arena[P[j].s + shared];
            }
        }
    }
    // build: games bottom-up, node v holds the loser, winners climb
    int win[2 * MERGE_KMAX];
    for (int j = 0; j < KP; j++) win[KP + j] = j;
    for (int v = KP - 1; v >= 1; v--) {
        const int a = win[2 * v], b = win[2 * v + 1];
        const int w = lcp_game(P, min(a, b), max(a, b), cached, arena, alen, words);
        win[v] = w;
        node[v] = w == a ? b : a;
    }
    int w = win[1];
    int64_t pos = cand_out[c];
    const int64_t stop = c2 >= 0 ? cand_out[c2] : R.off[K];
    for (; pos < stop; pos++) {
        out_h[pos] = P[w].s;
        out_l[pos] = P[w].h;
        // pull the winner's successor: its LCP and cached character are
        // relative to the string just emitted (lcpmerge.py:318-330)
        cur[w]++;
        if (cur[w] < lim[w]) {
            P[w].s = handles[cur[w]];
            P[w].h = lcps[cur[w]];
            if (cached) P[w].c = dchar[cur[w]];
        } else {
            P[w].s = -1;
            P[w].h = 0;
        }
        int x = w;
        for (int v = (KP + w) >> 1; v >= 1; v >>= 1) {
            const int y = node[v];
            const int lo = min(x, y), hi = max(x, y);
            const int win2 = lcp_game(P, lo, hi, cached, arena, alen, words);
            node[v] = win2 == lo ? hi : lo;
            x = win2;
        }
        w = x;
    }
    if (words) atomicAdd(words_ctr, (unsigned long long)words);
}

// First LCP of every job against the previous job's last string.
__global__ void k_merge_fix(const uint8_t* __restrict__ arena, int64_t alen,
                            const int32_t* __restrict__ order, int64_t ncand,
                            const int64_t* __restrict__ cand_out, int64_t shared,
                            const int64_t* __restrict__ out_h, int64_t* __restrict__ out_l,
                            unsigned long long* __restrict__ words_ctr) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ncand) return;
    const int64_t pos = cand_out[order[t]];
    if (pos == 0) {
        out_l[0] = shared;
        return;
    }
    unsigned words = 0;
    int64_t l;
    str_cmp_from(arena, alen, out_h[pos - 1], out_h[pos], shared, &l, words);
    out_l[pos] = l;
    if (words) atomicAdd(words_ctr, (unsigned long long)words);
}

}  // namespace s5g
