/*
 * oracle/s5_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference's S^5 hot path (strsort 0.1.0,
 * /root/reference/pkg/src/strsort/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` leg may load this code,
 * and only as the checker or the timed CPU baseline -- never as the product
 * path.  The product (paper_1403_2056_b200) never links or imports it.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py writes the fixtures; tests/test_oracle.py).
 *
 * One deliberate difference: draw_sample (ssss.py:76-82) uses numpy's PCG64
 * seeded with (seed, lo, hi, depth); we use a splitmix64 stream keyed by the
 * same tuple.  The sample only shapes splitter trees, never the output: the
 * result is the unique stable sort of the input handles.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WORD_CHARS 8
#define LCP_UNDEF (-1)
#define T_INSERTION 64       /* ssss.py:33, mkqs.py:26 */
#define OVERSAMPLE 2         /* ssss.py:32 */

typedef struct {
    int64_t char_cmps, word_fetches, merge_buffer_cmps, scratch_words;
    int64_t jobs_enqueued, jobs_executed, share_events;
} s5o_stats; /* counters.py:13-36 */

/* ------------------------------------------------------------------ */
/* word helpers: strset.py:152-206                                      */

/* Key at depth d for a string known to have length >= d
 * (the in-sort precondition; extract_keys strset.py:152-170). */
static inline uint64_t key_at(const uint8_t *buf, int64_t buflen, int64_t h, int64_t d)
{
    uint64_t k = 0;
    int64_t p = h + d;
    for (int j = 0; j < WORD_CHARS; j++, p++) {
        uint8_t c = p < buflen ? buf[p] : 0;
        if (c == 0) return j == 0 ? 0 : k << (8 * (WORD_CHARS - j));
        k = (k << 8) | c;
    }
    return k;
}

/* Exact extract_keys semantics for any depth: 0 when depth >= length. */
uint64_t s5o_extract_key(const uint8_t *buf, int64_t buflen, int64_t h, int64_t d)
{
    for (int64_t p = h; p < h + d; p++)
        if (p >= buflen || buf[p] == 0) return 0;
    return key_at(buf, buflen, h, d);
}

void s5o_extract_keys(const uint8_t *buf, int64_t buflen, const int64_t *handles,
                      int64_t n, int64_t d, uint64_t *out)
{
    for (int64_t i = 0; i < n; i++) out[i] = s5o_extract_key(buf, buflen, handles[i], d);
}

/* word_terminator_pos strset.py:187-191 */
int s5o_term_pos(uint64_t k)
{
    for (int i = 0; i < WORD_CHARS; i++)
        if (((k >> (8 * (WORD_CHARS - 1 - i))) & 0xff) == 0) return i;
    return WORD_CHARS;
}

/* shared_chars strset.py:194-206 */
int s5o_shared_chars(uint64_t a, uint64_t b)
{
    int i = 0;
    while (i < WORD_CHARS) {
        unsigned ca = (a >> (8 * (WORD_CHARS - 1 - i))) & 0xff;
        unsigned cb = (b >> (8 * (WORD_CHARS - 1 - i))) & 0xff;
        if (ca != cb || ca == 0) break;
        i++;
    }
    return i;
}

/* lcp strset.py:209-217 */
int64_t s5o_lcp(const uint8_t *buf, int64_t ha, int64_t hb)
{
    int64_t i = 0;
    for (;;) {
        uint8_t ca = buf[ha + i];
        if (ca == 0 || ca != buf[hb + i]) return i;
        i++;
    }
}

/* ------------------------------------------------------------------ */
/* splitter tree: ssss.py:67-146                                        */

int64_t s5o_tree_capacity(int64_t n, int64_t v)
{
    int64_t limit = n / 2 > 1 ? n / 2 : 1;
    if (v < limit) limit = v;
    int d = 0;
    while ((1LL << (d + 1)) - 1 <= limit) d++;
    int64_t cap = (1LL << d) - 1;
    return cap > 1 ? cap : 1;
}

typedef struct {
    int64_t v;
    uint64_t *tree;            /* v+1, index 0 unused, level order */
    uint64_t *inorder;         /* v */
    int64_t *node_to_inorder;  /* v+1 */
    int64_t *slcp;             /* v+1 */
    uint8_t *eq_final;         /* v */
    int64_t *eq_leftmost;      /* v */
    int64_t *term_pos;         /* v */
} tree_t;

static void fill_slots(uint64_t *inorder, const uint64_t *sample, int64_t slot_lo,
                       int64_t slot_hi, int64_t a, int64_t b, uint64_t parent)
{
    if (slot_lo >= slot_hi) return;
    int64_t mid = (slot_lo + slot_hi) / 2;
    if (a >= b) {
        /* subrange exhausted by duplicate skipping: reuse the parent pick */
        for (int64_t s = slot_lo; s < slot_hi; s++) inorder[s] = parent;
        return;
    }
    int64_t m = (a + b) / 2;
    uint64_t x = sample[m];
    inorder[mid] = x;
    int64_t b2 = m;
    while (b2 > a && sample[b2 - 1] == x) b2--;
    int64_t a2 = m + 1;
    while (a2 < b && sample[a2] == x) a2++;
    fill_slots(inorder, sample, slot_lo, mid, a, b2, x);
    fill_slots(inorder, sample, mid + 1, slot_hi, a2, b, x);
}

static void build_level(tree_t *t, int64_t node, int64_t lo, int64_t hi)
{
    if (lo >= hi) return;
    int64_t mid = (lo + hi) / 2;
    t->tree[node] = t->inorder[mid];
    t->node_to_inorder[node] = mid;
    build_level(t, 2 * node, lo, mid);
    build_level(t, 2 * node + 1, mid + 1, hi);
}

static void tree_finish(tree_t *t)
{
    int64_t v = t->v;
    memset(t->tree, 0, (v + 1) * sizeof(uint64_t));
    memset(t->node_to_inorder, 0, (v + 1) * sizeof(int64_t));
    build_level(t, 1, 0, v);
    memset(t->slcp, 0, (v + 1) * sizeof(int64_t));
    for (int64_t i = 1; i < v; i++) t->slcp[i] = s5o_shared_chars(t->inorder[i - 1], t->inorder[i]);
    for (int64_t i = 0; i < v; i++) {
        t->term_pos[i] = s5o_term_pos(t->inorder[i]);
        t->eq_final[i] = t->term_pos[i] < WORD_CHARS;
    }
    t->eq_leftmost[0] = 0;
    for (int64_t i = 1; i < v; i++)
        t->eq_leftmost[i] = t->inorder[i] == t->inorder[i - 1] ? t->eq_leftmost[i - 1] : i;
}

/* select_splitters ssss.py:85-146; sample must be sorted ascending. */
void s5o_select_splitters(const uint64_t *sample, int64_t count, int64_t v, uint64_t *tree,
                          uint64_t *inorder, int64_t *node_to_inorder, int64_t *slcp,
                          uint8_t *eq_final, int64_t *eq_leftmost, int64_t *term_pos)
{
    tree_t t = {v, tree, inorder, node_to_inorder, slcp, eq_final, eq_leftmost, term_pos};
    fill_slots(inorder, sample, 0, v, 0, count, sample[count / 2]);
    tree_finish(&t);
}

static int tree_levels(int64_t v)
{
    int l = 0;
    while ((1LL << l) < v + 1) l++;
    return l;
}

/* classify_keys ssss.py:149-181; variant 0 = unroll, 1 = equal */
int s5o_classify(const uint64_t *keys, int64_t n, int64_t v, const uint64_t *tree,
                 const uint64_t *inorder, const int64_t *node_to_inorder,
                 const int64_t *eq_leftmost, int variant, int64_t *out)
{
    int L = tree_levels(v);
    if (variant == 0) {
        for (int64_t i = 0; i < n; i++) {
            uint64_t k = keys[i];
            int64_t idx = 1;
            for (int l = 0; l < L; l++) idx = 2 * idx + (k > tree[idx]);
            int64_t leaf = idx - (v + 1);
            int64_t probe = leaf < v - 1 ? leaf : v - 1;
            out[i] = 2 * leaf + ((leaf < v) && k == inorder[probe]);
        }
        return 0;
    }
    if (variant == 1) {
        for (int64_t i = 0; i < n; i++) {
            uint64_t k = keys[i];
            int64_t idx = 1, bucket = -1;
            for (int l = 0; l < L; l++) {
                uint64_t val = tree[idx];
                if (bucket < 0 && k == val) bucket = 2 * eq_leftmost[node_to_inorder[idx]] + 1;
                int64_t step = 2 * idx + (k > val);
                idx = bucket >= 0 ? 1 : step;
            }
            out[i] = bucket >= 0 ? bucket : 2 * (idx - (v + 1));
        }
        return 0;
    }
    return -1; /* ValueError("unknown classify variant") */
}

/* distribute ssss.py:194-212: stable counting redistribution */
void s5o_distribute(const int64_t *handles, const int64_t *oracle, int64_t n,
                    int64_t num_buckets, int64_t *out, int64_t *bounds)
{
    memset(bounds, 0, (num_buckets + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) bounds[oracle[i] + 1]++;
    for (int64_t b = 0; b < num_buckets; b++) bounds[b + 1] += bounds[b];
    int64_t *pos = malloc((num_buckets + 1) * sizeof(int64_t));
    memcpy(pos, bounds, (num_buckets + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) out[pos[oracle[i]]++] = handles[i];
    free(pos);
}

/* ------------------------------------------------------------------ */
/* RNG (stand-in for numpy default_rng((seed, lo, hi, depth)))           */

static inline uint64_t splitmix64(uint64_t *s)
{
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t rng_seed(uint64_t seed, int64_t lo, int64_t hi, int64_t depth)
{
    uint64_t s = seed * 0x9E3779B97F4A7C15ULL;
    uint64_t st = s ^ (uint64_t)lo;
    st = splitmix64(&st) ^ (uint64_t)hi;
    st = splitmix64(&st) ^ (uint64_t)depth;
    return splitmix64(&st);
}

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

/* ------------------------------------------------------------------ */
/* LCP insertion sort, Alg. 5: basecase.py:67-116                        */

/* Sorts hs[0..n) (all sharing `depth` chars), writes absolute LCPs to
 * lcp_out[1..n) when non-NULL (lcp_out[0] untouched). */
static void lcp_insertion_core(const uint8_t *buf, int64_t *s, int64_t n, int64_t depth,
                               int64_t *lcp_out, s5o_stats *st)
{
    if (n <= 0) return;
    int64_t hbuf[T_INSERTION + 1];
    int64_t *h = n + 1 <= T_INSERTION + 1 ? hbuf : malloc((n + 1) * sizeof(int64_t));
    for (int64_t i = 0; i <= n; i++) h[i] = depth;
    for (int64_t j = 1; j < n; j++) {
        int64_t i = j, x = s[j], hp = depth;
        while (i > 0) {
            int64_t hi = h[i];
            if (hi < hp) break; /* case 1 */
            if (hi == hp) {     /* case 2 */
                int64_t p = hp;
                uint8_t cx, cy;
                for (;;) {
                    cx = buf[x + hp];
                    cy = buf[s[i - 1] + hp];
                    st->char_cmps++;
                    if (cx != 0 && cx == cy) { hp++; continue; }
                    break;
                }
                if (cx >= cy) { h[i] = hp; hp = p; break; }
            }
            s[i] = s[i - 1]; /* case 3 (or failed case 2) */
            h[i + 1] = h[i];
            i--;
        }
        s[i] = x;
        h[i + 1] = hp;
    }
    if (lcp_out)
        for (int64_t k = 1; k < n; k++) lcp_out[k] = h[k];
    if (h != hbuf) free(h);
}

void s5o_lcp_insertion_sort(const uint8_t *buf, int64_t *handles, int64_t n, int64_t depth,
                            int64_t *lcps, s5o_stats *st)
{
    s5o_stats dummy = {0};
    lcp_insertion_core(buf, handles, n, depth, lcps, st ? st : &dummy);
    if (lcps && n > 0) lcps[0] = LCP_UNDEF;
}

/* ------------------------------------------------------------------ */
/* caching multikey quicksort: mkqs.py:86-253                            */

/* _BlockReader: counts one word fetch per distinct (string, block) pair;
 * block 0 is seeded from the partitioning cache. */
typedef struct {
    int64_t handle, base;
    uint64_t bits[4];    /* blocks 0..255 */
    int64_t *extra;      /* blocks >= 256, sorted list */
    int64_t n_extra, cap_extra;
} blockreader_t;

static inline void br_touch(blockreader_t *r, int64_t pos, s5o_stats *st)
{
    int64_t blk = (pos - r->base) / WORD_CHARS;
    if (blk < 256) {
        uint64_t m = 1ULL << (blk & 63);
        if (!(r->bits[blk >> 6] & m)) { r->bits[blk >> 6] |= m; st->word_fetches++; }
        return;
    }
    for (int64_t i = 0; i < r->n_extra; i++)
        if (r->extra[i] == blk) return;
    if (r->n_extra == r->cap_extra) {
        r->cap_extra = r->cap_extra ? 2 * r->cap_extra : 16;
        r->extra = realloc(r->extra, r->cap_extra * sizeof(int64_t));
    }
    r->extra[r->n_extra++] = blk;
    st->word_fetches++;
}

/* _cached_insertion mkqs.py:121-172 */
static void cached_insertion(const uint8_t *buf, int64_t *wh, uint64_t *wc, int64_t lo,
                             int64_t hi, int64_t depth, int64_t *lcps, s5o_stats *st)
{
    int64_t n = hi - lo;
    blockreader_t rd[T_INSERTION];
    int64_t order[T_INSERTION], h[T_INSERTION + 1];
    for (int64_t k = 0; k < n; k++) {
        memset(&rd[k], 0, sizeof(blockreader_t));
        rd[k].handle = wh[lo + k];
        rd[k].base = depth;
        rd[k].bits[0] = 1; /* block 0 from the cache */
        order[k] = k;
    }
    for (int64_t k = 0; k <= n; k++) h[k] = depth;
    for (int64_t j = 1; j < n; j++) {
        int64_t i = j, x = order[j], hp = depth;
        while (i > 0) {
            int64_t hi_ = h[i];
            if (hi_ < hp) break;
            if (hi_ == hp) {
                int64_t p = hp, y = order[i - 1];
                uint8_t cx, cy;
                for (;;) {
                    br_touch(&rd[x], hp, st);
                    cx = buf[rd[x].handle + hp];
                    br_touch(&rd[y], hp, st);
                    cy = buf[rd[y].handle + hp];
                    st->char_cmps++;
                    if (cx != 0 && cx == cy) { hp++; continue; }
                    break;
                }
                if (cx >= cy) { h[i] = hp; hp = p; break; }
            }
            order[i] = order[i - 1];
            h[i + 1] = h[i];
            i--;
        }
        order[i] = x;
        h[i + 1] = hp;
    }
    int64_t th[T_INSERTION];
    uint64_t tc[T_INSERTION];
    for (int64_t k = 0; k < n; k++) { th[k] = wh[lo + order[k]]; tc[k] = wc[lo + order[k]]; }
    memcpy(wh + lo, th, n * sizeof(int64_t));
    memcpy(wc + lo, tc, n * sizeof(uint64_t));
    if (lcps)
        for (int64_t k = 1; k < n; k++) lcps[lo + k] = h[k];
    for (int64_t k = 0; k < n; k++) free(rd[k].extra);
}

static inline uint64_t median3(uint64_t a, uint64_t b, uint64_t c)
{
    if (a > b) { uint64_t t = a; a = b; b = t; }
    if (b > c) { b = c; }
    return a > b ? a : b;
}

typedef struct { int64_t lo, hi, d; } range3_t;

/* mkqs_cached_items mkqs.py:196-253 (stable ternary partition) */
static void mkqs_cached_items(const uint8_t *buf, int64_t buflen, int64_t *wh, uint64_t *wc,
                              int64_t lo0, int64_t hi0, int64_t d0, int64_t *lcps,
                              s5o_stats *st)
{
    int64_t cap = 64, top = 0;
    range3_t *stack = malloc(cap * sizeof(range3_t));
    int64_t tmpcap = 0;
    int64_t *th = NULL;
    uint64_t *tc = NULL;
    stack[top++] = (range3_t){lo0, hi0, d0};
    while (top) {
        range3_t r = stack[--top];
        int64_t lo = r.lo, hi = r.hi, d = r.d, n = hi - lo;
        if (n <= 1) continue;
        if (n < T_INSERTION) {
            cached_insertion(buf, wh, wc, lo, hi, d, lcps, st);
            continue;
        }
        uint64_t piv = median3(wc[lo], wc[lo + n / 2], wc[hi - 1]);
        if (n > tmpcap) {
            tmpcap = n;
            th = realloc(th, n * sizeof(int64_t));
            tc = realloc(tc, n * sizeof(uint64_t));
        }
        int64_t nlt = 0, neq = 0, k = 0;
        for (int64_t i = lo; i < hi; i++) nlt += wc[i] < piv, neq += wc[i] == piv;
        int64_t plt = 0, peq = nlt, pgt = nlt + neq;
        uint64_t left_max = 0, right_min = UINT64_MAX;
        for (int64_t i = lo; i < hi; i++) {
            uint64_t c = wc[i];
            if (c < piv) { k = plt++; if (c > left_max) left_max = c; }
            else if (c == piv) k = peq++;
            else { k = pgt++; if (c < right_min) right_min = c; }
            th[k] = wh[i];
            tc[k] = c;
        }
        memcpy(wh + lo, th, n * sizeof(int64_t));
        memcpy(wc + lo, tc, n * sizeof(uint64_t));
        int64_t b1 = lo + nlt, b2 = b1 + neq, ngt = hi - b2;
        if (lcps) {
            if (nlt) lcps[b1] = d + s5o_shared_chars(left_max, piv);
            if (ngt) lcps[b2] = d + s5o_shared_chars(piv, right_min);
        }
        if (top + 3 > cap) { cap *= 2; stack = realloc(stack, cap * sizeof(range3_t)); }
        if (ngt > 1) stack[top++] = (range3_t){b2, hi, d};
        if (neq > 1) {
            int tp = s5o_term_pos(piv);
            if (tp < WORD_CHARS) {
                if (lcps)
                    for (int64_t i = b1 + 1; i < b2; i++) lcps[i] = d + tp;
            } else {
                int64_t nd = d + WORD_CHARS;
                for (int64_t i = b1; i < b2; i++) wc[i] = key_at(buf, buflen, wh[i], nd);
                st->word_fetches += neq;
                stack[top++] = (range3_t){b1, b2, nd};
            }
        }
        if (nlt > 1) stack[top++] = (range3_t){lo, b1, d};
    }
    free(stack);
    free(th);
    free(tc);
}

/* mkqs_cached mkqs.py:256-272 */
void s5o_mkqs_cached(const uint8_t *buf, int64_t buflen, int64_t *handles, int64_t n,
                     int64_t depth, int64_t *lcps, s5o_stats *st)
{
    s5o_stats dummy = {0};
    if (!st) st = &dummy;
    uint64_t *wc = malloc((n > 0 ? n : 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < n; i++) wc[i] = key_at(buf, buflen, handles[i], depth);
    st->word_fetches += n;
    if (lcps)
        for (int64_t i = 0; i < n; i++) lcps[i] = LCP_UNDEF;
    mkqs_cached_items(buf, buflen, handles, wc, 0, n, depth, lcps, st);
    free(wc);
}

/* ------------------------------------------------------------------ */
/* S^5 driver: ssss.py:227-387                                           */

typedef struct {
    const uint8_t *buf;
    int64_t buflen;
    int64_t *cur, *other;
    uint64_t *cache;
    int64_t *lcps; /* NULL when !want_lcps */
    uint64_t seed;
    int variant;
    int64_t v, t_medium;
} s5ctx_t;

typedef struct { int64_t lo, hi, d; int in_cur; } item_t;

static void tree_alloc(tree_t *t, int64_t v)
{
    t->v = v;
    t->tree = malloc((v + 1) * sizeof(uint64_t));
    t->inorder = malloc(v * sizeof(uint64_t));
    t->node_to_inorder = malloc((v + 1) * sizeof(int64_t));
    t->slcp = malloc((v + 1) * sizeof(int64_t));
    t->eq_final = malloc(v);
    t->eq_leftmost = malloc(v * sizeof(int64_t));
    t->term_pos = malloc(v * sizeof(int64_t));
}

static void tree_free(tree_t *t)
{
    free(t->tree); free(t->inorder); free(t->node_to_inorder); free(t->slcp);
    free(t->eq_final); free(t->eq_leftmost); free(t->term_pos);
}

/* draw_sample + select_splitters for src[lo:hi] at depth d (ssss.py:284-289) */
static void make_tree(const s5ctx_t *c, const int64_t *src, int64_t lo, int64_t hi, int64_t d,
                      tree_t *t)
{
    int64_t n = hi - lo;
    int64_t v = s5o_tree_capacity(n, c->v);
    int64_t count = v * OVERSAMPLE + OVERSAMPLE - 1;
    uint64_t *sample = malloc(count * sizeof(uint64_t));
    uint64_t s = rng_seed(c->seed, lo, hi, d);
    for (int64_t j = 0; j < count; j++) {
        int64_t idx = (int64_t)(splitmix64(&s) % (uint64_t)n);
        sample[j] = key_at(c->buf, c->buflen, src[lo + idx], d);
    }
    qsort(sample, count, sizeof(uint64_t), cmp_u64);
    tree_alloc(t, v);
    s5o_select_splitters(sample, count, v, t->tree, t->inorder, t->node_to_inorder, t->slcp,
                         t->eq_final, t->eq_leftmost, t->term_pos);
    free(sample);
}

static void push_children(const s5ctx_t *c, const tree_t *t, const int64_t *bounds, int64_t lo,
                          int64_t d, int dst_in_cur, item_t **stack, int64_t *top,
                          int64_t *cap)
{
    int64_t k = 2 * t->v + 1;
    for (int64_t i = 0; i < k; i++) {
        int64_t clo = lo + bounds[i], chi = lo + bounds[i + 1], sz = chi - clo;
        if (sz == 0) continue;
        if ((i & 1) && t->eq_final[i / 2]) {
            if (!dst_in_cur) memcpy(c->cur + clo, c->other + clo, sz * sizeof(int64_t));
            if (c->lcps)
                for (int64_t j = clo + 1; j < chi; j++) c->lcps[j] = d + t->term_pos[i / 2];
            continue;
        }
        if (sz == 1) {
            if (!dst_in_cur) c->cur[clo] = c->other[clo];
            continue;
        }
        int64_t cd = (i & 1) ? d + t->term_pos[i / 2] : d + t->slcp[i / 2];
        if (*top == *cap) { *cap *= 2; *stack = realloc(*stack, *cap * sizeof(item_t)); }
        (*stack)[(*top)++] = (item_t){clo, chi, cd, dst_in_cur};
    }
}

/* s5_sort_items ssss.py:310-358 */
static void s5_sort_items(const s5ctx_t *c, const item_t *items, int64_t nitems, s5o_stats *st)
{
    int64_t cap = 256 + nitems, top = 0;
    item_t *stack = malloc(cap * sizeof(item_t));
    for (int64_t i = 0; i < nitems; i++) stack[top++] = items[i];
    while (top) {
        item_t it = stack[--top];
        int64_t lo = it.lo, hi = it.hi, d = it.d, n = hi - lo;
        const int64_t *src = it.in_cur ? c->cur : c->other;
        if (n < c->t_medium) {
            if (!it.in_cur) memcpy(c->cur + lo, src + lo, n * sizeof(int64_t));
            if (n < 2) continue;
            if (n < T_INSERTION) {
                lcp_insertion_core(c->buf, c->cur + lo, n, d, c->lcps ? c->lcps + lo : NULL, st);
            } else {
                for (int64_t i = lo; i < hi; i++) c->cache[i] = key_at(c->buf, c->buflen, c->cur[i], d);
                st->word_fetches += n;
                mkqs_cached_items(c->buf, c->buflen, c->cur, c->cache, lo, hi, d, c->lcps, st);
            }
            continue;
        }
        int64_t *dst = it.in_cur ? c->other : c->cur;
        tree_t t;
        make_tree(c, src, lo, hi, d, &t);
        int64_t k = 2 * t.v + 1;
        int64_t *oracle = malloc(n * sizeof(int64_t));
        uint64_t *keys = malloc(n * sizeof(uint64_t));
        for (int64_t i = 0; i < n; i++) keys[i] = key_at(c->buf, c->buflen, src[lo + i], d);
        s5o_classify(keys, n, t.v, t.tree, t.inorder, t.node_to_inorder, t.eq_leftmost,
                     c->variant, oracle);
        int64_t *bounds = malloc((k + 1) * sizeof(int64_t));
        s5o_distribute(src + lo, oracle, n, k, dst + lo, bounds);
        if (c->lcps) {
            /* _write_boundary_lcps ssss.py:242-263 via per-bucket min/max */
            uint64_t *bmin = malloc(k * sizeof(uint64_t)), *bmax = calloc(k, sizeof(uint64_t));
            for (int64_t b = 0; b < k; b++) bmin[b] = UINT64_MAX;
            for (int64_t i = 0; i < n; i++) {
                int64_t b = oracle[i];
                if (keys[i] < bmin[b]) bmin[b] = keys[i];
                if (keys[i] > bmax[b]) bmax[b] = keys[i];
            }
            int64_t prev = -1;
            for (int64_t b = 0; b < k; b++) {
                if (bounds[b + 1] == bounds[b]) continue;
                if (prev >= 0) c->lcps[lo + bounds[b]] = d + s5o_shared_chars(bmax[prev], bmin[b]);
                prev = b;
            }
            free(bmin); free(bmax);
        }
        free(oracle); free(keys);
        if (top + k >= cap) { cap = top + k + 256; stack = realloc(stack, cap * sizeof(item_t)); }
        push_children(c, &t, bounds, lo, d, !it.in_cur, &stack, &top, &cap);
        free(bounds);
        tree_free(&t);
    }
    free(stack);
}

/* s5_sort ssss.py:361-387.  out_handles receives the sorted handles;
 * out_lcps (nullable) the LCP array with lcps[0] = -1. */
int s5o_s5_sort(const uint8_t *buf, int64_t buflen, const int64_t *handles, int64_t n,
                int64_t depth, int variant, int64_t v, uint64_t seed, int64_t t_medium,
                int64_t *out_handles, int64_t *out_lcps, s5o_stats *st)
{
    if (variant != 0 && variant != 1) return -1;
    s5o_stats dummy = {0};
    if (!st) st = &dummy;
    memcpy(out_handles, handles, n * sizeof(int64_t));
    int64_t *other = malloc((n > 0 ? n : 1) * sizeof(int64_t));
    uint64_t *cache = calloc(n > 0 ? n : 1, sizeof(uint64_t));
    st->scratch_words += n;
    if (out_lcps)
        for (int64_t i = 0; i < n; i++) out_lcps[i] = LCP_UNDEF;
    s5ctx_t c = {buf, buflen, out_handles, other, cache, out_lcps, seed, variant, v, t_medium};
    item_t root = {0, n, depth, 1};
    if (n > 0) s5_sort_items(&c, &root, 1, st);
    if (out_lcps && n > 0) out_lcps[0] = LCP_UNDEF;
    free(other);
    free(cache);
    return 0;
}

/* ------------------------------------------------------------------ */
/* parallel S^5 (parallel.py:329-492), OpenMP threads stand in for the   */
/* forked WorkPool; the phased step and batching follow the reference.   */

int s5o_parallel_s5(const uint8_t *buf, int64_t buflen, const int64_t *handles, int64_t n,
                    int p, int variant, uint64_t seed, int64_t t_medium,
                    int64_t *out_handles, int64_t *out_lcps, s5o_stats *st)
{
    if (variant != 0 && variant != 1) return -1;
    s5o_stats dummy = {0};
    if (!st) st = &dummy;
    if (p < 1) p = 1;
    memcpy(out_handles, handles, n * sizeof(int64_t));
    if (out_lcps)
        for (int64_t i = 0; i < n; i++) out_lcps[i] = LCP_UNDEF;
    if (n == 0) return 0;
    int64_t *other = malloc(n * sizeof(int64_t));
    uint64_t *cache = calloc(n, sizeof(uint64_t));
    s5ctx_t c = {buf, buflen, out_handles, other, cache, out_lcps, seed, variant, 8191, t_medium};
    int64_t par_threshold = (n + p - 1) / p;
    if (par_threshold < T_INSERTION) par_threshold = T_INSERTION;
    int64_t pcap = 64, ptop = 0, scap = 1024, stop_ = 0;
    item_t *pending = malloc(pcap * sizeof(item_t));
    item_t *small = malloc(scap * sizeof(item_t));
    pending[ptop++] = (item_t){0, n, 0, 1};
    uint16_t *oracle = malloc(n * sizeof(uint16_t));
    uint64_t *keys = malloc(n * sizeof(uint64_t));
    while (ptop) {
        item_t it = pending[--ptop];
        int64_t lo = it.lo, hi = it.hi, d = it.d, nsub = hi - lo;
        if (nsub < par_threshold || nsub < 2 * T_INSERTION) {
            if (stop_ == scap) { scap *= 2; small = realloc(small, scap * sizeof(item_t)); }
            small[stop_++] = it;
            continue;
        }
        int64_t *src = it.in_cur ? c.cur : c.other;
        int64_t *dst = it.in_cur ? c.other : c.cur;
        tree_t t;
        make_tree(&c, src, lo, hi, d, &t);
        int64_t k = 2 * t.v + 1;
        int64_t *counts = calloc((size_t)p * k, sizeof(int64_t));
        uint64_t *bmin = malloc((size_t)p * k * sizeof(uint64_t));
        uint64_t *bmax = calloc((size_t)p * k, sizeof(uint64_t));
        for (int64_t i = 0; i < (int64_t)p * k; i++) bmin[i] = UINT64_MAX;
        #pragma omp parallel for num_threads(p) schedule(static, 1)
        for (int s = 0; s < p; s++) {
            int64_t slo = lo + (nsub * s) / p, shi = lo + (nsub * (s + 1)) / p;
            int64_t tmp[1];
            for (int64_t i = slo; i < shi; i++) {
                keys[i] = key_at(buf, buflen, src[i], d);
                s5o_classify(keys + i, 1, t.v, t.tree, t.inorder, t.node_to_inorder,
                             t.eq_leftmost, variant, tmp);
                oracle[i] = (uint16_t)tmp[0];
                counts[(int64_t)s * k + tmp[0]]++;
            }
        }
        /* interleaved prefix sum: bucket-major, shard-minor (parallel.py:379-385) */
        int64_t *bounds = malloc((k + 1) * sizeof(int64_t));
        int64_t run = 0;
        for (int64_t b = 0; b < k; b++) {
            bounds[b] = run;
            for (int s = 0; s < p; s++) {
                int64_t cnt = counts[(int64_t)s * k + b];
                counts[(int64_t)s * k + b] = run;
                run += cnt;
            }
        }
        bounds[k] = run;
        #pragma omp parallel for num_threads(p) schedule(static, 1)
        for (int s = 0; s < p; s++) {
            int64_t slo = lo + (nsub * s) / p, shi = lo + (nsub * (s + 1)) / p;
            int64_t *off = counts + (int64_t)s * k;
            uint64_t *mn = bmin + (int64_t)s * k, *mx = bmax + (int64_t)s * k;
            for (int64_t i = slo; i < shi; i++) {
                int b = oracle[i];
                dst[lo + off[b]++] = src[i];
                if (keys[i] < mn[b]) mn[b] = keys[i];
                if (keys[i] > mx[b]) mx[b] = keys[i];
            }
        }
        if (out_lcps) {
            int64_t prev = -1;
            uint64_t pmax = 0;
            for (int64_t b = 0; b < k; b++) {
                if (bounds[b + 1] == bounds[b]) continue;
                uint64_t mn = UINT64_MAX, mx = 0;
                for (int s = 0; s < p; s++) {
                    if (bmin[(int64_t)s * k + b] < mn) mn = bmin[(int64_t)s * k + b];
                    if (bmax[(int64_t)s * k + b] > mx) mx = bmax[(int64_t)s * k + b];
                }
                if (prev >= 0) out_lcps[lo + bounds[b]] = d + s5o_shared_chars(pmax, mn);
                prev = b;
                pmax = mx;
            }
        }
        /* route children (parallel.py:419-437) */
        for (int64_t i = 0; i < k; i++) {
            int64_t clo = lo + bounds[i], chi = lo + bounds[i + 1], sz = chi - clo;
            if (sz == 0) continue;
            int dst_in_cur = !it.in_cur;
            if ((i & 1) && t.eq_final[i / 2]) {
                if (!dst_in_cur) memcpy(c.cur + clo, c.other + clo, sz * sizeof(int64_t));
                if (out_lcps)
                    for (int64_t j = clo + 1; j < chi; j++) out_lcps[j] = d + t.term_pos[i / 2];
                continue;
            }
            if (sz == 1) {
                if (!dst_in_cur) c.cur[clo] = c.other[clo];
                continue;
            }
            int64_t cd = (i & 1) ? d + t.term_pos[i / 2] : d + t.slcp[i / 2];
            item_t ch = {clo, chi, cd, dst_in_cur};
            if (sz >= par_threshold) {
                if (ptop == pcap) { pcap *= 2; pending = realloc(pending, pcap * sizeof(item_t)); }
                pending[ptop++] = ch;
            } else {
                if (stop_ == scap) { scap *= 2; small = realloc(small, scap * sizeof(item_t)); }
                small[stop_++] = ch;
            }
        }
        free(counts); free(bmin); free(bmax); free(bounds);
        tree_free(&t);
    }
    free(oracle);
    free(keys);
    /* batch jobs over the small subproblems; dynamic scheduling stands in
     * for voluntary work sharing (parallel.py:439-445) */
    s5o_stats *tst = calloc(p, sizeof(s5o_stats));
    #pragma omp parallel for num_threads(p) schedule(dynamic, 1)
    for (int64_t i = 0; i < stop_; i++) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        s5_sort_items(&c, &small[i], 1, &tst[tid]);
        tst[tid].jobs_executed++;
    }
    for (int i = 0; i < p; i++) {
        st->char_cmps += tst[i].char_cmps;
        st->word_fetches += tst[i].word_fetches;
        st->jobs_executed += tst[i].jobs_executed;
    }
    st->jobs_enqueued += stop_;
    free(tst);
    free(pending);
    free(small);
    free(other);
    free(cache);
    if (out_lcps) out_lcps[0] = LCP_UNDEF;
    return 0;
}

/* ------------------------------------------------------------------ */
/* verification oracles: strset.py:220-309, plus the K11 certificate      */

/* lcp_array_oracle strset.py:220-240; returns -1 if sorted, else the first
 * violating index. */
int64_t s5o_lcp_array(const uint8_t *buf, const int64_t *handles, int64_t n, int64_t *out)
{
    if (n == 0) return -1;
    out[0] = LCP_UNDEF;
    for (int64_t i = 1; i < n; i++) {
        int64_t a = handles[i - 1], b = handles[i];
        int64_t h = s5o_lcp(buf, a, b);
        if (buf[a + h] > buf[b + h]) return i;
        out[i] = h;
    }
    return -1;
}

/* fill_dchar basecase.py:36-42 */
void s5o_fill_dchar(const uint8_t *buf, const int64_t *handles, const int64_t *lcps, int64_t n,
                    uint8_t *out)
{
    for (int64_t i = 0; i < n; i++) out[i] = buf[handles[i] + (lcps[i] < 0 ? 0 : lcps[i])];
}

typedef struct { int64_t key, idx; } pair_t;
static int cmp_pair(const void *a, const void *b)
{
    const pair_t *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : x->idx > y->idx;
}

/* K11 certificate: out_handles is the STABLE sort of in_handles by string
 * content and out_lcps (nullable) is its exact LCP array.
 * report[0] = status (0 ok, 1 not a permutation, 2 order violated,
 * 3 stability violated, 4 lcp mismatch), report[1] = first bad index. */
/* Stable parallel LSD radix sort of pairs by key (keys >= 0): the pairs
 * start in idx order, so equal keys stay in increasing idx order -- the
 * order cmp_pair gives. */
static void radix_pairs(pair_t *a, int64_t n)
{
    if (n < 2) return;
    int64_t mx = 0;
    #pragma omp parallel for reduction(max : mx)
    for (int64_t i = 0; i < n; i++) if (a[i].key > mx) mx = a[i].key;
    int bits = 0;
    while (bits < 63 && (mx >> bits)) bits++;
    pair_t *b = malloc(n * sizeof(pair_t));
    const int R = 11, B = 1 << R;
    int T = omp_get_max_threads();
    int64_t *cnt = malloc((size_t)T * B * sizeof(int64_t));
    for (int sh = 0; sh < bits; sh += R) {
        #pragma omp parallel num_threads(T)
        {
            int t = omp_get_thread_num(), nt = omp_get_num_threads();
            int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            int64_t *c = cnt + (size_t)t * B;
            memset(c, 0, B * sizeof(int64_t));
            for (int64_t i = lo; i < hi; i++) c[(a[i].key >> sh) & (B - 1)]++;
            #pragma omp barrier
            #pragma omp single
            {
                int64_t run = 0;
                for (int d = 0; d < B; d++)
                    for (int u = 0; u < nt; u++) {
                        int64_t x = cnt[(size_t)u * B + d];
                        cnt[(size_t)u * B + d] = run;
                        run += x;
                    }
            }
            for (int64_t i = lo; i < hi; i++) b[c[(a[i].key >> sh) & (B - 1)]++] = a[i];
        }
        memcpy(a, b, n * sizeof(pair_t));
    }
    free(cnt);
    free(b);
}

/* K11 certificate: verify (strset.py:250-281) -- the output is a
 * permutation of the input handles in non-descending content order --, plus
 * stability of equal strings and the exact LCP array (lcp_array_oracle,
 * strset.py:220-240).  O(n + L) string work, all host threads. */
int s5o_certify(const uint8_t *buf, const int64_t *in_handles, const int64_t *out_handles,
                const int64_t *out_lcps, int64_t n, int64_t *report)
{
    report[0] = 0;
    report[1] = -1;
    if (n == 0) return 0;
    /* input position of every output element (duplicate handles are
     * matched in increasing order, the favourable assignment) */
    pair_t *in = malloc(n * sizeof(pair_t)), *out = malloc(n * sizeof(pair_t));
    #pragma omp parallel for
    for (int64_t i = 0; i < n; i++) {
        in[i] = (pair_t){in_handles[i], i};
        out[i] = (pair_t){out_handles[i], i};
    }
    int neg = 0;
    #pragma omp parallel for reduction(| : neg)
    for (int64_t i = 0; i < n; i++) neg |= in[i].key < 0 || out[i].key < 0;
    if (neg) {
        qsort(in, n, sizeof(pair_t), cmp_pair);
        qsort(out, n, sizeof(pair_t), cmp_pair);
    } else {
        radix_pairs(in, n);
        radix_pairs(out, n);
    }
    int64_t *inpos = malloc(n * sizeof(int64_t));
    int64_t bad = INT64_MAX;
    #pragma omp parallel for reduction(min : bad)
    for (int64_t i = 0; i < n; i++) {
        if (in[i].key != out[i].key) { if (i < bad) bad = i; continue; }
        inpos[out[i].idx] = in[i].idx;
    }
    if (bad != INT64_MAX) {
        report[0] = 1; report[1] = out[bad].idx;
        free(in); free(out); free(inpos);
        return 1;
    }
    free(in);
    free(out);
    if (out_lcps && out_lcps[0] != LCP_UNDEF) { report[0] = 4; report[1] = 0; free(inpos); return 4; }
    /* first failing adjacent pair (smallest i), found by all threads */
    int64_t first = INT64_MAX;
    int code_at_first = 0;
    #pragma omp parallel
    {
        int64_t my = INT64_MAX;
        int mycode = 0;
        #pragma omp for schedule(static)
        for (int64_t i = 1; i < n; i++) {
            if (i >= my) continue;
            int64_t a = out_handles[i - 1], b = out_handles[i];
            int64_t h = s5o_lcp(buf, a, b);
            uint8_t ca = buf[a + h], cb = buf[b + h];
            int code = 0;
            if (ca > cb) code = 2;
            else if (ca == cb && a != b && inpos[i - 1] > inpos[i]) code = 3;
            else if (out_lcps && out_lcps[i] != h) code = 4;
            if (code && i < my) { my = i; mycode = code; }
        }
        #pragma omp critical
        if (my < first) { first = my; code_at_first = mycode; }
    }
    if (first != INT64_MAX) { report[0] = code_at_first; report[1] = first; }
    free(inpos);
    return (int)report[0];
}

/* Lengths of the strings at the given handles (terminator scan). */
void s5o_lengths(const uint8_t *buf, const int64_t *handles, int64_t n, int64_t *out)
{
    for (int64_t i = 0; i < n; i++) out[i] = (int64_t)strlen((const char *)buf + handles[i]);
}

/* dist_stats strset.py:290-309, from a sorted set and its exact LCP array:
 * D = sum min(len+1, max(h_i, h_{i+1})+1), L = sum lcps[1:].  `lens` are the
 * string lengths in sorted order. */
void s5o_dist_stats(const int64_t *lcps, const int64_t *lens, int64_t n, int64_t *D, int64_t *L)
{
    int64_t d = 0, l = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t left = i > 0 ? lcps[i] : 0, right = i + 1 < n ? lcps[i + 1] : 0;
        int64_t nb = left > right ? left : right;
        int64_t a = lens[i] + 1, b = nb + 1;
        d += a < b ? a : b;
        if (i > 0) l += lcps[i];
    }
    *D = d;
    *L = l;
}

/* ------------------------------------------------------------------ */
/* K-way LCP merge: lcp_compare / lcp_compare_cached (lcpmerge.py:57-140)
 * and the LoserTree tournament (lcpmerge.py:250-340), sequential.         */

typedef struct { int64_t s, h; int c; } mplayer;  /* handle (-1 = done), lcp, cached char */

/* game between players a < b; returns the winner, updates the loser */
static int m_game(const uint8_t *buf, mplayer *P, int a, int b, int cached, s5o_stats *st)
{
    mplayer *A = &P[a], *B = &P[b];
    if (A->s < 0) { A->h = 0; return b; }          /* lcpmerge.py:72-75 */
    if (B->s < 0) { B->h = 0; return a; }
    if (A->h < B->h) return b;                       /* lcpmerge.py:91-94 */
    if (A->h > B->h) return a;
    int64_t h = A->h;
    int xa, xb;
    if (cached) {                                    /* lcpmerge.py:117-135 */
        xa = A->c; xb = B->c;
        st->char_cmps++;
        if (xa != 0 && xa == xb) {
            h++;
            for (;;) {
                xa = buf[A->s + h]; xb = buf[B->s + h];
                st->char_cmps++; st->merge_buffer_cmps++;
                if (xa != 0 && xa == xb) { h++; continue; }
                break;
            }
        }
    } else {                                         /* lcpmerge.py:76-89 */
        for (;;) {
            xa = buf[A->s + h]; xb = buf[B->s + h];
            st->char_cmps++; st->merge_buffer_cmps++;
            if (xa != 0 && xa == xb) { h++; continue; }
            break;
        }
    }
    if (xa <= xb) { B->h = h; B->c = xb; return a; }
    A->h = h; A->c = xa;
    return b;
}

/* Merge k sorted runs (handles/lcps/dchar laid end to end, run j =
 * [run_off[j], run_off[j+1])) into out_h / out_l; out_l[0] = shared. */
void s5o_kway_merge(const uint8_t *buf, int k, const int64_t *run_off, const int64_t *handles,
                    const int64_t *lcps, const uint8_t *dchar, int64_t shared, int64_t *out_h,
                    int64_t *out_l, s5o_stats *st)
{
    int K = 1;
    while (K < k) K *= 2;
    mplayer *P = calloc((size_t)K, sizeof(mplayer));
    int64_t *cur = calloc((size_t)K, sizeof(int64_t)), *end = calloc((size_t)K, sizeof(int64_t));
    int *node = calloc((size_t)2 * K, sizeof(int));
    int cached = dchar != NULL;
    for (int j = 0; j < K; j++) {
        P[j].s = -1;
        if (j < k && run_off[j] < run_off[j + 1]) {
            cur[j] = run_off[j];
            end[j] = run_off[j + 1];
            P[j].s = handles[cur[j]];
            P[j].h = shared;
            P[j].c = cached ? buf[P[j].s + shared] : 0;
        }
    }
    /* bottom-up tournament: node[K + j] = j, inner nodes keep the loser */
    int *win = calloc((size_t)2 * K, sizeof(int));
    for (int j = 0; j < K; j++) win[K + j] = j;
    for (int v = K - 1; v >= 1; v--) {
        int a = win[2 * v], b = win[2 * v + 1];
        int lo = a < b ? a : b, hi = a < b ? b : a;
        int w = m_game(buf, P, lo, hi, cached, st);
        win[v] = w;
        node[v] = w == lo ? hi : lo;
    }
    int w = win[1];
    int64_t n = run_off[k] - run_off[0];
    for (int64_t pos = 0; pos < n; pos++) {
        out_h[pos] = P[w].s;
        out_l[pos] = P[w].h;
        cur[w]++;
        if (cur[w] < end[w]) {
            P[w].s = handles[cur[w]];
            P[w].h = lcps[cur[w]];
            P[w].c = cached ? dchar[cur[w]] : 0;
        } else {
            P[w].s = -1;
            P[w].h = 0;
        }
        int x = w;
        for (int v = (K + w) / 2; v >= 1; v /= 2) {
            int y = node[v];
            int lo = x < y ? x : y, hi = x < y ? y : x;
            int r = m_game(buf, P, lo, hi, cached, st);
            node[v] = r == lo ? hi : lo;
            x = r;
        }
        w = x;
    }
    free(P); free(cur); free(end); free(node); free(win);
}
