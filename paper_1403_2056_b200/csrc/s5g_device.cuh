// s5g_device.cuh -- device primitives of the B200 S^5 sorter (sm_100a).
//
// Word keys follow strset.py:152-206: the 8 characters at a depth, first
// character in the most significant byte, zeroed at and after the string's
// terminator, so unsigned comparison of keys == lexicographic comparison.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Checked builds (-DS5G_CHECKED, tools/build_variant.sh checked ...): device
// bounds checks on arena addresses, record / slot indices and output
// positions; a failed check prints its line and traps (the launch then
// fails with a CUDA error).  compute-sanitizer is not available on the GPU
// pool this repo is measured on; this is the stand-in.
#ifdef S5G_CHECKED
#include <cstdio>
#define S5G_CHECK(c)                                                                  \
    do {                                                                              \
        if (!(c)) {                                                                   \
            printf("s5g check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);         \
            __trap();                                                                 \
        }                                                                             \
    } while (0)
#else
#define S5G_CHECK(c) \
    do {             \
    } while (0)
#endif

namespace s5g {

constexpr int WORD = 8;
constexpr int VMAX = 8191;            // DEFAULT_V, ssss.py:31
constexpr int NBMAX = 2 * VMAX + 1;   // 16383 buckets
constexpr int LMAX = 13;              // levels of a v=8191 tree
constexpr int OVERSAMPLE = 2;         // alpha, ssss.py:32

constexpr uint64_t ONES = 0x0101010101010101ull;
constexpr uint64_t HIGHS = 0x8080808080808080ull;
constexpr uint64_t LOWS7 = 0x7f7f7f7f7f7f7f7full;

// Bit 7 of every zero byte of x (exact: no cross-byte carries).
__device__ __forceinline__ uint64_t zero_bytes(uint64_t x) {
    uint64_t t = ((x & LOWS7) + LOWS7) | x;
    return ~t & HIGHS;
}

__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}

// word_terminator_pos (strset.py:187-191): characters before the first 0.
__device__ __forceinline__ int term_pos(uint64_t key) {
    uint64_t z = zero_bytes(key);
    return z ? (__clzll(z) >> 3) : WORD;
}

// shared_chars (strset.py:194-206).
__device__ __forceinline__ int shared_chars(uint64_t a, uint64_t b) {
    return a == b ? term_pos(a) : (__clzll(a ^ b) >> 3);
}

// Mask a big-endian word after its first zero byte.
__device__ __forceinline__ uint64_t mask_terminated(uint64_t be) {
    uint64_t z = zero_bytes(be);
    if (!z) return be;
    int p = __clzll(z) >> 3;               // characters before the terminator
    return p ? (be & (~0ull << (64 - 8 * p))) : 0ull;
}

// 8 bytes at arena[pos..pos+8) as a little-endian word; bytes at or past
// arena_len read as 0.  Two aligned 8-byte loads + funnel shift: the arena is
// 8-byte aligned and readable to round_up(arena_len, 8) + 8.
__device__ __forceinline__ uint64_t load_word_le(const uint8_t* __restrict__ arena,
                                                 int64_t arena_len, int64_t pos) {
    int64_t a = pos & ~int64_t(7);
    int sh = (int)(pos & 7);
    S5G_CHECK(pos >= 0);
    uint64_t w0 = a < arena_len ? __ldg(reinterpret_cast<const unsigned long long*>(arena + a)) : 0ull;
    if (!sh) return w0;
    uint64_t w1 = (a + 8) < arena_len
                      ? __ldg(reinterpret_cast<const unsigned long long*>(arena + a + 8)) : 0ull;
    return (w0 >> (8 * sh)) | (w1 << (64 - 8 * sh));
}

// Key of the string at handle h at depth d, for a string of length >= d
// (the in-sort precondition: extract_keys strset.py:152-170).
__device__ __forceinline__ uint64_t load_key(const uint8_t* __restrict__ arena, int64_t arena_len,
                                             int64_t h, int64_t d) {
    return mask_terminated(bswap64(load_word_le(arena, arena_len, h + d)));
}

__device__ __forceinline__ uint64_t ld8_guard(const uint8_t* __restrict__ arena, int64_t alen,
                                              int64_t a) {
    S5G_CHECK(a >= 0);
    return a < alen ? __ldg(reinterpret_cast<const unsigned long long*>(arena + a)) : 0ull;
}

// The three words at depth d of the string at h (0 past the terminator):
// four aligned 8-byte loads, funnel shifts, byte swaps, exact masking.
__device__ __forceinline__ void load_words3(const uint8_t* __restrict__ arena, int64_t alen,
                                            int64_t h, int64_t d, uint64_t (&w)[3]) {
    const int64_t p = h + d, a = p & ~int64_t(7);
    const int sh = (int)(p & 7);
    const uint64_t x0 = ld8_guard(arena, alen, a), x1 = ld8_guard(arena, alen, a + 8),
                   x2 = ld8_guard(arena, alen, a + 16), x3 = sh ? ld8_guard(arena, alen, a + 24) : 0;
    const uint64_t l0 = sh ? (x0 >> (8 * sh)) | (x1 << (64 - 8 * sh)) : x0;
    const uint64_t l1 = sh ? (x1 >> (8 * sh)) | (x2 << (64 - 8 * sh)) : x1;
    const uint64_t l2 = sh ? (x2 >> (8 * sh)) | (x3 << (64 - 8 * sh)) : x2;
    w[0] = mask_terminated(bswap64(l0));
    w[1] = term_pos(w[0]) < WORD ? 0 : mask_terminated(bswap64(l1));
    w[2] = term_pos(w[1]) < WORD ? 0 : mask_terminated(bswap64(l2));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Position of sample j of `count` in a segment of n strings: stratified --
// one uniform pick inside each of `count` equal strata (draw_sample,
// ssss.py:76-82, picks uniformly at random; which positions are sampled
// never changes the output).  Consecutive samples fall in consecutive
// address ranges, so the random gathers of a large root sample share TLB
// entries instead of missing on nearly every one.
__device__ __forceinline__ int64_t sample_pos(uint64_t key0, int j, int count, int64_t n) {
    const int64_t a = (int64_t)j * n / count, b = (int64_t)(j + 1) * n / count;
    const int64_t w = b > a ? b - a : 1;
    return min(a + (int64_t)(splitmix64(key0 + j) % (uint64_t)w), n - 1);
}

// ---------------------------------------------------------------------------
// TMA-class 1-D bulk copies (cp.async.bulk) completing on an mbarrier.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// ---------------------------------------------------------------------------
// Block-wide scans over shared arrays.

template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* wsum, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < NT / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NT / 32) wsum[lane] = s;
    }
    __syncthreads();
    uint32_t base = w ? wsum[w - 1] : 0;
    if (total) *total = wsum[NT / 32 - 1];
    __syncthreads();
    return base + x - v;
}

// In-place exclusive scan of a[0..count) (any count); returns the total.
template <int NT>
__device__ uint32_t block_excl_scan_array(uint32_t* a, int count, uint32_t* wsum) {
    const int per = (count + NT - 1) / NT;
    const int beg = threadIdx.x * per;
    const int end = min(beg + per, count);
    uint32_t s = 0;
    for (int i = beg; i < end; i++) s += a[i];
    uint32_t total;
    uint32_t run = block_excl_sum<NT>(s, wsum, &total);
    for (int i = beg; i < end; i++) {
        uint32_t t = a[i];
        a[i] = run;
        run += t;
    }
    __syncthreads();
    return total;
}

template <int NT>
__device__ __forceinline__ uint32_t block_incl_max(uint32_t v, uint32_t* wsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, y);
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < NT / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s = max(s, y);
        }
        if (lane < NT / 32) wsum[lane] = s;
    }
    __syncthreads();
    uint32_t r = w ? max(wsum[w - 1], x) : x;
    __syncthreads();
    return r;
}

// Exclusive max over the threads before this one (0 for thread 0).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* wsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, y);
    }
    uint32_t ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = 0;
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < NT / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s = max(s, y);
        }
        if (lane < NT / 32) wsum[lane] = s;
    }
    __syncthreads();
    uint32_t r = w ? max(wsum[w - 1], ex) : ex;
    __syncthreads();
    return r;
}

}  // namespace s5g
