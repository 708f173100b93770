// s5g_gen.cu -- counter-based generator of the C5 corpus (BASELINE.json
// configs[4]: 2^28 unique strings, lengths U[32,200], 16-character prefix
// from a seeded 2^16-word vocabulary, lowercase filler, 6-character base-36
// counter).  Bench / test infrastructure, not part of the sort: it only
// produces inputs.  Built into its own libs5gen.so.
//
// Every byte of string i is a pure function of (seed, i, position), so
//  - the host (OpenMP) and device generators write identical bytes,
//  - a scaled corpus (n = 2^28 * scale) is a prefix of the full one,
//  - the full 31 GB arena is generated on the GPU in milliseconds instead of
//    minutes of numpy.
// Definition (frozen):
//   h0   = mix(mix(seed) ^ i)
//   len  = 32 + ((h0 >> 40) * 169 >> 24)                 U[32, 200]
//   word = h0 & 0xffff                                    vocabulary index
//   chars 0..15   : vocabulary word: y_q = mix(mix(seed ^ V) ^ (2 word + q)),
//                   char j of block q = 'a' + ((byte j of y_q) * 26 >> 8)
//   chars 16..len-7: filler: y = mix(mix(seed ^ F) ^ (i << 5 | p >> 3)),
//                   char p = 'a' + ((byte (p & 7) of y) * 26 >> 8)
//   chars len-6..len-1: i in base 36 ("0-9a-z"), most significant first
//   byte len: 0 terminator.  Strings are packed back to back.
#include <cuda_runtime.h>
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <string>

#include <cub/device/device_scan.cuh>

#include "s5g_gen.h"

namespace {

constexpr uint64_t VTAG = 0x5bd1e9955bd1e995ull, FTAG = 0xabcdef0123456789ull;

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64 finaliser
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint8_t letter(uint64_t y, int b) {
    return (uint8_t)('a' + ((((uint32_t)(y >> (8 * b))) & 255u) * 26u >> 8));
}

__host__ __device__ __forceinline__ uint64_t head(uint64_t seed, int64_t i) {
    return mix(mix(seed) ^ (uint64_t)i);
}

__host__ __device__ __forceinline__ int str_len(uint64_t h0) {
    return 32 + (int)(((h0 >> 40) * 169ull) >> 24);
}

// Byte p (0 <= p <= len) of string i; `y` caches the last 8-character
// hash block (blk = its index, -1 = none) across ascending positions.
struct Gen {
    uint64_t seed, i, h0, vseed, fseed;
    int len;
    uint64_t y;
    int64_t blk;
    __host__ __device__ Gen(uint64_t s, int64_t idx) : seed(s), i((uint64_t)idx) {
        h0 = head(s, idx);
        len = str_len(h0);
        vseed = mix(s ^ VTAG);
        fseed = mix(s ^ FTAG);
        blk = -1;
        y = 0;
    }
    __host__ __device__ __forceinline__ uint8_t at(int p) {
        if (p >= len) return 0;
        if (p < 16) {
            const int64_t b = p >> 3;  // vocabulary blocks 0, 1
            if (blk != b) {
                y = mix(vseed ^ (2 * (h0 & 0xffff) + (uint64_t)b));
                blk = b;
            }
            return letter(y, p & 7);
        }
        if (p >= len - 6) {
            uint64_t c = i;
            for (int k = len - 1; k > p; k--) c /= 36;
            const uint32_t d = (uint32_t)(c % 36);
            return (uint8_t)(d < 10 ? '0' + d : 'a' + d - 10);
        }
        const int64_t b = 2 + (p >> 3);  // filler blocks (>= 2 never clash with vocab)
        if (blk != b) {
            y = mix(fseed ^ (i << 5 | (uint64_t)(p >> 3)));
            blk = b;
        }
        return letter(y, p & 7);
    }
};

thread_local std::string g_err;

int fail(const std::string& m) {
    g_err = m;
    return -1;
}

__global__ void k_gen_len(uint64_t seed, int64_t n0, int64_t n, int64_t* __restrict__ len1) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) len1[k] = str_len(head(seed, n0 + k)) + 1;
}

// One thread per string: whole aligned 8-byte words inside the string are
// stored as u64, the (shared) edge words byte by byte.
__global__ void k_gen_fill(uint64_t seed, int64_t n0, int64_t n, const int64_t* __restrict__ off,
                           int64_t base, uint8_t* __restrict__ buf) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    Gen g(seed, n0 + k);
    const int64_t s = off[k] - base, e = s + g.len + 1;  // [s, e) incl. terminator
    int64_t a = (s + 7) & ~int64_t(7);
    const int64_t z = e & ~int64_t(7);
    for (int64_t q = s; q < (a < e ? a : e); q++) buf[q] = g.at((int)(q - s));
    for (int64_t q = a; q < z; q += 8) {
        uint64_t w = 0;
#pragma unroll
        for (int b = 0; b < 8; b++) w |= (uint64_t)g.at((int)(q + b - s)) << (8 * b);
        *reinterpret_cast<uint64_t*>(buf + q) = w;
    }
    for (int64_t q = (z > a ? z : a); q < e; q++) buf[q] = g.at((int)(q - s));
}

}  // namespace

extern "C" {

const char* s5gen_last_error(void) { return g_err.c_str(); }

int64_t s5gen_nodup_bytes(int64_t n0, int64_t n, uint64_t seed) {
    int64_t total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (int64_t k = 0; k < n; k++) total += str_len(head(seed, n0 + k)) + 1;
    return total;
}

int s5gen_nodup_host(int64_t n0, int64_t n, uint64_t seed, uint8_t* buf, int64_t* handles) {
    if (n < 0 || n0 < 0) return fail("negative size");
    if (n == 0) return 0;
    // offsets: per-thread block sums, then a serial scan of the blocks
    const int T = omp_get_max_threads();
    int64_t* part = new int64_t[T + 1]();
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        int64_t s = 0;
        for (int64_t k = lo; k < hi; k++) s += str_len(head(seed, n0 + k)) + 1;
        part[t + 1] = s;
#pragma omp barrier
#pragma omp single
        for (int u = 0; u < nt; u++) part[u + 1] += part[u];
        int64_t o = part[t];
        for (int64_t k = lo; k < hi; k++) {
            Gen g(seed, n0 + k);
            if (handles) handles[k] = o;
            if (buf) {
                for (int p = 0; p <= g.len; p++) buf[o + p] = g.at(p);
            }
            o += g.len + 1;
        }
    }
    delete[] part;
    return 0;
}

int s5gen_nodup_device(int64_t n0, int64_t n, uint64_t seed, uint8_t* buf, int64_t* handles,
                       void* stream) {
    if (n < 0 || n0 < 0) return fail("negative size");
    if (n == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)((n + 255) / 256);
    k_gen_len<<<grid, 256, 0, st>>>(seed, n0, n, handles);
    size_t tmp = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, handles, handles, n, st);
    void* d_tmp = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&d_tmp, tmp, st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp, handles, handles, n, st);
    if (e == cudaSuccess) e = cudaFreeAsync(d_tmp, st);
    if (e == cudaSuccess) {
        k_gen_fill<<<grid, 256, 0, st>>>(seed, n0, n, handles, 0, buf);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(std::string("cuda: ") + cudaGetErrorString(e));
    return 0;
}

}  // extern "C"
