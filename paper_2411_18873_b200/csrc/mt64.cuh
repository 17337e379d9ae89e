// std::mt19937_64 (libstdc++) on the device: seeding, one cooperative 312-word twist
// per CTA, the tempering output function, and libstdc++'s Lemire uniform draw.
#pragma once

#include <cstdint>

namespace etune_b200 {
namespace mt64 {

constexpr int kN = 312;
constexpr uint64_t kMatrixA = 0xb5026f5aa96619e9ull;
constexpr uint64_t kUpper = 0xffffffff80000000ull;
constexpr uint64_t kLower = 0x7fffffffull;

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71d67fffeda60000ull;
    y ^= (y << 37) & 0xfff7eee000000000ull;
    y ^= y >> 43;
    return y;
}

__device__ __forceinline__ uint64_t twist1(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t x = (cur & kUpper) | (next & kLower);
    return far ^ (x >> 1) ^ ((x & 1ull) ? kMatrixA : 0ull);
}

// mt19937_64(seed) state (f = 6364136223846793005); call from one thread.
__device__ __forceinline__ void seed_state(uint64_t* mt, uint64_t seed) {
    uint64_t v = seed;
    mt[0] = v;
    for (int i = 1; i < kN; ++i) {
        v = 6364136223846793005ull * (v ^ (v >> 62)) + uint64_t(i);
        mt[i] = v;
    }
}

// One in-place twist of the shared state by the whole CTA (blockDim >= 312):
// entries [0,156) read only old words; [156,311) read new [0,155]; 311 reads new 0/155.
// Ends with a barrier; the 312 fresh outputs are temper(mt[i]).
__device__ __forceinline__ void twist_block(uint64_t* mt) {
    const int tid = threadIdx.x;
    uint64_t cur = 0, nxt = 0;
    if (tid < kN) {
        cur = mt[tid];
        nxt = tid < kN - 1 ? mt[tid + 1] : 0;
    }
    __syncthreads();
    if (tid < 156) mt[tid] = twist1(cur, nxt, mt[tid + 156]);
    __syncthreads();
    if (tid >= 156 && tid < kN - 1) mt[tid] = twist1(cur, nxt, mt[tid - 156]);
    if (tid == kN - 1) {
        const uint64_t m0 = mt[0], m155 = mt[155];
        mt[kN - 1] = twist1(cur, m0, m155);
    }
    __syncthreads();
}

// uniform_int_distribution<size_t>(0, r-1) on one word without the rejection loop:
// returns the draw; *hazard is set when libstdc++ would reject this word and draw again.
__device__ __forceinline__ uint64_t lemire1(uint64_t x, uint64_t r, bool* hazard) {
    const uint64_t lo = x * r;
    if (lo < r) {
        const uint64_t thr = (0ull - r) % r;
        if (lo < thr) *hazard = true;
    }
    return __umul64hi(x, r);
}

}  // namespace mt64
}  // namespace etune_b200
