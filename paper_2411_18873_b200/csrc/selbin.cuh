// Fused selection's bucket function (score kernels -> sel_filter_kernel, sort.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace etune_b200 {

// SelHist with device-resident bounds -> kmin / shift (the same rule as the host's
// selection_buckets: the smallest shift that maps the key span onto kSelBins buckets)
__device__ __forceinline__ SelHist sel_resolve(SelHist s) {
    if (s.dbounds) {
        const uint64_t a = s.dbounds[0];
        uint64_t b = s.dbounds[1];
        if (!(b > a)) b = a + 1;
        const uint64_t span = b - a;
        // smallest sh with (span >> sh) < kSelBins (= 2^10): bit length of span minus 10
        const int bl = 64 - __clzll(static_cast<long long>(span));
        const uint32_t sh = bl > 10 ? uint32_t(bl - 10) : 0u;
        s.kmin = a;
        s.shift = sh;
    }
    return s;
}

// Bucket of a prediction for the fused selection (SelHist in kernels.hpp): monotone in
// the (score) order, so every key of a lower bucket is smaller than every key above it.
__device__ __forceinline__ uint32_t sel_bin(double p, const SelHist& s) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(p));
    const uint64_t key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    if (key < s.kmin) return 0u;
    const uint64_t d = (key - s.kmin) >> s.shift;
    return d < uint64_t(kSelBins - 1) ? uint32_t(d) : uint32_t(kSelBins - 1);
}

}  // namespace etune_b200
