// Host planner.  All per-candidate work that depends on one knob (or a pair of
// knobs) is tabulated here once per operator, so the device kernels reduce the
// reference's per-candidate counters.cpp/features.cpp arithmetic to table reads.
//
// Exactness argument (checked exhaustively by tests/test_gpu_parity.py):
//   glb_ld = grid*steps*bt_b*k_tile*(bt_m+bt_n)                     (counters.cpp:32-33)
//          = (B*M*N/(bt_m*bt_n)) * K * (bt_m+bt_n)   -> keyed by (bt_m, bt_n)
//   int_ops = shared_ld = grid*block*K*pt_b*(pt_m+pt_n)              (counters.cpp:37-38)
//          = (B*M*N/(pt_m*pt_n)) * K * (pt_m+pt_n)   -> keyed by (pt_m, pt_n)
// (integer identities; both sides are exact int64 whenever the final value fits, and
// build_plan rejects operators where 2*B*M*N*K could overflow).  log1p is then
// evaluated on the exact same int64->double value the reference passes to std::log1p.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

namespace etune_b200 {

std::vector<int64_t> divisors_of(int64_t e) {
    std::vector<int64_t> out;
    for (int64_t d = 1; d * d <= e; ++d) {
        if (e % d == 0) {
            out.push_back(d);
            if (d != e / d) out.push_back(e / d);
        }
    }
    std::sort(out.begin(), out.end());
    return out;
}

etune_status op_validate(const etune_op_spec& o, std::string* err) {
    auto bad = [&](const char* m) {
        *err = m;
        return ETUNE_ERR_VALIDATION;
    };
    if (o.kind == 0 || o.kind == 1) {
        if (o.batch < 1 || o.m < 1 || o.n < 1 || o.k < 1) return bad("matmul extents must all be >= 1");
        if (o.kind == 1 && o.m != 1) return bad("mv requires M == 1");
        return ETUNE_OK;
    }
    if (o.kind != 2) return bad("unknown operator kind");
    if (o.batch < 1 || o.height < 1 || o.width < 1 || o.in_channels < 1 || o.out_channels < 1 ||
        o.kernel_size < 1)
        return bad("conv extents must all be >= 1");
    if (o.stride < 1) return bad("conv stride must be >= 1");
    if (o.padding < 0) return bad("conv padding must be >= 0");
    const int64_t hs = o.height + 2 * o.padding - o.kernel_size;
    const int64_t ws = o.width + 2 * o.padding - o.kernel_size;
    if (hs < 0 || ws < 0 || hs % o.stride != 0 || ws % o.stride != 0)
        return bad("conv output extent (extent + 2*padding - kernel_size)/stride + 1 must be a positive integer");
    return ETUNE_OK;
}

void op_nest(const etune_op_spec& o, int64_t out[4]) {
    if (o.kind == 2) {
        const int64_t oh = (o.height + 2 * o.padding - o.kernel_size) / o.stride + 1;
        const int64_t ow = (o.width + 2 * o.padding - o.kernel_size) / o.stride + 1;
        out[0] = o.batch;
        out[1] = oh * ow;
        out[2] = o.out_channels;
        out[3] = o.in_channels * o.kernel_size * o.kernel_size;
    } else {
        out[0] = o.batch;
        out[1] = o.m;
        out[2] = o.n;
        out[3] = o.k;
    }
}

namespace {

uint64_t fnv_word(uint64_t h, uint64_t v) {
    for (int b = 0; b < 8; ++b) {
        h ^= (v >> (8 * b)) & 0xffu;
        h *= 1099511628211ull;
    }
    return h;
}

int index_of(const std::vector<int64_t>& sorted, int64_t v) {
    auto it = std::lower_bound(sorted.begin(), sorted.end(), v);
    return int(it - sorted.begin());
}

double lg(int64_t v) { return std::log1p(static_cast<double>(v)); }

template <typename T>
uint32_t put(std::vector<uint8_t>& blob, const T* data, size_t count) {
    const uint32_t off = align16(blob.size());
    blob.resize(off + sizeof(T) * count);
    if (count) std::memcpy(blob.data() + off, data, sizeof(T) * count);
    return off;
}

}  // namespace

etune_status build_plan(const etune_op_spec& op, const etune_device_config& dev,
                        const etune_space_limits& limits, PlanBuild* P, std::string* err) {
    if (etune_status st = op_validate(op, err)) return st;
    if (dev.num_sms < 1) {
        *err = "num_sms must be >= 1";
        return ETUNE_ERR_VALIDATION;
    }
    P->op = op;
    P->limits = limits;
    P->num_sms = dev.num_sms;
    P->dev = dev;
    int64_t nest[4];
    op_nest(op, nest);
    const int64_t B = nest[0], M = nest[1], N = nest[2], K = nest[3];
    const __int128 work = (__int128)B * M * N * K;
    if (work * 4 >= ((__int128)1 << 62)) {
        *err = "operator too large: 2*B*M*N*K would overflow the reference's int64 counters";
        return ETUNE_ERR_UNSUPPORTED;
    }
    PlanHdr& H = P->hdr;
    std::memset(&H, 0, sizeof(H));
    H.B = B;
    H.M = M;
    H.N = N;
    H.K = K;
    const int64_t outputs = B * M * N;
    H.flops = 2 * outputs * K;
    H.glb_st = outputs;
    H.num_sms = dev.num_sms;
    H.block_cap = int32_t(std::min<int64_t>(limits.max_block_threads, 1024));
    uint64_t h = 14695981039346656037ull;
    const int64_t* ow = &op.kind;
    for (int i = 0; i < 12; ++i) h = fnv_word(h, static_cast<uint64_t>(ow[i]));
    H.fnv_prefix = h;
    H.f0 = lg(H.flops);
    H.f3 = lg(H.glb_st);

    const int64_t ext[3] = {B, M, N};
    for (int d = 0; d < 3; ++d) {
        P->div[d] = divisors_of(ext[d]);
        if (P->div[d].size() > 65535 || ext[d] > 0xffffffffll) {
            *err = "extent has too many divisors / too large for 32-bit tiling records";
            return ETUNE_ERR_UNSUPPORTED;
        }
        H.nd[d] = int32_t(P->div[d].size());
        auto& T = P->til[d];
        T.clear();
        for (int64_t b : P->div[d]) {  // enumerate_dim_tilings, space.cpp:69-78
            const int64_t rest = ext[d] / b;
            for (int64_t t : divisors_of(rest)) {
                TilingRec r{};
                r.blocks = uint32_t(b);
                r.threads = uint32_t(t);
                r.pt = uint32_t(rest / t);
                r.db = uint16_t(index_of(P->div[d], b));
                r.dpt = uint16_t(index_of(P->div[d], rest / t));
                r.dbt = uint16_t(index_of(P->div[d], rest));
                T.push_back(r);
            }
        }
        if (T.size() > kMaxTilings) {
            *err = "more than 65536 tilings of one extent";
            return ETUNE_ERR_UNSUPPORTED;
        }
        H.nt[d] = int32_t(T.size());
    }
    P->divk = divisors_of(K);
    if (P->divk.size() > kMaxKDivisors) {
        *err = "reduction extent has more than 1024 divisors";
        return ETUNE_ERR_UNSUPPORTED;
    }
    H.ndk = int32_t(P->divk.size());

    // grid values: products of one divisor per dim
    const size_t nkey = size_t(H.nd[0]) * H.nd[1] * H.nd[2];
    if (nkey > (1u << 20)) {
        *err = "grid table too large";
        return ETUNE_ERR_UNSUPPORTED;
    }
    {
        std::vector<int64_t> vals;
        vals.reserve(nkey);
        for (int64_t a : P->div[0])
            for (int64_t b : P->div[1])
                for (int64_t c : P->div[2]) vals.push_back(a * b * c);
        std::vector<int64_t> sorted = vals;
        std::sort(sorted.begin(), sorted.end());
        sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
        if (sorted.size() > 65535) {
            *err = "too many distinct grid sizes";
            return ETUNE_ERR_UNSUPPORTED;
        }
        P->grid_values = sorted;
        P->gridkey.resize(nkey);
        for (size_t i = 0; i < nkey; ++i) P->gridkey[i] = uint16_t(index_of(sorted, vals[i]));
        H.ngrid = int32_t(sorted.size());
        P->grid.resize(sorted.size());
        for (size_t i = 0; i < sorted.size(); ++i) {  // counters.cpp:43-47, features.cpp:39-42
            const int64_t g = sorted[i];
            const int64_t active = std::min<int64_t>(g, dev.num_sms);
            P->grid[i].lg_grid = lg(g);
            P->grid[i].lg_active = lg(active);
            P->grid[i].a = static_cast<double>(active) / dev.num_sms;
        }
    }
    const int nd1 = H.nd[1], nd2 = H.nd[2];
    P->int2.resize(size_t(nd1) * nd2);
    P->glb2.resize(size_t(nd1) * nd2);
    for (int i = 0; i < nd1; ++i) {
        for (int j = 0; j < nd2; ++j) {
            const int64_t a = P->div[1][i], b = P->div[2][j];
            const int64_t q = outputs / (a * b);
            const int64_t x = q * K * (a + b);  // int_ops (pt keyed) / glb_ld (bt keyed)
            P->int2[size_t(i) * nd2 + j] = lg(x);
            P->glb2[size_t(i) * nd2 + j].lg_glb_ld = lg(x);
            P->glb2[size_t(i) * nd2 + j].f15 =
                static_cast<double>(H.flops) / static_cast<double>(x + H.glb_st + 1);
        }
    }
    P->block.resize(1025);
    for (int b = 0; b <= 1024; ++b) {
        P->block[b].lg_block = lg(b);
        P->block[b].b = std::min(1.0, static_cast<double>(b) / 256.0);
    }
    P->ptn.resize(nd2);
    for (int j = 0; j < nd2; ++j) P->ptn[j] = lg(P->div[2][j]);
    P->steps.resize(P->divk.size());
    for (size_t k = 0; k < P->divk.size(); ++k) P->steps[k] = lg(K / P->divk[k]);
    for (int c = 0; c < 4; ++c) P->lvl[c] = lg(8 + c);

    // enumeration knob lists (space.cpp:96-102)
    P->unroll_opts.clear();
    for (int64_t v = 1; v <= std::max<int64_t>(1, limits.max_unroll); v *= 2) P->unroll_opts.push_back(v);
    P->vec_opts.clear();
    for (int64_t v = 1; v <= std::min<int64_t>(4, std::max<int64_t>(1, limits.max_vectorize)); v *= 2)
        P->vec_opts.push_back(v);
    if (P->unroll_opts.size() > 16) {
        *err = "max_unroll above 2^15";
        return ETUNE_ERR_UNSUPPORTED;
    }
    H.max_unroll_log2 = int32_t(P->unroll_opts.size()) - 1;
    H.max_vec_log2 = int32_t(P->vec_opts.size()) - 1;

    // space size (count_schedules, space.cpp:152-160): legal = block <= cap,
    // unroll | k_tile, vectorize | pt_n; factorises over (tilings) x (k, unroll) x (vec).
    {
        int64_t ku = 0;
        for (int64_t kt : P->divk)
            for (int64_t u : P->unroll_opts) ku += (kt % u == 0);
        std::vector<int64_t> nvec_of_t2(P->til[2].size());
        for (size_t i = 0; i < P->til[2].size(); ++i) {
            int64_t c = 0;
            for (int64_t v : P->vec_opts) c += (P->til[2][i].pt % v == 0);
            nvec_of_t2[i] = c;
        }
        // count pairs of (t0, t1) by thread product, then combine with t2
        std::map<int64_t, int64_t> th01;
        for (const auto& a : P->til[0])
            for (const auto& b : P->til[1]) {
                const int64_t t = int64_t(a.threads) * b.threads;
                if (t <= H.block_cap) th01[t] += 1;
            }
        int64_t total = 0;
        for (size_t i = 0; i < P->til[2].size(); ++i) {
            const int64_t t2 = P->til[2][i].threads;
            int64_t pairs = 0;
            for (const auto& kv : th01)
                if (kv.first * t2 <= H.block_cap) pairs += kv.second;
            total += pairs * nvec_of_t2[i];
        }
        P->space_size = total * ku;
    }

    // ---- blob
    std::vector<uint8_t>& blob = P->blob;
    blob.assign(align16(sizeof(PlanHdr)), 0);
    for (int d = 0; d < 3; ++d) H.off_til[d] = put(blob, P->til[d].data(), P->til[d].size());
    H.off_divk = put(blob, P->divk.data(), P->divk.size());
    for (int d = 0; d < 3; ++d) {  // repair fit tables (reproduce); the breed kernels stage [0, off_gridkey)
        std::vector<uint32_t> tv;
        for (const TilingRec& r : P->til[d]) tv.push_back(r.threads);
        std::sort(tv.begin(), tv.end());
        tv.erase(std::unique(tv.begin(), tv.end()), tv.end());
        std::vector<uint32_t> start(1, 0u);
        std::vector<uint16_t> list;
        for (uint32_t lim : tv) {
            for (size_t j = 0; j < P->til[d].size(); ++j)
                if (P->til[d][j].threads <= lim) list.push_back(uint16_t(j));
            start.push_back(uint32_t(list.size()));
        }
        std::vector<uint8_t> blk(sizeof(FitHeader) + 4 * tv.size() + 4 * start.size() + 2 * list.size());
        FitHeader fh{int32_t(tv.size()), 0};
        size_t o = 0;
        std::memcpy(blk.data() + o, &fh, sizeof(fh));
        o += sizeof(fh);
        std::memcpy(blk.data() + o, tv.data(), 4 * tv.size());
        o += 4 * tv.size();
        std::memcpy(blk.data() + o, start.data(), 4 * start.size());
        o += 4 * start.size();
        if (!list.empty()) std::memcpy(blk.data() + o, list.data(), 2 * list.size());
        H.off_fit[d] = put(blob, blk.data(), blk.size());
    }
    H.off_gridkey = put(blob, P->gridkey.data(), P->gridkey.size());
    H.off_grid = put(blob, P->grid.data(), P->grid.size());
    H.off_int2 = put(blob, P->int2.data(), P->int2.size());
    H.off_glb2 = put(blob, P->glb2.data(), P->glb2.size());
    H.off_block = put(blob, P->block.data(), P->block.size());
    H.off_ptn = put(blob, P->ptn.data(), P->ptn.size());
    H.off_steps = put(blob, P->steps.data(), P->steps.size());
    H.off_lvl = put(blob, P->lvl, 4);
    blob.resize(align16(blob.size()));
    H.total = uint32_t(blob.size());
    std::memcpy(blob.data(), &H, sizeof(H));
    return ETUNE_OK;
}

}  // namespace etune_b200
