// TEST INFRASTRUCTURE: runs the forest compiler (forest.cpp) and the device scoring
// core (score_core.hpp, compiled here for the host) on the CPU, so the compiled
// class/leaf-mask tables can be checked against the oracle without a GPU.
// Never linked into libetune_cuda.so.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "forest.hpp"
#include "plan.hpp"
#include "score_core.hpp"

using namespace etune_b200;

static thread_local std::string g_err;

extern "C" const char* scc_last_error() { return g_err.c_str(); }

// returns 0 ok; stats_out[8] like etune_cu_forest_compile_stats.  keyed: score through the
// keyed form (KeyedHdr + key table, score_core.hpp keyed_sum) instead of the class tables.
static int score_impl(const int64_t* op_words, int num_sms, const int32_t* feature, const double* threshold,
                      const int32_t* left, const int32_t* right, const double* value, const int64_t* offsets,
                      int64_t num_trees, double base, double lr, const int64_t* sched, int64_t n, double* out,
                      int64_t* stats_out, int keyed) {
    etune_op_spec op;
    std::memcpy(&op, op_words, sizeof(op));
    etune_device_config d{};
    d.num_sms = num_sms;
    etune_space_limits l{1024, 8, 4};
    PlanBuild P;
    if (int st = build_plan(op, d, l, &P, &g_err)) return st;
    ForestHost F;
    const int64_t nn = offsets[num_trees];
    F.feature.assign(feature, feature + nn);
    F.threshold.assign(threshold, threshold + nn);
    F.left.assign(left, left + nn);
    F.right.assign(right, right + nn);
    F.value.assign(value, value + nn);
    F.offsets.assign(offsets, offsets + num_trees + 1);
    F.base = base;
    F.lr = lr;
    std::vector<uint8_t> blob;
    ScoreStats S;
    KeyedBuild KBd;
    if (int st = build_score_blob(F, P, &blob, &S, &g_err, keyed ? &KBd : nullptr, size_t(64) << 20,
                                  keyed == 2 ? 0 : size_t(64) << 20))
        return st;
    if (keyed && !KBd.ok) {
        g_err = "keyed form unavailable";
        return ETUNE_ERR_UNSUPPORTED;
    }
    struct alignas(16) KChunk { unsigned char b[16]; };
    std::vector<KChunk> kal(keyed ? (KBd.blob.size() + 15) / 16 : 0);
    if (keyed) std::memcpy(kal.data(), KBd.blob.data(), KBd.blob.size());
    const uint8_t* KB = keyed ? reinterpret_cast<const uint8_t*>(kal.data()) : nullptr;
    // 16-byte aligned copy, like the kernel's smem stage
    struct alignas(16) Chunk { unsigned char b[16]; };
    std::vector<Chunk> aligned((blob.size() + 15) / 16);
    std::memcpy(aligned.data(), blob.data(), blob.size());
    const uint8_t* B = reinterpret_cast<const uint8_t*>(aligned.data());
    const ScoreHdr& H = *reinterpret_cast<const ScoreHdr*>(B);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t* s = sched + 12 * i;
        uint32_t ti[3];
        for (int dd = 0; dd < 3; ++dd) {
            const auto& T = P.til[dd];
            auto it = std::find_if(T.begin(), T.end(), [&](const TilingRec& r) {
                return int64_t(r.blocks) == s[3 * dd] && int64_t(r.threads) == s[3 * dd + 1];
            });
            if (it == T.end()) {
                g_err = "tiling not found";
                return 4;
            }
            ti[dd] = uint32_t(it - T.begin());
        }
        const uint32_t k = uint32_t(std::lower_bound(P.divk.begin(), P.divk.end(), s[9]) - P.divk.begin());
        const uint32_t u = uint32_t(__builtin_ctzll(uint64_t(s[10])));
        const uint32_t v = uint32_t(__builtin_ctzll(uint64_t(s[11])));
        const uint64_t gnm = genome_pack(ti[0], ti[1], ti[2], k, u, v);
        if (keyed) {
            const KeyedHdr& KH = *reinterpret_cast<const KeyedHdr*>(KB);
            const Genome x = genome_unpack(gnm);
            const uint32_t kc = KB[KH.off_clskuv + (x.k * 16u + x.u) * 4u + x.v];
            const uint8_t* row = KBd.table.data() + size_t(keyed_row_index(KBd.params, KH, x, kc)) * size_t(KH.row_bytes);
            out[i] = keyed_finish(KH, KBd.params.kfull ? keyed_sum5(KB, KBd.params, row)
                                                       : keyed_sum(KB, KBd.params, row, kc));
            continue;
        }
        const CandClasses cc = candidate_classes(B, H, gnm);
        const TreeRec* trees = blob_at<TreeRec>(B, H.off_trees);
        const double sum = H.npairs > 0 ? forest_sum_pairs(B, H, blob_at<PairRec>(B, H.off_trees), cc.c)
                           : H.mask_bits == 32 ? forest_sum<uint32_t>(B, H, trees, cc.c)
                                               : forest_sum<uint64_t>(B, H, trees, cc.c);
        out[i] = finish_prediction(H, sum);
    }
    if (stats_out) {
        stats_out[0] = S.internal_nodes_in;
        stats_out[1] = S.tests_folded;
        stats_out[2] = S.lut_entries;
        stats_out[3] = S.max_leaves;
        stats_out[4] = S.total_leaves;
        stats_out[5] = int64_t(blob.size());
        stats_out[6] = S.channels_used;
        stats_out[7] = num_trees;
    }
    return 0;
}

extern "C" int scc_score(const int64_t* op_words, int num_sms, const int32_t* feature, const double* threshold,
                         const int32_t* left, const int32_t* right, const double* value, const int64_t* offsets,
                         int64_t num_trees, double base, double lr, const int64_t* sched, int64_t n, double* out,
                         int64_t* stats_out) {
    return score_impl(op_words, num_sms, feature, threshold, left, right, value, offsets, num_trees, base, lr, sched,
                      n, out, stats_out, 0);
}

extern "C" int scc_score_keyed8(const int64_t* op_words, int num_sms, const int32_t* feature, const double* threshold,
                                const int32_t* left, const int32_t* right, const double* value,
                                const int64_t* offsets, int64_t num_trees, double base, double lr,
                                const int64_t* sched, int64_t n, double* out, int64_t* stats_out) {
    return score_impl(op_words, num_sms, feature, threshold, left, right, value, offsets, num_trees, base, lr, sched,
                      n, out, stats_out, 2);
}

extern "C" int scc_score_keyed(const int64_t* op_words, int num_sms, const int32_t* feature, const double* threshold,
                               const int32_t* left, const int32_t* right, const double* value,
                               const int64_t* offsets, int64_t num_trees, double base, double lr,
                               const int64_t* sched, int64_t n, double* out, int64_t* stats_out) {
    return score_impl(op_words, num_sms, feature, threshold, left, right, value, offsets, num_trees, base, lr, sched,
                      n, out, stats_out, 1);
}
