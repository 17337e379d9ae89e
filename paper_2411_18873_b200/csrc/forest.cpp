// Forest compiler.
//
// The reference evaluates every tree by walking `f[feature] < threshold ? left : right`
// on FP64 features (energy_model.cpp:36-44).  For one operator every feature takes
// values from a small known set V_j (the plan's tables), so a test only matters
// through rho = #{v in V_j : v < thr}: for attainable x, x < thr <=> idx_j(x) < rho.
//   * rho == 0 or rho == |V_j|  -> the test is constant for this op: folded away.
//   * otherwise the distinct rho of feature j become its "effective thresholds" R_j,
//     bin_j(x) = #{rho in R_j : rho <= idx_j(x)} (fits a byte when |R_j| <= 254),
//     and the test becomes  bin_j(x) < r  with r = 1 + position of rho in R_j.
// Tests that a path already decides (same feature, nested ranks) are folded too.
// What remains is emitted as a perfect binary tree per reference tree (shallow
// leaves padded with always-right dummy tests, leaf value replicated) so the device
// walk is branch-free with a uniform trip count.  Leaf values are the reference's
// doubles, summed on device in the reference's tree order (energy_model.cpp:247).
#include "forest.hpp"

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>

namespace etune_b200 {

namespace {

template <typename T>
uint32_t put(std::vector<uint8_t>& blob, const T* data, size_t count) {
    const uint32_t off = align16(blob.size());
    blob.resize(off + sizeof(T) * count);
    if (count) std::memcpy(blob.data() + off, data, sizeof(T) * count);
    return off;
}

struct CNode {
    bool leaf = true;
    double value = 0.0;
    int feat = 0;
    int rprime = 0;  // test word rank (bin+1 domain)
    std::unique_ptr<CNode> kid[2];
    int depth() const { return leaf ? 0 : 1 + std::max(kid[0]->depth(), kid[1]->depth()); }
};

void sort_unique(std::vector<double>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
}

}  // namespace

etune_status forest_validate(const ForestHost& F, std::string* err) {
    const int64_t T = F.num_trees();
    if (T < 0) {
        *err = "tree_offsets must have num_trees+1 entries";
        return ETUNE_ERR_INVALID_ARGUMENT;
    }
    const int64_t nn = int64_t(F.feature.size());
    for (int64_t t = 0; t < T; ++t) {
        const int64_t b = F.offsets[t], e = F.offsets[t + 1];
        if (b < 0 || e > nn || e <= b) {
            *err = "model contains an empty or out-of-range tree";  // energy_model.cpp:326-328
            return ETUNE_ERR_IO;
        }
        for (int64_t i = b; i < e; ++i) {
            const int f = F.feature[i];
            if (f < -1 || f >= 16) {
                *err = "tree node feature index outside [-1, 16)";
                return ETUNE_ERR_SCHEMA_MISMATCH;
            }
            if (f >= 0) {
                const int64_t sz = e - b;
                if (F.left[i] < 0 || F.left[i] >= sz || F.right[i] < 0 || F.right[i] >= sz) {
                    *err = "tree node child index out of range";
                    return ETUNE_ERR_IO;
                }
            }
        }
    }
    return ETUNE_OK;
}

etune_status build_predict_blob(const ForestHost& F, std::vector<uint8_t>* blob, std::string* err) {
    if (etune_status st = forest_validate(F, err)) return st;
    PredictHdr H{};
    H.ntrees = int32_t(F.num_trees());
    H.nnodes = int32_t(F.feature.size());
    H.base = F.base;
    H.lr = F.lr;
    std::vector<int32_t> roots(size_t(H.ntrees));
    std::vector<GNode> nodes(F.feature.size());
    for (int64_t t = 0; t < H.ntrees; ++t) {
        const int64_t b = F.offsets[t];
        roots[t] = int32_t(b);
        for (int64_t i = b; i < F.offsets[t + 1]; ++i) {
            GNode& g = nodes[i];
            g.thr = F.threshold[i];
            g.feature = F.feature[i];
            g.left = F.feature[i] >= 0 ? int32_t(b + F.left[i]) : -1;
            g.right = F.feature[i] >= 0 ? int32_t(b + F.right[i]) : -1;
            g.pad = 0;
            g.value = F.value[i];
        }
    }
    blob->assign(align16(sizeof(PredictHdr)), 0);
    H.off_roots = put(*blob, roots.data(), roots.size());
    H.off_nodes = put(*blob, nodes.data(), nodes.size());
    blob->resize(align16(blob->size()));
    H.total = uint32_t(blob->size());
    std::memcpy(blob->data(), &H, sizeof(H));
    return ETUNE_OK;
}

etune_status build_score_blob(const ForestHost& F, const PlanBuild& P, std::vector<uint8_t>* blob,
                              ScoreStats* stats, std::string* err) {
    if (etune_status st = forest_validate(F, err)) return st;
    const PlanHdr& PH = P.hdr;

    // ---- attainable value sets V_j (supersets are fine: they only refine bins)
    std::vector<double> V[16];
    V[0] = {PH.f0};
    V[3] = {PH.f3};
    for (double x : P.int2) {
        V[1].push_back(x);
        V[4].push_back(x);
    }
    for (const GlbRec& g : P.glb2) {
        V[2].push_back(g.lg_glb_ld);
        V[5].push_back(g.lg_glb_ld);
        V[15].push_back(g.f15);
    }
    V[6] = {1.0, 2.0, 4.0};
    for (int u = 0; u < 16; ++u) V[7].push_back(double(int64_t(1) << u));
    for (double x : P.lvl) V[8].push_back(x);
    for (double x : P.ptn) V[9].push_back(x);
    for (double x : P.steps) V[10].push_back(x);
    for (const GridRec& g : P.grid) {
        V[11].push_back(g.lg_grid);
        V[14].push_back(g.lg_active);
    }
    for (int b = 0; b <= 1024; ++b) V[12].push_back(P.block[b].lg_block);
    for (const GridRec& g : P.grid)
        for (int b = 1; b <= 1024; ++b) V[13].push_back(g.a * P.block[b].b);
    for (auto& v : V) sort_unique(v);

    auto rho_of = [&](int j, double thr) {
        return int(std::lower_bound(V[j].begin(), V[j].end(), thr) - V[j].begin());
    };
    // ---- effective thresholds R_j
    std::vector<int> R[16];
    for (size_t i = 0; i < F.feature.size(); ++i) {
        const int j = F.feature[i];
        if (j < 0) continue;
        const int rho = rho_of(j, F.threshold[i]);
        if (rho > 0 && rho < int(V[j].size())) R[j].push_back(rho);
    }
    for (auto& r : R) {
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        if (r.size() > 254) {
            *err = "a feature has more than 254 effective split points for this operator "
                   "(byte bins); not supported by this build";
            return ETUNE_ERR_UNSUPPORTED;
        }
    }
    auto bin_of = [&](int j, double x) -> uint8_t {  // 1 + #(R_j <= idx(x))
        const int ix = rho_of(j, x);
        return uint8_t(1 + (std::upper_bound(R[j].begin(), R[j].end(), ix) - R[j].begin()));
    };

    // ---- compile trees
    ScoreStats S;
    int lo[16], hi[16];
    for (int j = 0; j < 16; ++j) {
        lo[j] = 1;
        hi[j] = int(R[j].size()) + 1;
    }
    std::function<std::unique_ptr<CNode>(int64_t, int64_t, int)> compile =
        [&](int64_t base, int64_t i, int guard) -> std::unique_ptr<CNode> {
        if (guard > 64) return nullptr;  // cycle
        auto node = std::make_unique<CNode>();
        const int j = F.feature[base + i];
        if (j < 0) {
            node->value = F.value[base + i];
            return node;
        }
        S.internal_nodes_in++;
        const int rho = rho_of(j, F.threshold[base + i]);
        if (rho == 0) {  // x < thr never: right
            S.tests_folded++;
            return compile(base, F.right[base + i], guard + 1);
        }
        if (rho == int(V[j].size())) {  // always left
            S.tests_folded++;
            return compile(base, F.left[base + i], guard + 1);
        }
        const int pos = int(std::lower_bound(R[j].begin(), R[j].end(), rho) - R[j].begin());
        const int rp = pos + 2;  // go right iff b'_j >= rp
        if (lo[j] >= rp) {
            S.tests_folded++;
            return compile(base, F.right[base + i], guard + 1);
        }
        if (hi[j] < rp) {
            S.tests_folded++;
            return compile(base, F.left[base + i], guard + 1);
        }
        node->leaf = false;
        node->feat = j;
        node->rprime = rp;
        const int save_lo = lo[j], save_hi = hi[j];
        hi[j] = rp - 1;
        node->kid[0] = compile(base, F.left[base + i], guard + 1);
        hi[j] = save_hi;
        lo[j] = rp;
        node->kid[1] = compile(base, F.right[base + i], guard + 1);
        lo[j] = save_lo;
        if (!node->kid[0] || !node->kid[1]) return nullptr;
        return node;
    };

    const int64_t T = F.num_trees();
    std::vector<TreeMeta> meta(static_cast<size_t>(T));
    std::vector<uint32_t> nodes;
    std::vector<double> leaves;
    for (int64_t t = 0; t < T; ++t) {
        auto root = compile(F.offsets[t], 0, 0);
        if (!root) {
            *err = "tree contains a cycle";
            return ETUNE_ERR_IO;
        }
        const int D = root->depth();
        if (D > 12) {
            *err = "tree deeper than 12 after partial evaluation; not supported by this build";
            return ETUNE_ERR_UNSUPPORTED;
        }
        S.max_depth = std::max(S.max_depth, D);
        S.sum_depth += D;
        meta[t].node_base = int32_t(nodes.size());
        meta[t].leaf_base = int32_t(leaves.size());
        meta[t].depth = D;
        meta[t].pad = 0;
        const size_t ni = (size_t(1) << D) - 1;
        const size_t nl = size_t(1) << D;
        const size_t nb = nodes.size(), lb = leaves.size();
        nodes.resize(nb + ni, 0x01000000u);
        leaves.resize(lb + nl, 0.0);
        S.perfect_slots += int64_t(ni);
        std::function<void(const CNode*, size_t, int)> emit = [&](const CNode* c, size_t slot, int level) {
            if (level == D) {
                leaves[lb + (slot - ni)] = c->value;
                return;
            }
            if (c->leaf) {  // dummy always-right test; replicate the leaf below
                nodes[nb + slot] = 0x01000000u;
                emit(c, 2 * slot + 1, level + 1);
                emit(c, 2 * slot + 2, level + 1);
                return;
            }
            const uint32_t pair = uint32_t(c->feat) >> 3;
            const uint32_t q = uint32_t(c->feat) & 7u;
            nodes[nb + slot] = (uint32_t(c->rprime) << 24) | (pair << 16) | (q * 0x1111u);
            emit(c->kid[0].get(), 2 * slot + 1, level + 1);
            emit(c->kid[1].get(), 2 * slot + 2, level + 1);
        };
        emit(root.get(), 0, 0);
    }

    // ---- bin tables
    ScoreHdr H{};
    H.K = PH.K;
    H.fnv_prefix = PH.fnv_prefix;
    H.base = F.base;
    H.lr = F.lr;
    H.ntrees = int32_t(T);
    H.max_depth = S.max_depth;
    for (int d = 0; d < 3; ++d) {
        H.nt[d] = PH.nt[d];
        H.nd[d] = PH.nd[d];
    }
    H.ndk = PH.ndk;
    H.ngrid = PH.ngrid;
    for (int j = 0; j < 16; ++j) H.bconst[j] = 1;
    H.bconst[0] = bin_of(0, PH.f0);
    H.bconst[3] = bin_of(3, PH.f3);

    std::vector<uint16_t> bgrid(P.grid.size());
    std::vector<double> grida(P.grid.size());
    for (size_t g = 0; g < P.grid.size(); ++g) {
        bgrid[g] = uint16_t(bin_of(11, P.grid[g].lg_grid) | (bin_of(14, P.grid[g].lg_active) << 8));
        grida[g] = P.grid[g].a;
    }
    std::vector<uint16_t> bint2(P.int2.size());
    for (size_t i = 0; i < P.int2.size(); ++i)
        bint2[i] = uint16_t(bin_of(1, P.int2[i]) | (bin_of(4, P.int2[i]) << 8));
    std::vector<uint32_t> bglb2(P.glb2.size());
    for (size_t i = 0; i < P.glb2.size(); ++i)
        bglb2[i] = uint32_t(bin_of(2, P.glb2[i].lg_glb_ld)) | (uint32_t(bin_of(5, P.glb2[i].lg_glb_ld)) << 8) |
                   (uint32_t(bin_of(15, P.glb2[i].f15)) << 16);
    std::vector<uint8_t> bblock(1025 + 15, 1);
    std::vector<double> blockb(1025);
    for (int b = 0; b <= 1024; ++b) {
        bblock[b] = bin_of(12, P.block[b].lg_block);
        blockb[b] = P.block[b].b;
    }
    std::vector<uint8_t> bptn(P.ptn.size());
    for (size_t i = 0; i < P.ptn.size(); ++i) bptn[i] = bin_of(9, P.ptn[i]);
    std::vector<uint8_t> bsteps(P.steps.size());
    for (size_t i = 0; i < P.steps.size(); ++i) bsteps[i] = bin_of(10, P.steps[i]);
    uint8_t small[32];
    std::memset(small, 1, sizeof(small));
    for (int c = 0; c < 4; ++c) small[c] = bin_of(8, P.lvl[c]);
    for (int u = 0; u < 16; ++u) small[4 + u] = bin_of(7, double(int64_t(1) << u));
    for (int v = 0; v < 3; ++v) small[20 + v] = bin_of(6, double(1 << v));
    std::vector<double> f13;
    for (int rho : R[13]) f13.push_back(V[13][size_t(rho)]);
    H.n13 = int32_t(f13.size());

    blob->assign(align16(sizeof(ScoreHdr)), 0);
    for (int d = 0; d < 3; ++d) H.off_til[d] = put(*blob, P.til[d].data(), P.til[d].size());
    H.off_divk = put(*blob, P.divk.data(), P.divk.size());
    H.off_gridkey = put(*blob, P.gridkey.data(), P.gridkey.size());
    H.off_bgrid = put(*blob, bgrid.data(), bgrid.size());
    H.off_grida = put(*blob, grida.data(), grida.size());
    H.off_bint2 = put(*blob, bint2.data(), bint2.size());
    H.off_bglb2 = put(*blob, bglb2.data(), bglb2.size());
    H.off_bblock = put(*blob, bblock.data(), bblock.size());
    H.off_blockb = put(*blob, blockb.data(), blockb.size());
    H.off_bptn = put(*blob, bptn.data(), bptn.size());
    H.off_bsteps = put(*blob, bsteps.data(), bsteps.size());
    H.off_small = put(*blob, small, 32);
    H.off_f13 = put(*blob, f13.data(), f13.size());
    H.off_meta = put(*blob, meta.data(), meta.size());
    H.off_nodes = put(*blob, nodes.data(), nodes.size());
    H.off_leaves = put(*blob, leaves.data(), leaves.size());
    blob->resize(align16(blob->size()));
    H.total = uint32_t(blob->size());
    std::memcpy(blob->data(), &H, sizeof(H));
    if (stats) *stats = S;
    return ETUNE_OK;
}

}  // namespace etune_b200
