// Forest compiler.
//
// The reference evaluates every tree by walking `f[feature] < threshold ? left : right`
// on FP64 features (energy_model.cpp:36-44).  For one operator each feature is a
// function of one small "channel key" of the candidate (etune_internal.hpp, Channel),
// whose value set is known exactly from the plan's tables.  So, per operator:
//   1. every key value of a channel is evaluated against every test of the forest on
//      that channel's features, with the exact doubles the reference would compare;
//      keys with identical outcome vectors form one class (u8);
//   2. per (tree, channel) a table class -> mask of the tree's leaves that remain
//      reachable (a node whose test goes right removes its left subtree's leaves);
//      tests whose outcome is the same for every attainable candidate (e.g. on the
//      constant features f0/f3) are folded into the tree's base mask;
//   3. on the device the exit leaf is the lowest set bit of the AND of the tree's
//      channel masks (QuickScorer's argument: the exit leaf survives every AND and
//      every leaf left of it lies in the left subtree of a node that went right).
// Leaf values are the reference's doubles, summed in tree order.
#include "forest.hpp"
#include "score_core.hpp"

#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
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

namespace {

// value of feature j for key `key` of its channel (only for j with a table-backed channel)
struct ChannelKeys {
    int nkeys[kNumChannels] = {0, 0, 0, 0, 0, 0, 0};
};

int channel_of(int j) {
    switch (j) {
    case 1: case 4: return kChInt;
    case 2: case 5: case 15: return kChGlb;
    case 11: case 14: return kChGrid;
    case 12: return kChBlk;
    case 13: return kChEff;
    case 6: case 7: case 10: return kChKuv;
    case 8: case 9: return kChLvp;
    default: return -1;  // f0, f3: constant over the operator
    }
}

}  // namespace

size_t debruijn_slot(int leaf, int mbits) {
    if (mbits == 32) return size_t((uint32_t(1u << leaf) * 0x077CB531u) >> 27);
    return size_t((uint64_t(1) << leaf) * 0x03f79d71b4ca8b09ull >> 58);
}

etune_status build_score_blob(const ForestHost& F, const PlanBuild& P, std::vector<uint8_t>* blob,
                              ScoreStats* stats, std::string* err, KeyedBuild* keyed, size_t max_table_bytes,
                              size_t max_full_bytes) {
    if (etune_status st = forest_validate(F, err)) return st;
    const PlanHdr& PH = P.hdr;
    const int nd1 = PH.nd[1], nd2 = PH.nd[2], ndk = PH.ndk;
    ScoreStats S;

    // ---- f13 (a(grid) * b(block)): the only feature computed on device; its class is
    // the number of effective f13 boundaries <= x (binary search in smem).
    std::vector<double> V13;
    for (const GridRec& g : P.grid)
        for (int b = 1; b <= 1024; ++b) V13.push_back(g.a * P.block[b].b);
    std::sort(V13.begin(), V13.end());
    V13.erase(std::unique(V13.begin(), V13.end()), V13.end());
    std::vector<double> f13b;  // boundaries V13[rho], rho in (0, |V13|)
    for (size_t i = 0; i < F.feature.size(); ++i) {
        if (F.feature[i] != 13) continue;
        const size_t rho = size_t(std::lower_bound(V13.begin(), V13.end(), F.threshold[i]) - V13.begin());
        if (rho > 0 && rho < V13.size()) f13b.push_back(V13[rho]);
    }
    std::sort(f13b.begin(), f13b.end());
    f13b.erase(std::unique(f13b.begin(), f13b.end()), f13b.end());

    // ---- feature value of (channel, key) for feature j
    const int nkeys[kNumChannels] = {nd1 * nd2, nd1 * nd2, PH.ngrid, 1025, int(f13b.size()) + 1, ndk * 64,
                                     4 * nd2};
    auto value = [&](int j, int key) -> double {
        switch (j) {
        case 1: case 4: return P.int2[size_t(key)];
        case 2: case 5: return P.glb2[size_t(key)].lg_glb_ld;
        case 15: return P.glb2[size_t(key)].f15;
        case 11: return P.grid[size_t(key)].lg_grid;
        case 14: return P.grid[size_t(key)].lg_active;
        case 12: return P.block[size_t(key)].lg_block;
        case 13: return key == 0 ? V13.front() : f13b[size_t(key - 1)];  // class representative
        case 10: return P.steps[size_t(key / 64)];
        case 7: return double(int64_t(1) << ((key / 4) % 16));
        case 6: return double(1 << (key % 4));
        case 8: return P.lvl[key / nd2];
        case 9: return P.ptn[size_t(key % nd2)];
        default: return 0.0;
        }
    };
    auto key_valid = [&](int c, int key) {  // kuv keys with v == 3 or k beyond K: unreachable
        if (c == kChKuv) return (key % 4) < 3;
        return true;
    };

    // ---- distinct tests per channel, then classes of keys by outcome signature
    std::vector<std::pair<int, double>> tests[kNumChannels];
    for (size_t i = 0; i < F.feature.size(); ++i) {
        const int j = F.feature[i];
        if (j < 0) continue;
        const int c = channel_of(j);
        if (c >= 0) tests[c].push_back({j, F.threshold[i]});
    }
    std::vector<std::vector<uint8_t>> cls(kNumChannels);
    std::vector<std::vector<int>> rep(kNumChannels);  // representative key per class
    for (int c = 0; c < kNumChannels; ++c) {
        auto& T = tests[c];
        std::sort(T.begin(), T.end());
        T.erase(std::unique(T.begin(), T.end()), T.end());
        std::map<std::vector<bool>, int> sig2cls;
        cls[c].assign(size_t(nkeys[c]), 0);
        for (int key = 0; key < nkeys[c]; ++key) {
            if (!key_valid(c, key)) continue;
            std::vector<bool> sig(T.size());
            for (size_t q = 0; q < T.size(); ++q) sig[q] = value(T[q].first, key) < T[q].second;
            auto it = sig2cls.find(sig);
            int id;
            if (it == sig2cls.end()) {
                id = int(sig2cls.size());
                sig2cls.emplace(std::move(sig), id);
                rep[c].push_back(key);
            } else {
                id = it->second;
            }
            if (id > 255) {
                *err = "more than 256 outcome classes on one feature channel for this operator";
                return ETUNE_ERR_UNSUPPORTED;
            }
            cls[c][size_t(key)] = uint8_t(id);
        }
        if (rep[c].empty()) rep[c].push_back(0);
    }

    // ---- per tree: leaves in order, left-subtree masks, per-channel LUTs
    const int64_t T = F.num_trees();
    if (T > kMaxParamTrees) {
        *err = "more than 1000 trees; not supported by this build";
        return ETUNE_ERR_UNSUPPORTED;
    }
    int max_leaves = 1;
    for (int64_t t = 0; t < T; ++t) {
        int nl = 0;
        for (int64_t i = F.offsets[t]; i < F.offsets[t + 1]; ++i) nl += F.feature[i] < 0;
        max_leaves = std::max(max_leaves, nl);
    }
    if (max_leaves > 64) {
        *err = "a tree has more than 64 leaves (max_depth > 6); not supported by this build";
        return ETUNE_ERR_UNSUPPORTED;
    }
    const int mbits = max_leaves <= 32 ? 32 : 64;
    const uint64_t full = mbits == 32 ? 0xffffffffull : ~0ull;

    std::vector<uint64_t> lut;  // mask words; word 0.. = shared all-ones table (256 entries)
    lut.assign(256, full);
    std::map<std::vector<uint64_t>, uint32_t> dedupe;
    std::vector<TreeRec> recs(static_cast<size_t>(T));
    std::vector<double> leaves;
    std::vector<std::vector<std::vector<uint64_t>>> tree_tl(static_cast<size_t>(T));  // pair mode input
    std::vector<uint32_t> tree_used(static_cast<size_t>(T), 0u);
    for (int64_t t = 0; t < T; ++t) {
        const int64_t b = F.offsets[t], e = F.offsets[t + 1];
        // in-order leaf numbering and left-subtree leaf masks (iterative DFS)
        std::vector<int> leaf_id(size_t(e - b), -1);
        std::vector<uint64_t> sub(size_t(e - b), 0);
        std::vector<double> lv;
        std::function<uint64_t(int64_t, int)> walk = [&](int64_t i, int guard) -> uint64_t {
            if (guard > 64) return 0;
            if (F.feature[b + i] < 0) {
                leaf_id[size_t(i)] = int(lv.size());
                lv.push_back(F.value[b + i]);
                return sub[size_t(i)] = uint64_t(1) << leaf_id[size_t(i)];
            }
            const uint64_t l = walk(F.left[b + i], guard + 1);
            const uint64_t r = walk(F.right[b + i], guard + 1);
            return sub[size_t(i)] = l | r;
        };
        walk(0, 0);
        uint64_t base = full;
        std::vector<std::vector<uint64_t>> tl(kNumChannels);
        std::vector<bool> used(kNumChannels, false);
        // visit reachable interior nodes
        std::vector<int64_t> stack = {0};
        while (!stack.empty()) {
            const int64_t i = stack.back();
            stack.pop_back();
            const int j = F.feature[b + i];
            if (j < 0) continue;
            S.internal_nodes_in++;
            const uint64_t lmask = sub[size_t(F.left[b + i])];
            const int c = channel_of(j);
            const double thr = F.threshold[b + i];
            if (c < 0) {  // constant feature
                const double x = (j == 0) ? PH.f0 : PH.f3;
                if (!(x < thr)) base &= ~lmask;
                S.tests_folded++;
            } else {
                // outcome per class (via representative key)
                bool all_left = true, all_right = true;
                std::vector<bool> right(rep[c].size());
                for (size_t k = 0; k < rep[c].size(); ++k) {
                    right[k] = !(value(j, rep[c][k]) < thr);
                    all_left &= !right[k];
                    all_right &= right[k];
                }
                if (all_left || all_right) {
                    S.tests_folded++;
                    if (all_right) base &= ~lmask;
                } else {
                    if (!used[c]) {
                        used[c] = true;
                        tl[c].assign(rep[c].size(), full);
                        S.channels_used |= 1 << c;
                    }
                    for (size_t k = 0; k < rep[c].size(); ++k)
                        if (right[k]) tl[c][k] &= ~lmask;
                }
            }
            stack.push_back(F.left[b + i]);
            stack.push_back(F.right[b + i]);
        }
        // fold the base mask into one channel table
        if (base != full) {
            int host = -1;
            for (int c = 0; c < kNumChannels; ++c)
                if (used[c]) {
                    host = c;
                    break;
                }
            if (host < 0) {  // nothing varies: private constant table on the smallest channel
                host = kChEff;
                for (int c = 0; c < kNumChannels; ++c)
                    if (rep[c].size() < rep[host].size()) host = c;
                used[host] = true;
                tl[host].assign(rep[host].size(), full);
            }
            for (auto& m : tl[host]) m &= base;
        }
        TreeRec& R = recs[size_t(t)];
        for (int c = 0; c < kNumChannels; ++c) {
            if (!used[c]) {
                R.lut[c] = 0;  // all-ones table
                continue;
            }
            auto it = dedupe.find(tl[c]);
            if (it != dedupe.end()) {
                R.lut[c] = it->second;
            } else {
                const uint32_t off = uint32_t(lut.size());
                lut.insert(lut.end(), tl[c].begin(), tl[c].end());
                dedupe.emplace(tl[c], off);
                R.lut[c] = off;
            }
            S.lut_entries += int64_t(tl[c].size());
        }
        uint32_t used_mask = 0;
        for (int c = 0; c < kNumChannels; ++c) used_mask |= uint32_t(used[c]) << c;
        tree_used[size_t(t)] = used_mask;
        tree_tl[size_t(t)] = tl;
        if (leaves.size() >= (1u << 24)) {
            *err = "forest has more than 2^24 leaves";
            return ETUNE_ERR_UNSUPPORTED;
        }
        R.meta = uint32_t(leaves.size()) | (used_mask << 24);
        // leaf l lives at its de Bruijn slot of (1 << l): the device turns the exit mask's
        // lowest set bit into the slot with AND/NEG/IMAD/SHF (no XU bit-scan)
        // and the block is split into the high words of all slots, then the low words:
        // 32-bit loads of distinct slots never share a bank (a 64-bit load of 32 slots spans
        // 256 B and conflicts), so each leaf value costs exactly two conflict-free wavefronts
        std::vector<uint32_t> words(size_t(2 * mbits), 0u);
        for (size_t l = 0; l < lv.size(); ++l) {
            uint64_t bits = 0;
            std::memcpy(&bits, &lv[l], 8);
            const size_t slot = debruijn_slot(int(l), mbits);
            words[slot] = uint32_t(bits >> 32);
            words[size_t(mbits) + slot] = uint32_t(bits);
        }
        std::vector<double> block(static_cast<size_t>(mbits));
        std::memcpy(block.data(), words.data(), words.size() * 4);
        leaves.insert(leaves.end(), block.begin(), block.end());
        S.total_leaves += int(lv.size());
        S.max_leaves = std::max(S.max_leaves, int(lv.size()));
    }

    // ---- pair mode (32-bit masks): trees 2p, 2p+1 share one record and 64-bit tables
    const bool paired = mbits == 32;
    std::vector<PairRec> precs;
    std::vector<uint64_t> plut;
    if (paired) {
        plut.assign(256, ~0ull);  // shared all-ones pair table
        std::map<std::vector<uint64_t>, uint32_t> pdedupe;
        const int64_t np = (T + 1) / 2;
        precs.resize(static_cast<size_t>(np));
        for (int64_t p = 0; p < np; ++p) {
            const size_t a = size_t(2 * p), b = size_t(2 * p + 1);
            const bool hasb = int64_t(b) < T;
            const uint32_t ua = tree_used[a], ub = hasb ? tree_used[b] : 0u;
            const uint32_t used = ua | ub;
            PairRec& PR = precs[size_t(p)];
            for (int c = 0; c < kNumChannels; ++c) {
                if (!((used >> c) & 1u)) {
                    PR.lut[c] = 0;
                    continue;
                }
                std::vector<uint64_t> tab(rep[c].size());
                for (size_t x = 0; x < tab.size(); ++x) {
                    const uint64_t ma = ((ua >> c) & 1u) ? tree_tl[a][size_t(c)][x] : 0xffffffffull;
                    const uint64_t mb = ((ub >> c) & 1u) ? tree_tl[b][size_t(c)][x] : 0xffffffffull;
                    tab[x] = (ma & 0xffffffffull) | (mb << 32);
                }
                auto it = pdedupe.find(tab);
                if (it != pdedupe.end()) {
                    PR.lut[c] = it->second;
                } else {
                    // a table that fits one 128-byte bank row is placed inside one, so a
                    // warp's loads of it are a single conflict-free wavefront
                    if (tab.size() <= 16 && (plut.size() % 16) + tab.size() > 16)
                        plut.resize((plut.size() + 15) / 16 * 16, ~0ull);
                    const uint32_t off = uint32_t(plut.size());
                    plut.insert(plut.end(), tab.begin(), tab.end());
                    pdedupe.emplace(tab, off);
                    PR.lut[c] = off;
                }
            }
            PR.meta_a = (recs[a].meta & 0xffffffu) | (used << 24);
            PR.meta_b = hasb ? ((recs[b].meta & 0xffffffu) | (1u << 31)) : 0u;
        }
    }

    // ---- blob
    ScoreHdr H{};
    H.K = PH.K;
    H.fnv_prefix = PH.fnv_prefix;
    H.base = F.base;
    H.lr = F.lr;
    H.ntrees = int32_t(T);
    H.mask_bits = mbits;
    for (int d = 0; d < 3; ++d) {
        H.nt[d] = PH.nt[d];
        H.nd[d] = PH.nd[d];
    }
    H.ndk = PH.ndk;
    H.ngrid = PH.ngrid;
    H.n13 = int32_t(f13b.size());
    H.npairs = 0;
    std::vector<double> grida(P.grid.size()), blockb(1025);
    for (size_t g = 0; g < P.grid.size(); ++g) grida[g] = P.grid[g].a;
    for (int b2 = 0; b2 <= 1024; ++b2) blockb[size_t(b2)] = P.block[size_t(b2)].b;

    blob->assign(align16(sizeof(ScoreHdr)), 0);
    for (int d = 0; d < 3; ++d) H.off_til[d] = put(*blob, P.til[d].data(), P.til[d].size());
    H.off_divk = put(*blob, P.divk.data(), P.divk.size());
    H.off_gridkey = put(*blob, P.gridkey.data(), P.gridkey.size());
    H.off_grida = put(*blob, grida.data(), grida.size());
    H.off_blockb = put(*blob, blockb.data(), blockb.size());
    H.off_f13 = put(*blob, f13b.data(), f13b.size());
    for (int c = 0; c < kNumChannels; ++c) H.off_cls[c] = put(*blob, cls[c].data(), cls[c].size());
    // tree records hold byte offsets from the blob start: reserve, then fill
    if (paired) {
        H.npairs = int32_t(precs.size());
        H.off_trees = put(*blob, precs.data(), precs.size());
        blob->resize((blob->size() + 127) & ~size_t(127));  // bank-row aligned (see the table placement)
        H.off_lut = put(*blob, plut.data(), plut.size());
    } else {
        H.off_trees = put(*blob, recs.data(), recs.size());
    }
    if (!paired) H.off_lut = put(*blob, lut.data(), lut.size());  // 64-bit masks
    H.off_leaves = put(*blob, leaves.data(), leaves.size());
    const uint32_t mbytes = uint32_t(mbits / 8);
    auto leaf_bytes = [&](uint32_t idx, uint32_t* out) {
        const uint32_t lb = H.off_leaves + idx * 8u;
        if (lb >= (1u << 24)) return false;
        *out = lb;
        return true;
    };
    if (paired) {
        for (PairRec& PR : precs) {
            const uint32_t used = PR.meta_a >> 24;
            for (int c = 0; c < kNumChannels; ++c) PR.lut[c] = H.off_lut + PR.lut[c] * 8u;
            uint32_t la = 0, lb = 0;
            if (!leaf_bytes(PR.meta_a & 0xffffffu, &la) || !leaf_bytes(PR.meta_b & 0xffffffu, &lb)) {
                *err = "compiled forest too large";
                return ETUNE_ERR_UNSUPPORTED;
            }
            PR.meta_a = la | (used << 24);
            PR.meta_b = (PR.meta_b >> 31) ? (lb | (1u << 31)) : 0u;
        }
        std::memcpy(blob->data() + H.off_trees, precs.data(), precs.size() * sizeof(PairRec));
    } else {
        for (TreeRec& R : recs) {
            const uint32_t used_mask = R.meta >> 24;
            for (int c = 0; c < kNumChannels; ++c) R.lut[c] = H.off_lut + R.lut[c] * mbytes;
            uint32_t lb = 0;
            if (!leaf_bytes(R.meta & 0xffffffu, &lb)) {
                *err = "compiled forest too large";
                return ETUNE_ERR_UNSUPPORTED;
            }
            R.meta = lb | (used_mask << 24);
        }
        std::memcpy(blob->data() + H.off_trees, recs.data(), recs.size() * sizeof(TreeRec));
    }
    blob->resize(align16(blob->size()));
    H.total = uint32_t(blob->size());
    std::memcpy(blob->data(), &H, sizeof(H));
    if (stats) *stats = S;

    // ---- keyed form: per tiling triple, each tree's AND of its non-Kuv channel masks,
    // as one byte per tree (the exit slot, or the index of the mask for Kuv trees)
    if (keyed) {
        keyed->ok = false;
        const int64_t nk = int64_t(PH.nt[0]) * PH.nt[1] * PH.nt[2];
        const int row_bytes = int((T + 15) / 16 * 16);
        if (mbits == 32 && T > 0 && T <= kKeyedMaxTrees && nk > 0 &&
            size_t(nk) * size_t(row_bytes) <= max_table_bytes) {
            keyed->nkeys = nk;
            int kb = 0;
            while ((int64_t(1) << kb) < nk) ++kb;
            keyed->key_bits = kb;
            keyed->table.assign(size_t(nk) * size_t(row_bytes), 0);
            std::vector<std::map<uint32_t, int>> mcode(static_cast<size_t>(T));
            std::vector<std::vector<uint32_t>> mlists(static_cast<size_t>(T));
            bool fits = true;
            const uint8_t* B = blob->data();  // the finished score blob: classes exactly as the device derives them
            for (int64_t t0 = 0; t0 < PH.nt[0] && fits; ++t0)
                for (int64_t t1 = 0; t1 < PH.nt[1] && fits; ++t1)
                    for (int64_t t2 = 0; t2 < PH.nt[2] && fits; ++t2) {
                        const CandClasses cc =
                            candidate_classes(B, H, genome_pack(uint32_t(t0), uint32_t(t1), uint32_t(t2), 0, 0, 0));
                        const int64_t key = (t0 * PH.nt[1] + t1) * PH.nt[2] + t2;
                        uint8_t* row = keyed->table.data() + size_t(key) * size_t(row_bytes);
                        for (int64_t t = 0; t < T; ++t) {
                            uint64_t m = full;
                            for (int c = 0; c < kNumChannels; ++c)
                                if (c != kChKuv && ((tree_used[size_t(t)] >> c) & 1u))
                                    m &= tree_tl[size_t(t)][size_t(c)][cc.c[c]];
                            const uint32_t m32 = uint32_t(m);
                            if ((tree_used[size_t(t)] >> kChKuv) & 1u) {
                                auto& mc = mcode[size_t(t)];
                                auto it = mc.find(m32);
                                int code;
                                if (it == mc.end()) {
                                    code = int(mc.size());
                                    if (code >= 256) {
                                        fits = false;
                                        break;
                                    }
                                    mc.emplace(m32, code);
                                    mlists[size_t(t)].push_back(m32);
                                } else {
                                    code = it->second;
                                }
                                row[t] = uint8_t(code);
                            } else {
                                // exit leaf = lowest set bit; unreachable keys (m == 0) never occur
                                row[t] = uint8_t(((m32 & (0u - m32)) * 0x077CB531u) >> 27);
                            }
                        }
                    }
            if (fits) {
                const int nkc = int(rep[kChKuv].size());
                std::vector<uint32_t> kuvtab(size_t(T) * size_t(nkc), 0xffffffffu);
                KeyedHdr K{};
                for (int64_t t = 0; t < T; ++t)
                    if ((tree_used[size_t(t)] >> kChKuv) & 1u) {
                        K.kuv_flags[t >> 5] |= 1u << (t & 31);
                        for (int x = 0; x < nkc; ++x)
                            kuvtab[size_t(t) * size_t(nkc) + size_t(x)] =
                                uint32_t(tree_tl[size_t(t)][kChKuv][size_t(x)]);
                    }
                K.K = PH.K;
                K.fnv_prefix = PH.fnv_prefix;
                K.base = F.base;
                K.lr = F.lr;
                K.ntrees = int32_t(T);
                K.row_bytes = row_bytes;
                K.nkc = nkc;
                for (int d = 0; d < 3; ++d) {
                    K.nt[d] = PH.nt[d];
                    K.nd[d] = PH.nd[d];
                }
                K.ndk = PH.ndk;
                std::vector<uint8_t>& kbl = keyed->blob;
                kbl.assign(align16(sizeof(KeyedHdr)), 0);
                // what the full form reads comes first (header, divisors of K, Kuv classes, leaf
                // blocks: the `full_bytes` prefix its kernel stages); tilings and the byte form's
                // mask lists follow
                K.off_divk = put(kbl, P.divk.data(), P.divk.size());
                K.off_clskuv = put(kbl, cls[kChKuv].data(), cls[kChKuv].size());
                K.off_leaves = put(kbl, leaves.data(), leaves.size());  // 32 doubles (256 B) per tree, tree order
                kbl.resize(align16(kbl.size()));
                K.full_bytes = uint32_t(kbl.size());
                for (int d = 0; d < 3; ++d) K.off_til[d] = put(kbl, P.til[d].data(), P.til[d].size());
                std::vector<uint32_t> mlist;
                std::vector<uint32_t> mstart(static_cast<size_t>(T), 0u);
                for (int64_t t = 0; t < T; ++t) {
                    mstart[size_t(t)] = uint32_t(mlist.size());
                    mlist.insert(mlist.end(), mlists[size_t(t)].begin(), mlists[size_t(t)].end());
                }
                if (mlist.empty()) mlist.push_back(0u);
                K.off_mlist = put(kbl, mlist.data(), mlist.size());
                for (int64_t t = 0; t < T; ++t) keyed->params.moff[t] = K.off_mlist + 4u * mstart[size_t(t)];
                K.off_kuvtab = put(kbl, kuvtab.data(), kuvtab.size());
                kbl.resize(align16(kbl.size()));
                K.total = uint32_t(kbl.size());
                std::memcpy(kbl.data(), &K, sizeof(K));
                for (int w = 0; w < 4; ++w) keyed->params.kuv_flags[w] = K.kuv_flags[w];
                keyed->params.off_kuvtab = K.off_kuvtab;
                for (int64_t t = 0; t < T; ++t) keyed->params.koff[t] = K.off_kuvtab + uint32_t(t) * uint32_t(nkc) * 4u;
                keyed->params.off_leaves = K.off_leaves;
                keyed->params.nkc = uint32_t(nkc);
                keyed->params.ntrees = uint32_t(T);
                keyed->params.kfull = 0;
                // full form: every (key, Kuv class) row holds exit slots only
                // 5-bit slots, 25 trees per 16-byte quad (slot j of a quad at bits [5j, 5j + 5)),
                // rows padded to whole 32-byte sectors (read with 256-bit loads)
                const int frow = int((T + 49) / 50 * 32);
                const size_t full_bytes = size_t(nk) * size_t(nkc) * size_t(frow);
                if (nkc > 0 && full_bytes <= max_full_bytes) {
                    std::vector<uint8_t> ft(full_bytes, 0);
                    for (int64_t key = 0; key < nk; ++key) {
                        const uint8_t* row = keyed->table.data() + size_t(key) * size_t(row_bytes);
                        for (int x = 0; x < nkc; ++x) {
                            uint32_t* fr =
                                reinterpret_cast<uint32_t*>(ft.data() + (size_t(key) * size_t(nkc) + size_t(x)) * size_t(frow));
                            for (int64_t t = 0; t < T; ++t) {
                                uint32_t slot = row[t];
                                if ((tree_used[size_t(t)] >> kChKuv) & 1u) {
                                    const uint32_t m = mlists[size_t(t)][row[t]] &
                                                       kuvtab[size_t(t) * size_t(nkc) + size_t(x)];
                                    slot = ((m & (0u - m)) * 0x077CB531u) >> 27;
                                }
                                const uint32_t q = uint32_t(t) / 25u, b = 5u * (uint32_t(t) % 25u), sh = b & 31u;
                                uint32_t* quad = fr + 4 * q;
                                quad[b >> 5] |= slot << sh;
                                if (sh > 27u) quad[(b >> 5) + 1] |= slot >> (32u - sh);
                            }
                        }
                    }
                    keyed->table.swap(ft);
                    keyed->params.kfull = 1;
                    for (int w = 0; w < 4; ++w) keyed->params.kuv_flags[w] = 0u;
                    K.row_bytes = frow;
                    std::memcpy(kbl.data(), &K, sizeof(K));
                }
                // candidate_id's FNV-1a state per key: operator prefix, then (blocks, threads,
                // pt) of the key's three tilings (space.cpp:12-45 word order), each word hashed as
                // 8 little-endian bytes
                keyed->khash.assign(size_t(nk), 0);
                for (int64_t key = 0; key < nk; ++key) {
                    const int64_t t2 = key % PH.nt[2], t1 = (key / PH.nt[2]) % PH.nt[1], t0 = key / (int64_t(PH.nt[2]) * PH.nt[1]);
                    const int64_t tt[3] = {t0, t1, t2};
                    uint64_t h = PH.fnv_prefix;
                    for (int d = 0; d < 3; ++d) {
                        const TilingRec& r = P.til[d][size_t(tt[d])];
                        for (uint32_t v : {r.blocks, r.threads, r.pt})
                            for (int b = 0; b < 8; ++b) {
                                h ^= (uint64_t(v) >> (8 * b)) & 0xffu;
                                h *= 1099511628211ull;
                            }
                    }
                    keyed->khash[size_t(key)] = h;
                }
                keyed->ok = true;
            }
        }
    }
    return ETUNE_OK;
}

}  // namespace etune_b200
