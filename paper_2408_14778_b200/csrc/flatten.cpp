// Host-side game validation + flattening (one O(V) pass family
// "a single complete game tree traversal"), then the B200 slot/tile layout.
//
//   1. Validate Def. 2.1: one root, parents in range, acyclic/connected,
//      action bijection 0..n-1 per decision node, infoset ids dense with one
//      owner and one |A(h)| per infoset, chance probabilities in [0,1] summing to
//      1 +- 1e-12, finite utilities, <= 2^23 nodes per infoset.
//   2. Canonical BFS order: node 0 is the root; depth-(d+1)
//      nodes are ordered by (canonical parent, incoming action).  The level graphs
//      L^(l) of P:176-178 become contiguous ranges level_ptr[l]..level_ptr[l+1]
//      and every decision node's children are contiguous (the CSR rows of G,
//      P:172-174, with implicit column indices).
//   3. Slots: decision nodes level by level, grouped by infoset in order of first
//      occurrence, so one backward tile owns whole infosets and the
//      per-infoset sums of Eq 3/5/7 finish inside one CTA.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "game.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace cfrb {

namespace {

bool fail(std::string& err, const std::string& m) {
    err = m;
    return false;
}

// E = 1 + ceil(log2(2*m)) = 2 + ceil(log2 m) for m > 0, else 1,
// evaluated on m itself: 2*m overflows for m > DBL_MAX / 2.  ilogb-based.
int exponent_for(double m) {
    if (!(m > 0.0)) return 1;
    int k = std::ilogb(m);                 // floor(log2 m) for normal m
    if (std::ldexp(1.0, k) < m) k += 1;    // ceil
    return 2 + k;
}

}  // namespace

namespace {
struct PhaseTimer {
    bool on = std::getenv("CFR_FLATTEN_VERBOSE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[flatten] %-12s %8.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
        t0 = t1;
    }
};
}  // namespace

// Tiles of each parent level: groups = maximal runs of equal infoset within the
// level's slots; a tile packs whole groups under the slot / pair / segment /
// staged-children limits; an oversized group is split (and its infoset deferred).
void build_tiles(Game& g, const std::vector<int64_t>& slot_h) {
    const int D = g.D;
    const int Pc = g.Pc;
    const int64_t H = g.H;
    // Groups = maximal runs of equal infoset within a level's slots.  Tiles pack
    // whole groups under the slot / pair / segment / staged-children limits.
    g.tile_ptr.assign(D + 1, 0);
    g.tiles.clear();
    g.segs.clear();
    // packing bound: >= the generic odd-stride row and the solver's chunked row
    auto row_elems = [&](int64_t s) -> int64_t { return (int64_t)g.s_n[s] * Pc + 2; };
    auto finish_tile = [&](TileH& t) {
        // generic staged layout: one row per slot, odd strides (conflict-free
        // per-thread row reads); the solver may re-lay uniform tiles in chunks
        int64_t off = 0;
        for (int64_t s = t.s0; s < t.s1; ++s) {
            g.s_coff[s] = (int32_t)std::min<int64_t>(off, INT32_MAX);
            off += ((int64_t)g.s_n[s] * Pc) | 1;
        }
        t.nch = (int32_t)std::min<int64_t>(off, INT32_MAX);
        t.staged = off <= kTileChildren ? 1 : 0;
        t.run0 = t.run1 = 0;
        t.seg1 = (int32_t)g.segs.size();
        g.tiles.push_back(t);
    };
    for (int L = 0; L < D; ++L) {
        g.tile_ptr[L] = (int64_t)g.tiles.size();
        const int64_t lo = g.slot_ptr[L], hi = g.slot_ptr[L + 1];
        TileH cur{lo, lo, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0, 0, 0, 0, 0};
        int64_t cur_ch = 0;
        auto close = [&]() {
            if (cur.s1 > cur.s0) finish_tile(cur);
            cur = TileH{cur.s1, cur.s1, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0, 0, 0, 0, 0};
            cur_ch = 0;
        };
        int64_t s = lo;
        while (s < hi) {
            int64_t e = s + 1;
            const int64_t h = slot_h[s];
            if (h >= 0)
                while (e < hi && slot_h[e] == h) ++e;
            const int64_t m = e - s;
            const int32_t n = (h >= 0) ? (int32_t)(g.qbase_int[h + 1] - g.qbase_int[h]) : 0;
            int64_t gch = 0;
            for (int64_t x = s; x < e; ++x) gch += row_elems(x);
            if (m > kTileSlots || n > kTilePairs) {
                // split group: its own chunks, accumulated globally (deferred)
                close();
                g.deferred[h] = 1;
                for (int64_t c0 = s; c0 < e; c0 += kTileSlots) {
                    const int64_t c1 = std::min(e, c0 + kTileSlots);
                    TileH t{c0, c1, (int32_t)g.segs.size(), 0, n, 0, 0, 0, 0, 0};
                    g.segs.push_back(SegH{h, c0, c1, 0, 0});
                    finish_tile(t);
                }
                cur = TileH{e, e, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0, 0, 0, 0, 0};
                cur_ch = 0;
                s = e;
                continue;
            }
            const int64_t segs_in = (int64_t)g.segs.size() - cur.seg0;
            if ((cur.s1 - cur.s0) + m > kTileSlots || cur.npairs + n > kTilePairs ||
                (h >= 0 && segs_in + 1 > kTileSegs) || (cur.s1 > cur.s0 && cur_ch + gch > kTileChildren))
                close();
            if (h >= 0) {
                g.segs.push_back(SegH{h, s, e, cur.npairs, g.deferred[h] ? 0 : 1});
                cur.npairs += n;
            }
            cur.s1 = e;
            cur_ch += gch;
            s = e;
        }
        close();
    }
    g.tile_ptr[D] = (int64_t)g.tiles.size();
    for (auto& sg : g.segs)
        if (g.deferred[sg.h]) sg.fused = 0;
    g.deferred_list.clear();
    g.dpos.assign(H, -1);
    g.dqbase.assign(1, 0);
    for (int64_t h = 0; h < H; ++h)
        if (g.deferred[h]) {
            g.dpos[h] = (int64_t)g.deferred_list.size();
            g.deferred_list.push_back(h);
            g.dqbase.push_back(g.dqbase.back() + (g.qbase_int[h + 1] - g.qbase_int[h]));
        }

}

bool build_game(const cfr_game_desc* d, Game& g, std::string& err) {
    PhaseTimer tm;
    const int64_t V = d->num_nodes;
    const int P = d->num_players;
    if (V < 1) return fail(err, "num_nodes must be >= 1");
    if (P < 1 || P > 16) return fail(err, "num_players must be in [1, 16]");
    if (!d->parent || !d->player || !d->infoset || !d->action || !d->chance_prob || !d->utility)
        return fail(err, "NULL array in cfr_game_desc");
    g.V = V;
    g.P = P;

    // ---------------------------------------------------------------- children
    // Parallel passes record the smallest offending node per error class, so the
    // message is deterministic; the slow sequential path is never needed.
    const int64_t NONE = INT64_MAX;
    int64_t e_parent = NONE, e_self = NONE, e_player = NONE, n_roots = 0, root = NONE;
    std::vector<int64_t> cstart(V + 1, 0);
#pragma omp parallel for schedule(static) reduction(min : e_parent, e_self, e_player, root) reduction(+ : n_roots)
    for (int64_t v = 0; v < V; ++v) {
        const int64_t p = d->parent[v];
        if (p < 0) {
            if (p != -1) e_parent = std::min(e_parent, v);
            else { ++n_roots; root = std::min(root, v); }
        } else if (p >= V) {
            e_parent = std::min(e_parent, v);
        } else if (p == v) {
            e_self = std::min(e_self, v);
        } else {
            __atomic_fetch_add(&cstart[p + 1], (int64_t)1, __ATOMIC_RELAXED);
        }
        const int32_t pl = d->player[v];
        if (pl < -1 || pl > P) e_player = std::min(e_player, v);
    }
    if (e_parent != NONE) return fail(err, "node " + std::to_string(e_parent) + ": parent must be -1 or a node id < V");
    if (e_self != NONE) return fail(err, "node " + std::to_string(e_self) + " is its own parent");
    if (e_player != NONE) return fail(err, "node " + std::to_string(e_player) + ": player out of range");
    if (n_roots == 0) return fail(err, "no root (parent == -1)");
    if (n_roots > 1) {
        int64_t r2 = NONE;
        for (int64_t v = root + 1; v < V && r2 == NONE; ++v)
            if (d->parent[v] == -1) r2 = v;
        return fail(err, "two roots: nodes " + std::to_string(root) + " and " + std::to_string(r2));
    }
    for (int64_t v = 0; v < V; ++v) cstart[v + 1] += cstart[v];
    std::vector<int64_t> clist(V > 1 ? V - 1 : 1, -1);
    int64_t e_action = NONE;
#pragma omp parallel for schedule(static) reduction(min : e_action)
    for (int64_t v = 0; v < V; ++v) {
        const int64_t p = d->parent[v];
        if (p < 0) continue;
        const int64_t n = cstart[p + 1] - cstart[p];
        const int32_t a = d->action[v];
        if (a < 0 || a >= n) e_action = std::min(e_action, v);
        else clist[cstart[p] + a] = v;
    }
    if (e_action != NONE) {
        const int64_t v = e_action, p = d->parent[v];
        return fail(err, "node " + std::to_string(v) + ": action " + std::to_string(d->action[v]) + " not in 0.." +
                             std::to_string(cstart[p + 1] - cstart[p] - 1) + " (action bijection, P:33)");
    }
    int64_t e_dup = NONE, e_term = NONE, e_dec = NONE, e_util = NONE;
    double max_u = 0.0;
#pragma omp parallel for schedule(static) reduction(min : e_dup, e_term, e_dec, e_util) reduction(max : max_u)
    for (int64_t v = 0; v < V; ++v) {
        const int64_t p = d->parent[v];
        if (p >= 0 && clist[cstart[p] + d->action[v]] != v) e_dup = std::min(e_dup, v);   // lost a race: duplicate
        const int64_t n = cstart[v + 1] - cstart[v];
        const int32_t pl = d->player[v];
        if (pl < 0 && n != 0) e_term = std::min(e_term, v);
        if (pl >= 0 && n == 0) e_dec = std::min(e_dec, v);
        if (pl < 0) {
            for (int j = 0; j < P; ++j) {
                const double u = d->utility[v * P + j];
                if (!std::isfinite(u)) e_util = std::min(e_util, v);
                else max_u = std::max(max_u, std::fabs(u));
            }
        }
    }
    if (e_dup != NONE)
        return fail(err, "node " + std::to_string(e_dup) + ": duplicate action " + std::to_string(d->action[e_dup]) +
                             " under parent " + std::to_string(d->parent[e_dup]));
    if (e_term != NONE) return fail(err, "terminal node " + std::to_string(e_term) + " has children");
    if (e_dec != NONE) return fail(err, "decision node " + std::to_string(e_dec) + " has no children");
    if (e_util != NONE) return fail(err, "terminal node " + std::to_string(e_util) + ": non-finite utility");
    g.max_abs_u = max_u;

    tm.mark("children");
    // ------------------------------------------------------- canonical BFS order
    // Level by level: children counts -> prefix sum -> parallel copy.
    std::vector<int64_t> order(V);
    std::vector<int64_t> canon_cb(V, -1);
    std::vector<int32_t> ncanon(V, 0);
    order[0] = root;
    g.level_ptr.assign(1, 0);
    g.level_ptr.push_back(1);
    {
        int64_t lo = 0, hi = 1;
        while (true) {
#pragma omp parallel for schedule(static)
            for (int64_t k = lo; k < hi; ++k) {
                const int64_t v = order[k];
                ncanon[k] = (int32_t)(cstart[v + 1] - cstart[v]);
            }
            int64_t tail = hi;
            for (int64_t k = lo; k < hi; ++k) {
                if (ncanon[k] > 0) {
                    canon_cb[k] = tail;
                    tail += ncanon[k];
                    if (tail > V) return fail(err, "tree has a cycle");
                }
            }
            if (tail == hi) break;
#pragma omp parallel for schedule(dynamic, 4096)
            for (int64_t k = lo; k < hi; ++k) {
                const int64_t v = order[k];
                const int64_t n = ncanon[k];
                for (int64_t a = 0; a < n; ++a) order[canon_cb[k] + a] = clist[cstart[v] + a];
            }
            lo = hi;
            hi = tail;
            g.level_ptr.push_back(hi);
        }
        if (hi != V)
            return fail(err, "tree is not connected: " + std::to_string(V - hi) +
                                 " node(s) unreachable from the root (cycle?)");
    }
    g.D = (int32_t)g.level_ptr.size() - 2;
    std::vector<int64_t>().swap(clist);
    std::vector<int64_t>().swap(cstart);
    g.canon_of_input.assign(V, 0);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < V; ++k) g.canon_of_input[order[k]] = k;

    tm.mark("bfs");
    // ------------------------------------------------------------ infoset checks
    int64_t H = 0, e_noinf = NONE, n_term = 0, n_chance = 0;
#pragma omp parallel for schedule(static) reduction(max : H) reduction(min : e_noinf) reduction(+ : n_term, n_chance)
    for (int64_t v = 0; v < V; ++v) {
        const int32_t pl = d->player[v];
        if (pl < 0) ++n_term;
        else if (pl == 0) ++n_chance;
        else {
            const int64_t h = d->infoset[v];
            if (h < 0) e_noinf = std::min(e_noinf, v);
            else H = std::max(H, h + 1);
        }
    }
    if (e_noinf != NONE) return fail(err, "player node " + std::to_string(e_noinf) + " has no infoset id");
    g.H = H;
    g.num_terminals = n_term;
    g.num_chance = n_chance;
    g.num_decision = V - n_term;
    std::vector<int32_t> nact(H, -1);
    std::vector<uint8_t> own(H, 0);
    std::vector<int64_t> members(H, 0);
    // any member's (|A|, owner) is written; a second pass checks all agree
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        const int32_t pl = d->player[v];
        if (pl < 1) continue;
        const int64_t h = d->infoset[v];
        __atomic_store_n(&nact[h], ncanon[k], __ATOMIC_RELAXED);
        __atomic_store_n(&own[h], (uint8_t)pl, __ATOMIC_RELAXED);
        __atomic_fetch_add(&members[h], (int64_t)1, __ATOMIC_RELAXED);
    }
    int64_t e_nact = NONE, e_own = NONE;
#pragma omp parallel for schedule(static) reduction(min : e_nact, e_own)
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        const int32_t pl = d->player[v];
        if (pl < 1) continue;
        const int64_t h = d->infoset[v];
        if (nact[h] != ncanon[k]) e_nact = std::min(e_nact, v);
        if (own[h] != pl) e_own = std::min(e_own, v);
    }
    if (e_nact != NONE)
        return fail(err, "infoset " + std::to_string(d->infoset[e_nact]) + ": nodes have different action counts (node " +
                             std::to_string(e_nact) + ")");
    if (e_own != NONE)
        return fail(err, "infoset " + std::to_string(d->infoset[e_own]) + ": nodes of different players (node " +
                             std::to_string(e_own) + ")");
    for (int64_t h = 0; h < H; ++h) {
        if (nact[h] < 0) return fail(err, "infoset ids are not dense: id " + std::to_string(h) + " unused");
        if (members[h] > (int64_t(1) << 23))
            return fail(err, "infoset " + std::to_string(h) + " has more than 2^23 nodes (exact-sum headroom)");
        g.max_infoset_nodes = std::max(g.max_infoset_nodes, members[h]);
    }
    g.qbase_caller.assign(H + 1, 0);
    for (int64_t h = 0; h < H; ++h) g.qbase_caller[h + 1] = g.qbase_caller[h] + nact[h];
    g.Q = g.qbase_caller[H];

    // chance probabilities (children of each chance node sum to 1 +- 1e-12)
    int64_t e_prob = NONE, e_sum = NONE;
#pragma omp parallel for schedule(static) reduction(min : e_prob, e_sum)
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        if (d->player[v] != 0) continue;
        double s = 0.0;
        for (int64_t c = canon_cb[k]; c < canon_cb[k] + ncanon[k]; ++c) {
            const double p = d->chance_prob[order[c]];
            if (!(p >= 0.0 && p <= 1.0)) e_prob = std::min(e_prob, order[c]);
            s += p;
        }
        if (!(std::fabs(s - 1.0) <= 1e-12)) e_sum = std::min(e_sum, v);
    }
    if (e_prob != NONE) return fail(err, "node " + std::to_string(e_prob) + ": chance probability outside [0, 1]");
    if (e_sum != NONE) {
        const int64_t k = g.canon_of_input[e_sum];
        double s = 0.0;
        for (int64_t c = canon_cb[k]; c < canon_cb[k] + ncanon[k]; ++c) s += d->chance_prob[order[c]];
        return fail(err, "chance node " + std::to_string(e_sum) + ": probabilities sum to " + std::to_string(s) + " != 1");
    }

    // zero-sum 2-player single-column storage (Appendix B-7)
    g.zero_sum_2p = false;
    if (P == 2) {
        int64_t nonzs = 0;
#pragma omp parallel for schedule(static) reduction(+ : nonzs)
        for (int64_t v = 0; v < V; ++v)
            if (d->player[v] < 0 && !(d->utility[v * 2 + 1] == -d->utility[v * 2])) ++nonzs;
        g.zero_sum_2p = (nonzs == 0);
    }
    g.Pc = g.zero_sum_2p ? 1 : P;

    tm.mark("infosets");
    // ------------------------------------------------------------------- slots
    // Level by level: decision nodes in canonical order get their "dec" index
    // (reach rows, forward pass); the same nodes grouped by infoset in order of
    // first occurrence get their slot (backward pass).  Internal infoset ids and
    // qbase_int follow first appearance in slot order; chance edges are numbered
    // in canonical order after the Q pairs of sigma_ext.
    const int D = g.D;
    const int Pc = g.Pc;
    g.ND = g.num_decision;
    g.NS = g.num_decision;
    const int64_t NS = g.NS;
    g.dec_ptr.assign(D + 1, 0);
    g.slot_ptr.assign(D + 1, 0);
    g.f_parent.assign(g.ND, -1);
    g.f_e.assign(g.ND, -1);
    g.f_pact.assign(g.ND, 0);
    g.s_node.resize(NS);
    g.s_cb.resize(NS);
    g.s_n.resize(NS);
    g.s_ebase.resize(NS);
    g.s_actor.resize(NS);
    g.s_dec.resize(NS);
    g.s_coff.assign(NS, 0);
    g.h_int_of_caller.assign(H, -1);
    g.h_caller_of_int.clear();
    g.h_caller_of_int.reserve(H);
    g.qbase_int.assign(H + 1, 0);
    g.owner_int.assign(H, 0);
    std::vector<uint8_t> defer_c(H, 0);     // by caller id
    std::vector<int32_t> lvl_of_h(H, -1);
    std::vector<int64_t> grp_of_h(H, -1);
    std::vector<int64_t> grp_count, grp_h;
    std::vector<int64_t> dec_k;              // canonical index of each decision node of the level
    std::vector<int64_t> node_grp;           // group of each decision node of the level
    std::vector<int64_t> ebase_dec(g.ND, -1);  // sigma_ext base of each decision node's children
    std::vector<int64_t> slot_h(NS, -1);     // internal infoset of each player slot
    std::vector<int64_t> dec_of_canon_lvl, prev_dec_of_canon;   // level-local canonical -> dec
    std::vector<int64_t> row_x;              // the level's decision nodes (dec_k indices) in row order
    g.chance_vals.clear();
    int64_t slot = 0, dec = 0, cnext = 0;
    const int64_t Qtot = g.Q;
    for (int L = 0; L < D; ++L) {
        const int64_t lo = g.level_ptr[L], hi = g.level_ptr[L + 1];
        g.dec_ptr[L] = dec;
        g.slot_ptr[L] = slot;
        // decision nodes of the level, canonical order (dec numbering)
        dec_k.clear();
        dec_of_canon_lvl.assign(hi - lo, -1);
        for (int64_t k = lo; k < hi; ++k)
            if (ncanon[k] > 0) {
                dec_of_canon_lvl[k - lo] = dec + (int64_t)dec_k.size();
                dec_k.push_back(k);
            }
        const int64_t nd = (int64_t)dec_k.size();
        // forward data from the parent (previous level)
        if (L > 0) {
            const int64_t plo = g.level_ptr[L - 1];
#pragma omp parallel for schedule(static)
            for (int64_t x = 0; x < nd; ++x) {
                const int64_t k = dec_k[x];
                const int64_t v = order[k];
                const int64_t pk = g.canon_of_input[d->parent[v]];
                const int64_t pd = prev_dec_of_canon[pk - plo];
                g.f_parent[dec + x] = pd;
                g.f_e[dec + x] = ebase_dec[pd] + d->action[v];
                g.f_pact[dec + x] = (uint8_t)d->player[order[pk]];
            }
        }
        // visiting order of the level's decision nodes: the device row order, i.e.
        // the previous level's slots in slot order, each slot's children in action
        // order.  Infosets are numbered, and their members ordered, by first
        // occurrence in this order, so the children of one parent and the users of
        // one parent-infoset edge (same sigma) sit close together in slot order --
        // the forward pass's parent-row and sigma gathers then hit in cache.
        row_x.clear();
        if (L == 0) {
            for (int64_t x = 0; x < nd; ++x) row_x.push_back(x);
        } else {
            const int64_t plo = g.slot_ptr[L - 1];
            for (int64_t ps = plo; ps < slot; ++ps) {
                const int64_t pk = g.s_node[ps];
                for (int64_t c = canon_cb[pk]; c < canon_cb[pk] + ncanon[pk]; ++c)
                    if (ncanon[c] > 0) row_x.push_back(dec_of_canon_lvl[c - lo] - dec);
            }
        }
        if ((int64_t)row_x.size() != nd) return fail(err, "internal: row order size mismatch");
        // groups: infosets in order of first occurrence, chance nodes alone
        grp_count.clear();
        grp_h.clear();
        node_grp.assign(nd, -1);
        for (int64_t xi = 0; xi < nd; ++xi) {
            const int64_t x = row_x[xi];
            const int64_t k = dec_k[x];
            const int64_t v = order[k];
            const int32_t pl = d->player[v];
            if (pl == 0) {
                node_grp[x] = (int64_t)grp_count.size();
                grp_count.push_back(1);
                grp_h.push_back(-1);
                ebase_dec[dec + x] = Qtot + cnext;
                for (int64_t a = 0; a < ncanon[k]; ++a) g.chance_vals.push_back(d->chance_prob[order[canon_cb[k] + a]]);
                cnext += ncanon[k];
                continue;
            }
            const int64_t h = d->infoset[v];
            if (lvl_of_h[h] != L) {
                if (lvl_of_h[h] >= 0) {
                    defer_c[h] = 1;  // infoset spans several depths
                    g.depth_homogeneous = false;
                }
                lvl_of_h[h] = L;
                grp_of_h[h] = (int64_t)grp_count.size();
                grp_count.push_back(0);
                grp_h.push_back(h);
            }
            node_grp[x] = grp_of_h[h];
            grp_count[grp_of_h[h]]++;
        }
        const int64_t ng = (int64_t)grp_count.size();
        for (int64_t gi = 0; gi < ng; ++gi) {
            const int64_t h = grp_h[gi];
            if (h >= 0 && g.h_int_of_caller[h] < 0) {
                const int64_t hi_ = (int64_t)g.h_caller_of_int.size();
                g.h_int_of_caller[h] = hi_;
                g.h_caller_of_int.push_back(h);
                g.qbase_int[hi_ + 1] = g.qbase_int[hi_] + nact[h];
                g.owner_int[hi_] = own[h];
            }
        }
        std::vector<int64_t> gfill(ng, 0);
        {
            int64_t acc = 0;
            for (int64_t gi = 0; gi < ng; ++gi) {
                gfill[gi] = acc;
                acc += grp_count[gi];
            }
        }
        for (int64_t xi = 0; xi < nd; ++xi) {
            const int64_t x = row_x[xi];
            const int64_t k = dec_k[x];
            const int64_t s = slot + gfill[node_grp[x]]++;
            const int64_t v = order[k];
            const int32_t pl = d->player[v];
            int64_t eb = ebase_dec[dec + x];
            if (pl >= 1) {
                const int64_t hint = g.h_int_of_caller[d->infoset[v]];
                eb = g.qbase_int[hint];
                ebase_dec[dec + x] = eb;
                slot_h[s] = hint;
            }
            g.s_node[s] = k;
            g.s_cb[s] = canon_cb[k];
            g.s_n[s] = ncanon[k];
            g.s_actor[s] = (uint8_t)pl;
            g.s_ebase[s] = eb;
            g.s_dec[s] = dec + x;
        }
        slot += nd;
        dec += nd;
        prev_dec_of_canon.swap(dec_of_canon_lvl);
    }
    g.dec_ptr[D] = dec;
    g.slot_ptr[D] = slot;
    if (slot != NS || dec != g.ND) return fail(err, "internal: slot count mismatch");
    if ((int64_t)g.h_caller_of_int.size() != H) return fail(err, "internal: infoset numbering");
    g.C = cnext;
    g.deferred.assign(H, 0);
    for (int64_t h = 0; h < H; ++h) g.deferred[g.h_int_of_caller[h]] = defer_c[h];

    tm.mark("slots");
    // ------------------------------------------------------------------- tiles
    build_tiles(g, slot_h);
    tm.mark("tiles");
    // ------------------------------------------------------------------ values
    g.util_c.resize((size_t)V * Pc);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        const bool term = d->player[v] < 0;
        for (int j = 0; j < Pc; ++j) g.util_c[(size_t)k * Pc + j] = term ? d->utility[v * P + j] : 0.0;
    }
    tm.mark("values");
    return true;
}

int game_exponent(double max_abs_u) { return exponent_for(max_abs_u); }

}  // namespace cfrb
