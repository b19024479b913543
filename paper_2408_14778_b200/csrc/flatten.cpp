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
#include <cmath>
#include <cstring>
#include <numeric>

#include "game.hpp"

namespace cfrb {

namespace {

bool fail(std::string& err, const std::string& m) {
    err = m;
    return false;
}

// E = 1 + ceil(log2(2*m)) for m > 0, else 1.  ilogb-based.
int exponent_for(double m) {
    if (!(m > 0.0)) return 1;
    const double x = 2.0 * m;
    int k = std::ilogb(x);                 // floor(log2 x) for normal x
    if (std::ldexp(1.0, k) < x) k += 1;    // ceil
    return 1 + k;
}

}  // namespace

bool build_game(const cfr_game_desc* d, Game& g, std::string& err) {
    const int64_t V = d->num_nodes;
    const int P = d->num_players;
    if (V < 1) return fail(err, "num_nodes must be >= 1");
    if (P < 1 || P > 16) return fail(err, "num_players must be in [1, 16]");
    if (!d->parent || !d->player || !d->infoset || !d->action || !d->chance_prob || !d->utility)
        return fail(err, "NULL array in cfr_game_desc");
    g.V = V;
    g.P = P;

    // ---------------------------------------------------------------- children
    int64_t root = -1;
    std::vector<int64_t> cstart(V + 1, 0);
    for (int64_t v = 0; v < V; ++v) {
        const int64_t p = d->parent[v];
        if (p < 0) {
            if (p != -1) return fail(err, "node " + std::to_string(v) + ": parent must be -1 or a node id");
            if (root >= 0) return fail(err, "two roots: nodes " + std::to_string(root) + " and " + std::to_string(v));
            root = v;
        } else {
            if (p >= V) return fail(err, "node " + std::to_string(v) + ": parent out of range");
            if (p == v) return fail(err, "node " + std::to_string(v) + " is its own parent");
            cstart[p + 1]++;
        }
        const int32_t pl = d->player[v];
        if (pl < -1 || pl > P) return fail(err, "node " + std::to_string(v) + ": player out of range");
    }
    if (root < 0) return fail(err, "no root (parent == -1)");
    for (int64_t v = 0; v < V; ++v) cstart[v + 1] += cstart[v];
    std::vector<int64_t> clist(V > 1 ? V - 1 : 1, -1);
    for (int64_t v = 0; v < V; ++v) {
        const int64_t p = d->parent[v];
        if (p < 0) continue;
        const int64_t n = cstart[p + 1] - cstart[p];
        const int32_t a = d->action[v];
        if (a < 0 || a >= n)
            return fail(err, "node " + std::to_string(v) + ": action " + std::to_string(a) +
                                 " not in 0.." + std::to_string(n - 1) + " (action bijection, P:33)");
        int64_t& slot = clist[cstart[p] + a];
        if (slot >= 0)
            return fail(err, "node " + std::to_string(v) + ": duplicate action " + std::to_string(a) + " under parent " +
                                 std::to_string(p));
        slot = v;
    }
    for (int64_t v = 0; v < V; ++v) {
        const int64_t n = cstart[v + 1] - cstart[v];
        const int32_t pl = d->player[v];
        if (pl < 0 && n != 0) return fail(err, "terminal node " + std::to_string(v) + " has children");
        if (pl >= 0 && n == 0) return fail(err, "decision node " + std::to_string(v) + " has no children");
        if (pl < 0) {
            for (int j = 0; j < P; ++j) {
                const double u = d->utility[v * P + j];
                if (!std::isfinite(u)) return fail(err, "terminal node " + std::to_string(v) + ": non-finite utility");
                g.max_abs_u = std::max(g.max_abs_u, std::fabs(u));
            }
        }
    }

    // ------------------------------------------------------- canonical BFS order
    std::vector<int64_t> order(V);
    order[0] = root;
    int64_t tail = 1;
    g.level_ptr.assign(1, 0);
    int64_t lvl_end = 1;
    g.level_ptr.push_back(1);
    std::vector<int64_t> canon_cb(V, -1);
    for (int64_t k = 0; k < tail; ++k) {
        if (k == lvl_end) {
            lvl_end = tail;
            g.level_ptr.push_back(tail);
        }
        const int64_t v = order[k];
        const int64_t n = cstart[v + 1] - cstart[v];
        if (n > 0) {
            canon_cb[k] = tail;
            if (tail + n > V) return fail(err, "tree has a cycle");
            for (int64_t a = 0; a < n; ++a) order[tail++] = clist[cstart[v] + a];
        }
    }
    if (tail != V) return fail(err, "tree is not connected: " + std::to_string(V - tail) + " node(s) unreachable from the root (cycle?)");
    if (g.level_ptr.back() != V) g.level_ptr.push_back(V);
    g.D = (int32_t)g.level_ptr.size() - 2;
    std::vector<int64_t>().swap(clist);
    std::vector<int64_t>().swap(cstart);
    g.canon_of_input.assign(V, 0);
    for (int64_t k = 0; k < V; ++k) g.canon_of_input[order[k]] = k;

    // ------------------------------------------------------------ infoset checks
    int64_t H = 0;
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        if (d->player[v] >= 1) {
            const int64_t h = d->infoset[v];
            if (h < 0) return fail(err, "player node " + std::to_string(v) + " has no infoset id");
            H = std::max(H, h + 1);
        }
    }
    g.H = H;
    std::vector<int32_t> nact(H, -1);
    std::vector<uint8_t> own(H, 0);
    std::vector<int64_t> members(H, 0);
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        const int32_t pl = d->player[v];
        if (pl < 0) {
            g.num_terminals++;
            continue;
        }
        if (pl == 0) {
            g.num_chance++;
            continue;
        }
        const int64_t h = d->infoset[v];
        members[h]++;
    }
    g.num_decision = V - g.num_terminals;
    // children counts per canonical node
    std::vector<int32_t> ncanon(V, 0);
    {
        // canon_cb is monotone over decision nodes; n = next cb - cb
        int64_t prev = -1;
        for (int64_t k = 0; k < V; ++k) {
            if (canon_cb[k] >= 0) {
                if (prev >= 0) ncanon[prev] = (int32_t)(canon_cb[k] - canon_cb[prev]);
                prev = k;
            }
        }
        if (prev >= 0) ncanon[prev] = (int32_t)(V - canon_cb[prev]);
    }
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        const int32_t pl = d->player[v];
        if (pl < 1) continue;
        const int64_t h = d->infoset[v];
        if (nact[h] < 0) {
            nact[h] = ncanon[k];
            own[h] = (uint8_t)pl;
        } else {
            if (nact[h] != ncanon[k])
                return fail(err, "infoset " + std::to_string(h) + ": nodes have different action counts (node " +
                                     std::to_string(v) + ")");
            if (own[h] != pl) return fail(err, "infoset " + std::to_string(h) + ": nodes of different players");
        }
    }
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
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        if (d->player[v] != 0) continue;
        double s = 0.0;
        for (int64_t c = canon_cb[k]; c < canon_cb[k] + ncanon[k]; ++c) {
            const double p = d->chance_prob[order[c]];
            if (!(p >= 0.0 && p <= 1.0))
                return fail(err, "node " + std::to_string(order[c]) + ": chance probability outside [0, 1]");
            s += p;
        }
        if (std::fabs(s - 1.0) > 1e-12)
            return fail(err, "chance node " + std::to_string(v) + ": probabilities sum to " + std::to_string(s) + " != 1");
    }

    // zero-sum 2-player single-column storage (Appendix B-7)
    g.zero_sum_2p = false;
    if (P == 2) {
        bool zs = true;
        for (int64_t v = 0; v < V && zs; ++v)
            if (d->player[v] < 0 && !(d->utility[v * 2 + 1] == -d->utility[v * 2])) zs = false;
        g.zero_sum_2p = zs;
    }
    g.Pc = g.zero_sum_2p ? 1 : P;

    // ------------------------------------------------------------------- slots
    const int D = g.D;
    g.slot_ptr.assign(D + 1, 0);
    g.NS = g.num_decision;
    const int64_t NS = g.NS;
    g.s_node.resize(NS);
    g.s_cb.resize(NS);
    g.s_n.resize(NS);
    g.s_ebase.resize(NS);
    g.s_actor.resize(NS);
    g.s_parent.resize(NS);
    g.s_e.resize(NS);
    g.s_pact.resize(NS);
    g.h_int_of_caller.assign(H, -1);
    g.h_caller_of_int.clear();
    g.h_caller_of_int.reserve(H);
    g.deferred.assign(H, 0);
    std::vector<int32_t> lvl_of_h(H, -1);
    std::vector<int64_t> grp_of_h(H, -1);   // group index within the current level
    std::vector<int64_t> par_slot_next, e_next;   // for the next level, indexed by node - level_ptr[L+1]
    std::vector<uint8_t> pact_next;
    // parent info for level 0: root only
    int64_t slot = 0;
    int64_t cnext = 0;                        // chance edges assigned so far
    std::vector<int64_t> grp_first, grp_count, grp_h;  // per group of the level
    std::vector<int64_t> node_grp;                      // per decision node of the level (level order)
    std::vector<int64_t> cur_par_slot(1, -1), cur_e(1, -1);
    std::vector<uint8_t> cur_pact(1, 0);
    g.chance_vals.clear();
    for (int L = 0; L < D; ++L) {
        const int64_t lo = g.level_ptr[L], hi = g.level_ptr[L + 1];
        g.slot_ptr[L] = slot;
        grp_first.clear();
        grp_count.clear();
        grp_h.clear();
        node_grp.assign(hi - lo, -1);
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t v = order[k];
            const int32_t pl = d->player[v];
            if (pl < 0) continue;
            if (pl == 0) {
                node_grp[k - lo] = (int64_t)grp_count.size();
                grp_first.push_back(k);
                grp_count.push_back(1);
                grp_h.push_back(-1);
                continue;
            }
            const int64_t h = d->infoset[v];
            if (lvl_of_h[h] != L) {
                if (lvl_of_h[h] >= 0) {
                    g.deferred[h] = 1;  // infoset spans several depths
                    g.depth_homogeneous = false;
                }
                lvl_of_h[h] = L;
                grp_of_h[h] = (int64_t)grp_count.size();
                grp_first.push_back(k);
                grp_count.push_back(0);
                grp_h.push_back(h);
            }
            node_grp[k - lo] = grp_of_h[h];
            grp_count[grp_of_h[h]]++;
        }
        // group start slots
        const int64_t ng = (int64_t)grp_count.size();
        std::vector<int64_t> gstart(ng + 1, 0);
        for (int64_t gi = 0; gi < ng; ++gi) gstart[gi + 1] = gstart[gi] + grp_count[gi];
        std::vector<int64_t> gfill(gstart.begin(), gstart.end() - 1);
        // internal infoset ids in order of first appearance in slot order
        for (int64_t gi = 0; gi < ng; ++gi) {
            const int64_t h = grp_h[gi];
            if (h >= 0 && g.h_int_of_caller[h] < 0) {
                g.h_int_of_caller[h] = (int64_t)g.h_caller_of_int.size();
                g.h_caller_of_int.push_back(h);
            }
        }
        // place nodes into slots
        const int64_t nlo = g.level_ptr[L + 1];
        const int64_t nhi = g.level_ptr[L + 2];
        par_slot_next.assign(nhi - nlo, -1);
        e_next.assign(nhi - nlo, -1);
        pact_next.assign(nhi - nlo, 0);
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t gi = node_grp[k - lo];
            if (gi < 0) continue;
            const int64_t s = slot + gfill[gi]++;
            const int64_t v = order[k];
            const int32_t pl = d->player[v];
            g.s_node[s] = k;
            g.s_cb[s] = canon_cb[k];
            g.s_n[s] = ncanon[k];
            g.s_actor[s] = (uint8_t)pl;
            g.s_parent[s] = cur_par_slot[k - lo];
            g.s_e[s] = cur_e[k - lo];
            g.s_pact[s] = cur_pact[k - lo];
            // children edge probabilities base (filled below for players via qbase_int)
            if (pl == 0) {
                g.s_ebase[s] = -1 - cnext;  // provisional: chance edge offset, fixed after Q known
                for (int64_t a = 0; a < ncanon[k]; ++a) g.chance_vals.push_back(d->chance_prob[order[canon_cb[k] + a]]);
                cnext += ncanon[k];
            } else {
                g.s_ebase[s] = d->infoset[v];  // provisional: caller infoset, fixed below
            }
            for (int64_t a = 0; a < ncanon[k]; ++a) {
                const int64_t c = canon_cb[k] + a - nlo;
                par_slot_next[c] = s;
                pact_next[c] = (uint8_t)pl;
                // provisional edge id: chance -> -1 - (chance edge), player -> (caller infoset h, a) packed later
                e_next[c] = (pl == 0) ? (-1 - (cnext - ncanon[k] + a)) : a;
            }
        }
        slot += gstart[ng];
        // next level's decision nodes inherit parent slot / edge / parent actor
        cur_par_slot.assign(nhi - nlo, -1);
        cur_e.assign(nhi - nlo, -1);
        cur_pact.assign(nhi - nlo, 0);
        for (int64_t c = 0; c < nhi - nlo; ++c) {
            cur_par_slot[c] = par_slot_next[c];
            cur_e[c] = e_next[c];
            cur_pact[c] = pact_next[c];
        }
    }
    g.slot_ptr[D] = slot;
    if (slot != NS) return fail(err, "internal: slot count mismatch");
    g.C = cnext;

    // internal qbase and owner
    g.qbase_int.assign(H + 1, 0);
    g.owner_int.assign(H, 0);
    for (int64_t hi = 0; hi < H; ++hi) {
        const int64_t h = g.h_caller_of_int[hi];
        g.qbase_int[hi + 1] = g.qbase_int[hi] + nact[h];
        g.owner_int[hi] = own[h];
    }
    // finalize edge indices into sigma_ext = [sigma (Q, internal order) | chance (C)]
    for (int64_t s = 0; s < NS; ++s) {
        if (g.s_actor[s] == 0) g.s_ebase[s] = g.Q + (-1 - g.s_ebase[s]);
        else g.s_ebase[s] = g.qbase_int[g.h_int_of_caller[g.s_ebase[s]]];
        const int64_t p = g.s_parent[s];
        if (p < 0) {
            g.s_e[s] = -1;
        } else if (g.s_pact[s] == 0) {
            g.s_e[s] = g.Q + (-1 - g.s_e[s]);
        } else {
            g.s_e[s] = g.s_ebase[p] + g.s_e[s];
        }
    }
    // deferred flags are per caller id so far; convert to internal ids
    {
        std::vector<uint8_t> dint(H, 0);
        for (int64_t h = 0; h < H; ++h) dint[g.h_int_of_caller[h]] = g.deferred[h];
        g.deferred.swap(dint);
    }

    // ------------------------------------------------------------------- tiles
    // Groups are maximal runs of equal infoset within a level's slots.
    g.tile_ptr.assign(D + 1, 0);
    g.tiles.clear();
    g.segs.clear();
    std::vector<int64_t> slot_h(NS, -1);  // internal infoset of each player slot
    for (int64_t s = 0; s < NS; ++s)
        if (g.s_actor[s] >= 1) slot_h[s] = g.h_int_of_caller[d->infoset[order[g.s_node[s]]]];
    for (int L = 0; L < D; ++L) {
        g.tile_ptr[L] = (int64_t)g.tiles.size();
        const int64_t lo = g.slot_ptr[L], hi = g.slot_ptr[L + 1];
        TileH cur{lo, lo, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0};
        auto close = [&]() {
            if (cur.s1 > cur.s0) {
                cur.seg1 = (int32_t)g.segs.size();
                g.tiles.push_back(cur);
            }
            cur = TileH{cur.s1, cur.s1, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0};
        };
        int64_t s = lo;
        while (s < hi) {
            int64_t e = s + 1;
            const int64_t h = slot_h[s];
            if (h >= 0)
                while (e < hi && slot_h[e] == h) ++e;
            const int64_t m = e - s;
            const int32_t n = (h >= 0) ? (int32_t)(g.qbase_int[h + 1] - g.qbase_int[h]) : 0;
            const bool too_big = (m > kTileSlots) || (n > kTilePairs);  // split: accumulate globally
            if (too_big) {
                // split group: its own chunks, accumulated globally (deferred)
                close();
                g.deferred[h] = 1;
                for (int64_t c0 = s; c0 < e; c0 += kTileSlots) {
                    const int64_t c1 = std::min(e, c0 + kTileSlots);
                    TileH t{c0, c1, (int32_t)g.segs.size(), 0, n, 0};
                    g.segs.push_back(SegH{h, c0, c1, 0, 0});
                    t.seg1 = (int32_t)g.segs.size();
                    g.tiles.push_back(t);
                }
                cur = TileH{e, e, (int32_t)g.segs.size(), (int32_t)g.segs.size(), 0, 0};
                s = e;
                continue;
            }
            const int64_t segs_in = (int64_t)g.segs.size() - cur.seg0;
            if ((cur.s1 - cur.s0) + m > kTileSlots || cur.npairs + n > kTilePairs ||
                (h >= 0 && segs_in + 1 > kTileSegs))
                close();
            if (h >= 0) {
                g.segs.push_back(SegH{h, s, e, cur.npairs, g.deferred[h] ? 0 : 1});
                cur.npairs += n;
            }
            cur.s1 = e;
            s = e;
        }
        close();
    }
    g.tile_ptr[D] = (int64_t)g.tiles.size();
    // segments of deferred infosets are never fused
    for (auto& sg : g.segs)
        if (g.deferred[sg.h]) sg.fused = 0;
    g.deferred_list.clear();
    for (int64_t h = 0; h < H; ++h)
        if (g.deferred[h]) g.deferred_list.push_back(h);

    // ------------------------------------------------------------------ values
    const int Pc = g.Pc;
    g.util_c.assign((size_t)V * Pc, 0.0);
    for (int64_t k = 0; k < V; ++k) {
        const int64_t v = order[k];
        if (d->player[v] >= 0) continue;
        for (int j = 0; j < Pc; ++j) g.util_c[(size_t)k * Pc + j] = d->utility[v * P + j];
    }
    return true;
}

int game_exponent(double max_abs_u) { return exponent_for(max_abs_u); }

}  // namespace cfrb
