// Multi-GPU level sharding.
//
// In canonical BFS order the descendants of a contiguous range of depth-k nodes
// form a contiguous range at every deeper depth.  Depths 0..cut (the trunk) are
// replicated on every rank; the decision nodes of depth `cut` are split into
// `world` contiguous ranges balanced by subtree size, and rank r owns all
// descendants of its range (P:403's trunk/subtree chunking, without making the
// trunk a bottleneck: it is recomputed redundantly).
//
// Exchanges per iteration (done by the solver):
//   1. after the backward pass of depth `cut` (the owned cut parents): the values
//      of all cut-level decision nodes (each row nonzero on exactly one rank ->
//      a sum-allreduce is exact);
//   2. after the trunk backward pass: the exact int64 slice sums of the deferred
//      infosets (spanning ranks, spanning depths or split over tiles); trunk tiles
//      contribute on rank 0 only.  Integer sums make the result bit-identical to
//      one GPU and to the oracle for any world size.
#include <algorithm>
#include <string>

#include "game.hpp"

namespace cfrb {

bool build_shard(const Game& F, int rank, int world, Game& G, ShardInfo& info, std::string& err) {
    info = ShardInfo{};
    info.rank = rank;
    info.world = world;
    const int D = F.D;
    // ---- choose the cut: the shallowest depth with >= 2*world decision nodes that
    // still has deeper decision nodes below it
    int cut = -1;
    for (int l = 1; l < D; ++l) {
        if (F.dec_ptr[l + 1] - F.dec_ptr[l] >= 2 * (int64_t)world) {
            cut = l;
            break;
        }
    }
    if (world <= 1) cut = -1;
    info.cut = cut;

    // slot of every decision node
    std::vector<int64_t> slot_of_dec(F.ND, -1);
    for (int64_t s = 0; s < F.NS; ++s) slot_of_dec[F.s_dec[s]] = s;

    // ---- owner of every decision node (-1 = trunk, replicated)
    std::vector<int32_t> owner(F.ND, -1);
    if (cut >= 0) {
        // subtree sizes (nodes), bottom-up in dec order
        std::vector<int64_t> size(F.ND, 0);
        for (int64_t d = 0; d < F.ND; ++d) size[d] = 1 + F.s_n[slot_of_dec[d]];
        for (int64_t d = F.ND - 1; d >= 0; --d) {
            const int64_t p = F.f_parent[d];
            if (p >= 0) size[p] += size[d] - 1;
        }
        const int64_t c0 = F.dec_ptr[cut], c1 = F.dec_ptr[cut + 1];
        int64_t total = 0;
        for (int64_t d = c0; d < c1; ++d) total += size[d];
        int64_t acc = 0;
        for (int64_t d = c0; d < c1; ++d) {
            // rank r takes the nodes whose cumulative-size midpoint falls in its share
            const int64_t mid = acc + size[d] / 2;
            int r = (int)std::min<int64_t>(world - 1, (mid * world) / std::max<int64_t>(total, 1));
            owner[d] = r;
            acc += size[d];
        }
        // keep ranges contiguous and non-decreasing (midpoint rule already is)
        for (int64_t d = F.dec_ptr[cut + 1]; d < F.ND; ++d) owner[d] = owner[F.f_parent[d]];
    }

    // ---- local node ranges per depth
    G = Game{};
    G.P = F.P;
    G.Pc = F.Pc;
    G.zero_sum_2p = F.zero_sum_2p;
    G.D = D;
    G.max_abs_u = F.max_abs_u;
    G.depth_homogeneous = F.depth_homogeneous;
    G.H = F.H;
    G.Q = F.Q;
    G.C = F.C;
    G.h_int_of_caller = F.h_int_of_caller;
    G.h_caller_of_int = F.h_caller_of_int;
    G.qbase_int = F.qbase_int;
    G.qbase_caller = F.qbase_caller;
    G.owner_int = F.owner_int;
    G.chance_vals = F.chance_vals;
    std::vector<int64_t> lo(D + 1), hi(D + 1);
    for (int l = 0; l <= D; ++l) {
        if (cut < 0 || l <= cut) {
            lo[l] = F.level_ptr[l];
            hi[l] = F.level_ptr[l + 1];
        } else {
            // children of the owned decision nodes of depth l-1 (contiguous)
            int64_t a = -1, b = -1;
            for (int64_t d = F.dec_ptr[l - 1]; d < F.dec_ptr[l]; ++d)
                if (owner[d] == rank) {
                    const int64_t s = slot_of_dec[d];
                    if (a < 0) a = F.s_cb[s];
                    b = F.s_cb[s] + F.s_n[s];
                }
            if (a < 0) a = b = F.level_ptr[l];
            lo[l] = a;
            hi[l] = b;
        }
    }
    G.level_ptr.assign(D + 2, 0);
    for (int l = 0; l <= D; ++l) G.level_ptr[l + 1] = G.level_ptr[l] + (hi[l] - lo[l]);
    G.V = G.level_ptr[D + 1];
    info.local_level_nodes.assign(D + 1, 0);
    for (int l = 0; l <= D; ++l) {
        info.local_level_nodes[l] = hi[l] - lo[l];
        if (cut >= 0 && l > cut) info.owned_nodes += hi[l] - lo[l];
    }
    // canonical (global) node k of depth l -> local node index
    std::vector<int64_t> lvl_of_slotlevel;  // unused helper placeholder
    auto to_local = [&](int l, int64_t k) -> int64_t { return G.level_ptr[l] + (k - lo[l]); };
    G.util_c.assign((size_t)G.V * G.Pc, 0.0);
    for (int l = 0; l <= D; ++l)
        for (int64_t k = lo[l]; k < hi[l]; ++k)
            for (int j = 0; j < G.Pc; ++j)
                G.util_c[(size_t)to_local(l, k) * G.Pc + j] = F.util_c[(size_t)k * F.Pc + j];
    G.num_terminals = 0;
    G.num_chance = 0;

    // ---- local decision nodes (dec order): trunk + owned
    std::vector<int64_t> ldec(F.ND, -1);
    G.dec_ptr.assign(D + 1, 0);
    int64_t nd = 0;
    for (int l = 0; l < D; ++l) {
        G.dec_ptr[l] = nd;
        for (int64_t d = F.dec_ptr[l]; d < F.dec_ptr[l + 1]; ++d)
            if (cut < 0 || l <= cut || owner[d] == rank) ldec[d] = nd++;
    }
    G.dec_ptr[D] = nd;
    G.ND = nd;
    G.num_decision = nd;
    G.f_parent.assign(nd, -1);
    G.f_e.assign(nd, -1);
    G.f_pact.assign(nd, 0);
    for (int64_t d = 0; d < F.ND; ++d) {
        const int64_t x = ldec[d];
        if (x < 0) continue;
        G.f_parent[x] = F.f_parent[d] >= 0 ? ldec[F.f_parent[d]] : -1;
        G.f_e[x] = F.f_e[d];
        G.f_pact[x] = F.f_pact[d];
        if (F.s_actor[slot_of_dec[d]] == 0) G.num_chance++;
    }

    // ---- local slots: every trunk parent of depth < cut, owned parents at depth >= cut
    auto slot_kept = [&](int L, int64_t s) -> bool {
        if (cut < 0 || L < cut) return true;
        return owner[F.s_dec[s]] == rank;
    };
    G.slot_ptr.assign(D + 1, 0);
    int64_t ns = 0;
    for (int L = 0; L < D; ++L)
        for (int64_t s = F.slot_ptr[L]; s < F.slot_ptr[L + 1]; ++s) ns += slot_kept(L, s) ? 1 : 0;
    G.NS = ns;
    G.s_node.resize(ns);
    G.s_cb.resize(ns);
    G.s_n.resize(ns);
    G.s_ebase.resize(ns);
    G.s_actor.resize(ns);
    G.s_dec.resize(ns);
    G.s_coff.assign(ns, 0);
    std::vector<int64_t> slot_h(ns, -1);
    {
        // internal infoset of each global player slot
        int64_t x = 0;
        for (int L = 0; L < D; ++L) {
            G.slot_ptr[L] = x;
            for (int64_t s = F.slot_ptr[L]; s < F.slot_ptr[L + 1]; ++s) {
                if (!slot_kept(L, s)) continue;
                G.s_node[x] = to_local(L, F.s_node[s]);
                G.s_cb[x] = to_local(L + 1, F.s_cb[s]);
                G.s_n[x] = F.s_n[s];
                G.s_ebase[x] = F.s_ebase[s];
                G.s_actor[x] = F.s_actor[s];
                G.s_dec[x] = ldec[F.s_dec[s]];
                if (F.s_actor[s] >= 1) {
                    // s_ebase of a player slot is qbase_int[h]: recover h by search
                    const int64_t eb = F.s_ebase[s];
                    const int64_t h = std::upper_bound(F.qbase_int.begin(), F.qbase_int.end(), eb) - F.qbase_int.begin() - 1;
                    slot_h[x] = h;
                }
                ++x;
            }
        }
        G.slot_ptr[D] = x;
    }

    // ---- deferred set: identical on every rank (compact exchange layout)
    G.deferred = F.deferred;
    if (cut >= 0) {
        std::vector<int32_t> first(F.H, -1);
        for (int L = cut; L < D; ++L)
            for (int64_t s = F.slot_ptr[L]; s < F.slot_ptr[L + 1]; ++s) {
                if (F.s_actor[s] < 1) continue;
                const int64_t eb = F.s_ebase[s];
                const int64_t h = std::upper_bound(F.qbase_int.begin(), F.qbase_int.end(), eb) - F.qbase_int.begin() - 1;
                const int32_t r = owner[F.s_dec[s]];
                if (first[h] < 0) first[h] = r;
                else if (first[h] != r) G.deferred[h] = 1;   // spans ranks
            }
    }
    build_tiles(G, slot_h);
    if (G.deferred_list != F.deferred_list && cut < 0) {
        err = "internal: deferred set changed";
        return false;
    }

    // ---- exchange metadata
    info.tile_contrib.assign(G.tiles.size(), 1);
    if (cut >= 0)
        for (int L = 0; L < cut; ++L)
            for (int64_t t = G.tile_ptr[L]; t < G.tile_ptr[L + 1]; ++t) info.tile_contrib[t] = (rank == 0) ? 1 : 0;
    if (cut >= 0) {
        for (int64_t d = F.dec_ptr[cut]; d < F.dec_ptr[cut + 1]; ++d) {
            info.cut_row.push_back(to_local(cut, F.s_node[slot_of_dec[d]]));
            info.cut_owned.push_back(owner[d] == rank ? 1 : 0);
        }
    }
    // readback reporter: trunk and deferred infosets -> rank 0; shard-local -> owner
    info.report.assign(F.H, 0);
    {
        std::vector<int32_t> rep(F.H, 0);
        if (cut >= 0)
            for (int L = cut; L < D; ++L)
                for (int64_t s = F.slot_ptr[L]; s < F.slot_ptr[L + 1]; ++s) {
                    if (F.s_actor[s] < 1) continue;
                    const int64_t eb = F.s_ebase[s];
                    const int64_t h =
                        std::upper_bound(F.qbase_int.begin(), F.qbase_int.end(), eb) - F.qbase_int.begin() - 1;
                    if (!G.deferred[h]) rep[h] = owner[F.s_dec[s]];
                }
        for (int64_t h = 0; h < F.H; ++h) info.report[h] = (rep[h] == rank) ? 1 : 0;
    }
    G.num_terminals = G.V - G.ND;
    G.max_infoset_nodes = F.max_infoset_nodes;
    G.canon_of_input.clear();
    return true;
}

}  // namespace cfrb
