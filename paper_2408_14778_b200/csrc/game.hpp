// Internal (product-side) representation of a flattened game.  Built once on the
// host by flatten.cpp (SURVEY.md Appendix B-1 canonical BFS + DESIGN.md §5 slot
// layout), uploaded by solver.cu.  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cfr_b200.h"

namespace cfrb {

// Backward-pass work unit: a run of slots [s0, s1) of one level holding whole
// infoset groups (or one chunk of an oversized group), plus its segments.
struct TileH {
    int64_t s0, s1;        // slot range
    int32_t seg0, seg1;    // segments [seg0, seg1) in Game::segs
    int32_t npairs;        // sum of |A(h)| over the tile's segments
    int32_t nch;           // staged child elements (padded rows), <= kTileChildren if staged
    int32_t run0, run1;    // (unused, 0)
    int32_t staged;        // 1: children staged in shared memory
    int32_t pad;
};


// A segment = the member slots [sb, se) of internal infoset h inside one tile.
struct SegH {
    int64_t h;             // internal infoset id
    int64_t sb, se;        // member slots inside the tile
    int32_t pair_off;      // offset of (h, 0) in the tile's pair numbering
    int32_t fused;         // 1: all members here, single depth -> update in-tile
};

constexpr int kTileSlots = 128;     // parents per tile (= threads per CTA)
constexpr int kTilePairs = 512;     // (infoset, action) pairs per tile
constexpr int kTileSegs = 64;       // segments (infosets) per tile
constexpr int kTileChildren = 2816; // staged child values (R elements, padded rows)

struct Game {
    // ---- input-level facts
    int64_t V = 0;
    int32_t P = 0;
    int32_t Pc = 0;          // value columns stored on device (1 if zero-sum 2p)
    bool zero_sum_2p = false;
    int32_t D = 0;           // max depth
    int64_t num_terminals = 0, num_chance = 0, num_decision = 0;
    int64_t max_infoset_nodes = 0;
    bool depth_homogeneous = true;
    double max_abs_u = 0.0;  // over the double inputs

    // ---- canonical flattening (Appendix B-1)
    std::vector<int64_t> canon_of_input;  // [V]
    std::vector<int64_t> level_ptr;       // [D+2] canonical node ranges per depth

    // ---- decision nodes in canonical order ("dec" index): forward pass + reach
    int64_t ND = 0;
    std::vector<int64_t> dec_ptr;         // [D+1]: decision nodes of depth l in [dec_ptr[l], dec_ptr[l+1])
    std::vector<int64_t> f_parent;        // [ND] dec index of the parent (-1 root)
    std::vector<int64_t> f_e;             // [ND] sigma_ext index of the incoming edge
    std::vector<uint8_t> f_pact;          // [ND] actor of the parent

    // ---- slots: decision nodes, level-major, infoset-grouped
    int64_t NS = 0;
    std::vector<int64_t> slot_ptr;        // [D+1]: slots of depth L in [slot_ptr[L], slot_ptr[L+1])
    std::vector<int64_t> s_node;          // canonical node index
    std::vector<int64_t> s_cb;            // canonical index of first child
    std::vector<int32_t> s_n;             // number of children
    std::vector<int64_t> s_ebase;         // base of the children's edge probs in sigma_ext
    std::vector<uint8_t> s_actor;         // 0 chance, 1..P player
    std::vector<int64_t> s_dec;           // dec index (reach row)
    std::vector<int32_t> s_coff;          // tile-local offset of the staged child row

    // ---- infosets, internal numbering (order of first appearance in slot order)
    int64_t H = 0, Q = 0, C = 0;          // infosets, pairs, chance edges
    std::vector<int64_t> h_int_of_caller, h_caller_of_int;
    std::vector<int64_t> qbase_int;       // [H+1]
    std::vector<int64_t> qbase_caller;    // [H+1]
    std::vector<uint8_t> owner_int;       // [H]
    std::vector<uint8_t> deferred;        // [H] 1: accumulate globally, update after the pass
    std::vector<int64_t> deferred_list;   // internal ids, ascending
    std::vector<int64_t> dpos;            // [H] index in deferred_list or -1
    std::vector<int64_t> dqbase;          // [ndef + 1] compact pair base of each deferred infoset
    std::vector<double> chance_vals;      // [C], sigma_ext[Q + c]

    // ---- backward tiles
    std::vector<int64_t> tile_ptr;        // [D+1]: tiles of parent depth L
    std::vector<TileH> tiles;
    std::vector<SegH> segs;

    // ---- values
    std::vector<double> util_c;           // [V * Pc] canonical rows (terminals; 0 elsewhere)
};

// Multi-GPU level sharding.  Depths 0..cut are
// the replicated trunk; every deeper node belongs to the rank that owns its
// depth-`cut` ancestor.  The per-rank view is itself a Game (local canonical
// numbering), plus the exchange metadata below.
struct ShardInfo {
    int rank = 0, world = 1;
    int cut = -1;                          // -1: nothing sharded (every rank redundant)
    std::vector<int64_t> cut_row;          // local U row of every cut-level decision node
    std::vector<uint8_t> cut_owned;        // 1 if this rank computes it
    std::vector<uint8_t> tile_contrib;     // per local tile: adds deferred partial sums
    std::vector<uint8_t> report;           // [H] 1 if this rank reports the infoset in readbacks
    std::vector<int64_t> local_level_nodes;// nodes per depth on this rank
    int64_t owned_nodes = 0;               // nodes of depths > cut owned here
};
bool build_shard(const Game& full, int rank, int world, Game& local, ShardInfo& info, std::string& err);
// store.cpp: shard files
std::string shard_path(const std::string& prefix, int rank, int world);
bool save_shard(const std::string& path, const Game& full, const Game& local, const ShardInfo& info, std::string& err);
bool load_shard(const std::string& path, Game& head, Game& local, ShardInfo& info, std::string& err);

// flatten.cpp
bool build_game(const cfr_game_desc* d, Game& g, std::string& err);
// (re)build tiles + segments + deferred list from the slot arrays; slot_h[s] =
// internal infoset of player slot s, -1 for chance
void build_tiles(Game& g, const std::vector<int64_t>& slot_h);
// E = 1 + ceil(log2(2 max|u|)) (exact-accumulation exponent)
int game_exponent(double max_abs_u);

}  // namespace cfrb

struct cfr_game {
    cfrb::Game g;
    // per (rank, world) shard views, built on first use (solver workspace sizing
    // and creation share them)
    struct Shard {
        cfrb::Game local;
        cfrb::ShardInfo info;
    };
    std::map<std::pair<int, int>, std::shared_ptr<Shard>> shards;
    bool shard_only = false;   // loaded from a shard file: `g` holds only the header facts
};

// error plumbing shared by the product's translation units
void cfrb_set_error(const std::string& msg);
