// Shard files: the per-rank view of a level-sharded game, written
// once by one process and loaded by each rank, so that N ranks on one host do not
// each flatten (and hold) the whole ~1e9-node tree.  Binary, little-endian,
// "CFRSHRD1" magic + field-by-field records; a loaded shard carries the header
// facts of the full game needed by cfr_game_info / readbacks.
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>

#include "game.hpp"

namespace cfrb {
namespace {

struct Writer {
    FILE* f;
    bool ok = true;
    template <class T>
    void pod(const T& x) {
        static_assert(std::is_trivially_copyable<T>::value, "pod");
        ok = ok && std::fwrite(&x, sizeof(T), 1, f) == 1;
    }
    template <class T>
    void vec(const std::vector<T>& v) {
        const uint64_t n = v.size();
        pod(n);
        if (n) ok = ok && std::fwrite(v.data(), sizeof(T), n, f) == n;
    }
};
struct Reader {
    FILE* f;
    bool ok = true;
    template <class T>
    void pod(T& x) {
        ok = ok && std::fread(&x, sizeof(T), 1, f) == 1;
    }
    template <class T>
    void vec(std::vector<T>& v) {
        uint64_t n = 0;
        pod(n);
        if (!ok || n > (uint64_t(1) << 40)) { ok = false; return; }
        v.resize(n);
        if (n) ok = ok && std::fread(v.data(), sizeof(T), n, f) == n;
    }
};

template <class IO, class G>
void game_fields(IO& io, G& g) {
    io.pod(g.V); io.pod(g.P); io.pod(g.Pc); io.pod(g.zero_sum_2p); io.pod(g.D);
    io.pod(g.num_terminals); io.pod(g.num_chance); io.pod(g.num_decision); io.pod(g.max_infoset_nodes);
    io.pod(g.depth_homogeneous); io.pod(g.max_abs_u);
    io.vec(g.level_ptr);
    io.pod(g.ND); io.vec(g.dec_ptr); io.vec(g.f_parent); io.vec(g.f_e); io.vec(g.f_pact);
    io.pod(g.NS); io.vec(g.slot_ptr); io.vec(g.s_node); io.vec(g.s_cb); io.vec(g.s_n); io.vec(g.s_ebase);
    io.vec(g.s_actor); io.vec(g.s_dec); io.vec(g.s_coff);
    io.pod(g.H); io.pod(g.Q); io.pod(g.C);
    io.vec(g.h_int_of_caller); io.vec(g.h_caller_of_int); io.vec(g.qbase_int); io.vec(g.qbase_caller);
    io.vec(g.owner_int); io.vec(g.deferred); io.vec(g.deferred_list); io.vec(g.dpos); io.vec(g.dqbase);
    io.vec(g.chance_vals); io.vec(g.tile_ptr); io.vec(g.tiles); io.vec(g.segs); io.vec(g.util_c);
}
template <class IO, class S>
void info_fields(IO& io, S& s) {
    io.pod(s.rank); io.pod(s.world); io.pod(s.cut);
    io.vec(s.cut_row); io.vec(s.cut_owned); io.vec(s.tile_contrib); io.vec(s.report); io.vec(s.local_level_nodes);
    io.pod(s.owned_nodes);
}

const char kMagic[8] = {'C', 'F', 'R', 'S', 'H', 'R', 'D', '2'};
// The file stores raw TileH / SegH records: their sizes are part of the format, so
// a layout change is rejected on load instead of being read as corrupt data.
struct FormatTag {
    uint32_t version = 2;
    uint32_t tile_bytes = (uint32_t)sizeof(TileH);
    uint32_t seg_bytes = (uint32_t)sizeof(SegH);
    uint32_t pad = 0;
};

}  // namespace

std::string shard_path(const std::string& prefix, int rank, int world) {
    return prefix + ".r" + std::to_string(rank) + "of" + std::to_string(world) + ".cfrshard";
}

bool save_shard(const std::string& path, const Game& full, const Game& local, const ShardInfo& info, std::string& err) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) { err = "cannot open " + path + " for writing"; return false; }
    Writer w{f};
    w.ok = std::fwrite(kMagic, 1, 8, f) == 8;
    const FormatTag tag;
    w.ok = w.ok && std::fwrite(&tag, sizeof(tag), 1, f) == 1;
    // header of the full game (info / caller-order readbacks)
    Game head;
    head.V = full.V; head.P = full.P; head.Pc = full.Pc; head.zero_sum_2p = full.zero_sum_2p; head.D = full.D;
    head.num_terminals = full.num_terminals; head.num_chance = full.num_chance; head.num_decision = full.num_decision;
    head.max_infoset_nodes = full.max_infoset_nodes; head.depth_homogeneous = full.depth_homogeneous;
    head.max_abs_u = full.max_abs_u; head.level_ptr = full.level_ptr; head.H = full.H; head.Q = full.Q; head.C = full.C;
    head.h_int_of_caller = full.h_int_of_caller; head.h_caller_of_int = full.h_caller_of_int;
    head.qbase_int = full.qbase_int; head.qbase_caller = full.qbase_caller; head.owner_int = full.owner_int;
    game_fields(w, head);
    game_fields(w, const_cast<Game&>(local));
    info_fields(w, const_cast<ShardInfo&>(info));
    const bool closed = std::fclose(f) == 0;   // always close, then combine
    const bool ok = w.ok && closed;
    if (!ok) {
        err = "write failed: " + path;
        std::remove(path.c_str());   // no partial shard file left behind
    }
    return ok;
}

bool load_shard(const std::string& path, Game& head, Game& local, ShardInfo& info, std::string& err) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) { err = "cannot open " + path; return false; }
    Reader r{f};
    char magic[8];
    r.ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kMagic, 8) == 0;
    if (!r.ok) { std::fclose(f); err = "bad magic (or an older shard format) in " + path; return false; }
    FormatTag tag, want;
    r.ok = std::fread(&tag, sizeof(tag), 1, f) == 1 && tag.version == want.version &&
           tag.tile_bytes == want.tile_bytes && tag.seg_bytes == want.seg_bytes;
    if (!r.ok) { std::fclose(f); err = "shard format version / record layout mismatch in " + path; return false; }
    game_fields(r, head);
    game_fields(r, local);
    info_fields(r, info);
    std::fclose(f);
    if (!r.ok) err = "truncated or corrupt shard file " + path;
    return r.ok;
}

}  // namespace cfrb

extern "C" {

cfr_status cfr_game_save_shards(const cfr_game* g, int32_t world, const char* prefix) {
    if (!g || !prefix || world < 2) { cfrb_set_error("bad argument"); return CFR_ERR_INVALID_ARG; }
    for (int r = 0; r < world; ++r) {
        cfrb::Game local;
        cfrb::ShardInfo info;
        std::string err;
        if (!cfrb::build_shard(g->g, r, world, local, info, err)) { cfrb_set_error("shard: " + err); return CFR_ERR_INVALID_TREE; }
        if (!cfrb::save_shard(cfrb::shard_path(prefix, r, world), g->g, local, info, err)) {
            cfrb_set_error(err);
            return CFR_ERR_INVALID_ARG;
        }
    }
    return CFR_OK;
}

cfr_status cfr_game_load_shard(const char* prefix, int32_t rank, int32_t world, cfr_game** out) {
    if (!prefix || !out || world < 2 || rank < 0 || rank >= world) { cfrb_set_error("bad argument"); return CFR_ERR_INVALID_ARG; }
    *out = nullptr;
    cfr_game* G = new cfr_game();
    auto sh = std::make_shared<cfr_game::Shard>();
    std::string err;
    if (!cfrb::load_shard(cfrb::shard_path(prefix, rank, world), G->g, sh->local, sh->info, err)) {
        delete G;
        cfrb_set_error(err);
        return CFR_ERR_INVALID_ARG;
    }
    if (sh->info.rank != rank || sh->info.world != world) {
        delete G;
        cfrb_set_error("shard file " + cfrb::shard_path(prefix, rank, world) + " holds rank " +
                       std::to_string(sh->info.rank) + " of " + std::to_string(sh->info.world));
        return CFR_ERR_INVALID_ARG;
    }
    G->shard_only = true;
    G->shards.emplace(std::make_pair(rank, world), sh);
    *out = G;
    return CFR_OK;
}

}  // extern "C"
