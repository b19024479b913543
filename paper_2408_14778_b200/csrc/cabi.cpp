// Game half of the C ABI (include/cfr_b200.h) + error plumbing.
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "game.hpp"

namespace {
thread_local std::string g_last_error;
}

void cfrb_set_error(const std::string& msg) { g_last_error = msg; }

extern "C" {

const char* cfr_status_string(cfr_status s) {
    switch (s) {
        case CFR_OK: return "CFR_OK";
        case CFR_ERR_INVALID_ARG: return "CFR_ERR_INVALID_ARG";
        case CFR_ERR_INVALID_TREE: return "CFR_ERR_INVALID_TREE";
        case CFR_ERR_UNSUPPORTED: return "CFR_ERR_UNSUPPORTED";
        case CFR_ERR_CUDA: return "CFR_ERR_CUDA";
        case CFR_ERR_NCCL: return "CFR_ERR_NCCL";
        case CFR_ERR_OOM: return "CFR_ERR_OOM";
        case CFR_ERR_NUMERICAL: return "CFR_ERR_NUMERICAL";
    }
    return "CFR_ERR_UNKNOWN";
}

const char* cfr_last_error(void) { return g_last_error.c_str(); }

cfr_status cfr_game_create(const cfr_game_desc* desc, cfr_game** out) {
    if (!desc || !out) {
        cfrb_set_error("NULL argument");
        return CFR_ERR_INVALID_ARG;
    }
    *out = nullptr;
    try {
        cfr_game* g = new cfr_game();
        std::string err;
        if (!cfrb::build_game(desc, g->g, err)) {
            delete g;
            cfrb_set_error(err);
            return CFR_ERR_INVALID_TREE;
        }
        *out = g;
        return CFR_OK;
    } catch (const std::bad_alloc&) {
        cfrb_set_error("host allocation failed while flattening the game");
        return CFR_ERR_OOM;
    } catch (const std::exception& e) {
        cfrb_set_error(std::string("internal error: ") + e.what());
        return CFR_ERR_INVALID_ARG;
    }
}

void cfr_game_destroy(cfr_game* g) { delete g; }

cfr_status cfr_game_info(const cfr_game* gg, cfr_game_info_t* o) {
    if (!gg || !o) {
        cfrb_set_error("NULL argument");
        return CFR_ERR_INVALID_ARG;
    }
    const cfrb::Game& g = gg->g;
    o->num_nodes = g.V;
    o->num_terminals = g.num_terminals;
    o->num_decision = g.num_decision;
    o->num_chance = g.num_chance;
    o->num_infosets = g.H;
    o->num_pairs = g.Q;
    o->num_players = g.P;
    o->depth = g.D;
    o->max_infoset_nodes = g.max_infoset_nodes;
    o->depth_homogeneous = g.depth_homogeneous ? 1 : 0;
    o->zero_sum_2p = g.zero_sum_2p ? 1 : 0;
    return CFR_OK;
}

cfr_status cfr_game_qbase(const cfr_game* gg, int64_t* qbase) {
    if (!gg || !qbase) {
        cfrb_set_error("NULL argument");
        return CFR_ERR_INVALID_ARG;
    }
    std::memcpy(qbase, gg->g.qbase_caller.data(), gg->g.qbase_caller.size() * sizeof(int64_t));
    return CFR_OK;
}

cfr_status cfr_game_canonical(const cfr_game* gg, int64_t* canon_of_input, int64_t* level_ptr) {
    if (!gg) {
        cfrb_set_error("NULL argument");
        return CFR_ERR_INVALID_ARG;
    }
    const cfrb::Game& g = gg->g;
    if (canon_of_input && gg->shard_only) {
        cfrb_set_error("canonical order is not stored in a shard file");
        return CFR_ERR_UNSUPPORTED;
    }
    if (canon_of_input) std::memcpy(canon_of_input, g.canon_of_input.data(), g.V * sizeof(int64_t));
    if (level_ptr) std::memcpy(level_ptr, g.level_ptr.data(), g.level_ptr.size() * sizeof(int64_t));
    return CFR_OK;
}

}  // extern "C"
