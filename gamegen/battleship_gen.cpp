// Battleship game-tree generator (test / bench INPUTS only; no CFR arithmetic).
//
// The paper's Experiment 2 workload (Table 5 at P:570-602,
// Table 7 rows at P:676-698): OpenSpiel's battleship with parameters (board
// width, board height, ship sizes, shots per player), ship values all 1
// (P:570 caption).  Rules (reading Q20; they reproduce Table 7's node,
// terminal and infoset counts, tests/test_gamegen.py):
//   * placement: ship k = 0, 1, ... is placed by player 1, then by player 2;
//     a ship of size 1 has one placement per cell, a longer one a horizontal and
//     a vertical placement per fitting cell; ships of one player do not overlap;
//   * shooting: players alternate (player 1 first), num_shots shots each, any of
//     the W*H cells (repeated shots allowed); a player whose ships are all sunk
//     ends the game at once;
//   * a ship cell counts as hit once: a repeated shot on it is reported as a hit
//     again but sinks nothing new;
//   * observations: a player sees its own placements, every shot's cell, and
//     whether its own shots hit; a ship's sinking is announced to the shooter;
//   * utility: u_i = (opponent ships sunk by i) - loss_multiplier * (own ships
//     sunk), OpenSpiel's default loss_multiplier = 2 (general-sum).
// Nodes are emitted in DFS pre-order (any order is valid input, Def. 2.1).
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

struct Params {
    int W, H, S, shots;
    int size[8];
    double loss;
};

struct Gen {
    Params p;
    std::vector<int64_t> parent;
    std::vector<int32_t> player, action;
    std::vector<int64_t> infoset;
    std::vector<double> util;
    std::unordered_map<std::string, int64_t> ids;
    // state
    int cells_of[2][8][8];   // [player][ship][k] cell indices of placed ships
    int placed[2];
    int hits[2][8];          // hits taken by [player][ship]
    int sunk[2];
    int shots_done[2];
    std::vector<int> board[2];   // cell -> ship index + 1 (0 = water)
    std::vector<int> struck[2];  // cell -> times shot (a ship cell counts as hit once)
    std::string key[2];          // observation history of each player

    int64_t emit(int64_t par, int act) {
        parent.push_back(par);
        action.push_back(act);
        player.push_back(-1);
        infoset.push_back(-1);
        util.push_back(0.0);
        util.push_back(0.0);
        return (int64_t)parent.size() - 1;
    }
    void decision(int64_t v, int pl) {
        std::string k = key[pl - 1];
        k.push_back((char)pl);
        auto it = ids.find(k);
        int64_t id;
        if (it == ids.end()) {
            id = (int64_t)ids.size();
            ids.emplace(k, id);
        } else {
            id = it->second;
        }
        player[v] = pl;
        infoset[v] = id;
    }
    void terminal(int64_t v) {
        player[v] = -1;
        util[2 * v] = (double)sunk[1] - p.loss * (double)sunk[0];
        util[2 * v + 1] = (double)sunk[0] - p.loss * (double)sunk[1];
    }
    // legal placements of player pl's next ship: lists of cells
    std::vector<std::vector<int>> placements(int pl) {
        std::vector<std::vector<int>> out;
        const int k = placed[pl];
        const int sz = p.size[k];
        const std::vector<int>& b = board[pl];
        for (int o = 0; o < (sz == 1 ? 1 : 2); ++o)
            for (int r = 0; r < p.H; ++r)
                for (int c = 0; c < p.W; ++c) {
                    if (o == 0 && c + sz > p.W) continue;
                    if (o == 1 && r + sz > p.H) continue;
                    std::vector<int> cells;
                    bool ok = true;
                    for (int j = 0; j < sz && ok; ++j) {
                        const int cell = o == 0 ? r * p.W + c + j : (r + j) * p.W + c;
                        if (b[cell]) ok = false;
                        cells.push_back(cell);
                    }
                    if (ok) out.push_back(cells);
                }
        return out;
    }
    void place_phase(int64_t v, int turn) {
        // turn = 2k + (pl - 1): ship k of player pl
        if (turn == 2 * p.S) {
            shoot(v, 0);
            return;
        }
        const int pl = turn & 1;
        decision(v, pl + 1);
        const auto opts = placements(pl);
        for (int a = 0; a < (int)opts.size(); ++a) {
            const int64_t c = emit(v, a);
            const int k = placed[pl];
            for (int j = 0; j < (int)opts[a].size(); ++j) {
                board[pl][opts[a][j]] = k + 1;
                cells_of[pl][k][j] = opts[a][j];
            }
            placed[pl]++;
            key[pl].push_back('P');
            key[pl].push_back((char)a);
            place_phase(c, turn + 1);
            key[pl].resize(key[pl].size() - 2);
            placed[pl]--;
            for (int cell : opts[a]) board[pl][cell] = 0;
        }
    }
    void shoot(int64_t v, int turn) {
        const int pl = turn & 1;   // shooter
        if (shots_done[0] == p.shots && shots_done[1] == p.shots) {
            terminal(v);
            return;
        }
        decision(v, pl + 1);
        const int op = pl ^ 1;
        for (int cell = 0; cell < p.W * p.H; ++cell) {
            const int64_t c = emit(v, cell);
            const int ship = board[op][cell];   // 0 = water
            const bool fresh = struck[op][cell]++ == 0;
            int sunk_now = 0;
            if (ship && fresh) {
                hits[op][ship - 1]++;
                if (hits[op][ship - 1] == p.size[ship - 1]) { sunk[op]++; sunk_now = 1; }
            }
            shots_done[pl]++;
            const size_t l0 = key[pl].size(), l1 = key[op].size();
            key[pl].push_back('S');
            key[pl].push_back((char)cell);
            key[pl].push_back((char)(ship ? (sunk_now ? 2 : 1) : 0));
            key[op].push_back('O');
            key[op].push_back((char)cell);
            if (sunk[op] == p.S) terminal(c);
            else shoot(c, turn + 1);
            key[pl].resize(l0);
            key[op].resize(l1);
            shots_done[pl]--;
            if (ship && fresh) {
                if (sunk_now) sunk[op]--;
                hits[op][ship - 1]--;
            }
            struck[op][cell]--;
        }
    }
};

}  // namespace

extern "C" {

void* battleship_generate(int W, int H, const int* sizes, int S, int shots, double loss) {
    if (W < 1 || H < 1 || W * H > 120 || S < 1 || S > 8 || shots < 1) return nullptr;
    Gen* g = new Gen();
    g->p.W = W;
    g->p.H = H;
    g->p.S = S;
    g->p.shots = shots;
    g->p.loss = loss;
    for (int k = 0; k < S; ++k) g->p.size[k] = sizes[k];
    g->board[0].assign(W * H, 0);
    g->board[1].assign(W * H, 0);
    g->struck[0].assign(W * H, 0);
    g->struck[1].assign(W * H, 0);
    g->placed[0] = g->placed[1] = 0;
    g->sunk[0] = g->sunk[1] = 0;
    g->shots_done[0] = g->shots_done[1] = 0;
    std::memset(g->hits, 0, sizeof(g->hits));
    const int64_t root = g->emit(-1, -1);
    g->place_phase(root, 0);
    return g;
}

int64_t battleship_num_nodes(void* h) { return (int64_t)static_cast<Gen*>(h)->parent.size(); }

int64_t battleship_num_infosets(void* h) { return (int64_t)static_cast<Gen*>(h)->ids.size(); }

void battleship_copy(void* h, int64_t* parent, int32_t* player, int64_t* infoset, int32_t* action, double* util) {
    Gen* g = static_cast<Gen*>(h);
    const size_t V = g->parent.size();
    std::memcpy(parent, g->parent.data(), V * sizeof(int64_t));
    std::memcpy(player, g->player.data(), V * sizeof(int32_t));
    std::memcpy(infoset, g->infoset.data(), V * sizeof(int64_t));
    std::memcpy(action, g->action.data(), V * sizeof(int32_t));
    std::memcpy(util, g->util.data(), V * 2 * sizeof(double));
}

void battleship_free(void* h) { delete static_cast<Gen*>(h); }

}  // extern "C"
