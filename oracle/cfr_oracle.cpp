// ============================================================================
// CPU ORACLE for arXiv 2408.14778 -- TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.  It shares no code, header, table or
// helper with the CUDA product (paper_2408_14778_b200/); it reads the same
// C-ABI input arrays (gamegen/) and nothing else.
//
// What it computes: plain recursive, simultaneous-update CFR and CFR+ (and the
// discounted variants LCFR / DCFR of reading Q18) following
// the paper's DEFINITIONS step by step (SURVEY.md §8(c) "Oracle per iteration"):
//   * Eq 1   u_check(v,i): recursive expected payoff, children summed
//                        in ascending action order starting from +0.
//   * Eq 2   pi_check(v,i): path product, own actions replaced by 1.
//   * Eq 4  pi_hat(v,i): path product of player i's own actions
//                        (reading Q1: the recursion's pi_check is a typo for pi_hat).
//   * Eq 3/6/7 r~(h,a) in the cancelled form
//                        sum_{d in h} pi_check(d,i) * (u(child(d,a),i) - u(d,i))
//                        (reading Q2: never divide by pi~).
//   * Eq 5 pi_bar(h) = sum_{d in h} pi_hat(d,i).
//   * Eq 8/15 regrets stored CUMULATIVELY (reading Q4);
//                        CFR+: R <- max(R + r~, +0) (reading Q6).
//   * Eq 9 regret matching, uniform 1/|A(h)| when sum of positives = 0.
//   * Eq 10 average strategy as the quotient of running sums
//                        S_num / S_den (reading Q5), weight w_t = 1 (CFR) or t (CFR+).
//   * Cross-node sums (the per-infoset sums of Eq 3/5/7 and the BR sums) are
//     accumulated EXACTLY as three 40-bit int64 slices (reading Q8, SURVEY.md
//     Appendix B-4), so their value does not depend on summation order.
//   * FP environment (reading Q9): IEEE RNE, no FMA contraction
//     (-ffp-contract=off), no fast-math.  f32 mode (reading Q14): inputs rounded
//     to float once, all state float, sliced sums decoded to double then float.
//   * Readbacks: EV under sigma_bar, best response with ties to the
//     lowest action, NashConv = sum_i (BR_i - EV_i), exploitability = NashConv/P.
// ============================================================================
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

namespace {

thread_local std::string g_err;
constexpr int kMaxP = 16;
constexpr int kSlices = 3;   // K = 3 slices of 40 bits

// ---- exact accumulation (Appendix B-4), written independently of the product --
inline void slice_add(int64_t* acc, double x, int E) {
    for (int k = 1; k <= kSlices; ++k) {
        double scaled = std::ldexp(x, 40 * k - E);      // exact power-of-two scaling
        long long c = std::llrint(scaled);               // round half to even
        acc[k - 1] += (int64_t)c;
        x = x - std::ldexp((double)c, E - 40 * k);       // exact remainder
    }
}
inline double slice_decode(const int64_t* acc, int E) {
    double a = std::ldexp((double)acc[0], E - 40);
    double b = std::ldexp((double)acc[1], E - 80);
    double c = std::ldexp((double)acc[2], E - 120);
    return (a + b) + c;
}

struct Game {
    int64_t V = 0;
    int P = 0;
    int64_t root = -1;
    std::vector<int64_t> cstart;   // [V+1] children of v at clist[cstart[v] .. cstart[v+1])
    std::vector<int64_t> clist;    // ordered by incoming action
    std::vector<int32_t> player;
    std::vector<int64_t> infoset;
    std::vector<double> cprob;
    std::vector<double> util;      // [V*P]
    int64_t H = 0, Q = 0;
    std::vector<int64_t> qbase;    // [H+1], caller infoset order
    std::vector<int32_t> nact;     // [H]
    std::vector<int32_t> owner;    // [H]
    std::vector<int64_t> mstart, mlist;  // members of each infoset
    int E = 1;
};

template <class R>
struct Solver {
    const Game& g;
    std::vector<R> cprob, util;    // inputs rounded to R once (Q14)
    std::vector<R> sigma, regret, snum, sden;
    std::vector<int64_t> acc_r, acc_p;
    std::vector<R> stk;            // scratch stack for child values
    size_t sp = 0;
    int64_t t = 0;
    int variant = 0;

    explicit Solver(const Game& gg) : g(gg) {
        cprob.resize(g.V);
        util.resize(g.V * (size_t)g.P);
        for (int64_t v = 0; v < g.V; ++v) cprob[v] = (R)g.cprob[v];
        for (size_t k = 0; k < util.size(); ++k) util[k] = (R)g.util[k];
        sigma.assign(g.Q, (R)0);
        regret.assign(g.Q, (R)0);
        snum.assign(g.Q, (R)0);
        sden.assign(g.H, (R)0);
        acc_r.assign(g.Q * kSlices, 0);
        acc_p.assign(g.H * kSlices, 0);
        // sigma^(T=1) = 1/|A(h)|
        for (int64_t h = 0; h < g.H; ++h)
            for (int64_t q = g.qbase[h]; q < g.qbase[h + 1]; ++q) sigma[q] = (R)1 / (R)g.nact[h];
    }

    R* push(int64_t n) {
        if (sp + n > stk.size()) stk.resize(std::max(stk.size() * 2, sp + n + 1024));
        R* p = stk.data() + sp;
        sp += n;
        return p;
    }

    // One recursive CFR visit (Eq 1, 2, 4, 7 cancelled form, 5).  pc = pi_check(v,.)
    // (Eq 2), ph = pi_hat(v,.) (Eq 4); out = u_check(v,.) (Eq 1).
    void walk(int64_t v, const R* pc, const R* ph, R* out) {
        const int P = g.P;
        const int pl = g.player[v];
        if (pl < 0) {
            for (int j = 0; j < P; ++j) out[j] = util[v * P + j];
            return;
        }
        const int64_t c0 = g.cstart[v], n = g.cstart[v + 1] - g.cstart[v];
        R pc2[kMaxP], ph2[kMaxP], cv[kMaxP];
        for (int j = 0; j < P; ++j) out[j] = (R)0;
        if (pl == 0) {  // chance: sigma_0 multiplies every player's pi_check (Eq 2)
            for (int64_t a = 0; a < n; ++a) {
                const int64_t c = g.clist[c0 + a];
                const R s = cprob[c];
                for (int j = 0; j < P; ++j) { pc2[j] = pc[j] * s; ph2[j] = ph[j]; }
                walk(c, pc2, ph2, cv);
                for (int j = 0; j < P; ++j) out[j] = out[j] + s * cv[j];
            }
            return;
        }
        const int i = pl - 1;
        const int64_t h = g.infoset[v], qb = g.qbase[h];
        const size_t mark = sp;
        R* ci = push(n);
        for (int64_t a = 0; a < n; ++a) {
            const int64_t c = g.clist[c0 + a];
            const R s = sigma[qb + a];
            for (int j = 0; j < P; ++j) {
                pc2[j] = (j != i) ? pc[j] * s : pc[j];
                ph2[j] = (j == i) ? ph[j] * s : ph[j];
            }
            walk(c, pc2, ph2, cv);
            ci = stk.data() + mark;  // stack may have grown
            for (int j = 0; j < P; ++j) out[j] = out[j] + s * cv[j];
            ci[a] = cv[i];
        }
        ci = stk.data() + mark;
        const R cf = pc[i];
        for (int64_t a = 0; a < n; ++a) {
            const R term = cf * (ci[a] - out[i]);
            slice_add(&acc_r[(qb + a) * kSlices], (double)term, g.E);
        }
        slice_add(&acc_p[h * kSlices], (double)ph[i], 1);
        sp = mark;
    }

    // Per-infoset update: Eq 10 running sums, Eq 8/15 cumulative regret (CFR or
    // CFR+), Eq 9 regret matching.  Variants 2 (linear CFR) and 3 (DCFR with
    // alpha = 3/2, beta = 0, gamma = 2) apply Brown & Sandholm's discounting to
    // Eq 14 / Eq 15 as P:399 suggests (reading Q18): after iteration t's terms are
    // added, positive regrets are multiplied by t^a/(t^a+1), the others by
    // t^b/(t^b+1), and both average-strategy sums by (t/(t+1))^g.
    void update_infoset(int64_t h) {
        const int64_t qb = g.qbase[h], n = g.nact[h];
        const R pibar = (R)slice_decode(&acc_p[h * kSlices], 1);
        const R w = (variant == 1 || variant == 4) ? (R)t : (R)1;
        const R wp = w * pibar;
        // discount factors of iteration t (only correctly rounded operations)
        const R tt = (R)t;
        R dpos = (R)1, dneg = (R)1, dsum = (R)1;
        if (variant == 2) {            // LCFR: alpha = beta = gamma = 1
            const R f = tt / (tt + (R)1);
            dpos = f;
            dneg = f;
            dsum = f;
        } else if (variant == 3) {     // DCFR(3/2, 0, 2): t^(3/2) = t * sqrt(t), t^0 = 1
            const R a = tt * std::sqrt(tt);
            dpos = a / (a + (R)1);
            dneg = (R)1 / ((R)1 + (R)1);
            const R f = tt / (tt + (R)1);
            dsum = f * f;
        }
        for (int64_t a = 0; a < n; ++a) {
            const int64_t q = qb + a;
            const R rt = (R)slice_decode(&acc_r[q * kSlices], g.E);
            if (variant == 0) {
                regret[q] = regret[q] + rt;
            } else if (variant == 1 || variant == 4) {
                const R x = regret[q] + rt;
                regret[q] = (x > (R)0) ? x : (R)0;
            } else {
                const R x = regret[q] + rt;
                regret[q] = (x > (R)0) ? x * dpos : x * dneg;
            }
            if (variant == 2 || variant == 3) snum[q] = (snum[q] + wp * sigma[q]) * dsum;
            else snum[q] = snum[q] + wp * sigma[q];
        }
        if (variant == 2 || variant == 3) sden[h] = (sden[h] + wp) * dsum;
        else sden[h] = sden[h] + wp;
        R z = (R)0;
        for (int64_t a = 0; a < n; ++a) {
            const R r = regret[qb + a];
            z = z + ((r > (R)0) ? r : (R)0);
        }
        for (int64_t a = 0; a < n; ++a) {
            const R r = regret[qb + a];
            const R pos = (r > (R)0) ? r : (R)0;
            sigma[qb + a] = (z > (R)0) ? pos / z : (R)1 / (R)n;
        }
    }

    // One iteration.  Simultaneous updates (variants 0-3): one walk, every infoset
    // updated.  Variant 4 = CFR+ with ALTERNATING updates (Tammelin's published
    // form, reading Q19): for players i = 1..P in turn, a full walk under the
    // current profile (already holding the players updated earlier this
    // iteration), then only player i's infosets are updated (RM+, w_t = t).
    void iterate() {
        t += 1;
        const int passes = (variant == 4) ? g.P : 1;
        for (int pass = 1; pass <= passes; ++pass) {
            std::fill(acc_r.begin(), acc_r.end(), 0);
            std::fill(acc_p.begin(), acc_p.end(), 0);
            R pc[kMaxP], ph[kMaxP], out[kMaxP];
            for (int j = 0; j < g.P; ++j) { pc[j] = (R)1; ph[j] = (R)1; }
            sp = 0;
            walk(g.root, pc, ph, out);
            for (int64_t h = 0; h < g.H; ++h)
                if (variant != 4 || g.owner[h] == pass) update_infoset(h);
        }
    }

    void average(std::vector<R>& avg) const {
        avg.resize(g.Q);
        for (int64_t h = 0; h < g.H; ++h)
            for (int64_t q = g.qbase[h]; q < g.qbase[h + 1]; ++q)
                avg[q] = (sden[h] > (R)0) ? snum[q] / sden[h] : (R)1 / (R)g.nact[h];
    }

    // Eq 1 under an arbitrary profile `st` (values only).
    void value(int64_t v, const std::vector<R>& st, R* out) const {
        const int P = g.P;
        const int pl = g.player[v];
        if (pl < 0) {
            for (int j = 0; j < P; ++j) out[j] = util[v * P + j];
            return;
        }
        R cv[kMaxP];
        for (int j = 0; j < P; ++j) out[j] = (R)0;
        const int64_t c0 = g.cstart[v], n = g.cstart[v + 1] - g.cstart[v];
        for (int64_t a = 0; a < n; ++a) {
            const int64_t c = g.clist[c0 + a];
            const R s = (pl == 0) ? cprob[c] : st[g.qbase[g.infoset[v]] + a];
            value(c, st, cv);
            for (int j = 0; j < P; ++j) out[j] = out[j] + s * cv[j];
        }
    }

    // ---- best response of player `bi` (1-based) against profile st ----------
    std::vector<R> cfr_reach;      // pi_check(v, bi) under st (Eq 2)
    std::vector<R> memo;
    std::vector<uint8_t> have;
    std::vector<int32_t> br_act;   // per infoset: -1 unknown, -2 in progress
    int bi = 0;
    const std::vector<R>* bst = nullptr;
    bool br_error = false;

    void reach_walk(int64_t v, R pc) {
        cfr_reach[v] = pc;
        const int pl = g.player[v];
        if (pl < 0) return;
        const int64_t c0 = g.cstart[v], n = g.cstart[v + 1] - g.cstart[v];
        for (int64_t a = 0; a < n; ++a) {
            const int64_t c = g.clist[c0 + a];
            R s = (pl == 0) ? cprob[c] : (*bst)[g.qbase[g.infoset[v]] + a];
            reach_walk(c, (pl == bi) ? pc : pc * s);
        }
    }

    int32_t best_action(int64_t h) {
        if (br_act[h] >= 0) return br_act[h];
        if (br_act[h] == -2) { br_error = true; return 0; }   // imperfect recall cycle
        br_act[h] = -2;
        const int64_t n = g.nact[h];
        std::vector<int64_t> acc(n * kSlices, 0);
        for (int64_t m = g.mstart[h]; m < g.mstart[h + 1]; ++m) {
            const int64_t d = g.mlist[m];
            const R cf = cfr_reach[d];
            for (int64_t a = 0; a < n; ++a) {
                const R val = br_value(g.clist[g.cstart[d] + a]);
                const R term = cf * val;
                slice_add(&acc[a * kSlices], (double)term, g.E);
            }
        }
        int32_t best = 0;
        R bv = (R)slice_decode(&acc[0], g.E);
        for (int64_t a = 1; a < n; ++a) {
            const R x = (R)slice_decode(&acc[a * kSlices], g.E);
            if (x > bv) { bv = x; best = (int32_t)a; }
        }
        br_act[h] = best;
        return best;
    }

    R br_value(int64_t v) {
        if (have[v]) return memo[v];
        const int pl = g.player[v];
        R out;
        if (pl < 0) {
            out = util[v * g.P + (bi - 1)];
        } else if (pl == bi) {
            const int32_t a = best_action(g.infoset[v]);
            out = br_value(g.clist[g.cstart[v] + a]);
        } else {
            out = (R)0;
            const int64_t c0 = g.cstart[v], n = g.cstart[v + 1] - g.cstart[v];
            for (int64_t a = 0; a < n; ++a) {
                const int64_t c = g.clist[c0 + a];
                const R s = (pl == 0) ? cprob[c] : (*bst)[g.qbase[g.infoset[v]] + a];
                out = out + s * br_value(c);
            }
        }
        memo[v] = out;
        have[v] = 1;
        return out;
    }

    bool best_response(const std::vector<R>& st, int player, R* value_out, int32_t* actions) {
        bi = player;
        bst = &st;
        br_error = false;
        cfr_reach.assign(g.V, (R)0);
        memo.assign(g.V, (R)0);
        have.assign(g.V, 0);
        br_act.assign(g.H, -1);
        reach_walk(g.root, (R)1);
        *value_out = br_value(g.root);
        if (actions) for (int64_t h = 0; h < g.H; ++h) actions[h] = br_act[h];
        return !br_error;
    }
};

struct Handle {
    Game g;
    int precision = 64;
    void* solver = nullptr;
    ~Handle() {
        if (precision == 32) delete (Solver<float>*)solver;
        else delete (Solver<double>*)solver;
    }
};

bool build_game(Game& g, int64_t V, int P, const int64_t* parent, const int32_t* player,
                const int64_t* infoset, const int32_t* action, const double* cprob, const double* util) {
    if (V <= 0 || P < 1 || P > kMaxP) { g_err = "bad V or P"; return false; }
    g.V = V; g.P = P;
    g.player.assign(player, player + V);
    g.infoset.assign(infoset, infoset + V);
    g.cprob.assign(cprob, cprob + V);
    g.util.assign(util, util + V * (size_t)P);
    g.cstart.assign(V + 1, 0);
    for (int64_t v = 0; v < V; ++v) {
        if (parent[v] < 0) {
            if (g.root >= 0) { g_err = "two roots"; return false; }
            g.root = v;
        } else {
            if (parent[v] >= V) { g_err = "parent out of range"; return false; }
            g.cstart[parent[v] + 1]++;
        }
    }
    if (g.root < 0) { g_err = "no root"; return false; }
    for (int64_t v = 0; v < V; ++v) g.cstart[v + 1] += g.cstart[v];
    g.clist.assign(V, -1);
    for (int64_t v = 0; v < V; ++v) {
        if (parent[v] < 0) continue;
        const int64_t p = parent[v];
        const int64_t n = g.cstart[p + 1] - g.cstart[p];
        if (action[v] < 0 || action[v] >= n) { g_err = "action out of range at node " + std::to_string(v); return false; }
        int64_t& slot = g.clist[g.cstart[p] + action[v]];
        if (slot != -1) { g_err = "duplicate action at node " + std::to_string(v); return false; }
        slot = v;
    }
    int64_t H = 0;
    for (int64_t v = 0; v < V; ++v) {
        const int64_t n = g.cstart[v + 1] - g.cstart[v];
        if (player[v] < 0 && n != 0) { g_err = "terminal with children"; return false; }
        if (player[v] >= 0 && n == 0) { g_err = "decision node without children"; return false; }
        if (player[v] > P) { g_err = "bad player"; return false; }
        if (player[v] >= 1) {
            if (infoset[v] < 0) { g_err = "player node without infoset"; return false; }
            H = std::max(H, infoset[v] + 1);
        }
    }
    g.H = H;
    g.nact.assign(H, -1);
    g.owner.assign(H, -1);
    std::vector<int64_t> cnt(H + 1, 0);
    for (int64_t v = 0; v < V; ++v) {
        if (player[v] < 1) continue;
        const int64_t h = infoset[v];
        const int32_t n = (int32_t)(g.cstart[v + 1] - g.cstart[v]);
        if (g.nact[h] < 0) { g.nact[h] = n; g.owner[h] = player[v]; }
        else if (g.nact[h] != n || g.owner[h] != player[v]) { g_err = "inconsistent infoset " + std::to_string(h); return false; }
        cnt[h + 1]++;
    }
    g.qbase.assign(H + 1, 0);
    for (int64_t h = 0; h < H; ++h) {
        if (g.nact[h] < 0) { g_err = "infoset ids not dense"; return false; }
        g.qbase[h + 1] = g.qbase[h] + g.nact[h];
    }
    g.Q = g.qbase[H];
    g.mstart.assign(H + 1, 0);
    for (int64_t h = 0; h < H; ++h) g.mstart[h + 1] = g.mstart[h] + cnt[h + 1];
    g.mlist.assign(g.mstart[H], 0);
    std::vector<int64_t> fill(g.mstart.begin(), g.mstart.end() - 1);
    for (int64_t v = 0; v < V; ++v)
        if (player[v] >= 1) g.mlist[fill[infoset[v]]++] = v;
    return true;
}

template <class R>
int compute_E(const Game& g) {
    // E = 1 + ceil(log2(2 * max|u|)) over the utilities rounded to R (Appendix B-4)
    double m = 0.0;
    for (int64_t v = 0; v < g.V; ++v)
        if (g.player[v] < 0)
            for (int j = 0; j < g.P; ++j) m = std::max(m, std::fabs((double)(R)g.util[v * g.P + j]));
    if (m == 0.0) return 1;
    // ceil(log2(2m)) = 1 + ceil(log2 m), taken on m (2m overflows above DBL_MAX / 2)
    int e;
    const double f = std::frexp(m, &e);   // m = f * 2^e, f in [0.5, 1)
    const int ceil_log2 = (f == 0.5) ? e - 1 : e;
    return 2 + ceil_log2;
}

}  // namespace

template <class R>
static void run_impl(Solver<R>* s, int32_t variant, int64_t T) {
    s->variant = variant;
    for (int64_t k = 0; k < T; ++k) s->iterate();
}

template <class R>
static void state_impl(Solver<R>* s, double* sigma, double* regret, double* snum, double* sden,
                       double* avg, int64_t* t) {
    const Game& g = s->g;
    for (int64_t q = 0; q < g.Q; ++q) {
        if (sigma) sigma[q] = (double)s->sigma[q];
        if (regret) regret[q] = (double)s->regret[q];
        if (snum) snum[q] = (double)s->snum[q];
    }
    if (sden) for (int64_t hh = 0; hh < g.H; ++hh) sden[hh] = (double)s->sden[hh];
    if (avg) {
        std::vector<R> a;
        s->average(a);
        for (int64_t q = 0; q < g.Q; ++q) avg[q] = (double)a[q];
    }
    if (t) *t = s->t;
}

template <class R>
static std::vector<R> pick(Solver<R>* s, int32_t which, const double* strategy) {
    std::vector<R> st;
    if (which == 0) s->average(st);
    else if (which == 1) st = s->sigma;
    else { st.resize(s->g.Q); for (int64_t q = 0; q < s->g.Q; ++q) st[q] = (R)strategy[q]; }
    return st;
}

template <class R>
static void ev_impl(Solver<R>* s, int32_t which, const double* strategy, double* out) {
    std::vector<R> st = pick(s, which, strategy);
    R o[kMaxP];
    s->value(s->g.root, st, o);
    for (int j = 0; j < s->g.P; ++j) out[j] = (double)o[j];
}

template <class R>
static int br_impl(Solver<R>* s, int32_t which, const double* strategy, int32_t player, double* value,
                   int32_t* actions) {
    std::vector<R> st = pick(s, which, strategy);
    R v;
    if (!s->best_response(st, player, &v, actions)) { g_err = "best response: infoset cycle (imperfect recall)"; return 1; }
    *value = (double)v;
    return 0;
}

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

void* oracle_create(int64_t V, int32_t P, const int64_t* parent, const int32_t* player,
                    const int64_t* infoset, const int32_t* action, const double* cprob,
                    const double* util, int32_t precision) {
    Handle* hd = new Handle();
    if (!build_game(hd->g, V, P, parent, player, infoset, action, cprob, util)) { delete hd; return nullptr; }
    hd->precision = precision;
    if (precision == 32) {
        hd->g.E = compute_E<float>(hd->g);
        hd->solver = new Solver<float>(hd->g);
    } else {
        hd->g.E = compute_E<double>(hd->g);
        hd->solver = new Solver<double>(hd->g);
    }
    return hd;
}

void oracle_destroy(void* h) { delete (Handle*)h; }

void oracle_dims(void* hp, int64_t* out /* V, P, H, Q, E, root */) {
    Handle* h = (Handle*)hp;
    out[0] = h->g.V; out[1] = h->g.P; out[2] = h->g.H; out[3] = h->g.Q; out[4] = h->g.E; out[5] = h->g.root;
}

void oracle_qbase(void* hp, int64_t* qbase) {
    Handle* h = (Handle*)hp;
    std::copy(h->g.qbase.begin(), h->g.qbase.end(), qbase);
}


int oracle_run(void* hp, int32_t variant, int64_t T) {
    Handle* h = (Handle*)hp;
    if (variant < 0 || variant > 4) { g_err = "bad variant"; return 1; }
    if (h->precision == 32) run_impl((Solver<float>*)h->solver, variant, T);
    else run_impl((Solver<double>*)h->solver, variant, T);
    return 0;
}


void oracle_state(void* hp, double* sigma, double* regret, double* snum, double* sden, double* avg, int64_t* t) {
    Handle* h = (Handle*)hp;
    if (h->precision == 32) state_impl((Solver<float>*)h->solver, sigma, regret, snum, sden, avg, t);
    else state_impl((Solver<double>*)h->solver, sigma, regret, snum, sden, avg, t);
}

// which: 0 = average strategy, 1 = current strategy, 2 = `strategy` argument


void oracle_expected_values(void* hp, int32_t which, const double* strategy, double* out) {
    Handle* h = (Handle*)hp;
    if (h->precision == 32) ev_impl((Solver<float>*)h->solver, which, strategy, out);
    else ev_impl((Solver<double>*)h->solver, which, strategy, out);
}


int oracle_best_response(void* hp, int32_t which, const double* strategy, int32_t player, double* value,
                         int32_t* actions) {
    Handle* h = (Handle*)hp;
    if (player < 1 || player > h->g.P) { g_err = "bad player"; return 1; }
    if (h->precision == 32) return br_impl((Solver<float>*)h->solver, which, strategy, player, value, actions);
    return br_impl((Solver<double>*)h->solver, which, strategy, player, value, actions);
}

// NashConv = sum_i (BR_i - EV_i) (ascending i, in double); exploitability = NashConv / P
int oracle_exploitability(void* hp, int32_t which, const double* strategy, double* nash_conv,
                          double* expl, double* br, double* ev) {
    Handle* h = (Handle*)hp;
    const int P = h->g.P;
    double evs[kMaxP];
    oracle_expected_values(hp, which, strategy, evs);
    double nc = 0.0;
    for (int i = 1; i <= P; ++i) {
        double b;
        if (oracle_best_response(hp, which, strategy, i, &b, nullptr)) return 1;
        if (br) br[i - 1] = b;
        nc = nc + (b - evs[i - 1]);
    }
    if (ev) for (int j = 0; j < P; ++j) ev[j] = evs[j];
    *nash_conv = nc;
    *expl = nc / (double)P;
    return 0;
}

// Exact-accumulation primitive exposed for its own pin tests.
void oracle_slice_sum(const double* x, int64_t n, int32_t E, int64_t* acc3, double* decoded) {
    acc3[0] = acc3[1] = acc3[2] = 0;
    for (int64_t k = 0; k < n; ++k) slice_add(acc3, x[k], E);
    *decoded = slice_decode(acc3, E);
}

}  // extern "C"
