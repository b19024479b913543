"""Pins of the CPU oracle against what the paper and the mathematics fix
(not against itself).  CPU only.  See DESIGN.md §3 for the list and citations."""
from fractions import Fraction
import itertools
import math

import numpy as np
import pytest

import gamegen
import oracle


# ----------------------------------------------------------------- structure
TABLE7 = {  # PAPER.md Table 7: nodes, terminals, infosets
    "kuhn": (58, 30, 12),
    "kuhn3": (617, 312, 48),
    "leduc": (9457, 5520, 936),
    "liars_dice": (294883, 147420, 24576),
}


@pytest.mark.parametrize("name", sorted(TABLE7))
def test_table7_counts(name):
    d = gamegen.by_name(name)
    assert (d.num_nodes, d.num_terminals, d.num_infosets) == TABLE7[name]


def test_goofspiel_and_synthetic_counts():
    d = gamegen.goofspiel()
    assert (d.num_nodes, d.num_terminals, d.num_infosets) == (55731, 14400, 9948)
    c = gamegen.synthetic_counts(40)
    assert (c["V"], c["T"], c["H"], c["Q"], c["D"]) == (965153641, 916896000, 1206440, 24128800, 11)
    for n in (1, 2, 3):
        d = gamegen.synthetic(n_types=n)
        c = gamegen.synthetic_counts(n)
        assert (d.num_nodes, d.num_terminals, d.num_infosets) == (c["V"], c["T"], c["H"])


def _sparsities(d):
    """PAPER.md Table 8 quantities from the game arrays."""
    V = d.num_nodes
    o = oracle.Oracle(d)
    Q, H = o.Q, o.H
    par = d.parent
    player_children = int(np.sum((par >= 0) & (d.player[np.maximum(par, 0)] >= 1)))
    depth = np.zeros(V, dtype=np.int64)
    order = np.argsort(par)  # parents before children is not guaranteed: iterate
    changed = True
    while changed:
        nd = np.where(par >= 0, depth[np.maximum(par, 0)] + 1, 0)
        changed = not np.array_equal(nd, depth)
        depth = nd
    D = int(depth.max())
    s_mqv = 1 - player_children / (Q * V)
    s_mhq = 1 - Q / (H * Q)
    s_g = 1 - (V - 1) / (V * V)
    s_l = np.mean([1 - np.sum(depth == l) / (V * V) for l in range(1, D + 1)])
    return [round(100 * x, 1) for x in (s_mqv, s_mhq, s_l, s_g)], D


def test_table8_kuhn_sparsities():
    sp, D = _sparsities(gamegen.kuhn(2))
    assert D == 5
    assert sp == [96.6, 91.7, 99.7, 98.3]


def test_table8_kuhn3_sparsities():
    sp, _ = _sparsities(gamegen.kuhn(3))
    assert sp[0] == 99.0 and sp[1] == 97.9 and sp[3] == 99.8  # P:718 ("99.9+" for L)
    assert sp[2] >= 99.9


# ------------------------------------------------------- exact accumulation
def test_slice_sum_order_free_and_accurate():
    rng = np.random.default_rng(0)
    for E in (1, 2, 3, 7):
        x = rng.uniform(-1, 1, size=2000) * 2.0 ** (E - 1) * rng.choice([1, 1e-3, 1e-9, 1e-17], size=2000)
        acc, dec = oracle.slice_sum(x, E)
        for s in range(3):
            acc2, dec2 = oracle.slice_sum(rng.permutation(x), E)
            assert np.array_equal(acc, acc2) and dec == dec2
        exact = sum(Fraction(float(v)) for v in x)
        bound = len(x) * Fraction(2) ** (E - 121) + abs(exact) * Fraction(2) ** -51 + Fraction(2) ** (E - 200)
        assert abs(Fraction(dec) - exact) <= bound
        accn, decn = oracle.slice_sum(-x, E)
        assert np.array_equal(accn, -acc) and decn == -dec


def test_slice_sum_on_grid_values_exact():
    x = np.array([0.5, 0.25, -0.125, 1.5, 3.0 * 2.0 ** -100])
    acc, dec = oracle.slice_sum(x, 2)
    assert dec == float(sum(Fraction(v) for v in x))


# ------------------------------------------------------------ closed forms
def _kuhn_equilibrium(d, alpha):
    """Kuhn equilibrium family (alpha in [0, 1/3]); returns sigma in qbase order."""
    keys = d.meta["infoset_keys"]
    bet = {}
    J, Qc, K = 0, 1, 2
    bet[(1, (J, ()))] = alpha
    bet[(1, (Qc, ()))] = 0.0
    bet[(1, (K, ()))] = 3 * alpha
    bet[(1, (J, (0, 1)))] = 0.0
    bet[(1, (Qc, (0, 1)))] = alpha + 1.0 / 3.0
    bet[(1, (K, (0, 1)))] = 1.0
    bet[(2, (J, (0,)))] = 1.0 / 3.0
    bet[(2, (J, (1,)))] = 0.0
    bet[(2, (Qc, (0,)))] = 0.0
    bet[(2, (Qc, (1,)))] = 1.0 / 3.0
    bet[(2, (K, (0,)))] = 1.0
    bet[(2, (K, (1,)))] = 1.0
    s = np.zeros(2 * len(keys))
    for h, k in enumerate(keys):
        s[2 * h + 1] = bet[k]
        s[2 * h] = 1.0 - bet[k]
    return s


@pytest.mark.parametrize("alpha", [0.0, 1.0 / 6.0, 1.0 / 3.0])
def test_kuhn_equilibrium_value(alpha):
    d = gamegen.kuhn(2)
    o = oracle.Oracle(d)
    s = _kuhn_equilibrium(d, alpha)
    ev = o.expected_values(s)
    assert abs(ev[0] + 1.0 / 18.0) <= 1e-15 and abs(ev[1] - 1.0 / 18.0) <= 1e-15
    ex = o.exploitability(s)
    assert abs(ex["nash_conv"]) <= 1e-15


def test_kuhn_uniform_closed_forms():
    o = oracle.Oracle(gamegen.kuhn(2))
    assert np.allclose(o.expected_values("current"), [0.125, -0.125], rtol=0, atol=1e-15)
    ex = o.exploitability("current")
    assert abs(ex["br"][0] - 0.5) <= 1e-15 and abs(ex["br"][1] - 5.0 / 12.0) <= 1e-15
    assert abs(ex["nash_conv"] - 11.0 / 12.0) <= 1e-15


def test_chance_only_game_value_zero():
    for P in (1, 2):
        o = oracle.Oracle(gamegen.chance_pm1(P))
        assert np.all(o.expected_values("current") == 0.0)


def test_single_decision_regret_and_rm():
    """payoffs (1, 0): r~ = (0.5, -0.5), sigma^(2) = (1, 0); sigma_bar(1) = sigma^(1)."""
    o = oracle.Oracle(gamegen.single_decision()).run(1, 0)
    st = o.state()
    assert np.array_equal(st["regret"], [0.5, -0.5])
    assert np.array_equal(st["sigma"], [1.0, 0.0])
    assert np.array_equal(st["avg"], [0.5, 0.5])
    o.run(1, 0)
    assert np.array_equal(o.state()["sigma"], [1.0, 0.0])


# ------------------------------------------------- brute force on tiny trees
def _tree(d):
    ch = [[] for _ in range(d.num_nodes)]
    for v in np.argsort(d.action, kind="stable"):
        p = d.parent[v]
        if p >= 0:
            ch[p].append(int(v))
    for p in range(d.num_nodes):
        ch[p].sort(key=lambda c: d.action[c])
    root = int(np.nonzero(d.parent < 0)[0][0])
    return ch, root


def _pure_strategies(d, o, player):
    hs = [h for h in range(o.H) if d.player[np.nonzero(d.infoset == h)[0][0]] == player]
    n = [int(o.qbase[h + 1] - o.qbase[h]) for h in hs]
    for choice in itertools.product(*[range(k) for k in n]):
        yield hs, choice


def test_best_response_equals_pure_strategy_enumeration():
    """Brute-force BR (PAPER.md P:59 max over Sigma_j; pure strategies suffice)."""
    d = gamegen.kuhn(2)
    o = oracle.Oracle(d)
    rng = np.random.default_rng(3)
    profiles = [None]
    for _ in range(4):
        s = np.zeros(o.Q)
        for h in range(o.H):
            w = rng.uniform(0.05, 1, size=o.qbase[h + 1] - o.qbase[h])
            s[o.qbase[h]:o.qbase[h + 1]] = w / w.sum()
        profiles.append(s)
    for prof in profiles:
        base = o.current_strategy() if prof is None else prof
        for pl in (1, 2):
            best = -math.inf
            for hs, choice in _pure_strategies(d, o, pl):
                s = base.copy()
                for h, a in zip(hs, choice):
                    s[o.qbase[h]:o.qbase[h + 1]] = 0.0
                    s[o.qbase[h] + a] = 1.0
                best = max(best, o.expected_values(s)[pl - 1])
            val, _ = o.best_response(pl, base)
            assert abs(val - best) <= 1e-12
            assert val >= o.expected_values(base)[pl - 1] - 1e-15


def _eq7_bruteforce(d, o, sigma):
    """r~(h,a) from the LITERAL Eq 6/7 with the override profile
    sigma|h->a, pi_check by Eq 2 and pi_hat by Eq 4 -- plain Python."""
    ch, root = _tree(d)
    P = d.num_players
    qb = o.qbase

    def prob(v, a, prof):
        pl = d.player[v]
        c = ch[v][a]
        return d.chance_prob[c] if pl == 0 else prof[qb[d.infoset[v]] + a]

    def value(v, prof):
        if d.player[v] < 0:
            return d.utility[v].copy()
        return sum(prob(v, a, prof) * value(c, prof) for a, c in enumerate(ch[v]))

    pc = {}
    ph = {}

    def reach(v, rc, rh):
        pc[v], ph[v] = rc, rh
        if d.player[v] < 0:
            return
        pl = d.player[v]
        for a, c in enumerate(ch[v]):
            s = prob(v, a, sigma)
            reach(c, [rc[j] * (s if pl != j + 1 else 1.0) for j in range(P)],
                  [rh[j] * (s if pl == j + 1 else 1.0) for j in range(P)])

    reach(root, [1.0] * P, [1.0] * P)
    rt = np.zeros(o.Q)
    pibar = np.zeros(o.H)
    for h in range(o.H):
        members = [int(v) for v in np.nonzero((d.infoset == h) & (d.player >= 1))[0]]
        i = int(d.player[members[0]])
        n = int(qb[h + 1] - qb[h])
        pibar[h] = sum(ph[m][i - 1] for m in members)
        base = sum(pc[m][i - 1] * value(m, sigma)[i - 1] for m in members)
        for a in range(n):
            over = sigma.copy()
            over[qb[h]:qb[h + 1]] = 0.0
            over[qb[h] + a] = 1.0
            rt[qb[h] + a] = sum(pc[m][i - 1] * value(m, over)[i - 1] for m in members) - base
    return rt, pibar


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 5, 8])
def test_iteration_one_matches_literal_eq7_eq5_eq9(seed):
    d = gamegen.random_game(seed, num_players=2 + seed % 2, max_nodes=300)
    o = oracle.Oracle(d)
    sigma1 = o.current_strategy()
    rt, pibar = _eq7_bruteforce(d, o, sigma1)
    o.run(1, 0)
    st = o.state()
    assert np.allclose(st["regret"], rt, rtol=0, atol=1e-13)
    assert np.allclose(st["sden"], pibar, rtol=0, atol=1e-13)      # w_1 = 1: S_den = pi_bar
    assert np.array_equal(st["avg"], sigma1)                       # sigma_bar(1) = sigma^(1)
    # Eq 9 applied to the literal regrets
    for h in range(o.H):
        r = rt[o.qbase[h]:o.qbase[h + 1]]
        pos = np.maximum(r, 0)
        want = pos / pos.sum() if pos.sum() > 1e-12 else np.full(len(r), 1.0 / len(r))
        assert np.allclose(st["sigma"][o.qbase[h]:o.qbase[h + 1]], want, atol=1e-9)


def test_cfr_plus_linear_weights_and_rm_plus():
    """Reading Q6: R <- max(R + r~, 0); S_num += t * pi_bar * sigma (w_t = t)."""
    d = gamegen.random_game(4, max_nodes=300)
    o = oracle.Oracle(d).run(1, 1)
    st1 = o.state()
    sig2 = st1["sigma"].copy()
    rt2, pibar2 = _eq7_bruteforce(d, o, sig2)
    o.run(1, 1)
    st2 = o.state()
    assert np.all(st2["regret"] >= 0)
    assert np.allclose(st2["regret"], np.maximum(st1["regret"] + rt2, 0), atol=1e-12)
    want_sden = st1["sden"] + 2 * pibar2
    assert np.allclose(st2["sden"], want_sden, atol=1e-12)
    h_of_q = np.repeat(np.arange(o.H), np.diff(o.qbase))
    assert np.allclose(st2["snum"], st1["snum"] + 2 * pibar2[h_of_q] * sig2, atol=1e-12)


# ------------------------------------------------------------- convergence
def test_kuhn_1000_value_and_2eps_bound():
    """BASELINE configs[0]: EV1 -> -1/18; |EV1 - v*| <= NashConv."""
    o = oracle.Oracle(gamegen.kuhn(2)).run(1000, 0)
    ev = o.expected_values()
    nc = o.exploitability()["nash_conv"]
    assert abs(ev[0] + 1.0 / 18.0) <= 1e-4
    assert abs(ev[0] + 1.0 / 18.0) <= nc
    assert ev[0] + ev[1] == 0.0


@pytest.mark.parametrize("game,variant", [("kuhn", 0), ("kuhn", 1), ("kuhn3", 0)])
def test_checkpoint_monotone_exploitability(game, variant):
    """SPEC S:665 / PAPER Fig 3: NashConv of sigma_bar falls at checkpoints."""
    o = oracle.Oracle(gamegen.by_name(game))
    vals = []
    done = 0
    for T in (10, 100, 1000, 5000):
        o.run(T - done, variant)
        done = T
        vals.append(o.exploitability()["nash_conv"])
    assert all(b < a for a, b in zip(vals, vals[1:])), vals
    assert vals[-1] < 1e-2


def test_f32_vs_f64_kuhn():
    a = oracle.Oracle(gamegen.kuhn(2), 64).run(1000, 0).average_strategy()
    b = oracle.Oracle(gamegen.kuhn(2), 32).run(1000, 0).average_strategy()
    assert np.max(np.abs(a - b)) <= 1e-3
    assert not np.array_equal(a, b)


def test_leduc_cfr_plus_value_bound():
    """Leduc value ~ -0.0856 (literature, not in PAPER.md): |EV1 - v| <= NashConv."""
    o = oracle.Oracle(gamegen.leduc()).run(500, 1)
    ex = o.exploitability()
    assert abs(ex["ev"][0] + 0.0856) <= ex["nash_conv"]
    assert ex["nash_conv"] < 0.05


def test_goofspiel_symmetric_value_bound():
    o = oracle.Oracle(gamegen.goofspiel()).run(100, 1)
    ex = o.exploitability()
    assert abs(ex["ev"][0]) <= ex["nash_conv"]


# ---- discounted variants (reading Q18: Brown & Sandholm's discounting of
# Eq 14 / Eq 15).  LCFR = DCFR(1, 1, 1), DCFR = DCFR(3/2, 0, 2).
BIASED_RPS = [[0.0, -1.0, 2.0], [1.0, 0.0, -1.0], [-1.0, 1.0, 0.0]]


@pytest.mark.parametrize("variant,power", [(2, 1), (3, 2)])
def test_discounted_average_is_polynomially_weighted(variant, power):
    """Unrolling the discount (S + x_t) * (t/(t+1))^g gives S_T = sum_t x_t t^g / (T+1)^g:
    the average strategy is the t^g-weighted average of the iterates (pi_bar is
    constant in a matrix game, so it cancels).  The recursion in the oracle must
    reproduce that closed form from its own recorded iterates."""
    d = gamegen.matrix_game(BIASED_RPS)
    o = oracle.Oracle(d, precision=64)
    T = 60
    sig = []
    for _ in range(T):
        sig.append(o.state()["sigma"].copy())
        o.run(1, variant)
    w = np.array([(t + 1) ** power for t in range(T)], dtype=np.float64)
    want = (w[:, None] * np.array(sig)).sum(0) / w.sum()
    got = o.average_strategy()
    assert np.allclose(got, want, rtol=1e-12, atol=1e-14), (got, want)
    # the iterates genuinely change and mix (the weighting is exercised)
    S = np.array(sig)
    assert ((S > 0.05) & (S < 0.95)).any() and np.abs(S[T // 2] - S[-1]).max() > 1e-3


def test_lcfr_regret_is_linearly_weighted():
    """LCFR: R_T = sum_t t r~_t / (T+1).  With the opponent fixed to its recorded
    strategies, player 1's instantaneous regrets in a matrix game are
    r~_t(i) = (A sigma2_t)_i - sigma1_t . A sigma2_t (Eq 7 at the root, pi_check = 1)."""
    A = np.array(BIASED_RPS)
    d = gamegen.matrix_game(BIASED_RPS)
    o = oracle.Oracle(d, precision=64)
    qb = o.qbase
    T = 40
    acc = np.zeros(3)
    for t in range(1, T + 1):
        s = o.state()["sigma"]
        # infoset ids follow the builder's order: 0 = rows (player 1), 1 = cols (player 2)
        s1, s2 = s[qb[0]:qb[1]], s[qb[1]:qb[2]]
        ua = A @ s2
        acc += t * (ua - s1 @ ua)
        o.run(1, 2)
    R1 = o.state()["regret"][qb[0]:qb[1]]
    assert np.allclose(R1, acc / (T + 1), rtol=1e-11, atol=1e-13), (R1, acc / (T + 1))


@pytest.mark.parametrize("variant", [2, 3])
def test_discounted_variants_converge_on_kuhn(variant):
    d = gamegen.kuhn(2)
    o = oracle.Oracle(d, precision=64)
    nc = []
    for T in (10, 100, 1000):
        o.run(T - o.state()["t"], variant)
        nc.append(o.exploitability()["nash_conv"])
    assert nc[0] > nc[1] > nc[2] and nc[2] < 2.5e-2, nc   # simultaneous updates: ~vanilla rate
    ev = o.expected_values()[0]
    assert abs(ev + 1.0 / 18.0) <= nc[2], (ev, nc)


# ---- CFR+ with alternating updates (variant 4, reading Q19)
def test_alternating_equals_simultaneous_for_one_player():
    """With one player there is nothing to alternate: variant 4 == CFR+ bit for bit."""
    d = gamegen.single_decision()
    a = oracle.Oracle(d).run(7, 4).state()
    b = oracle.Oracle(d).run(7, 1).state()
    for k in ("sigma", "regret", "snum", "sden"):
        assert np.array_equal(a[k], b[k]), k


def test_alternating_first_iteration_matrix_game():
    """Iteration 1 on a matrix game by direct enumeration: player 1 updates against
    the uniform column mix; player 2 then updates against player 1's NEW strategy."""
    A = np.array(BIASED_RPS)
    d = gamegen.matrix_game(BIASED_RPS)
    o = oracle.Oracle(d).run(1, 4)
    qb = o.qbase
    st = o.state()
    s2 = np.full(3, 1 / 3)
    u1 = A @ s2
    r1 = np.maximum(u1 - np.full(3, 1 / 3) @ u1, 0.0)
    s1_new = r1 / r1.sum()
    u2 = -(s1_new @ A)                     # player 2's payoff per column
    r2 = np.maximum(u2 - s2 @ u2, 0.0)
    s2_new = r2 / r2.sum() if r2.sum() > 0 else np.full(3, 1 / 3)
    assert np.allclose(st["regret"][qb[0]:qb[1]], r1, atol=1e-14)
    assert np.allclose(st["regret"][qb[1]:qb[2]], r2, atol=1e-14)   # members weighted by pi_check = sigma1_new(row)
    assert np.allclose(st["sigma"][qb[0]:qb[1]], s1_new, atol=1e-14)
    assert np.allclose(st["sigma"][qb[1]:qb[2]], s2_new, atol=1e-14)


def test_alternating_cfr_plus_converges_faster_on_kuhn():
    d = gamegen.kuhn(2)
    alt = oracle.Oracle(d).run(1000, 4).exploitability()["nash_conv"]
    sim = oracle.Oracle(d).run(1000, 1).exploitability()["nash_conv"]
    assert alt < sim and alt < 3e-3, (alt, sim)


@pytest.mark.parametrize("n_types,seed", [(2, 1), (3, 4)])
def test_sampled_first_iteration_regrets_match_full_oracle(n_types, seed):
    """oracle/sampled.py (used at full size, where the full oracle cannot run) against
    the full oracle: R^1 of every sampled deepest-level infoset, CFR and CFR+."""
    from oracle.sampled import first_iteration_regrets, qbase
    d = gamegen.synthetic(n_types=n_types, seed=seed)
    q = qbase(d)
    assert np.array_equal(q, oracle.Oracle(d).qbase)
    dec = np.flatnonzero(d.player > 0)
    rng = np.random.default_rng(seed)
    hs = np.unique(d.infoset[rng.choice(dec[-len(dec) // 10:], 40, replace=False)])
    for plus in (False, True):
        reg = oracle.Oracle(d).run(1, int(plus)).state()["regret"]
        res = first_iteration_regrets(d, hs, plus)
        for h in hs:
            ref = reg[q[h]:q[h + 1]]
            assert np.allclose(res[h], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max()), h
            assert np.abs(ref).max() > 0


# ------------------------------------------------------------- f32 mode (Q14)
# Reading Q14 ("both 64-bit and 32-bit floating-point data types"): in f32
# mode the utilities and sigma_0 are rounded to binary32 ONCE at load, all state
# is binary32, and every exact slice sum is decoded to binary64 and rounded ONCE
# to binary32.  The two games below are built so that each of those two rules
# changes a result macroscopically (a strategy or an ulp-exact regret).

def _one_decision(payoffs):
    b = gamegen.Builder("one_decision", 1)
    r = b.node(-1, -1)
    b.set_player(r, 1, "root", len(payoffs))
    for a, u in enumerate(payoffs):
        b.set_terminal(b.node(r, a), [u])
    return b.build(zero_sum=False)


def test_f32_rounds_utilities_once_at_load():
    """Payoffs (1 + 2^-30, 1): in binary64 action 0 is strictly better by 2^-30,
    so r~ = (+2^-31, -2^-31) (Eq 7, sigma^1 uniform) and sigma^2 = (1, 0) (Eq 9).
    Rounded to binary32 first, both payoffs are 1: r~ = (0, 0), sigma^2 uniform
    (Eq 9, z = 0).  An f32 mode that kept binary64 inputs would give (1, 0)."""
    d = _one_decision([1.0 + 2.0 ** -30, 1.0])
    s64 = oracle.Oracle(d, 64).run(1, 0).state()
    assert np.array_equal(s64["regret"], [2.0 ** -31, -(2.0 ** -31)])
    assert np.array_equal(s64["sigma"], [1.0, 0.0])
    s32 = oracle.Oracle(d, 32).run(1, 0).state()
    assert np.array_equal(s32["regret"], [0.0, 0.0])
    assert np.array_equal(s32["sigma"], [0.5, 0.5])


def _hidden_chance_decision():
    """Chance (1/2, 1/4, 1/4) -> one player-1 infoset (the outcome is hidden) with
    two actions; payoffs (2, -2), (3*2^-24, -3*2^-24) twice (all exact in binary32).
    Under sigma^1 every u(d) = 0, so the Eq 7 terms of action 0 are
    1/2 * 2 = 1 and 1/4 * 3*2^-24 = 0.75*2^-24 (twice)."""
    b = gamegen.Builder("hidden_chance", 1)
    r = b.node(-1, -1)
    b.set_chance(r)
    small = 3.0 * 2.0 ** -24
    for k, (p, u) in enumerate(((0.5, 2.0), (0.25, small), (0.25, small))):
        v = b.node(r, k, p)
        b.set_player(v, 1, "hidden", 2)
        b.set_terminal(b.node(v, 0), [u])
        b.set_terminal(b.node(v, 1), [-u])
    return b.build(zero_sum=False)


def test_f32_exact_sum_decoded_then_rounded_once():
    """r~(h, 0) = 1 + 1.5*2^-24 exactly (binary64 holds it).  Rounded once to
    binary32 that is 1 + 2^-23 (0.75 ulp rounds up); a running binary32 sum in
    node order gives 1 (each 0.375-ulp term rounds away).  The result may not
    depend on the node order (reading Q8)."""
    d = _hidden_chance_decision()
    r64 = oracle.Oracle(d, 64).run(1, 0).state()["regret"]
    assert r64[0] == 1.0 + 1.5 * 2.0 ** -24 and r64[1] == -r64[0]
    for desc in (d, d.shuffled(1), d.shuffled(2)):
        r32 = oracle.Oracle(desc, 32).run(1, 0).state()["regret"]
        assert r32[0] == 1.0 + 2.0 ** -23 and r32[1] == -r32[0], r32
    naive = np.float32(0)
    for t in (1.0, 0.75 * 2.0 ** -24, 0.75 * 2.0 ** -24):
        naive = np.float32(naive + np.float32(t))
    assert naive == np.float32(1.0)   # the order-dependent answer the rule excludes


def test_f32_kuhn_uniform_closed_forms():
    """Kuhn under sigma^1 in binary32: EV = (1/8, -1/8), BR = (1/2, 5/12),
    NashConv = 11/12, each within a few binary32 ulps (payoffs are
    small integers; only 1/3 and 1/2 are rounded)."""
    o = oracle.Oracle(gamegen.kuhn(2), 32)
    ulp = 2.0 ** -24
    ev = o.expected_values("current")
    assert abs(ev[0] - 0.125) <= 8 * ulp and abs(ev[1] + 0.125) <= 8 * ulp
    ex = o.exploitability("current")
    assert abs(ex["br"][0] - 0.5) <= 16 * ulp and abs(ex["br"][1] - 5.0 / 12.0) <= 16 * ulp
    assert abs(ex["nash_conv"] - 11.0 / 12.0) <= 32 * ulp
    # every readback is a binary32 number
    for x in list(ev) + list(ex["br"]):
        assert float(np.float32(x)) == x


def _eq7_bruteforce_f32(d, o, sigma):
    """_eq7_bruteforce in binary32 arithmetic: inputs rounded once (Q14), every
    product and sum a binary32 operation (plain Python over np.float32 scalars)."""
    f = np.float32
    ch, root = _tree(d)
    P = d.num_players
    qb = o.qbase
    util = d.utility.astype(np.float32)
    cp = d.chance_prob.astype(np.float32)
    sig = np.asarray(sigma, dtype=np.float32)

    def prob(v, a, prof):
        c = ch[v][a]
        return cp[c] if d.player[v] == 0 else prof[qb[d.infoset[v]] + a]

    def value(v, prof):
        if d.player[v] < 0:
            return util[v].copy()
        out = np.zeros(P, dtype=np.float32)
        for a, c in enumerate(ch[v]):
            out = (out + prob(v, a, prof) * value(c, prof)).astype(np.float32)
        return out

    pc, ph = {}, {}

    def reach(v, rc, rh):
        pc[v], ph[v] = rc, rh
        if d.player[v] < 0:
            return
        pl = d.player[v]
        for a, c in enumerate(ch[v]):
            s = prob(v, a, sig)
            reach(c, [f(rc[j] * (s if pl != j + 1 else f(1))) for j in range(P)],
                  [f(rh[j] * (s if pl == j + 1 else f(1))) for j in range(P)])

    reach(root, [f(1)] * P, [f(1)] * P)
    rt = np.zeros(o.Q)
    for h in range(o.H):
        members = [int(v) for v in np.nonzero((d.infoset == h) & (d.player >= 1))[0]]
        i = int(d.player[members[0]])
        n = int(qb[h + 1] - qb[h])
        # the literal Eq 6/7: sum_d pi_check(d) u(sigma|h->a, d) - sum_d pi_check(d) u(sigma, d)
        base = f(0)
        for m in members:
            base = f(base + f(pc[m][i - 1] * value(m, sig)[i - 1]))
        for a in range(n):
            over = sig.copy()
            over[qb[h]:qb[h + 1]] = 0
            over[qb[h] + a] = 1
            tot = f(0)
            for m in members:
                tot = f(tot + f(pc[m][i - 1] * value(m, over)[i - 1]))
            rt[qb[h] + a] = float(f(tot - base))
    return rt


@pytest.mark.parametrize("seed", [0, 1, 2, 5])
def test_f32_iteration_one_matches_literal_eq7_in_binary32(seed):
    """The f32 oracle's first-iteration regrets against the LITERAL Eq 6/7 evaluated
    in binary32 (a different formula: override profiles, no cancellation).  The two
    differ only by binary32 rounding: |d| <= 64 ulp(1) * max|u| (depth <= 6 sums of
    <= 4 terms on each side).  Every regret is a binary32 number, and it is within
    the same scale of the binary64 oracle's."""
    d = gamegen.random_game(seed, num_players=2 + seed % 2, max_nodes=300)
    o32 = oracle.Oracle(d, 32)
    sigma1 = o32.current_strategy()
    lit = _eq7_bruteforce_f32(d, o32, sigma1)
    got = o32.run(1, 0).state()["regret"]
    umax = float(np.abs(d.utility).max())
    assert np.all(np.abs(got - lit) <= 64 * 2.0 ** -24 * umax), np.abs(got - lit).max()
    for x in got:
        assert float(np.float32(x)) == x
    r64 = oracle.Oracle(d, 64).run(1, 0).state()["regret"]
    assert np.all(np.abs(got - r64) <= 64 * 2.0 ** -24 * umax)


@pytest.mark.parametrize("n_types,seed", [(2, 1), (3, 4)])
def test_sampled_pibar_rm_and_uniform_ev_match_full_oracle(n_types, seed):
    """oracle/sampled.py's pi_bar (Eq 5), regret matching (Eq 9) of the sampled R^1
    and the uniform-profile EV against the full oracle after one iteration."""
    from oracle.sampled import first_iteration_pibar, first_iteration_regrets, qbase, regret_matching, uniform_ev
    d = gamegen.synthetic(n_types=n_types, seed=seed)
    q = qbase(d)
    dec = np.flatnonzero(d.player > 0)
    rng = np.random.default_rng(seed)
    hs = np.unique(d.infoset[rng.choice(dec[-len(dec) // 10:], 30, replace=False)])
    for plus in (False, True):
        o = oracle.Oracle(d).run(1, int(plus))
        st = o.state()
        pib = first_iteration_pibar(d, hs)
        r1 = first_iteration_regrets(d, hs, plus)
        for h in hs:
            assert abs(st["sden"][h] - pib[h]) <= 1e-15 * pib[h] and pib[h] > 0
            assert np.allclose(st["sigma"][q[h]:q[h + 1]], regret_matching(r1[h]), rtol=1e-12, atol=1e-13)
        ev, mag = uniform_ev(d)
        assert np.all(np.abs(o.expected_values() - ev) <= 1e-14 * mag), (o.expected_values(), ev)
        assert np.all(mag > 0) and abs(ev[0] + ev[1]) <= 1e-15 * mag[0]


def _depths(d):
    dep = np.full(d.num_nodes, -1)
    order = []
    root = int(np.nonzero(d.parent < 0)[0][0])
    dep[root] = 0
    ch = [[] for _ in range(d.num_nodes)]
    for v in range(d.num_nodes):
        if d.parent[v] >= 0:
            ch[d.parent[v]].append(v)
    stack = [root]
    while stack:
        v = stack.pop()
        for c in ch[v]:
            dep[c] = dep[v] + 1
            stack.append(c)
    return dep


@pytest.mark.parametrize("seed", [5, 11, 33, 34])
def test_best_response_on_depth_spanning_infosets_equals_enumeration(seed):
    """Reading Q17: on perfect-recall games whose infosets pool nodes of different
    depths, the oracle's memoised recursive BR equals the max over every pure
    strategy of the player (max over Sigma_j; pure strategies suffice)."""
    d = gamegen.random_game(seed, num_players=2, span_depths=True, max_depth=5, max_nodes=80)
    dep = _depths(d)
    spans = [h for h in range(d.num_infosets) if len(set(dep[d.infoset == h])) > 1]
    assert spans, "fixture must pool nodes of several depths"
    o = oracle.Oracle(d)
    rng = np.random.default_rng(seed)
    base = np.zeros(o.Q)
    for h in range(o.H):
        w = rng.uniform(0.05, 1, size=o.qbase[h + 1] - o.qbase[h])
        base[o.qbase[h]:o.qbase[h + 1]] = w / w.sum()
    for pl in (1, 2):
        best = -math.inf
        for hs, choice in _pure_strategies(d, o, pl):
            s = base.copy()
            for h, a in zip(hs, choice):
                s[o.qbase[h]:o.qbase[h + 1]] = 0.0
                s[o.qbase[h] + a] = 1.0
            best = max(best, o.expected_values(s)[pl - 1])
        val, _ = o.best_response(pl, base)
        assert abs(val - best) <= 1e-12, (pl, val, best)


def test_exact_sums_near_the_largest_double():
    """Appendix B-4's exponent E = 1 + ceil(log2(2 max|u|)) evaluated without
    overflow: with payoffs (B, -B), B = 1.5e308 (2B is not finite), iteration 1 of
    vanilla CFR gives v = 0, r~ = (B, -B) exactly (S:529's closed form scaled), and
    sigma^(2) = (1, 0); iteration 2's term -B - B overflows (Eq 7)."""
    from gamegen.desc import Builder

    B = 1.5e308
    b = Builder("big", 1)
    r = b.node(-1, -1)
    b.set_player(r, 1, "root", 2)
    for a, u in enumerate((B, -B)):
        c = b.node(r, a)
        b.set_terminal(c, [u])
    o = oracle.Oracle(b.build(zero_sum=False)).run(1, 0)
    st = o.state()
    assert st["regret"].tolist() == [B, -B]
    assert st["sigma"].tolist() == [1.0, 0.0]
    assert o.expected_values("current").tolist() == [B]
