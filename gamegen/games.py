"""Real-game fixtures (structure pinned by PAPER.md Table 7,
P:659-673).  Pure game rules -> GameDesc arrays; no CFR arithmetic."""
from __future__ import annotations

import numpy as np

from .desc import Builder, GameDesc


# --------------------------------------------------------------------------- Kuhn
def kuhn(num_players: int = 2) -> GameDesc:
    """Kuhn poker with P+1 cards, chained chance deals (P:659 rows kuhn_poker /
    kuhn_poker(players=3): 58/30/12 and 617/312/48).  Actions: 0 pass, 1 bet.
    A bet ends the game once every other player responded once (#actions = P + index
    of first bettor); otherwise the game ends when all P passed."""
    P = num_players
    cards = P + 1
    b = Builder(f"kuhn{P}", P)

    def betting(v, hand, hist):
        n = len(hist)
        first_bet = hist.index(1) if 1 in hist else None
        done = (first_bet is None and n == P) or (first_bet is not None and n == P + first_bet)
        if done:
            contrib = [1] * P
            if first_bet is None:
                contenders = list(range(P))
            else:
                contenders = []
                for k in range(first_bet, n):
                    pl = k % P
                    if hist[k] == 1:
                        contrib[pl] += 1
                        contenders.append(pl)
            winner = max(contenders, key=lambda p: hand[p])
            pot = sum(contrib)
            u = [-contrib[p] for p in range(P)]
            u[winner] = pot - contrib[winner]
            b.set_terminal(v, u)
            return
        pl = n % P
        b.set_player(v, pl + 1, (hand[pl], tuple(hist)), 2)
        for a in (0, 1):
            c = b.node(v, a)
            betting(c, hand, hist + [a])

    def deal(v, hand):
        b.set_chance(v)
        remaining = [c for c in range(cards) if c not in hand]
        for a, card in enumerate(remaining):
            c = b.node(v, a, 1.0 / len(remaining))
            if len(hand) + 1 < P:
                deal(c, hand + [card])
            else:
                betting(c, hand + [card], [])

    root = b.node(-1, -1)
    deal(root, [])
    return b.build(zero_sum=True)


# -------------------------------------------------------------------------- Leduc
def leduc() -> GameDesc:
    """Leduc hold'em (P:665 row leduc_poker: 9,457 nodes / 5,520 terminals / 936
    infosets).  6 cards J,J,Q,Q,K,K (rank = card // 2); raise 2 then 4; <= 2 raises
    per round; legal order fold, call, raise (fold only facing a bet)."""
    b = Builder("leduc", 2)
    raise_size = (2, 4)

    def showdown(hand, public, contrib):
        def strength(c):
            return (1 if c // 2 == public // 2 else 0, c // 2)
        s0, s1 = strength(hand[0]), strength(hand[1])
        if s0 > s1:
            return [contrib[1], -contrib[1]]
        if s1 > s0:
            return [-contrib[0], contrib[0]]
        return [0.0, 0.0]

    def betting(v, hand, public, rnd, hists, contrib, raises):
        cur = hists[rnd]
        pl = len(cur) % 2
        facing = contrib[1 - pl] > contrib[pl]
        legal = []
        if facing:
            legal.append("f")
        legal.append("c")
        if raises < 2:
            legal.append("r")
        key = (hand[pl], public, tuple(hists[0]), tuple(hists[1]))
        b.set_player(v, pl + 1, key, len(legal))
        for a, act in enumerate(legal):
            c = b.node(v, a)
            nh = [list(hists[0]), list(hists[1])]
            nh[rnd].append(act)
            nc = list(contrib)
            if act == "f":
                u = [0.0, 0.0]
                u[pl] = -contrib[pl]
                u[1 - pl] = contrib[pl]
                b.set_terminal(c, u)
            elif act == "c":
                nc[pl] = nc[1 - pl]
                if len(nh[rnd]) >= 2:
                    if rnd == 0:
                        b.set_chance(c)
                        rem = [x for x in range(6) if x not in hand]
                        for pa, card in enumerate(rem):
                            cc = b.node(c, pa, 1.0 / len(rem))
                            betting(cc, hand, card, 1, nh, nc, 0)
                    else:
                        b.set_terminal(c, showdown(hand, public, nc))
                else:
                    betting(c, hand, public, rnd, nh, nc, raises)
            else:  # raise
                nc[pl] = nc[1 - pl] + raise_size[rnd]
                betting(c, hand, public, rnd, nh, nc, raises + 1)

    root = b.node(-1, -1)
    b.set_chance(root)
    for a1 in range(6):
        c1 = b.node(root, a1, 1.0 / 6.0)
        b.set_chance(c1)
        rem = [x for x in range(6) if x != a1]
        for a2, card2 in enumerate(rem):
            c2 = b.node(c1, a2, 1.0 / 5.0)
            betting(c2, (a1, card2), -1, 0, [[], []], [1, 1], 0)
    return b.build(zero_sum=True)


# ---------------------------------------------------------------------- Liar's dice
def liars_dice(faces: int = 6) -> GameDesc:
    """Liar's dice, 1 die x `faces` per player (P:669 row liars_dice: 294,883 /
    147,420 / 24,576).  Bids 0..2*faces-1 quantity-major, strictly increasing;
    'liar' (last action index) legal after the first bid.  Reading (R16):
    the highest face is wild; the caller wins iff count(face) < quantity."""
    nb = 2 * faces
    b = Builder("liars_dice", 2)

    def node(v, dice, hist):
        pl = len(hist) % 2
        last = hist[-1] if hist else -1
        legal = list(range(last + 1, nb)) + (["liar"] if hist else [])
        b.set_player(v, pl + 1, (dice[pl], tuple(hist)), len(legal))
        for a, act in enumerate(legal):
            c = b.node(v, a)
            if act == "liar":
                q, f = last // faces + 1, last % faces + 1
                cnt = sum(1 for d in dice if d == f or d == faces)
                caller_wins = cnt < q
                u = [0.0, 0.0]
                u[pl] = 1.0 if caller_wins else -1.0
                u[1 - pl] = -u[pl]
                b.set_terminal(c, u)
            else:
                node(c, dice, hist + [act])

    root = b.node(-1, -1)
    b.set_chance(root)
    for d1 in range(1, faces + 1):
        c1 = b.node(root, d1 - 1, 1.0 / faces)
        b.set_chance(c1)
        for d2 in range(1, faces + 1):
            c2 = b.node(c1, d2 - 1, 1.0 / faces)
            node(c2, (d1, d2), [])
    return b.build(zero_sum=True)


# ------------------------------------------------------------------------ Goofspiel
def goofspiel(num_cards: int = 5) -> GameDesc:
    """Goofspiel, descending point cards, imperfect information, turn-based
    (55,731 nodes / 14,400 terminals / 9,948 infosets for 5
    cards).  P1 bids, then P2 bids without seeing it; infoset = (own past bids,
    public outcome sequence); win/loss returns."""
    n = num_cards
    b = Builder(f"goofspiel{n}", 2)

    def p1(v, h1, h2, outcomes, pts):
        hand = sorted(set(range(1, n + 1)) - set(h1))
        b.set_player(v, 1, (tuple(h1), tuple(outcomes)), len(hand))
        for a, card in enumerate(hand):
            c = b.node(v, a)
            p2(c, h1 + [card], h2, outcomes, pts)

    def p2(v, h1, h2, outcomes, pts):
        hand = sorted(set(range(1, n + 1)) - set(h2))
        b.set_player(v, 2, (tuple(h2), tuple(outcomes)), len(hand))
        turn = len(h2)
        prize = n - turn
        for a, card in enumerate(hand):
            c = b.node(v, a)
            c1 = h1[-1]
            np_ = list(pts)
            if c1 > card:
                oc = "W"
                np_[0] += prize
            elif c1 < card:
                oc = "L"
                np_[1] += prize
            else:
                oc = "T"
            if turn + 1 == n:
                s = float(np.sign(np_[0] - np_[1]))
                b.set_terminal(c, [s, -s])
            else:
                p1(c, h1, h2 + [card], outcomes + [oc], np_)

    root = b.node(-1, -1)
    p1(root, [], [], [], [0, 0])
    return b.build(zero_sum=True)


# ------------------------------------------------------------------- tiny fixtures
def chance_pm1(num_players: int = 2) -> GameDesc:
    """Root chance 0.5/0.5 to two terminals with payoffs +-1: EV 0."""
    b = Builder("chance_pm1", num_players)
    r = b.node(-1, -1)
    b.set_chance(r)
    for a, s in enumerate((1.0, -1.0)):
        c = b.node(r, a, 0.5)
        u = [s] + [-s] * (num_players - 1) if num_players > 1 else [s]
        b.set_terminal(c, u)
    return b.build(zero_sum=num_players == 2)


def single_decision() -> GameDesc:
    """One player-1 decision with two actions paying (1, 0)."""
    b = Builder("single_decision", 1)
    r = b.node(-1, -1)
    b.set_player(r, 1, "root", 2)
    for a, u in enumerate((1.0, 0.0)):
        c = b.node(r, a)
        b.set_terminal(c, [u])
    return b.build(zero_sum=False)


def signal_game() -> GameDesc:
    """Chance picks a state (0.5/0.5); P1 observes it and sends one of two messages;
    P2 sees only the message and replies.  15 nodes, 8 terminals, general-sum."""
    b = Builder("signal", 2)
    r = b.node(-1, -1)
    b.set_chance(r)
    for st in (0, 1):
        s = b.node(r, st, 0.5)
        b.set_player(s, 1, ("state", st), 2)
        for m in (0, 1):
            mv = b.node(s, m)
            b.set_player(mv, 2, ("msg", m), 2)
            for rep in (0, 1):
                t = b.node(mv, rep)
                match = 1.0 if rep == st else 0.0
                b.set_terminal(t, [2.0 * match - (0.5 if m == 1 else 0.0), match + 0.25 * rep])
    return b.build(zero_sum=False)


# ------------------------------------------------------------------- random games
def random_game(seed: int, max_depth: int = 6, max_branching: int = 4, num_players: int = 2,
                chance_fraction: float = 0.2, terminal_ramp: float = 0.6, pool: int = 2,
                zero_sum: bool | None = None, max_nodes: int = 4000, span_depths: bool = False) -> GameDesc:
    """Seeded random perfect-recall game (SPEC S:128-162 idea): infosets pool
    same-depth nodes of one player with the same own (infoset, action) history and a
    random bucket in [0, pool); |A(h)| is a function of that history so pooled nodes
    agree.  Payoffs uniform in [-1, 1] (zero-sum when P = 2 and zero_sum).
    span_depths: the depth is left out of the pooling key, so one infoset may hold
    nodes of several depths (still perfect recall: pooled nodes share the player's
    own history, and a member's descendants always extend it)."""
    rng = np.random.default_rng(seed)
    P = num_players
    if zero_sum is None:
        zero_sum = (P == 2 and seed % 2 == 0)
    b = Builder(f"random{seed}", P)
    nact_of: dict = {}
    count = [0]

    def gen(v, depth, own):
        count[0] += 1
        term = depth >= max_depth or count[0] > max_nodes or (
            depth > 0 and rng.random() < terminal_ramp * depth / max_depth)
        if term:
            u = rng.uniform(-1.0, 1.0, size=P)
            u = np.round(u * 64.0) / 64.0
            if zero_sum:
                u[1] = -u[0]
            b.set_terminal(v, list(u))
            return
        if rng.random() < chance_fraction:
            b.set_chance(v)
            k = int(rng.integers(2, max_branching + 1))
            w = rng.uniform(0.1, 1.0, size=k)
            p = w / w.sum()
            for a in range(k):
                c = b.node(v, a, float(p[a]))
                gen(c, depth + 1, own)
            return
        pl = int(rng.integers(1, P + 1))
        dkey = -1 if span_depths else depth
        hkey = (pl, dkey, own[pl])
        if hkey not in nact_of:
            nact_of[hkey] = int(rng.integers(1 if rng.random() < 0.1 else 2, max_branching + 1))
        k = nact_of[hkey]
        bucket = int(rng.integers(0, pool))
        key = (dkey, own[pl], bucket)
        b.set_player(v, pl, key, k)
        h = b.infoset[v]
        for a in range(k):
            c = b.node(v, a)
            nown = dict(own)
            nown[pl] = own[pl] + ((h, a),)
            gen(c, depth + 1, nown)

    r = b.node(-1, -1)
    gen(r, 0, {p: () for p in range(1, P + 1)})
    return b.build(zero_sum=bool(zero_sum))


def matrix_game(A, name: str = "matrix") -> GameDesc:
    """Two-player zero-sum normal-form game as a tree: player 1 picks a row at the
    root, player 2 (one infoset: it does not see the row) picks a column; payoff
    (A[r][c], -A[r][c]).  Strategies stay mixed, so CFR variants differ."""
    A = [list(map(float, row)) for row in A]
    m, k = len(A), len(A[0])
    b = Builder(name, 2)
    r = b.node(-1, -1)
    b.set_player(r, 1, "rows", m)
    for i in range(m):
        c = b.node(r, i)
        b.set_player(c, 2, "cols", k)
        for j in range(k):
            t = b.node(c, j)
            b.set_terminal(t, [A[i][j], -A[i][j]])
    return b.build(zero_sum=True)
