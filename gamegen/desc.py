"""GameDesc container and a tiny node builder (no CFR arithmetic here)."""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np


@dataclass
class GameDesc:
    name: str
    num_players: int
    parent: np.ndarray
    player: np.ndarray
    infoset: np.ndarray
    action: np.ndarray
    chance_prob: np.ndarray
    utility: np.ndarray  # [V, P]
    meta: dict = field(default_factory=dict)

    @property
    def num_nodes(self) -> int:
        return int(self.parent.shape[0])

    @property
    def num_infosets(self) -> int:
        return int(self.infoset.max()) + 1 if (self.infoset >= 0).any() else 0

    @property
    def num_terminals(self) -> int:
        return int((self.player == -1).sum())

    def shuffled(self, seed: int) -> "GameDesc":
        """Same game, nodes renumbered by a random permutation (root anywhere)."""
        rng = np.random.default_rng(seed)
        V = self.num_nodes
        perm = rng.permutation(V)          # new position -> old id
        new_of_old = np.empty(V, dtype=np.int64)
        new_of_old[perm] = np.arange(V, dtype=np.int64)
        par = self.parent[perm]
        par = np.where(par >= 0, new_of_old[np.maximum(par, 0)], -1)
        return GameDesc(self.name + f"~{seed}", self.num_players, par.astype(np.int64),
                        self.player[perm].copy(), self.infoset[perm].copy(), self.action[perm].copy(),
                        self.chance_prob[perm].copy(), self.utility[perm].copy(), dict(self.meta))

    def relabel_infosets(self, seed: int) -> "GameDesc":
        """Same game with the caller's infoset ids permuted (tests qbase mapping)."""
        H = self.num_infosets
        rng = np.random.default_rng(seed)
        p = rng.permutation(H).astype(np.int64)
        inf = np.where(self.infoset >= 0, p[np.maximum(self.infoset, 0)], -1)
        return GameDesc(self.name + f"^{seed}", self.num_players, self.parent.copy(), self.player.copy(),
                        inf.astype(np.int64), self.action.copy(), self.chance_prob.copy(),
                        self.utility.copy(), dict(self.meta))


class Builder:
    """Append-only node list.  Infoset keys are interned to dense ids in order of
    first appearance; the key must include the owning player."""

    def __init__(self, name: str, num_players: int):
        self.name = name
        self.P = num_players
        self.parent: list[int] = []
        self.player: list[int] = []
        self.infoset: list[int] = []
        self.action: list[int] = []
        self.chance: list[float] = []
        self.util: list[tuple] = []
        self._ids: dict = {}
        self._nact: dict = {}

    def node(self, parent: int, action: int, chance_prob: float = 0.0) -> int:
        self.parent.append(parent)
        self.player.append(-1)
        self.infoset.append(-1)
        self.action.append(action)
        self.chance.append(chance_prob)
        self.util.append((0.0,) * self.P)
        return len(self.parent) - 1

    def set_chance(self, v: int):
        self.player[v] = 0

    def set_player(self, v: int, player: int, key, n_actions: int):
        k = (player, key)
        if k not in self._ids:
            self._ids[k] = len(self._ids)
            self._nact[k] = n_actions
        elif self._nact[k] != n_actions:
            raise ValueError(f"infoset {k} has inconsistent action counts")
        self.player[v] = player
        self.infoset[v] = self._ids[k]

    def set_terminal(self, v: int, utility):
        assert len(utility) == self.P
        self.player[v] = -1
        self.util[v] = tuple(float(x) for x in utility)

    def build(self, **meta) -> GameDesc:
        keys = [None] * len(self._ids)
        for k, i in self._ids.items():
            keys[i] = k
        meta.setdefault("infoset_keys", keys)
        return GameDesc(
            self.name, self.P,
            np.asarray(self.parent, dtype=np.int64),
            np.asarray(self.player, dtype=np.int32),
            np.asarray(self.infoset, dtype=np.int64),
            np.asarray(self.action, dtype=np.int32),
            np.asarray(self.chance, dtype=np.float64),
            np.asarray(self.util, dtype=np.float64).reshape(len(self.parent), self.P),
            dict(meta),
        )
