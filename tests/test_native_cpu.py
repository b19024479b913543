"""CPU-side tests of the C-ABI library: it loads, exports every symbol the header
declares, canonicalises bit-exactly like an independent Python BFS, and validates
inputs (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import gamegen
import paper_2408_14778_b200 as pb
from paper_2408_14778_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cfr_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cfr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = pb.load()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cfr_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def python_bfs(d):
    """Independent canonical order: BFS from the root with
    children in ascending incoming-action order."""
    V = d.num_nodes
    children = [[] for _ in range(V)]
    for v in range(V):
        p = int(d.parent[v])
        if p >= 0:
            children[p].append((int(d.action[v]), v))
    root = int(np.nonzero(d.parent < 0)[0][0])
    order = [root]
    level_ptr = [0, 1]
    frontier = [root]
    while frontier:
        nxt = []
        for v in frontier:
            nxt.extend(c for _, c in sorted(children[v]))
        if nxt:
            order.extend(nxt)
            level_ptr.append(len(order))
        frontier = nxt
    canon = np.empty(V, dtype=np.int64)
    canon[np.asarray(order)] = np.arange(V)
    return canon, np.asarray(level_ptr, dtype=np.int64)


@pytest.mark.parametrize("name", ["kuhn", "kuhn3", "leduc", "goofspiel", "random:3", "random:11"])
@pytest.mark.parametrize("shuffle", [False, True])
def test_canonical_flattening_bit_exact(name, shuffle):
    d = gamegen.by_name(name)
    if shuffle:
        d = d.shuffled(17)
    g = pb.Game(d)
    canon, lp = g.canonical()
    want_c, want_lp = python_bfs(d)
    assert np.array_equal(canon, want_c)
    assert np.array_equal(lp, want_lp)
    assert g.D == len(want_lp) - 2
    qb = g.qbase()
    nact = np.zeros(d.num_infosets, dtype=np.int64)
    for v in np.nonzero(d.player >= 1)[0]:
        nact[d.infoset[v]] = np.sum(d.parent == v)
    assert np.array_equal(qb, np.concatenate([[0], np.cumsum(nact)]))


def test_game_info_table7():
    for name, (V, T, H) in {"kuhn": (58, 30, 12), "kuhn3": (617, 312, 48), "leduc": (9457, 5520, 936)}.items():
        g = pb.Game(gamegen.by_name(name))
        assert (g.info["num_nodes"], g.info["num_terminals"], g.info["num_infosets"]) == (V, T, H)
        assert g.info["depth_homogeneous"] == 1
    assert pb.Game(gamegen.kuhn(2)).info["zero_sum_2p"] == 1
    assert pb.Game(gamegen.kuhn(2)).info["depth"] == 5
    assert pb.Game(gamegen.signal_game()).info["zero_sum_2p"] == 0


def _bad(d, **changes):
    import copy
    e = copy.deepcopy(d)
    for k, (idx, val) in changes.items():
        getattr(e, k)[idx] = val
    return e


def test_validation_errors():
    d = gamegen.kuhn(2)
    cases = [
        _bad(d, parent=(5, -1)),                       # two roots
        _bad(d, action=(5, 7)),                        # action out of range
        _bad(d, chance_prob=(1, 0.6)),                 # chance probs don't sum to 1
        _bad(d, player=(int(np.nonzero(d.player == -1)[0][0]), 1)),  # "player" node w/o children
        _bad(d, parent=(3, 3)),                        # self-parent
    ]
    u = d.utility.copy()
    u[np.nonzero(d.player == -1)[0][0], 0] = np.nan
    e = _bad(d)
    e.utility = u
    cases.append(e)
    for bad in cases:
        with pytest.raises(pb.NativeError) as ei:
            pb.Game(bad)
        assert ei.value.name in ("CFR_ERR_INVALID_TREE", "CFR_ERR_INVALID_ARG")
        assert len(str(ei.value)) > 20


def test_chance_060_060_rejected():
    """chance node with children 0.6, 0.6 is invalid."""
    b = gamegen.Builder("bad", 1)
    r = b.node(-1, -1)
    b.set_chance(r)
    for a in range(2):
        c = b.node(r, a, 0.6)
        b.set_terminal(c, [1.0])
    with pytest.raises(pb.NativeError, match="sum"):
        pb.Game(b.build())


def test_one_node_game():
    """a single terminal root is valid (D = 0)."""
    b = gamegen.Builder("one", 1)
    r = b.node(-1, -1)
    b.set_terminal(r, [0.0])
    g = pb.Game(b.build())
    assert g.D == 0 and g.V == 1 and g.H == 0


def test_status_strings():
    L = pb.load()
    assert L.cfr_status_string(0) == b"CFR_OK"
    assert L.cfr_status_string(7) == b"CFR_ERR_NUMERICAL"


def test_solver_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = pb.Game(gamegen.kuhn(2))
    with pytest.raises(RuntimeError, match="CUDA"):
        pb.Solver(g)


def test_shard_files_roundtrip(tmp_path):
    """DESIGN.md §9 shard files: one writer, each rank loads its own view."""
    g = pb.Game(gamegen.goofspiel())
    prefix = str(tmp_path / "goof")
    g.save_shards(4, prefix)
    for r in range(4):
        h = pb.Game.load_shard(prefix, r, 4)
        assert (h.V, h.H, h.Q, h.D) == (g.V, g.H, g.Q, g.D)
        assert np.array_equal(h.qbase(), g.qbase())
        assert h.shard_info(r, 4) == g.shard_info(r, 4)
        with pytest.raises(pb.NativeError):
            h.shard_info((r + 1) % 4, 4)
        with pytest.raises(pb.NativeError):
            h.canonical()
    with pytest.raises(pb.NativeError):
        pb.Game.load_shard(str(tmp_path / "missing"), 0, 4)
