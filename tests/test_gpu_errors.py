"""Error paths of the C ABI on the GPU: NaN / Inf detection (CFR_ERR_NUMERICAL,
SPEC S:469 via SURVEY §8(b): "returns CFR_ERR_NUMERICAL and sets cfr_last_error
with the iteration index on NaN/Inf").

The first iteration that overflows follows in closed form from Eq 1 and Eq 7 on
games built for it (the oracle's exact slice sums have no defined value for a
non-finite term, so it is not the reference here); the device must report
exactly that iteration, through each kernel family."""
import dataclasses

import numpy as np
import pytest

import gamegen
import paper_2408_14778_b200 as pb
from gamegen.desc import Builder

pytestmark = pytest.mark.gpu

CFR_ERR_NUMERICAL = 7


def overflow_decision(big: float):
    """One player-1 decision of a zero-sum 2-player game paying (+big, -big).
    Iteration 1 (uniform): v = 0, regrets (big, -big) are finite; iteration 2
    (sigma = (1, 0) for vanilla CFR): v = big and the term of action 1 is
    -big - big = -inf (Eq 7)."""
    b = Builder("overflow", 2)
    r = b.node(-1, -1)
    b.set_player(r, 1, "root", 2)
    for a, u in enumerate((big, -big)):
        c = b.node(r, a)
        b.set_terminal(c, [u, -u])
    return b.build(zero_sum=True)


def saturated(desc, big: float):
    """Every utility replaced by +-big (its sign): a node whose children mix signs
    has |u(child) - v| > big for some child, which overflows for big > max/2."""
    return dataclasses.replace(desc, utility=np.sign(desc.utility) * big, name=desc.name + f"~{big:g}")


def expect_numerical(desc, variant: str, precision: int, flags: int, t_run: int, t_bad: int):
    s = pb.Solver(pb.Game(desc), variant=variant, precision=precision, flags=flags)
    with pytest.raises(pb.NativeError) as ei:
        s.run(t_run)
    assert ei.value.status == CFR_ERR_NUMERICAL, ei.value
    assert f"iteration {t_bad}" in str(ei.value), (str(ei.value), t_bad)
    return s


@pytest.mark.parametrize("precision,big", [(64, 1.5e308), (32, 3.0e38)])
@pytest.mark.parametrize("flags", [0, pb.FLAG_NO_TINY, pb.FLAG_NO_TINY | pb.FLAG_NO_GRAPH])
def test_overflow_reports_iteration(cuda, precision, big, flags):
    expect_numerical(overflow_decision(big), "cfr", precision, flags, 5, 2)   # overflow_decision's closed form


def test_finite_run_is_ok(cuda):
    """The same game at a harmless scale runs clean (no false positive)."""
    s = pb.Solver(pb.Game(overflow_decision(1.0)), variant="cfr", precision=64)
    s.run(5)
    assert s.iteration == 5


@pytest.mark.parametrize("precision,big", [(64, 1.7e308), (32, 3.3e38)])
def test_overflow_streaming_kernel(cuda, precision, big):
    """Saturated synthetic through k_bwd_stream (forced): the device flags the
    oracle's first non-finite iteration."""
    desc = saturated(gamegen.synthetic(n_types=2, seed=1), big)
    # iteration 1 (uniform sigma, every reach > 0): a deepest decision node whose
    # terminal children carry both signs, unevenly, has a term u - v (Eq 7) beyond
    # the largest finite value (v = Eq 1 under the uniform strategy)
    term = desc.player == -1
    par, u = desc.parent[term], desc.utility[term, 0]
    s1 = np.bincount(par, weights=u / big, minlength=desc.num_nodes)
    cnt = np.bincount(par, minlength=desc.num_nodes)
    leaf_parents = (cnt > 0) & (cnt == np.bincount(desc.parent[desc.parent >= 0], minlength=desc.num_nodes))
    v = np.where(cnt > 0, s1 / np.maximum(cnt, 1), 0.0) * big
    fmax = float(np.finfo(np.float64 if precision == 64 else np.float32).max)
    assert (np.abs(u - v[par]) > fmax)[leaf_parents[par]].any()
    s = expect_numerical(desc, "cfr", precision, pb.FLAG_FORCE_STREAM, 6, 1)
    assert "k_bwd_stream" in s.level_kernels()


@pytest.mark.parametrize("precision,big", [(64, 1.7e308), (32, 3.3e38)])
@pytest.mark.parametrize("name", ["leduc", "goofspiel"])
def test_overflow_subtree_mode(cuda, name, precision, big):
    """A saturated game through the subtree mode (k_sub + k_sub_update, the default
    for these games) reports the same first non-finite iteration as the per-level
    kernels (CFR_FLAG_NO_SUBTREE)."""
    desc = saturated(gamegen.by_name(name), big)
    ref = pb.Solver(pb.Game(desc), variant="cfr", precision=precision, flags=pb.FLAG_NO_SUBTREE)
    with pytest.raises(pb.NativeError) as ei:
        ref.run(8)
    assert ei.value.status == CFR_ERR_NUMERICAL, ei.value
    import re
    t_bad = int(re.search(r"iteration (\d+)", str(ei.value)).group(1))
    s = expect_numerical(desc, "cfr", precision, 0, 8, t_bad)
    assert "k_sub" in s.level_kernels()
