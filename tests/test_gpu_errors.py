"""Error paths of the C ABI on the GPU: NaN / Inf detection (CFR_ERR_NUMERICAL,
SPEC S:469 via SURVEY §8(b): "returns CFR_ERR_NUMERICAL and sets cfr_last_error
with the iteration index on NaN/Inf").

The first iteration whose state holds a non-finite value is taken from the
ORACLE, run one iteration at a time on the same game; the device must report
exactly that iteration, through each kernel family."""
import dataclasses

import numpy as np
import pytest

import gamegen
import oracle
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


def scaled(desc, factor: float):
    return dataclasses.replace(desc, utility=desc.utility * factor, name=desc.name + f"*{factor:g}")


def first_bad_iteration(desc, variant: int, precision: int, t_max: int) -> int:
    o = oracle.Oracle(desc, precision=precision)
    for t in range(1, t_max + 1):
        o.run(1, variant)
        st = o.state()
        if not all(np.isfinite(st[k]).all() for k in ("sigma", "regret")):
            return t
    return 0


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
    desc = overflow_decision(big)
    t_bad = first_bad_iteration(desc, 0, precision, 5)
    assert t_bad == 2   # the closed form in overflow_decision's docstring
    expect_numerical(desc, "cfr", precision, flags, 5, t_bad)


def test_finite_run_is_ok(cuda):
    """The same game at a harmless scale runs clean (no false positive)."""
    s = pb.Solver(pb.Game(overflow_decision(1.0)), variant="cfr", precision=64)
    s.run(5)
    assert s.iteration == 5


@pytest.mark.parametrize("precision,factor", [(64, 1.7e308), (32, 3.3e38)])
def test_overflow_streaming_kernel(cuda, precision, factor):
    """Scaled synthetic through k_bwd_stream (forced): the device flags the oracle's
    first non-finite iteration."""
    desc = scaled(gamegen.synthetic(n_types=2, seed=1), factor)
    t_bad = first_bad_iteration(desc, 0, precision, 6)
    assert t_bad > 0
    s = expect_numerical(desc, "cfr", precision, pb.FLAG_FORCE_STREAM, 6, t_bad)
    assert "k_bwd_stream" in s.level_kernels()
