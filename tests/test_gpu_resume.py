"""Checkpoint / resume (include/cfr_b200.h cfr_solver_set_state): a
solver restored from get_state() after T1 iterations and run T2 more holds the same
bits as one run T1 + T2 without stopping, and as the oracle at T1 + T2."""
import numpy as np
import pytest

import gamegen
import oracle
import paper_2408_14778_b200 as pb
from tests.parity import assert_same

pytestmark = pytest.mark.gpu


def _resume(desc, variant, precision, T1, T2, flags=0):
    g = pb.Game(desc)
    a = pb.Solver(g, variant=variant, precision=precision, flags=flags).run(T1)
    st = a.state()
    b = pb.Solver(g, variant=variant, precision=precision, flags=flags)
    b.set_state(T1, st["regret"], st["snum"], st["sden"])
    assert b.iteration == T1
    assert np.array_equal(b.current_strategy(), a.current_strategy())
    b.run(T2)
    ref = pb.Solver(g, variant=variant, precision=precision, flags=flags).run(T1 + T2)
    sb, sr = b.state(), ref.state()
    for k in ("regret", "snum", "sden"):
        assert np.array_equal(sb[k], sr[k]), k
    assert np.array_equal(b.average_strategy(), ref.average_strategy())
    assert np.array_equal(b.current_strategy(), ref.current_strategy())
    return b


@pytest.mark.parametrize("name", ["kuhn", "leduc", "goofspiel"])
@pytest.mark.parametrize("variant", [0, 1, 3, 4])
def test_resume_bit_identical(cuda, name, variant):
    desc = gamegen.by_name(name)
    b = _resume(desc, variant, 64, 17, 13)
    o = oracle.Oracle(desc).run(30, variant)
    assert_same("average strategy", b.average_strategy(), o.average_strategy(), 64)


@pytest.mark.parametrize("precision", [64, 32])
def test_resume_streaming_and_tile_kernels(cuda, precision):
    desc = gamegen.synthetic(n_types=3, seed=7)
    _resume(desc, 1, precision, 3, 2, flags=pb.FLAG_FORCE_STREAM)
    _resume(gamegen.leduc(), 0, precision, 40, 25, flags=pb.FLAG_NO_TINY)


def test_resume_rejects_bad_arguments(cuda):
    s = pb.Solver(pb.Game(gamegen.kuhn()), variant="cfr", precision=64)
    with pytest.raises(ValueError):
        s.set_state(1, np.zeros(3), np.zeros(s.Q), np.zeros(s.H))
    with pytest.raises(pb.NativeError):
        s.set_state(-1, np.zeros(s.Q), np.zeros(s.Q), np.zeros(s.H))
