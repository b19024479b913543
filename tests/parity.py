"""Parity helpers: run the CPU oracle and the CUDA path (through the C ABI) on the
same seeded game and compare element by element.

Bar (BASELINE.json north_star): sigma_bar and expected values within 1e-10
relative in fp64 and 1e-4 in fp32.  Under the arithmetic contract of DESIGN.md §4
both sides perform the same IEEE operations, so the comparison asserts IEEE
equality (max relative difference 0, i.e. strictly inside the north-star bar);
the tolerance check is asserted as well so a failure message reports both.
"""
from __future__ import annotations

import numpy as np

import oracle
import paper_2408_14778_b200 as pb

TOL = {64: 1e-10, 32: 1e-4}


def rel_diff(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    d = np.abs(a - b) / den
    d[(a == b)] = 0.0
    return float(d.max())


def assert_same(name, got, want, precision, exact=True):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, f"{name}: shape {got.shape} vs {want.shape}"
    rd = rel_diff(got, want)
    assert rd <= TOL[precision], f"{name}: max relative diff {rd:.3e} > {TOL[precision]:.0e}"
    if exact:
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (f"{name}: {bad.size} entries differ bitwise (max rel {rd:.3e}); first at "
                               f"{bad[0]}: got {got[bad[0]]!r} want {want[bad[0]]!r}")
    return rd


def run_pair(desc, variant: int, precision: int, T: int, device=None, flags=0, checks=("all",),
             oracle_obj=None, solver=None):
    """Run T iterations on both sides; compare state and readbacks.  Returns diffs."""
    o = oracle_obj if oracle_obj is not None else oracle.Oracle(desc, precision=precision)
    o.run(T, variant)
    if solver is None:
        g = pb.Game(desc)
        solver = pb.Solver(g, variant=int(variant), precision=precision,
                           device=device or "cuda", flags=flags)
    solver.run(T)
    assert solver.iteration == o.state()["t"]
    os_ = o.state()
    ss = solver.state()
    out = {}
    out["sigma"] = assert_same("current strategy", solver.current_strategy(), os_["sigma"], precision)
    out["regret"] = assert_same("regret", ss["regret"], os_["regret"], precision)
    out["snum"] = assert_same("S_num", ss["snum"], os_["snum"], precision)
    out["sden"] = assert_same("S_den", ss["sden"], os_["sden"], precision)
    out["avg"] = assert_same("average strategy", solver.average_strategy(), os_["avg"], precision)
    out["ev"] = assert_same("EV(avg)", solver.expected_values("average"), o.expected_values(), precision)
    out["ev_cur"] = assert_same("EV(current)", solver.expected_values("current"), o.expected_values("current"),
                                precision)
    if "all" in checks or "br" in checks:
        # the device best response is general (any infoset structure, any world
        # size): an unsupported status is a failure, never a skip
        se = solver.exploitability()
        oe = o.exploitability()
        out["br"] = assert_same("BR", se["br"], oe["br"], precision)
        out["nash_conv"] = assert_same("NashConv", [se["nash_conv"]], [oe["nash_conv"]], precision)
    return out, solver, o
