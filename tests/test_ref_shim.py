"""Pin tests/ref_shim.py (the stand-in for the reference's loop front end
used by the GPU plugin-route test) against the REAL reference's `_drive`
(loop.py:198-224) in the build container: both drive the same recording
executor through the same begin/step/finish/abort sequence and return the
same reports.  Skipped where /root/reference is absent (the GPU box)."""

import os
import sys

import pytest

import ref_shim as S

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


class Recorder:
    def __init__(self, values, fail_at=None):
        self.values, self.fail_at, self.log = values, fail_at, []

    def begin(self, plan, grid):
        self.log.append(("begin", plan.k, plan.indexed, plan.delta is not None))
        return {"i": 0}

    def step(self, run):
        run["i"] += 1
        self.log.append(("step", run["i"]))
        if run["i"] == self.fail_at:
            raise KeyError("boom")
        return self.values[run["i"] - 1]

    def finish(self, run):
        self.log.append(("finish", run["i"]))
        return "out", "ledger"

    def abort(self, run):
        self.log.append(("abort", run["i"]))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import stencilkit.loop as L
    import stencilkit

    return stencilkit, L


SCENARIOS = [
    dict(cond=lambda v, it, s: v < 0.5, values=[3.0, 2.0, 1.0, 0.4, 0.1], mi=None),
    dict(cond=lambda v, it, s: v < 0.5, values=[3.0, 2.0, 1.0, 0.9], mi=3),
    dict(cond=lambda v, it, s: it >= 2, values=[5, 6, 7], mi=None),
    dict(cond=lambda v, it, s: s >= 3, values=[1, 1, 1, 1, 1], mi=None, state=True),
    dict(cond=lambda v, it, s: False, values=[1, 2, 3], mi=None, fail=2),
]


@pytest.mark.parametrize("sc", SCENARIOS)
def test_shim_drive_matches_reference(sc):
    sk_ref, L = _ref()
    outs = []
    for mod, mk_op, mk_state in (
            (L, lambda: sk_ref.max_combinator(0.0), lambda: L.LoopState(
                init=lambda: 0, update=lambda s, it, v: s + 1)),
            (S, lambda: S.max_combinator(0.0), lambda: S.LoopState(
                init=lambda: 0, update=lambda s, it, v: s + 1))):
        rec = Recorder(sc["values"], sc.get("fail"))
        state = mk_state() if sc.get("state") else None
        try:
            if state is None:
                out, rep = mod.loop_stencil_reduce_d(1, lambda nb, e: 0, lambda a, b: a,
                                                     mk_op(), sc["cond"], "grid", executor=rec,
                                                     max_iterations=sc["mi"])
            else:
                out, rep = mod.loop_stencil_reduce_s(1, lambda nb, e: 0, mk_op(), sc["cond"],
                                                     state, "grid", executor=rec,
                                                     max_iterations=sc["mi"])
            res = (out, rep.iterations, rep.final_reduce, rep.exhausted, rep.copies)
        except KeyError:
            res = "raised"
        outs.append((res, rec.log))
    assert outs[0] == outs[1]
