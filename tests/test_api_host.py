"""Host-side API mirror (no GPU): ``write_iteration_log`` and the result
records against the reference's own functions when the reference is
importable (the build container), and against a pinned text otherwise."""

import numpy as np

from tests.conftest import needs_reference


def _result(mod, log):
    return mod.SolveResult(x=np.zeros(2), y=np.zeros(1), z=np.zeros(2),
                           status=mod.SolveStatus.OPTIMAL, objective=1.0, kkt=None,
                           iterations=32, restarts=1, solve_time=0.1, sigma_final=2.0,
                           lam=1.01, residual_log=log)


LOG = [{"iteration": 16, "epoch": 0, "rel_primal": 0.125, "rel_dual": 1e-3,
        "rel_box": 0.0, "rel_gap": 3.0000000000000004e-05, "sigma": 0.98},
       {"iteration": 32, "epoch": 1, "rel_primal": 1.5e-17, "rel_dual": 2.5e-4,
        "rel_box": 1e-300, "rel_gap": float("nan"), "sigma": 1.6782757095248741}]

PINNED = ("solve_id,iteration,epoch,rel_primal,rel_dual,rel_box,rel_gap,sigma\r\n"
          "a,16,0,0.125,0.001,0.0,3.0000000000000004e-05,0.98\r\n"
          "a,32,1,1.5e-17,0.00025,1e-300,nan,1.6782757095248741\r\n"
          "b,16,0,0.125,0.001,0.0,3.0000000000000004e-05,0.98\r\n"
          "b,32,1,1.5e-17,0.00025,1e-300,nan,1.6782757095248741\r\n")


def test_write_iteration_log_pinned(tmp_path):
    from paper_2510_10891_b200 import hprlp
    p = tmp_path / "mine.csv"
    r = _result(hprlp, LOG)
    hprlp.write_iteration_log(str(p), r, "a")       # creates the file with a header
    hprlp.write_iteration_log(str(p), r, "b")       # appends without one
    assert p.read_bytes().decode() == PINNED


@needs_reference
def test_write_iteration_log_matches_reference(tmp_path):
    from scuckit import hprlp as ref
    from paper_2510_10891_b200 import hprlp
    a, b = tmp_path / "mine.csv", tmp_path / "ref.csv"
    for sid in ("x", "y"):
        hprlp.write_iteration_log(str(a), _result(hprlp, LOG), sid)
        ref.write_iteration_log(str(b), _result(ref, LOG), sid)
    assert a.read_bytes() == b.read_bytes()


@needs_reference
def test_result_records_match_reference_fields():
    """The mirror's records carry the reference's fields (the drop-in reads
    them by name: lp_backends.py:37-40, fixing.py:164-176)."""
    import dataclasses
    from scuckit import hprlp as ref
    from paper_2510_10891_b200 import hprlp
    for name in ("SolverConfig", "KktResidual", "SolveResult"):
        mine = [f.name for f in dataclasses.fields(getattr(hprlp, name))]
        theirs = [f.name for f in dataclasses.fields(getattr(ref, name))]
        assert mine[:len(theirs)] == theirs, name
    assert [s.value for s in hprlp.SolveStatus] == [s.value for s in ref.SolveStatus]
    val = lambda v: v.value if hasattr(v, "value") else v          # noqa: E731
    mine = {f.name: val(getattr(hprlp.SolverConfig(), f.name))
            for f in dataclasses.fields(hprlp.SolverConfig)}
    theirs = {f.name: val(getattr(ref.SolverConfig(), f.name))
              for f in dataclasses.fields(ref.SolverConfig)}
    assert mine == theirs
