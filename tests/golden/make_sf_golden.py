"""A completed end-to-end successive-fixing run of the UNMODIFIED reference
driver (``scuckit.driver.run``, driver.py:203-324: two-stage transmission
filtering, successive fixing, presolve, B&B) on a small synthetic instance
that finishes on the CPU (12 buses, 6 units, 6 periods, seed 5, initial
outputs capped at the shutdown limit), recorded in the build container:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_sf_golden.py

tests/test_dropin_fixing.py::test_driver_run_completes_like_reference replays
it with the LP solves, presolve, flow screen and model builder routed to the
B200 path by ``hprlp.install()`` and compares the final MILP objective,
status, commitment, monitored set and per-pass records.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import driver, parse_instance  # noqa: E402

from paper_2510_10891_b200 import scuc  # noqa: E402

ARGS = dict(n_buses=12, n_gens=6, n_lines=18, n_periods=6, seed=5, shutdown_feasible=True)


def record(rep) -> dict:
    d = rep.to_json_dict()
    d.pop("timings")
    return d


def main():
    doc = scuc.generate_instance(**ARGS)
    rep = driver.run(parse_instance(doc), driver.DriverConfig(time_limit=600.0))
    out = {"instance": ARGS, "report": record(rep), "wall_s": rep.total_time}
    with open(os.path.join(HERE, "sf_small.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out["report"]["status"], out["report"]["objective"], rep.total_time)


if __name__ == "__main__":
    main()
