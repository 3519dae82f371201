"""Golden C1 solve at tolerance 1e-6 from the UNMODIFIED reference (build
container only; ~17 min):  python tests/golden/make_c1_1e6_golden.py
The reference ends in numerical-failure (its dual iterate overflows after
548 restarts); tests/test_gpu_parity.py checks the engine fails at the same
iteration with the same best objective."""
import sys, time, json
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
from scuckit import hprlp
from scuckit.lp_kernel import SparseMatrix, StandardFormLp
from paper_2510_10891_b200 import scuc
doc = scuc.generate_instance(**scuc.CONFIGS["C1"])
lpa = scuc.build_relaxation(doc, scuc.all_base_triples(doc))
lp = StandardFormLp(matrix=SparseMatrix(lpa.csr()), rhs=lpa.rhs, cost=lpa.cost, lower=lpa.lower, upper=lpa.upper, n_eq=lpa.n_eq, offset=lpa.offset)
t = time.time()
r = hprlp.solve(lp, hprlp.SolverConfig(tolerance=1e-6, ruiz=False, max_iterations=400000))
print(json.dumps({"status": r.status.value, "iterations": r.iterations, "restarts": r.restarts, "objective": r.objective, "seconds": time.time() - t, "fp64_fallback": getattr(r, "fp64_fallback", None)}))
