python - > gpurun_out/probe_det.txt 2>&1 <<'PY'
import time, hashlib
from threadpoolctl import threadpool_limits
from paper_2510_10891_b200 import scuc
for nt in (1, 8):
    with threadpool_limits(nt):
        t=time.time(); doc,mon,lp=scuc.build_config("C2"); print("C2", nt, lp.digest(), time.time()-t)
doc = scuc.generate_instance(**scuc.CONFIGS["C4"])
mon = scuc.sample_monitored(doc, 1000, 4)
inst = scuc.Instance(doc); net = inst.net
lines = sorted({inst.line_pos[l] for l,t,k in mon})
print(len(lines))
with threadpool_limits(8):
    t=time.time(); rows = scuc._ptdf_rows_direct(net.n_b, net.fb, net.tb, net.react, net.ref, lines); print("C4 ptdf cpu 8 thr", time.time()-t)
print(hashlib.sha256(rows.tobytes()).hexdigest())
PY
