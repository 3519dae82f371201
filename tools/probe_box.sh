lscpu | head -20 > gpurun_out/box_cpu.txt; nproc >> gpurun_out/box_cpu.txt; free -g >> gpurun_out/box_cpu.txt
python -c "import numpy; numpy.show_config()" >> gpurun_out/box_cpu.txt 2>&1
python - >> gpurun_out/box_cpu.txt 2>&1 <<'PY'
import time
from paper_2510_10891_b200 import scuc
for name in ("C1","C2"):
    t=time.time(); doc,mon,lp=scuc.build_config(name); print(name, lp.digest(), lp.shape, lp.nnz, time.time()-t)
t=time.time(); doc,mon,lp=scuc.build_config("C4", device="cuda"); print("C4", lp.digest(), lp.shape, lp.nnz, time.time()-t)
PY
