# round-2 batch an: committed build vs FP64-paired epilogues (dual loads + primal columns; FP32 SASS unchanged); GPU suite on the new default
bash tools/ab_bench.sh tools/ab_base.so tools/ab_new.so 2 > gpurun_out/r2an_ab64.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r2an_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2an_pytest.log
