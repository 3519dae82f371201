mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_screen.py -m gpu -x -q > gpurun_out/scr2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/scr2_pytest.log
for r in 128 168 255; do HPR_LIB=build/lib_r$r.so timeout 600 python tools/screen_bench.py --cpu 0 > gpurun_out/scr2_r$r.json 2> gpurun_out/scr2_r$r.err; done
timeout 900 python tools/screen_bench.py > gpurun_out/scr2_c4.json 2> gpurun_out/scr2_c4.err
echo DONE
