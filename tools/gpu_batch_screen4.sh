mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_screen.py -m gpu -x -q > gpurun_out/scr4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/scr4_pytest.log
timeout 600 python tools/screen_bench.py > gpurun_out/scr4_c4.json 2> gpurun_out/scr4_c4.err
timeout 300 python tools/screen_bench.py --buses 1354 --gens 260 --lines 1991 --periods 24 > gpurun_out/scr4_c2.json 2> gpurun_out/scr4_c2.err
timeout 300 python tools/screen_bench.py --buses 6468 --gens 399 --lines 9000 --periods 36 > gpurun_out/scr4_c3.json 2> gpurun_out/scr4_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:screen_product -c 1 -o gpurun_out/scr4_c4 -f python tools/screen_bench.py --cpu 0 --reps 1 > gpurun_out/scr4_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:screen_ --csv --log-file gpurun_out/scr4_launches.csv python tools/screen_bench.py --cpu 0 --reps 2 > gpurun_out/scr4_ncu2.log 2>&1
echo DONE
