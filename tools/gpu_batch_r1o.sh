mkdir -p gpurun_out
timeout 300 python tools/screen_bench.py > gpurun_out/r1o_base.json 2>&1
for v in mt8_kb16_s3 mt4_kb16_s2 mt2_kb16_s3; do HPR_LIB=build/lib_$v.so timeout 300 python tools/screen_bench.py > gpurun_out/r1o_$v.json 2>&1; done
timeout 300 python tools/screen_bench.py > gpurun_out/r1o_base2.json 2>&1
echo DONE
