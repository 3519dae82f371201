mkdir -p gpurun_out
timeout 300 python tools/screen_bench.py --cpu 0 > gpurun_out/r1l_base.json 2>&1
for v in kb16_s4 kb32_s3 kb32_s2 kb8_s4; do HPR_LIB=build/lib_$v.so timeout 300 python tools/screen_bench.py --cpu 0 > gpurun_out/r1l_$v.json 2>&1; done
timeout 300 python tools/screen_bench.py --cpu 0 > gpurun_out/r1l_base2.json 2>&1
echo DONE
