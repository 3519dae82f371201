mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_screen.py -m gpu -x -q > gpurun_out/r1i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1i_pytest.log
timeout 600 python tools/batch_probe.py --config C1 --copies 8 > gpurun_out/r1i_batch_c1.json 2> gpurun_out/r1i_batch_c1.err
timeout 600 python tools/batch_probe.py --config C2 --copies 8 > gpurun_out/r1i_batch_c2.json 2> gpurun_out/r1i_batch_c2.err
timeout 600 python tools/batch_probe.py --config C1 --copies 16 --workers 16 > gpurun_out/r1i_batch_c1_16.json 2> gpurun_out/r1i_batch_c1_16.err
echo DONE
