mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_screen.py tests/test_gpu_batch.py -m gpu -x -q > gpurun_out/r1m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1m_pytest.log
timeout 600 python tools/screen_bench.py > gpurun_out/r1m_c4.json 2> gpurun_out/r1m_c4.err
echo DONE
