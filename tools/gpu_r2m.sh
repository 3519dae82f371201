# round-2 batch m: halt flag gated to the queued loop only; full GPU suite; C4 bench
python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
python -m pytest tests -m gpu -x -q > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2m_pytest.log
python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2m_bench2.json 2> gpurun_out/r2m_bench2.err
