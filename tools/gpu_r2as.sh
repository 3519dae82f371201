# round-2 batch as: round-end rehearsal on HEAD (GPU suite, smoke, default bench, reference arm)
python -m pytest tests -m gpu -x -q > gpurun_out/r2as_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2as_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2as_smoke.log 2>&1
python bench.py > gpurun_out/r2as_bench.json 2> gpurun_out/r2as_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2as_ref.json 2> gpurun_out/r2as_ref.err
