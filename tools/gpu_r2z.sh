# round-2 batch z: driver-contract checks: smoke(); bench under torchrun (1 rank); reference arm under torchrun
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2z_smoke.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 5 --warmup 3 --no-screen > gpurun_out/r2z_torchrun.log 2>&1; echo "rc $?" >> gpurun_out/r2z_torchrun.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r2z_torchrun_ref.log 2>&1; echo "rc $?" >> gpurun_out/r2z_torchrun_ref.log
