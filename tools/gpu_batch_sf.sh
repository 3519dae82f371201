# SF end-to-end (reference driver.run), GPU backend (LP on the B200 + native presolve) vs CPU
mkdir -p gpurun_out
for cfg in C1 C2; do
  timeout 1300 python tools/sf_e2e.py --backend cpu --config $cfg --time-limit 1200 --shutdown-feasible --out gpurun_out/sf_${cfg}_cpu.json > gpurun_out/sf_${cfg}_cpu.log 2>&1 &
  CPID=$!
  timeout 1300 python tools/sf_e2e.py --backend gpu --config $cfg --time-limit 1200 --shutdown-feasible --out gpurun_out/sf_${cfg}_gpu.json > gpurun_out/sf_${cfg}_gpu.log 2>&1; echo sf_${cfg}_gpu=$?
  tail -c 400 gpurun_out/sf_${cfg}_gpu.log
  wait $CPID; echo sf_${cfg}_cpu=$?
  tail -c 400 gpurun_out/sf_${cfg}_cpu.log
done
