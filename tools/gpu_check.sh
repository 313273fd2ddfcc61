#!/bin/bash
# One GPU session: gpu tests, bench at EP=1 and at every EP the box has
# (torchrun), phase stamps at the largest EP.  Outputs in gpurun_out/.
# usage: tools/gpu_check.sh [config] [stamps]
CFG=${1:-decode}
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --config $CFG --no-cpu-baseline > gpurun_out/bench_${CFG}_ep1.json 2> gpurun_out/bench_${CFG}_ep1.err
N=2
while [ $N -le $NG ]; do
  timeout 300 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config $CFG --gpus $N --no-cpu-baseline > gpurun_out/bench_${CFG}_ep$N.json 2> gpurun_out/bench_${CFG}_ep$N.err
  N=$((N*2))
done
if [ "${2:-stamps}" = stamps ]; then
  timeout 300 $TR --nproc-per-node $NG --master-port 29650 tools/prof_torchrun.py --config $CFG --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/stamps_${CFG}_ep$NG.txt
fi
for f in gpurun_out/bench_${CFG}_ep*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], 'warm', d.get('p50_l2_warm_us'), d['kernel_us'], 'e2e', d['e2e']['value'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
