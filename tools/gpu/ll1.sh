# line-flagged dispatch rows: parity (release + checked) and A/B vs TXB_NO_LL=1 on the same box
mkdir -p gpurun_out/ll1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -x -k "line_flagged" > gpurun_out/ll1/pytest_ll.log 2>&1; echo "rc=$?" >> gpurun_out/ll1/pytest_ll.log; tail -15 gpurun_out/ll1/pytest_ll.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do for M in ll noll; do
  if [ $M = noll ]; then export TXB_NO_LL=1; else unset TXB_NO_LL; fi
  timeout 300 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config decode --gpus $N --no-cpu-baseline > gpurun_out/ll1/bench_ep${N}_$M.json 2> gpurun_out/ll1/bench_ep${N}_$M.err
  python -c "
import json; d=json.loads(open('gpurun_out/ll1/bench_ep${N}_$M.json').read().strip().splitlines()[-1]); print('EP$N $M', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))" 2>&1 | tail -1
done; done
unset TXB_NO_LL
timeout 300 $TR --nproc-per-node 2 --master-port 29652 tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > gpurun_out/ll1/stamps_ep2.txt
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -x -k "line_flagged or dsv3_decode or checked_build" > gpurun_out/ll1/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/ll1/pytest_checked.log; tail -5 gpurun_out/ll1/pytest_checked.log
