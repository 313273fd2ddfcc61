# same-box A/B at EP=2/4 (decode), 2 runs each, then stamps with B and the multi-GPU parity tests on B
OUT=gpurun_out/$1; A=$2; B=$3; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do for rep in 1 2; do for L in A B; do
  LIB=$([ $L = A ] && echo $A || echo $B)
  TXB200_LIB=$PWD/$LIB timeout 300 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config decode --gpus $N --no-cpu-baseline > $OUT/b_ep${N}_${L}_$rep.json 2> $OUT/b_ep${N}_${L}_$rep.err
  python -c "
import json; d=json.loads(open('$OUT/b_ep${N}_${L}_$rep.json').read().strip().splitlines()[-1]); print('EP$N $L rep$rep', d['value'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
done; done; done
TXB200_LIB=$PWD/$B timeout 900 python -m pytest tests/test_multigpu.py tests/test_moe_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
