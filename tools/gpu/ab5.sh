# same-box A/B at EP=1 (decode, kimi) and EP=2 (decode), 2 runs each; parity of B
OUT=gpurun_out/$1; A=$2; B=$3; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2; do for L in A B; do
  LIB=$([ $L = A ] && echo $A || echo $B)
  for CFG in decode kimi; do
    TXB200_LIB=$PWD/$LIB timeout 300 python bench.py --config $CFG --no-cpu-baseline > $OUT/b1_${CFG}_${L}_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$OUT/b1_${CFG}_${L}_$rep.json').read().strip().splitlines()[-1]); print('EP1 $CFG $L rep$rep', d['value'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
  done
  TXB200_LIB=$PWD/$LIB timeout 300 $TR --nproc-per-node 2 --master-port 29602 bench.py --config decode --gpus 2 --no-cpu-baseline > $OUT/b2_${L}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/b2_${L}_$rep.json').read().strip().splitlines()[-1]); print('EP2 decode $L rep$rep', d['value'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
done; done
TXB200_LIB=$PWD/$B timeout 900 python -m pytest tests/test_multigpu.py tests/test_moe_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
