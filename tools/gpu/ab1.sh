# same-box A/B at EP=1: bench decode/kimi x3 each, stamps; usage: bash tools/gpu/ab1.sh <outdir> <libA> <libB>
OUT=gpurun_out/$1; A=$2; B=$3; mkdir -p $OUT
for rep in 1 2 3; do for L in A B; do
  LIB=$([ $L = A ] && echo $A || echo $B)
  for CFG in decode kimi; do
  TXB200_LIB=$PWD/$LIB timeout 300 python bench.py --config $CFG --no-cpu-baseline > $OUT/bench_${CFG}_${L}_$rep.json 2> $OUT/bench_${CFG}_${L}_$rep.err
  python -c "
import json; d=json.loads(open('$OUT/bench_${CFG}_${L}_$rep.json').read().strip().splitlines()[-1]); print('$CFG $L rep$rep', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
  done
done; done
for L in A B; do LIB=$([ $L = A ] && echo $A || echo $B); TXB200_LIB=$PWD/$LIB timeout 300 python tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP > $OUT/stamps_ep1_$L.txt; done
timeout 900 python -m pytest tests/test_moe_gpu.py -m gpu -q -p no:cacheprovider -x > $OUT/pytest_moe.log 2>&1; tail -2 $OUT/pytest_moe.log
