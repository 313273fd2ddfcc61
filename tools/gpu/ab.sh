# same-box A/B of two library builds: stamps + bench decode at EP=2 and EP=4
# usage: bash tools/gpu/ab.sh <outdir> <libA> <libB>
OUT=gpurun_out/$1; A=$2; B=$3; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do for L in A B; do
  LIB=$([ $L = A ] && echo $A || echo $B)
  TXB200_LIB=$PWD/$LIB timeout 300 $TR --nproc-per-node $N --master-port $((29650+N)) tools/prof_torchrun.py --reps 50 2>&1 | grep -v OMP | grep -v '^\*' > $OUT/stamps_ep${N}_$L.txt
  for rep in 1 2; do
  TXB200_LIB=$PWD/$LIB timeout 600 $TR --nproc-per-node $N --master-port $((29600+N)) bench.py --config decode --gpus $N --no-cpu-baseline > $OUT/bench_ep${N}_${L}_$rep.json 2> $OUT/bench_ep${N}_${L}_$rep.err
  python -c "
import json; d=json.loads(open('$OUT/bench_ep${N}_${L}_$rep.json').read().strip().splitlines()[-1]); print('EP$N $L rep$rep', d['value'], d['kernel_us'], 'flushed', d.get('p50_flushed_step_us'), 'span', d.get('p50_kernel_span_us'))"
  done
done; done
