# checked-build sweep: torchrun benches across configs, count device-side check failures
mkdir -p gpurun_out/sweep
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so
run() {  # name, command...
  local name=$1; shift
  timeout 400 "$@" > gpurun_out/sweep/$name.txt 2>&1
  echo "$name rc=$? fails=$(grep -c 'txb check failed' gpurun_out/sweep/$name.txt)"
}
for i in 1 2; do run decode_ep1_$i python bench.py --no-cpu-baseline --steps 60; done
run prefill_ep1 python bench.py --config prefill --no-cpu-baseline --steps 20
run kimi_ep1 python bench.py --config kimi --no-cpu-baseline --steps 60
for N in 2 4; do
  for i in 1 2 3; do run kimi_ep${N}_$i $TR --nproc-per-node $N --master-port $((29700+N+10*i)) bench.py --config kimi --gpus $N --steps 60 --no-cpu-baseline; done
  for i in 1 2; do run decode_p32_ep${N}_$i $TR --nproc-per-node $N --master-port $((29750+N+10*i)) bench.py --config decode --private 32 --gpus $N --steps 60 --no-cpu-baseline; done
  run prefill_ep$N $TR --nproc-per-node $N --master-port $((29790+N)) bench.py --config prefill --gpus $N --steps 20 --no-cpu-baseline
done
grep -h "txb check failed" gpurun_out/sweep/*.txt | sort | uniq -c | head
