tools/gpu_check.sh kimi nostamps
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2; do timeout 200 $TR --nproc-per-node 2 --master-port $((29890+i)) bench.py --config kimi --gpus 2 --no-cpu-baseline > gpurun_out/kk_$i.json 2> gpurun_out/kk_$i.err; echo "kimi ep2 run $i rc=$?"; done
