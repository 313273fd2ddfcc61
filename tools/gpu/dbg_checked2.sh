# checked build under torchrun IPC, no phase syncs, repeated
mkdir -p gpurun_out/dbg
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2 3 4 5 6; do for CFG in decode kimi; do
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 200 $TR --nproc-per-node 2 --master-port $((29611+i)) bench.py --config $CFG --gpus 2 --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/dbg/fix_${CFG}_$i.txt 2>&1
echo "run $CFG $i rc=$? fails=$(grep -c 'check failed' gpurun_out/dbg/fix_${CFG}_$i.txt)"; grep "check failed" gpurun_out/dbg/fix_${CFG}_$i.txt | head -3
done; done
