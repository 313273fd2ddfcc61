# checked build under torchrun IPC: which bench phase trips the combine row check
mkdir -p gpurun_out/dbg
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export TXB_BENCH_TRACE=1
for CFG in decode kimi; do
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 300 $TR --nproc-per-node 2 --master-port 29611 bench.py --config $CFG --gpus 2 --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/dbg/checked_$CFG.txt 2>&1
echo "$CFG rc=$?"; grep -c "check failed" gpurun_out/dbg/checked_$CFG.txt; grep "mark\|check failed" gpurun_out/dbg/checked_$CFG.txt | head -30
done
