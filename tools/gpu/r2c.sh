# EP=2 phase stamps with and without the private round; EP=1 stamps
mkdir -p gpurun_out/r2c
for P in 0 32 128; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/prof_torchrun.py --reps 50 --private $P > gpurun_out/r2c/stamps_ep2_p$P.txt 2>&1
done
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2c/stamps_ep1.txt 2>&1
tail -5 gpurun_out/r2c/*.txt
