mkdir -p gpurun_out/r2d
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2d/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d/pytest.log
tail -3 gpurun_out/r2d/pytest.log
for P in 0 32; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/prof_torchrun.py --reps 50 --private $P > gpurun_out/r2d/stamps_ep2_p$P.txt 2>&1
done
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2d/stamps_ep1.txt 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready,launch --reps 3 > gpurun_out/r2d/kv_vec.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready --tma --reps 3 > gpurun_out/r2d/kv_tma.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes ready --grid 32 --reps 3 > gpurun_out/r2d/kv_vec_g32.json 2>&1
timeout 600 python tools/bench_kv_stream.py --modes paced --layer-us 12 --grid 32 --reps 2 > gpurun_out/r2d/kv_paced.json 2>&1
tail -2 gpurun_out/r2d/kv*.json | cut -c1-600
