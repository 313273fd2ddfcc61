mkdir -p gpurun_out/r2r
# KV stream (one persistent kernel) and the per-step copy kernel: plain runs first, then ncu
timeout 600 python tools/bench_kv_stream.py --modes ready --reps 2 > gpurun_out/r2r/kv_ready.json 2>&1; tail -c 400 gpurun_out/r2r/kv_ready.json
timeout 600 python tools/bench_kv.py --steps 20 > gpurun_out/r2r/kv_steps.json 2>&1; tail -c 600 gpurun_out/r2r/kv_steps.json
timeout 900 ncu --set full --clock-control none -k regex:"k_kv_stream" -c 1 -o gpurun_out/r2r/kv_stream python tools/bench_kv_stream.py --modes ready --reps 1 > gpurun_out/r2r/ncu_kv_stream.log 2>&1; tail -2 gpurun_out/r2r/ncu_kv_stream.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum --clock-control none -k regex:"k_copy_jobs|k_kv_stream" -c 6 --csv --log-file gpurun_out/r2r/kv_nvlink.csv python tools/bench_kv.py --steps 4 > gpurun_out/r2r/ncu_kv_nvl.log 2>&1; tail -2 gpurun_out/r2r/ncu_kv_nvl.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dispatch_roles|k_combine_fused" -s 40 -c 2 -o gpurun_out/r2r/ep1_full python bench.py --steps 25 --warmup 3 --no-cpu-baseline > gpurun_out/r2r/ncu_ep1.log 2>&1; tail -2 gpurun_out/r2r/ncu_ep1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2r/launches_ep1.csv python bench.py --steps 25 --warmup 3 --no-cpu-baseline > gpurun_out/r2r/ncu_launch.log 2>&1; tail -1 gpurun_out/r2r/ncu_launch.log
