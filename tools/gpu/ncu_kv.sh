mkdir -p gpurun_out/ncukv
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,smsp__pcsamp_warps_issue_stalled_membar,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_drain,smsp__pcsamp_sample_count,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:k_kv_stream -c 1 python tools/bench_kv_stream.py --modes ready --reps 1 > gpurun_out/ncukv/stream.txt 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:pages2 -c 3 ./tools/micro/peer_width > gpurun_out/ncukv/micro.txt 2>&1
grep -E "k_kv_stream|pages2|gpu__time|dram__|nvltx|stalled|sample_count|inst_executed|lts__" gpurun_out/ncukv/stream.txt | head -20
grep -E "pages2|gpu__time|dram__|nvltx|stalled|sample_count|inst_executed|lts__" gpurun_out/ncukv/micro.txt | tail -14
