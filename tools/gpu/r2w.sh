mkdir -p gpurun_out/r2w
timeout 300 python tools/prof_torchrun.py --reps 50 --noflush > gpurun_out/r2w/stamps_ep1_noflush.txt 2>&1
timeout 300 python tools/prof_torchrun.py --reps 50 > gpurun_out/r2w/stamps_ep1_flush.txt 2>&1
for f in gpurun_out/r2w/stamps_ep1_noflush.txt gpurun_out/r2w/stamps_ep1_flush.txt; do echo $f; grep -v nan $f | grep "CTA" | head -24; done
