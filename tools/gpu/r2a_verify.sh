set -x
nvidia-smi -L
mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/pytest.log
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py decode1 > gpurun_out/r2a/san_${t}_decode1.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/san_${t}_decode1.log
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize.py prefill1 > gpurun_out/r2a/san_racecheck_prefill1.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/san_racecheck_prefill1.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize.py gated2 decode1 > gpurun_out/r2a/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/san_memcheck.log
tail -3 gpurun_out/r2a/*.log
