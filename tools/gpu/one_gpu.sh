# what the driver runs on one GPU: suite, smoke, bench (both arms)
mkdir -p gpurun_out/one
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/one/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/one/pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/one/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/one/smoke.log)"
timeout 600 python bench.py > gpurun_out/one/bench.json 2> gpurun_out/one/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/one/bench.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/one/ref.json 2> gpurun_out/one/ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/one/ref.json; echo
