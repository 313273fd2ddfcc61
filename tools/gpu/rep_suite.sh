# repeated full GPU suite (flake hunt): release x2, checked x1
mkdir -p gpurun_out/rep
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rep/pytest_$i.log 2>&1; echo "release $i rc=$? $(tail -1 gpurun_out/rep/pytest_$i.log)"
done
TXB200_LIB=$PWD/paper_2510_27656_b200/libtxb200_checked.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rep/pytest_checked.log 2>&1; echo "checked rc=$? $(tail -1 gpurun_out/rep/pytest_checked.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rep/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/rep/smoke.log)"
