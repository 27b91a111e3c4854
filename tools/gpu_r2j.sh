mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_checked.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so NOEV=1 timeout 600 python tools/trace_ring.py g28 > gpurun_out/trace_steal.log 2>&1
