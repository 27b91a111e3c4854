mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so timeout 300 python tools/trace_finalize.py 3 22 > gpurun_out/trace_fin_c3.log 2>&1
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so timeout 300 python tools/trace_ring.py a22 > gpurun_out/trace_ring_c3.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -3 gpurun_out/pytest_gpu.log
