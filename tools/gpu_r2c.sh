mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so timeout 300 python tools/trace_ring.py a22 > gpurun_out/trace_ring_c3.log 2>&1
for t in 4 8 12 16; do HOOD_STAGE_THREADS=$t timeout 600 python bench.py --steps 5 --warmup 2 --cpu-seconds 0.1 --no-kernel-events > gpurun_out/bench_c4_t$t.json 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 6 -c 1 \
   -o gpurun_out/prof_c3b -f python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c3b.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
