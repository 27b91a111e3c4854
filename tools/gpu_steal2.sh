#!/bin/bash
# multi-steal + adaptive claims: parity, bench config 4 (x2), steal counts, warp exit spread
mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2/pytest.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --cpu-seconds 0.01 --no-e2e > gpurun_out/s2/bench_c4_$i.json 2> gpurun_out/s2/bench_c4_$i.err; done
python tools/steal_diag.py > gpurun_out/s2/steal_diag.log 2>&1
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so NOEV=1 timeout 600 python tools/trace_ring.py g28 > gpurun_out/s2/trace_ring.log 2>&1
