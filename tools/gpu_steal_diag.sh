python tools/steal_diag.py > gpurun_out/steal_diag.log 2>&1
HOOD_STEAL=0 python tools/steal_diag.py >> gpurun_out/steal_diag.log 2>&1
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so NOEV=1 timeout 600 python tools/trace_ring.py g28 > gpurun_out/trace_steal.log 2>&1
