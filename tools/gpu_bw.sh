mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/adv_sweep.py 6 > gpurun_out/adv_sweep.log 2>&1
python tools/time_shapes.py > gpurun_out/shapes_new.log 2>&1
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_prev.so python tools/time_shapes.py > gpurun_out/shapes_prev.log 2>&1
