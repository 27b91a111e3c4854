mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python tools/time_dent.py > gpurun_out/time_dent.log 2>&1
python tools/time_shapes.py > gpurun_out/shapes_new.log 2>&1
for c in 3 2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py >> gpurun_out/bench_fin.log; done
