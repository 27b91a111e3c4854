mkdir -p gpurun_out
timeout 900 python tools/adv_sweep.py 12 > gpurun_out/adv_sweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 5 3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 0.5 --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
tail -5 gpurun_out/pytest_gpu.log
