mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 3 2 5; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 0.5 --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -30 gpurun_out/pytest_gpu.log
