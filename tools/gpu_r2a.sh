# Round-2 first pass: parity tests, config-4 bench line, config-3 ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --cpu-seconds 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ring_hull|finalize_kernel" --launch-skip 6 -c 2 \
   -o gpurun_out/prof_c3 -f python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
