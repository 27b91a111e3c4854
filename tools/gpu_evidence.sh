# Round evidence on one B200: parity tests, default bench line (+ reference
# arm), ncu launch list of the bench command, ncu full captures of the ring
# kernel (configs 2 and 5) and of finalize.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 2 > gpurun_out/bench_c$c.json 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_hull -s 2 -c 1 -o gpurun_out/prof_ring_c2 -f \
  python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_ring_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_hull -s 2 -c 1 -o gpurun_out/prof_ring_c5 -f \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_ring_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_hull -s 2 -c 1 -o gpurun_out/prof_ring_c4 -f \
  python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_ring_c4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:finalize -s 2 -c 1 -o gpurun_out/prof_fin_c2 -f \
  python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_fin_c2.log 2>&1
ls -la gpurun_out
