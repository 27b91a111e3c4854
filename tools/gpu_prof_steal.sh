mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 3 -c 1 -o gpurun_out/prof_c4_steal -f python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c4s.log 2>&1
HOOD_STEAL=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 3 -c 1 -o gpurun_out/prof_c4_nosteal -f python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c4ns.log 2>&1
