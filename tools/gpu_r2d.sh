mkdir -p gpurun_out
timeout 300 python tools/h2d_register.py > gpurun_out/h2d_register.log 2>&1
for c in 4 8 32 64; do HOOD_STAGE_CHUNK_MB=$c timeout 600 python bench.py --steps 5 --warmup 2 --cpu-seconds 0.1 --no-kernel-events > gpurun_out/bench_c4_c$c.json 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 3 -c 1 \
   -o gpurun_out/prof_c3b -f python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c3b.log 2>&1
