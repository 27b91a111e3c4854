mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
oracle/_dropin/acceptance > gpurun_out/dropin_acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/dropin_acceptance.log
HOOD_BENCH_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --steps 10 --warmup 3 --cpu-seconds 0.1 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 3 -c 1 \
   -o gpurun_out/prof_c5 -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c5.log 2>&1
tail -8 gpurun_out/pytest_gpu.log
