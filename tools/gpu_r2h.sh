mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 5 2 3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 0.5 --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,gpu__time_duration.sum -k regex:"ring_hull" --launch-skip 3 -c 1 python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_c5_conf.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
