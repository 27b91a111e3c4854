# Round-2 evidence pass: parity, bench lines of every config (default = config 4
# with e2e), the reference arm, the ncu launch list of the default bench, one
# ncu --set full capture per config's ring kernel (+ config-2 finalize), traces.
set -x
mkdir -p gpurun_out/ev
nvidia-smi > gpurun_out/ev/nvidia_smi.txt 2>&1
lscpu > gpurun_out/ev/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 1200 python bench.py --steps 30 --warmup 5 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference_c4.json 2> gpurun_out/ev/bench_reference_c4.err
for c in 1 2 3 5; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --cpu-seconds 5 > gpurun_out/ev/bench_c$c.json 2> gpurun_out/ev/bench_c$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --cpu-seconds 0.01 > gpurun_out/ev/ncu_launches.log 2>&1
for c in 2 3 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ring_hull" --launch-skip 3 -c 1 -o gpurun_out/ev/prof_ring_c$c -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ev/ncu_ring_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"finalize" --launch-skip 3 -c 1 -o gpurun_out/ev/prof_fin_c2 -f python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ev/ncu_fin_c2.log 2>&1
export HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_trace.so
NOEV=1 timeout 600 python tools/trace_ring.py 24 g28 a22 b > gpurun_out/ev/trace_ring.log 2>&1
timeout 300 python tools/trace_finalize.py 2 > gpurun_out/ev/trace_fin_c2.log 2>&1
unset HOOD_B200_LIB
for c in 3 4; do timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum -k regex:"ring_hull|finalize" --launch-skip 6 -c 2 python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ev/ncu_dfma_c$c.log 2>&1; done
python tools/steal_diag.py > gpurun_out/ev/steal_diag.log 2>&1
python tools/time_dent.py > gpurun_out/ev/time_dent.log 2>&1
bash tools/gpu_checked.sh
