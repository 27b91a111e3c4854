# (Needs the commit that added HOOD_FORCE_INSTANCE; the switch was removed after this A/B.)
# A/B for config 5: the LEAN ring kernel (one warp per instance) vs the
# CTA-cooperative instance kernel (TMA tiles of 4 instances, CTA merge tree).
mkdir -p gpurun_out
HOOD_FORCE_INSTANCE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "batched or block_lengths or config5 or acceptance_full" > gpurun_out/pytest_inst.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_inst.log
: > gpurun_out/ab_inst.log
for r in 1 2 3; do for t in 0 1; do
  HOOD_FORCE_INSTANCE=$t timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/inst=$t /" >> gpurun_out/ab_inst.log
done; done
for c in 3 4; do timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum -k regex:"ring_hull|finalize" --launch-skip 6 -c 2 python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/ncu_dfma_c$c.log 2>&1; done
tail -2 gpurun_out/pytest_inst.log
