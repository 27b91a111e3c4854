# Tail-stealing parameters (claim size G, smallest steal): config 4 kernel and step.
mkdir -p gpurun_out
: > gpurun_out/ab_steal_params.log
D=$PWD/paper_1203_5004_b200/lib
for r in 1 2 3; do
  for v in base st4_4 st4_8 st16_8; do
    if [ $v = base ]; then lib=$D/libhood_b200.so; else lib=$D/libhood_b200_$v.so; fi
    HOOD_B200_LIB=$lib timeout 300 python bench.py --config 4 --steps 10 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/$v /" >> gpurun_out/ab_steal_params.log
  done
done
HOOD_B200_LIB=$D/libhood_b200_st4_4.so timeout 600 python -m pytest tests -m gpu -q -k "stealing or config4" > gpurun_out/pytest_st44.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_st44.log
