# A/B: the batched (LEAN) ring variant's block width and register cap on config 5
mkdir -p gpurun_out/leanu
V=$PWD/paper_1203_5004_b200/lib/var
for n in u4r80 u4r96; do
  HOOD_B200_LIB=$V/$n.so timeout 600 python -m pytest tests -m gpu -q -x -k "config or batched or acceptance or adversarial or padded or block_len or known" > gpurun_out/leanu/pytest_$n.log 2>&1; echo "rc=$?" >> gpurun_out/leanu/pytest_$n.log
done
: > gpurun_out/leanu/ab.log
for r in 1 2; do for n in u8r128 u8r96 u4r128 u4r96 u4r80 u4r72; do
  HOOD_B200_LIB=$V/$n.so timeout 300 python bench.py --config 5 --steps 30 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/$n /" >> gpurun_out/leanu/ab.log
done; done
for n in u8r128 u4r80; do
  HOOD_B200_LIB=$V/$n.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_hull --launch-skip 6 -c 1 -o gpurun_out/leanu/prof_$n -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-kernel-events --cpu-seconds 0.01 > gpurun_out/leanu/ncu_$n.log 2>&1
done
