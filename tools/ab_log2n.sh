mkdir -p gpurun_out/ab
V=$PWD/paper_1203_5004_b200/lib/var
: > gpurun_out/ab/pf26.log
for r in 1 2 3; do for lg in 26 27; do for n in A B; do
  HOOD_B200_LIB=$V/$n.so timeout 300 python bench.py --config 4 --log2n $lg --steps 30 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/$n $lg /" >> gpurun_out/ab/pf26.log
done; done; done
