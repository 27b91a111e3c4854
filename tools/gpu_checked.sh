# The GPU suite against the bounds-checked build (-DHOOD_CHECKED: device
# invariant checks that trap) in place of compute-sanitizer (closed on the pool).
mkdir -p gpurun_out
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_checked.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_checked.log
HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_checked.so timeout 900 python tools/adv_sweep.py 4 > gpurun_out/adv_sweep_checked.log 2>&1; echo "rc=$?" >> gpurun_out/adv_sweep_checked.log
for c in 1 2 3 4 5; do HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_checked.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --cpu-seconds 0.01 2>&1 | tail -1 | python tools/benchline.py >> gpurun_out/bench_checked.log; done
tail -3 gpurun_out/pytest_checked.log
