# Same-box comparison of several libraries: tools/abc_run.sh "A B C" config...
vs=$1; shift
for rep in 1 2; do for c in "$@"; do for v in $vs; do
  HOOD_B200_LIB=paper_1203_5004_b200/lib/var/$v.so timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --cpu-seconds 0.05 2>&1 | tail -1 | python tools/benchline.py "$v" | cut -c1-110
done; done; done
