# Ring shapes x libraries on one box: tools/shape_ab.sh "A B" "118 128" config...
vs=$1; rs=$2; shift 2
for c in "$@"; do for v in $vs; do for r in $rs; do
  HOOD_RING=$r HOOD_B200_LIB=paper_1203_5004_b200/lib/var/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --cpu-seconds 0.05 2>&1 | tail -1 | python tools/benchline.py "$v R=$r" | cut -c1-110
done; done; done
