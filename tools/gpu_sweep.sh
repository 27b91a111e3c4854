for v in "r128 118" "r128 128" "r104 124" "r128 124" "default 118" "default 128"; do set -- $v
  lib=paper_1203_5004_b200/lib/var/libhood_$1.so; [ "$1" = default ] && lib=""
  for c in 2 5 4; do HOOD_B200_LIB=$lib HOOD_RING=$2 timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-seconds 0.05 2>&1 | tail -1 | python tools/benchline.py "$1 R=$2"; done
done
