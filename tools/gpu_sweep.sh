# Register cap x ring shape sweep (configs 2 and 5), kernel time only.
for r in 168 128 104 96; do for d in 12 13 22 23; do for c in 2 5; do
  HOOD_B200_LIB=paper_1203_5004_b200/lib/var/libhood_r$r.so HOOD_RING=$d timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-seconds 0.05 2>&1 | tail -1 | python tools/benchline.py "r=$r R=$d"
done; done; done
