# ncu full capture of the ring kernel on config $1 (default 2) -> gpurun_out/prof_$2.ncu-rep
c=${1:-2}; tag=${2:-c$c}
timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/plain_$tag.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_hull -s 2 -c 1 -o gpurun_out/prof_$tag -f \
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --cpu-seconds 0.1 > gpurun_out/ncu_$tag.log 2>&1
tail -3 gpurun_out/ncu_$tag.log
