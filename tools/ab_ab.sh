# same-box A/B of lib/var/A.so (before) vs lib/var/B.so (after) on the given configs
# usage: bash tools/ab_ab.sh "4 3" [rounds] [tag] ["A B C"]
mkdir -p gpurun_out/ab
cfgs=${1:-"4"}; rounds=${2:-3}; tag=${3:-ab}; vars=${4:-"A B"}
V=$PWD/paper_1203_5004_b200/lib/var
: > gpurun_out/ab/$tag.log
for r in $(seq $rounds); do for c in $cfgs; do for n in $vars; do
  st=40; [ $c = 4 ] && st=20
  HOOD_B200_LIB=$V/$n.so timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/$n /" >> gpurun_out/ab/$tag.log
done; done; done
