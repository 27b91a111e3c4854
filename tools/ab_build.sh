# Build the ring library from a git revision (A) and from the working tree (B)
# into paper_1203_5004_b200/lib/var/{A,B}.so for same-box A/B timing.
set -e
rev=${1:-HEAD}
tmp=$(mktemp -d)
mkdir -p $tmp/pkg/csrc $tmp/include
git show $rev:include/hood_b200.h > $tmp/include/hood_b200.h
srcA=""
for f in hood_kernels.cu hood_capi.cu hood_kernels.cuh hood_device.cuh hood_host.cpp; do
  if git show $rev:paper_1203_5004_b200/csrc/$f > $tmp/pkg/csrc/$f 2>/dev/null; then
    case $f in *.cu|*.cpp) srcA="$srcA $tmp/pkg/csrc/$f";; esac
  fi
done
mkdir -p paper_1203_5004_b200/lib/var
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared --expt-relaxed-constexpr -I include"
$NV -o paper_1203_5004_b200/lib/var/A.so $srcA &
$NV -o paper_1203_5004_b200/lib/var/B.so paper_1203_5004_b200/csrc/hood_kernels.cu paper_1203_5004_b200/csrc/hood_capi.cu paper_1203_5004_b200/csrc/hood_host.cpp &
wait
rm -rf $tmp
