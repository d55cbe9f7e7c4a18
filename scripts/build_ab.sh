#!/bin/bash
# Build the library of git revision $1 into ab/libtprod_$1.so for A/B timing (TPROD_LIB=...).
set -e
rev=${1:-HEAD}
d=/tmp/ab_$rev; rm -rf $d; mkdir -p $d/csrc $d/include
git -C /root/repo archive $rev paper_1806_07247_b200/csrc include | tar -x -C $d
mkdir -p /root/repo/ab
objs=""
for f in $d/paper_1806_07247_b200/csrc/*.cu; do
  o=$d/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I$d/include -c $f -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/ab/libtprod_$rev.so $objs -ldl
echo built /root/repo/ab/libtprod_$rev.so
