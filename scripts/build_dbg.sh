# debug build of libtprod.so with -D$1 into ab/dbg/libtprod.so (load with TPROD_LIB=ab/dbg/libtprod.so)
set -e
cd "$(dirname "$0")/.."
objs=""
for f in paper_1806_07247_b200/csrc/*.cu; do
  o=ab/dbg/$(basename $f).o
  if [ "$(basename $f)" = "$2" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -D$1 -Iinclude -c $f -o $o
  else
    cp paper_1806_07247_b200/build/$(basename $f).o $o
  fi
  objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/dbg/libtprod.so $objs -ldl
