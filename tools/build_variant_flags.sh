#!/bin/bash
# A/B variant of libffspmv.so with extra compile flags for the units that
# see them (default: runs.cu, runs_build.cpp, abi.cpp; the other objects come
# from build/ffspmv):
#   tools/build_variant_flags.sh <name> "<flags>" [unit ...]
set -e
name=$1; flags=$2; shift 2
units="$*"; [ -z "$units" ] && units="runs.cu runs_build.cpp abi.cpp"
R=/root/repo; C=$R/paper_1004_3719_b200/csrc
W=/tmp/varf_$name; rm -rf $W; mkdir -p $W
GEN="-gencode arch=compute_100a,code=sm_100a"
objs=""
for s in $(cd $C; ls *.cu *.cpp); do
  if [[ " $units " == *" $s "* ]]; then
    if [[ $s == *.cu ]]; then
      /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo $GEN $flags -Xptxas -v -Xcompiler -fPIC,-fvisibility=hidden -I $C -c $C/$s -o $W/$s.o > $W/ptxas_$s.log 2>&1
    else
      g++ -std=c++17 -O3 -fPIC -fvisibility=hidden $flags -I /usr/local/cuda/include -I $C -c $C/$s -o $W/$s.o
    fi
    objs="$objs $W/$s.o"
  else
    objs="$objs $R/build/ffspmv/$s.o"
  fi
done
mkdir -p $R/tools/variants
/usr/local/cuda/bin/nvcc -shared $GEN -cudart static -o $R/tools/variants/lib$name.so $objs -Xlinker --exclude-libs,ALL -ldl
echo built $R/tools/variants/lib$name.so
