#!/bin/bash
# Like build_variant.sh but recompiles only the named .cu (the other objects
# come from build/ffspmv): tools/build_variant_one.sh <name> <unit.cu> <file> <modified copy>
set -e
name=$1; unit=$2; file=$3; mod=$4
R=/root/repo; C=$R/paper_1004_3719_b200/csrc
W=/tmp/var_$name; rm -rf $W; mkdir -p $W/csrc; cp $C/* $W/csrc/; cp $mod $W/csrc/$file
GEN="-gencode arch=compute_100a,code=sm_100a"
objs=""
for s in $(cd $C; ls *.cu); do
  if [ "$s" = "$unit" ]; then
    /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo $GEN -Xptxas -v -Xcompiler -fPIC,-fvisibility=hidden -I $W/csrc -c $W/csrc/$s -o $W/$s.o > $W/ptxas.log 2>&1
    objs="$objs $W/$s.o"
  else
    objs="$objs $R/build/ffspmv/$s.o"
  fi
done
for s in $(cd $C; ls *.cpp); do objs="$objs $R/build/ffspmv/$s.o"; done
mkdir -p $R/tools/variants
/usr/local/cuda/bin/nvcc -shared $GEN -cudart static -o $R/tools/variants/lib$name.so $objs -Xlinker --exclude-libs,ALL
echo built $R/tools/variants/lib$name.so
