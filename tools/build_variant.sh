#!/bin/bash
# Builds an A/B variant of libffspmv.so from a modified copy of one source
# file: tools/build_variant.sh <name> <file.cu|.cuh> <modified copy>
# (reuses build/ffspmv objects for everything else; output tools/variants/lib<name>.so)
set -e
name=$1; file=$2; mod=$3
R=/root/repo; C=$R/paper_1004_3719_b200/csrc
W=/tmp/var_$name; rm -rf $W; mkdir -p $W/csrc; cp $C/* $W/csrc/; cp $mod $W/csrc/$file
GEN="-gencode arch=compute_100a,code=sm_100a"
objs=""
for s in $(cd $C; ls *.cu); do
  if [ "$s" = "$file" ] || grep -q "include \"$file\"" $C/$s; then
    /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo $GEN -Xcompiler -fPIC,-fvisibility=hidden -I $W/csrc -c $W/csrc/$s -o $W/$s.o
    objs="$objs $W/$s.o"
  else
    objs="$objs $R/build/ffspmv/$s.o"
  fi
done
for s in $(cd $C; ls *.cpp); do objs="$objs $R/build/ffspmv/$s.o"; done
mkdir -p $R/tools/variants
/usr/local/cuda/bin/nvcc -shared $GEN -cudart static -o $R/tools/variants/lib$name.so $objs -Xlinker --exclude-libs,ALL
echo built $R/tools/variants/lib$name.so
