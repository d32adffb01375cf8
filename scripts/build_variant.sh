#!/bin/bash
# Build a variant of libs2w.so with extra nvcc flags for one translation unit
# (development aid for A/B timing on the GPU box via S2W_LIB).
#   scripts/build_variant.sh NAME SRC.cu "-DFOO=1 ..."
# -> lib_var/NAME/libs2w.so (other objects from build/, i.e. run `make` first)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
mkdir -p build_var/$name lib_var/$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xptxas -v -Iinclude $flags \
  -c paper_1211_1680_b200/csrc/$src -o build_var/$name/${src%.cu}.o 2> build_var/$name/ptxas.log \
  || (cat build_var/$name/ptxas.log; false)
objs=""
for o in build/*.o; do
  b=$(basename $o)
  if [ "$b" = "${src%.cu}.o" ]; then objs="$objs build_var/$name/$b"; else objs="$objs $o"; fi
done
nvcc $ARCH -shared -o lib_var/$name/libs2w.so $objs -lcudart_static -lrt -lpthread -ldl
echo "built lib_var/$name/libs2w.so"
