#!/bin/bash
# Build a variant of libisg.so with extra nvcc flags for ONE source file, for A/B timing:
#   tools/build_variant.sh <name> <file.cu> <flags...>  ->  build/variants/libisg_<name>.so
# Run with ISG_LIB_PATH=build/variants/libisg_<name>.so.  Needs the regular build first.
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p build/variants
objs=()
for o in build/isg/*.o; do
  if [ "$(basename "$o" .o)" = "$(basename "$src" .cu)" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC,-fopenmp -I include "$@" -c "paper_2403_14244_b200/csrc/$src" \
      -o "build/variants/${name}.o"
    objs+=("build/variants/${name}.o")
  else
    objs+=("$o")
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC,-fopenmp \
  -o "build/variants/libisg_${name}.so" "${objs[@]}" -ldl -lgomp
echo "build/variants/libisg_${name}.so"
