#!/bin/bash
# Build a variant of libisg.so with extra nvcc flags for ONE source file, for A/B timing:
#   tools/build_variant.sh <name> <file.cu> <flags...>  ->  build/variants/libisg_<name>.so
#   (<file.cu> = ALL: every source gets the flags, for macros shared through headers)
# Run with ISG_LIB_PATH=build/variants/libisg_<name>.so.  Needs the regular build first.
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p build/variants
objs=()
for o in build/isg/*.o; do
  if [ "$src" = ALL ] || [ "$(basename "$o" .o)" = "$(basename "$src" .cu)" ]; then
    f=paper_2403_14244_b200/csrc/$(basename "$o" .o).cu
    extra=""; [ "$(basename "$o")" = k_adapt.o ] && extra="-fmad=false"
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC,-fopenmp -I include $extra "$@" -c "$f" \
      -o "build/variants/${name}_$(basename "$o")"
    objs+=("build/variants/${name}_$(basename "$o")")
  else
    objs+=("$o")
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC,-fopenmp \
  -o "build/variants/libisg_${name}.so" "${objs[@]}" -ldl -lgomp
echo "build/variants/libisg_${name}.so"
