#!/bin/bash
# A/B timing of library variants built by tools/build_variant.sh (run on the GPU box):
#   tools/ab_variants.sh <config> <steps> base <name>...  ->  gpurun_out/v_<name>.jsonl
# "base" is the regular in-tree libisg.so.
cd "$(dirname "$0")/.."
cfg=$1; steps=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset ISG_LIB_PATH; else export ISG_LIB_PATH=$PWD/build/variants/libisg_$v.so; fi
  python bench.py --config "$cfg" --no-cpu --steps "$steps" > "gpurun_out/v_$v.jsonl" 2> "gpurun_out/v_$v.err"
done
