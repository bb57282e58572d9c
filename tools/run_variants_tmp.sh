for v in base nopf; do
  if [ $v = base ]; then unset ISG_LIB_PATH; else export ISG_LIB_PATH=$PWD/build/variants/libisg_$v.so; fi
  python bench.py --config c3 --no-cpu --steps 200 > gpurun_out/v_$v.jsonl 2>gpurun_out/v_$v.err
done
