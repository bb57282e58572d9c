#!/bin/bash
# Round-end measurement evidence (run on the GPU box): bench lines of every config, the ncu
# launch lists of C3 and C5 train steps, and one `--set full` capture of a C3 train step.
#   tools/profile_round.sh <outdir under gpurun_out/>
set -x
cd "$(dirname "$0")/.."
out=gpurun_out/$1
mkdir -p "$out"
nvidia-smi -L > "$out/host.txt"; nproc >> "$out/host.txt"; lscpu | grep "Model name" >> "$out/host.txt"
python bench.py > "$out/bench_c3.jsonl" 2> "$out/bench_c3.err"
python bench.py --config c2 > "$out/bench_c2.jsonl" 2> "$out/bench_c2.err"
python bench.py --config c1 > "$out/bench_c1.jsonl" 2> "$out/bench_c1.err"
python bench.py --config c4 --steps 20 > "$out/bench_c4.jsonl" 2> "$out/bench_c4.err"
python bench.py --config c5 --steps 20 > "$out/bench_c5.jsonl" 2> "$out/bench_c5.err"
python bench.py --deterministic --no-cpu > "$out/bench_c3_deterministic.jsonl" 2> "$out/bench_c3_det.err"
python bench.py --loss l1_dssim --no-cpu > "$out/bench_c3_dssim.jsonl" 2> "$out/bench_c3_dssim.err"
python bench.py --no-graph --no-cpu > "$out/bench_c3_nograph.jsonl" 2> "$out/bench_c3_nograph.err"
python bench.py --impl reference --steps 3 > "$out/bench_reference.jsonl" 2> "$out/bench_reference.err"
python bench.py --impl reference --config c2 > "$out/bench_reference_c2.jsonl" 2> "$out/bench_reference_c2.err"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file "$out/launches_c3_train.csv" python tools/profile_step.py --steps 3 --const-target > "$out/ncu_l3.log" 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file "$out/launches_c5_train.csv" python tools/profile_step.py --steps 2 --config c5 --const-target > "$out/ncu_l5.log" 2>&1
ncu --set full --clock-control none --import-source on -o "$out/ncu_step" \
  python tools/profile_step.py --steps 1 --const-target > "$out/ncu_full.log" 2>&1
