#!/bin/bash
# Round profile capture (run under gpurun on one B200): bench lines, ncu launch lists, and one
# `ncu --set full` capture of the dominant kernel of configs 1 and 3.  Outputs in gpurun_out/prof/.
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 600 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config 3 --steps 10 --virtual-k 1 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --virtual-k 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -s 4 -c 2 \
  -o $O/full_c1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --virtual-k 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_c3.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_kernel -s 3 -c 4 \
  -o $O/full_conv python tools/breakdown.py units 0,0,3 4 32 112 > /dev/null 2>&1
ls -la $O
