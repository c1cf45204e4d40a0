#!/bin/bash
# Round profile capture (run under gpurun on one B200): bench lines, ncu launch lists, and `ncu --set full`
# captures of the dominant kernels of configs 1 and 3.  Outputs in gpurun_out/prof/ (copy the summaries to
# profiles/).  Usage: tools/profile_round.sh
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 600 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config 3 --steps 10 --virtual-k 1 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 2 --virtual-k 1 > $O/bench_c2.json 2> $O/bench_c2.err
# configs[1]: launch list of the bench command, full capture of its two GEMMs
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --virtual-k 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -s 4 -c 2 \
  -o $O/full_c1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --virtual-k 1 > /dev/null 2>&1
# configs[3]: launch list of one step (tools/breakdown.py launches the bench's kernels one by one)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_c3.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
# full captures: stage-0 1x1 GEMMs (the dominant 1x1 data gradient with its fused add+mask epilogue) of a
# 2-unit stage-0 WResNet (batch 32, 56x56), and the stage-2 3x3 convolution kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -c 16 \
  -o $O/full_c3_gemm python tools/breakdown.py units 2 4 32 224 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_kernel -s 3 -c 4 \
  -o $O/full_c3_conv python tools/breakdown.py units 0,0,3 4 32 112 > /dev/null 2>&1
# export the judged metrics as CSV + markdown summaries and drop the large reports (gpurun copies back <= 64 MiB)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
for f in full_c1 full_c3_gemm full_c3_conv; do
  ncu -i $O/$f.ncu-rep --page raw --csv --metrics $M > $O/ncu_$f.csv 2>/dev/null
  python tools/ncu_summary.py $O/$f.ncu-rep > $O/ncu_$f.md 2>&1
done
rm -f $O/full_c3_gemm.ncu-rep $O/full_c3_conv.ncu-rep
ls -la $O
du -sh $O
