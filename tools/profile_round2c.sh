#!/bin/bash
# Round-2 (third session) profile capture under gpurun, one B200: the bench line, the ncu launch list of the
# headline step, and ncu --set full captures (per-launch DRAM traffic) of the three workloads' dominant kernels:
# WResNet stage-0 1x1 data gradient with the fused add+mask epilogue (wide chunks, MODE 45), the LSTM batched
# input-gradient GEMM L.dx (2-CTA pairs), the FC weight gradient with the fused momentum-SGD epilogue.
# Outputs in gpurun_out/prof3/ (summaries are copied to profiles/).
set -x
O=gpurun_out/prof3
mkdir -p $O
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c3_k1.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
fi
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_bf16_kernel<(\(int\))?256, (\(bool\))?(0|false), (\(bool\))?(1|true), (\(int\))?45,' -c 4 \
  -o $O/full_c3_dgrad python tools/breakdown.py units 2 4 32 224 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_bf16_kernel<(\(int\))?256, (\(bool\))?(0|false), (\(bool\))?(1|true), (\(int\))?16,' -c 2 \
  -o $O/full_c2_dx python tools/breakdown.py lstm 1 4096 20 128 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_bf16_kernel<(\(int\))?256, (\(bool\))?(1|true), (\(bool\))?(1|true), (\(int\))?19,' -c 2 \
  -o $O/full_c1_wgrad python tools/breakdown.py 1 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
for f in full_c3_dgrad full_c2_dx full_c1_wgrad; do
  ncu -i $O/$f.ncu-rep --page raw --csv --metrics $M > $O/ncu_$f.csv 2>/dev/null
  python tools/ncu_summary.py $O/$f.ncu-rep > $O/ncu_$f.md 2>&1
done
rm -f $O/*.ncu-rep
ls -la $O
