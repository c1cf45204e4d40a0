#!/bin/bash
# Round-2 profile capture (under gpurun, one B200): bench lines (headline WResNet-152-4 with FC / LSTM as
# other_workloads), ncu launch lists, ncu --set full of the dominant GEMM class (stage-0 1x1 data gradient with
# fused add + mask), the 3x3 convolutions, and the MultiFetch / reduce piece kernels of a k = 8 plan.
# Outputs in gpurun_out/prof2/ (summaries are copied to profiles/).
set -x
O=gpurun_out/prof2
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c3_k1.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
K=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_c3_k8.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -c 16 \
  -o $O/full_c3_gemm python tools/breakdown.py units 2 4 32 224 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_kernel -s 3 -c 4 \
  -o $O/full_c3_conv python tools/breakdown.py units 0,0,3 4 32 112 > /dev/null 2>&1
K=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pieces -c 12 \
  -o $O/full_pieces_k8 python tools/breakdown.py units 2 4 32 224 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
for f in full_c3_gemm full_c3_conv full_pieces_k8; do
  ncu -i $O/$f.ncu-rep --page raw --csv --metrics $M > $O/ncu_$f.csv 2>/dev/null
  python tools/ncu_summary.py $O/$f.ncu-rep > $O/ncu_$f.md 2>&1
done
rm -f $O/*.ncu-rep
ls -la $O
