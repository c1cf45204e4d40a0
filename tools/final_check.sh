#!/bin/bash
# End-of-round check under gpurun (one B200): the GPU test suite, smoke(), the bench line (default config),
# the reference arm, and the ncu launch list of the headline step.  Outputs in gpurun_out/final/.
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c3_k1.csv \
  python tools/breakdown.py 3 > /dev/null 2>&1
tail -2 $O/gputest.log; tail -1 $O/smoke.log
