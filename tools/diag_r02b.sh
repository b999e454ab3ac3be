#!/bin/bash
# re-entry check of the round-2 state + where the consumer time goes at configs 1-2
O=gpurun_out/d1; mkdir -p $O
source tools/sweep.sh
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
D=paper_2405_15573_b200/_build/libuhmv_diag.so
for c in 2 1 3; do
ARGS="--config $c"
ENVV="X=1" run "c$c base"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1" run "c$c nocompute"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=3" run "c$c nocompute-nogather"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1 UHMV_DEBUG_SKIP_WAITS=1" run "c$c nocompute-nowaits"
ENVV="UHMV_LIB=$D UHMV_DEBUG_SKIP_WAITS=1" run "c$c nowaits"
ENVV="UHMV_PROFILE=1" run "c$c prof"
done > $O/diag.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o $O/full_bulk_cfg2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_b2.log 2>&1
echo done
