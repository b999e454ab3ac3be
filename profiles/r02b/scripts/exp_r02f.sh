#!/bin/bash
O=gpurun_out/e4; mkdir -p $O
source tools/sweep.sh
D=paper_2405_15573_b200/_build/libuhmv_diag.so
{
for c in 2 3; do
ARGS="--config $c"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1 UHMV_PROFILE=1" run "c$c nocompute prof"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=3 UHMV_PROFILE=1" run "c$c nocompute-nogather prof"
ENVV="UHMV_LIB=$D UHMV_PROFILE=1" run "c$c prof"
done
ARGS="--config 2 --view near"
ENVV="X=1" run "c2 near-only"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1" run "c2 near-only nocompute"
ARGS="--config 2 --view far"
ENVV="X=1" run "c2 far-only"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1" run "c2 far-only nocompute"
ARGS="--config 3 --view near"
ENVV="X=1" run "c3 near-only"
ARGS="--config 3 --view far"
ENVV="X=1" run "c3 far-only"
} > $O/exp.txt 2>&1
echo done
