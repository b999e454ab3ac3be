#!/bin/bash
# cheap knobs after nacc1: warp-per-row threshold, NEAR rows per op, no-split share, interleave
O=gpurun_out/e10; mkdir -p $O
source tools/sweep.sh
{
for c in 2 1; do
ARGS="--config $c --steps 60"
ENVV="X=1" run "c$c base"
ENVV="UHMV_WIDE_COLS=128" run "c$c wide128"
ENVV="UHMV_WIDE_COLS=64" run "c$c wide64"
ENVV="UHMV_WIDE_COLS=200" run "c$c wide200"
ENVV="UHMV_ROWS_PER_CHUNK=10" run "c$c rpc10"
ENVV="UHMV_ROWS_PER_CHUNK=8" run "c$c rpc8"
ENVV="UHMV_NOSPLIT=0.5" run "c$c nosplit.5"
ENVV="UHMV_NOSPLIT=0.2" run "c$c nosplit.2"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.1,0.2,0.4" run "c$c near.3.1.2.4"
ENVV="UHMV_NEAR_INTERLEAVE=0.1,0.1,0.3,0.5" run "c$c near.1.1.3.5"
ENVV="UHMV_NEAR_INTERLEAVE=0.25,0.15,0.25,0.35" run "c$c near.25.15.25.35"
ENVV="UHMV_NEAR_INTERLEAVE=0.1,0.05,0.15,0.7" run "c$c near.1.05.15.7"
ENVV="X=1" run "c$c base again"
done
} > $O/exp.txt 2>&1
echo done
