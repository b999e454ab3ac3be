#!/bin/bash
# config 2 with the four-phase chain: nearfield shares and op granularity, 3 repeats of the candidates
O=gpurun_out/e14; mkdir -p $O
source tools/sweep.sh
{
ARGS="--config 2 --steps 100"
for r in 1 2 3; do
ENVV="X=1" run "c2 default r$r"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.2,0.0,0.6" run "c2 near.2.2.0.6 r$r"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.2,0.0,0.5" run "c2 near.3.2.0.5 r$r"
done
ENVV="UHMV_NEAR_INTERLEAVE=0.4,0.2,0.0,0.4" run "c2 near.4.2.0.4"
ENVV="UHMV_NEAR_INTERLEAVE=0.25,0.25,0.0,0.5" run "c2 near.25.25.0.5"
ENVV="UHMV_NEAR_INTERLEAVE=0.15,0.25,0.0,0.6" run "c2 near.15.25.0.6"
ENVV="UHMV_FAR_ROWS=20" run "c2 far20"
ENVV="UHMV_SPLIT_P1_OUT=96" run "c2 p1o96"
ENVV="UHMV_SPLIT_Z_ROWS=16" run "c2 z16rows"
ENVV="UHMV_Z_ELEMS=16384" run "c2 z16k"
} > $O/exp.txt 2>&1
echo done
