#!/bin/bash
# tail filler (a 5th nearfield share behind the FAR ops) and the cost of the output memset
O=gpurun_out/e6; mkdir -p $O
source tools/sweep.sh
D=paper_2405_15573_b200/_build/libuhmv_diag.so
{
ARGS="--config 2"
ENVV="X=1" run "c2 base"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=4" run "c2 nomemset"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.2,0.4,0.1" run "c2 tail.1"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.2,0.3,0.2" run "c2 tail.2"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.2,0.2,0.3" run "c2 tail.3"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.2,0.3,0.2 UHMV_Z_ELEMS=12288" run "c2 tail.2 z12k"
ENVV="UHMV_NEAR_INTERLEAVE=0.1,0.1,0.2,0.4,0.2 UHMV_Z_ELEMS=12288" run "c2 tail.2b z12k"
ARGS="--config 1"
ENVV="X=1" run "c1 base"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=4" run "c1 nomemset"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.6,0.2" run "c1 tail.2"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.4,0.4" run "c1 tail.4"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.2,0.6" run "c1 tail.6"
ARGS="--config 3"
ENVV="X=1" run "c3 base"
ENVV="UHMV_NEAR_INTERLEAVE=0.35,0.1,0.2,0.3,0.05" run "c3 tail.05"
ENVV="UHMV_NEAR_INTERLEAVE=0.35,0.1,0.2,0.25,0.1" run "c3 tail.1"
ARGS="--config 4"
ENVV="X=1" run "c4 base"
ENVV="UHMV_NEAR_INTERLEAVE=0.35,0.1,0.2,0.3,0.05" run "c4 tail.05"
} > $O/exp.txt 2>&1
echo done
