#!/bin/bash
# config 1 nearfield shares with the product-biased stored form (default below 1 GB)
O=gpurun_out/e12; mkdir -p $O
source tools/sweep.sh
{
ARGS="--config 1 --steps 100"
ENVV="X=1" run "c1 default"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.0,0.7" run "c1 near.2.1.0.7"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.2,0.0,0.5" run "c1 near.3.2.0.5"
ENVV="UHMV_NEAR_INTERLEAVE=0.1,0.1,0.0,0.8" run "c1 near.1.1.0.8"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.1,0.1,0.5" run "c1 near.3.1.1.5"
ENVV="UHMV_NEAR_INTERLEAVE=0.4,0.2,0.0,0.4" run "c1 near.4.2.0.4"
ENVV="X=1" run "c1 default again"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.1,0.0,0.7" run "c1 near.2.1.0.7 again"
ARGS="--config 2 --steps 100"
ENVV="X=1" run "c2 default"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.2,0.0,0.5" run "c2 near.3.2.0.5"
ENVV="UHMV_NEAR_INTERLEAVE=0.2,0.2,0.0,0.6" run "c2 near.2.2.0.6"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.1,0.1,0.5" run "c2 near.3.1.1.5"
} > $O/exp.txt 2>&1
echo done
