#!/bin/bash
# adjoint of configs 1-2 with the product-biased stored form: nearfield shares
O=gpurun_out/e15; mkdir -p $O
source tools/sweep.sh
{
for c in 2 1; do
ARGS="--config $c --steps 100 --adjoint"
ENVV="X=1" run "c$c adj default"
ENVV="UHMV_FACTOR_BIAS=1" run "c$c adj bias1"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.2,0.1,0.2,0.5" run "c$c adj .2.1.2.5"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.3,0.2,0.3,0.2" run "c$c adj .3.2.3.2"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.1,0.1,0.3,0.5" run "c$c adj .1.1.3.5"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.5,0.2,0.2,0.1" run "c$c adj .5.2.2.1"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.2,0.2,0.4,0.2" run "c$c adj .2.2.4.2"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.05,0.05,0.1,0.8" run "c$c adj .05.05.1.8"
ENVV="X=1" run "c$c adj default again"
done
} > $O/exp.txt 2>&1
echo done
