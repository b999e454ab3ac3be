#!/bin/bash
# ordered output (NEAR stores, FAR waits + adds: no memset, no atomics): full GPU suite + A/B
O=gpurun_out/e7; mkdir -p $O
source tools/sweep.sh
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
{
for c in 2 1 3 4; do
ARGS="--config $c"
ENVV="UHMV_W_ORDER=0" run "c$c atomic+memset"
ENVV="X=1" run "c$c ordered"
ARGS="--config $c --adjoint"
ENVV="UHMV_W_ORDER=0" run "c$c adj atomic+memset"
ENVV="X=1" run "c$c adj ordered"
done
ARGS="--config 2"
ENVV="UHMV_Z_ELEMS=12288" run "c2 ordered z12k"
ENVV="UHMV_Z_ELEMS=12288 UHMV_NEAR_INTERLEAVE=0.1,0.1,0.2,0.6" run "c2 ordered z12k near.6"
ENVV="UHMV_NEAR_INTERLEAVE=0.1,0.1,0.2,0.6" run "c2 ordered near.6"
ENVV="UHMV_NEAR_INTERLEAVE=0.3,0.1,0.2,0.4" run "c2 ordered near.4"
} > $O/exp.txt 2>&1
echo done
