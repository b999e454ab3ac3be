#!/bin/bash
# stored form of the coupling: product form for more blocks (no U phase in the forward chain)
O=gpurun_out/e11; mkdir -p $O
source tools/sweep.sh
UHMV_FACTOR_BIAS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -q -m gpu -x > $O/pytest_product.log 2>&1; echo "rc=$?" >> $O/pytest_product.log
{
for c in 2 1 3; do
ARGS="--config $c --steps 60"
ENVV="X=1" run "c$c bias1"
ENVV="UHMV_FACTOR_BIAS=0.75" run "c$c bias.75"
ENVV="UHMV_FACTOR_BIAS=0.5" run "c$c bias.5"
ENVV="UHMV_FACTOR_BIAS=0" run "c$c bias0"
ENVV="UHMV_FACTOR_BIAS=0 UHMV_Z_ELEMS=12288" run "c$c bias0 z12k"
ENVV="UHMV_FACTOR_BIAS=0 UHMV_Z_ELEMS=8192" run "c$c bias0 z8k"
ENVV="UHMV_FACTOR_BIAS=0 UHMV_NEAR_INTERLEAVE=0.2,0.1,0.0,0.7" run "c$c bias0 near.2.1.0.7"
ENVV="UHMV_FACTOR_BIAS=0 UHMV_NEAR_INTERLEAVE=0.3,0.2,0.0,0.5" run "c$c bias0 near.3.2.0.5"
ARGS="--config $c --steps 60 --adjoint"
ENVV="X=1" run "c$c adj bias1"
ENVV="UHMV_FACTOR_BIAS=0" run "c$c adj bias0"
done
} > $O/exp.txt 2>&1
UHMV_FACTOR_BIAS=0 timeout 300 python tools/timeline.py 2 fwd full > $O/timeline_c2_product.txt 2>&1
UHMV_FACTOR_BIAS=0 timeout 300 python tools/timeline.py 1 fwd full > $O/timeline_c1_product.txt 2>&1
echo done
