#!/bin/bash
# adjoint copy at the large configs (forced on): adjoint lines of configs 3-4 + full-size parity
O=gpurun_out/e18; mkdir -p $O
source tools/sweep.sh
{
ARGS="--config 4 --adjoint --steps 30"
ENVV="X=1" run "c4 adj no-copy"
ENVV="UHMV_ADJ_COPY=1" run "c4 adj copy"
ENVV="UHMV_ADJ_COPY=1 UHMV_NEAR_INTERLEAVE_ADJ=0.35,0.1,0.2,0.35" run "c4 adj copy fwd-shares"
ARGS="--config 3 --adjoint --steps 50"
ENVV="X=1" run "c3 adj no-copy"
ENVV="UHMV_ADJ_COPY=1" run "c3 adj copy"
ENVV="UHMV_ADJ_COPY=1 UHMV_NEAR_INTERLEAVE_ADJ=0.35,0.1,0.2,0.35" run "c3 adj copy fwd-shares"
ARGS="--config 3 --steps 50"
ENVV="UHMV_ADJ_COPY=1" run "c3 fwd copy"
ARGS="--config 4 --steps 30"
ENVV="UHMV_ADJ_COPY=1" run "c4 fwd copy"
} > $O/exp.txt 2>&1
UHMV_ADJ_COPY=1 timeout 900 python -m pytest tests/test_gpu_workloads.py tests/test_gpu_parity.py -q -m gpu -x > $O/pytest_copy_large.log 2>&1; echo "rc=$?" >> $O/pytest_copy_large.log
echo done
