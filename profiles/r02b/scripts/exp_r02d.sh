#!/bin/bash
# pipelined producer (next op's ticket -> order -> header -> records chain behind the copies)
O=gpurun_out/e2; mkdir -p $O
source tools/sweep.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_symmetric.py -q -m gpu -x > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
D=paper_2405_15573_b200/_build/libuhmv_diag.so
{
for c in 2 1 3 4; do
ARGS="--config $c"
ENVV="X=1" run "c$c pipe"
ENVV="UHMV_PROFILE=1" run "c$c pipe prof"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1" run "c$c pipe nocompute"
done
ARGS="--config 3 --adjoint"; ENVV="X=1" run "c3adj pipe"
ARGS="--config 4 --adjoint"; ENVV="X=1" run "c4adj pipe"
ARGS="--config 3 --format h"; ENVV="X=1" run "c3H pipe"
ARGS="--config 3 --format sym"; ENVV="X=1" run "c3sym pipe"
} > $O/exp.txt 2>&1
timeout 300 python tools/timeline.py 2 fwd > $O/timeline_c2.txt 2>&1
timeout 300 python tools/timeline.py 1 fwd > $O/timeline_c1.txt 2>&1
echo done
