#!/bin/bash
# A/B: pipelined producer vs plain producer, 3 repeats each, same box
O=gpurun_out/e8; mkdir -p $O
source tools/sweep.sh
P0=paper_2405_15573_b200/_build/libuhmv_pipe0.so
{
for rep in 1 2; do
for c in 1 2 3; do
ARGS="--config $c --steps 100"
ENVV="UHMV_LIB=$P0" run "c$c pipe0 r$rep"
ENVV="X=1" run "c$c pipe1 r$rep"
done
done
ARGS="--config 4"
ENVV="UHMV_LIB=$P0" run "c4 pipe0"
ENVV="X=1" run "c4 pipe1"
ARGS="--config 3 --adjoint"
ENVV="UHMV_LIB=$P0" run "c3adj pipe0"
ENVV="X=1" run "c3adj pipe1"
} > $O/exp.txt 2>&1
echo done
