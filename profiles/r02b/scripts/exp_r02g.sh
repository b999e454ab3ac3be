#!/bin/bash
# chain shortening at configs 1-3: byte-threshold splits of the long Z / U ops
O=gpurun_out/e5; mkdir -p $O
source tools/sweep.sh
{
for c in 2 1; do
for v in "" "--view far"; do
ARGS="--config $c $v"
ENVV="X=1" run "c$c $v base"
ENVV="UHMV_Z_ELEMS=12288" run "c$c $v z12k"
ENVV="UHMV_Z_ELEMS=8192" run "c$c $v z8k"
ENVV="UHMV_Z_ELEMS=6144" run "c$c $v z6k"
ENVV="UHMV_Z_ELEMS=4096" run "c$c $v z4k"
ENVV="UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096" run "c$c $v z8k u4k"
ENVV="UHMV_Z_ELEMS=6144 UHMV_U_ELEMS=3072" run "c$c $v z6k u3k"
ENVV="UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096 UHMV_SPLIT_P1_OUT=96" run "c$c $v z8k u4k p1o96"
ENVV="UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096 UHMV_FAR_ROWS=20" run "c$c $v z8k u4k far20"
done
done
ARGS="--config 3"
ENVV="UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096" run "c3 z8k u4k"
ENVV="UHMV_Z_ELEMS=16384 UHMV_U_ELEMS=8192" run "c3 z16k u8k"
ARGS="--config 3 --view far"
ENVV="UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096" run "c3 far z8k u4k"
} > $O/exp.txt 2>&1
UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096 timeout 300 python tools/timeline.py 2 fwd full > $O/timeline_c2_z8k_u4k.txt 2>&1
UHMV_Z_ELEMS=8192 UHMV_U_ELEMS=4096 timeout 300 python tools/timeline.py 2 fwd far > $O/timeline_c2_far_z8k_u4k.txt 2>&1
timeout 300 python tools/timeline.py 2 fwd far > $O/timeline_c2_far.txt 2>&1
echo done
