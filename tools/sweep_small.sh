#!/bin/bash
# configs 1-2 (chain-latency-bound): op-splitting / interleave sweep + timelines
source tools/sweep.sh
O=gpurun_out/small; mkdir -p $O
for c in 1 2; do
ARGS="--config $c"
ENVV="X=1" run "c$c base"
ENVV="UHMV_SPLIT_Z_ROWS=8" run "c$c z8"
ENVV="UHMV_SPLIT_Z_ROWS=4" run "c$c z4"
ENVV="UHMV_FAR_ROWS=16" run "c$c far16"
ENVV="UHMV_FAR_ROWS=32" run "c$c far32"
ENVV="UHMV_SPLIT_P1_OUT=64" run "c$c p1o64"
ENVV="UHMV_SPLIT_U_COLS=64" run "c$c u64"
ENVV="UHMV_SPLIT_Z_ROWS=8 UHMV_FAR_ROWS=32 UHMV_SPLIT_P1_OUT=64" run "c$c combo"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c$c nearlate"
ENVV="UHMV_NEAR_INTERLEAVE=0.6,0.1,0.1,0.2" run "c$c nearearly"
ENVV="UHMV_PROFILE=1" run "c$c prof"
timeout 300 python tools/timeline.py $c fwd > $O/timeline_c$c.txt 2>&1
UHMV_SPLIT_Z_ROWS=8 UHMV_FAR_ROWS=32 UHMV_SPLIT_P1_OUT=64 timeout 300 python tools/timeline.py $c fwd > $O/timeline_c${c}_combo.txt 2>&1
done
