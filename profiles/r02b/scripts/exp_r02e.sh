#!/bin/bash
# stage-ring geometry at configs 1-2 (bytes in flight per SM vs stage granularity)
O=gpurun_out/e3; mkdir -p $O
source tools/sweep.sh
D=paper_2405_15573_b200/_build/libuhmv_diag.so
{
for c in 2 1; do
ARGS="--config $c"
ENVV="X=1" run "c$c base"
ENVV="UHMV_STAGE_ELEMS=1120" run "c$c st1120"
ENVV="UHMV_STAGE_ELEMS=1200" run "c$c st1200"
ENVV="UHMV_STAGE_ELEMS=704" run "c$c st704"
ENVV="UHMV_STAGE_ELEMS=600" run "c$c st600"
ENVV="UHMV_STAGE_ELEMS=840" run "c$c st840"
ENVV="UHMV_BULK_CTAS=2" run "c$c ctas2"
ENVV="UHMV_BULK_CTAS=2 UHMV_STAGE_ELEMS=1120" run "c$c ctas2 st1120"
ENVV="UHMV_BULK_CTAS=2 UHMV_STAGE_ELEMS=704" run "c$c ctas2 st704"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1 UHMV_STAGE_ELEMS=1120" run "c$c nocompute st1120"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1 UHMV_STAGE_ELEMS=704" run "c$c nocompute st704"
ENVV="UHMV_LIB=$D UHMV_DEBUG_FLAGS=1 UHMV_BULK_CTAS=2" run "c$c nocompute ctas2"
done
} > $O/exp.txt 2>&1
echo done
