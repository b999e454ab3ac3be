source tools/sweep.sh
O=gpurun_out/small2; mkdir -p $O
for c in 1 2; do
ARGS="--config $c"
ENVV="X=1" run "c$c base"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c$c nearlate"
ENVV="UHMV_SPLIT_Z_ROWS=8 UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c$c z8 nearlate"
ENVV="UHMV_SPLIT_Z_ROWS=13 UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c$c z13 nearlate"
ENVV="UHMV_SPLIT_Z_ROWS=8 UHMV_FAR_ROWS=32 UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c$c z8 far32 nearlate"
ENVV="UHMV_SPLIT_Z_ROWS=8 UHMV_NEAR_INTERLEAVE=0.0,0.0,0.0,1.0" run "c$c z8 nearlast"
ENVV="UHMV_NEAR_INTERLEAVE=0.0,0.0,0.0,1.0" run "c$c nearlast"
done > $O/sweep.txt 2>&1
