source tools/sweep.sh
for c in 1 2; do
ARGS="--config $c"
ENVV="X=1" run "c$c base"
ENVV="UHMV_BULK_CTAS=2" run "c$c ctas2"
ENVV="UHMV_BULK_CTAS=1" run "c$c ctas1"
ENVV="UHMV_ROWS_PER_CHUNK=8" run "c$c rpc8"
ENVV="UHMV_NEAR_INTERLEAVE=0.5,0.1,0.2,0.2" run "c$c inter"
done
