source tools/sweep.sh
mkdir -p gpurun_out/o
for c in 1 2; do for m in bulk fused phased; do ARGS="--config $c --mode $m"; ENVV="X=1" run "c$c $m"; done; done > gpurun_out/o/sweep.txt 2>&1
