# adjoint nearfield interleave shares (whole-leaf NEAR ops are long: 90 us at configs 3-4)
source tools/sweep.sh
O=gpurun_out/adj; mkdir -p $O
for c in 4 3; do ARGS="--config $c --adjoint"
for iv in "0.4,0.15,0.3,0.15" "0.6,0.2,0.2,0.0" "0.5,0.2,0.3,0.0" "0.5,0.15,0.25,0.1" "0.7,0.1,0.2,0.0" "0.3,0.3,0.3,0.1"; do
  ENVV="UHMV_NEAR_INTERLEAVE_ADJ=$iv" run "adj c$c $iv"
done; done > $O/sweep.txt 2>&1
