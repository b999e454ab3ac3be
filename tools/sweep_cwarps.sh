# consumer warps per CTA: the default build (4 + 1 producer, 3 CTAs/SM) vs a 7 + 1 build at
# 2 CTAs/SM (14 consumer warps per SM instead of 12); usage: bash tools/sweep_cwarps.sh OUT
set -u
O=${1:-gpurun_out/cw}; mkdir -p $O
source tools/sweep.sh
for c in 1 2 3; do ARGS="--config $c"; ENVV="X=1" run "w4 c$c"; done > $O/sweep.txt 2>&1
UHMV_NVCC_EXTRA="-DUHMV_CWARPS=7" python -c "import __graft_entry__ as g; g.build()" > $O/build7.log 2>&1
UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=28 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x -k "device_matches or bit_identical or host_io or peer" > $O/pytest_w7.log 2>&1; echo rc=$? >> $O/pytest_w7.log
for c in 1 2 3; do ARGS="--config $c"
  ENVV="UHMV_BULK_CTAS=2" run "w7 c$c rpc16"
  ENVV="UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=28" run "w7 c$c rpc28"
  ENVV="UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=28 UHMV_STAGE_ELEMS=2816" run "w7 c$c rpc28 st2816"
done >> $O/sweep.txt 2>&1
ARGS="--config 3 --format sym"; ENVV="UHMV_BULK_CTAS=2" run "w7 sym3" >> $O/sweep.txt 2>&1
ARGS="--config 4"; ENVV="UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=28" run "w7 c4 rpc28" >> $O/sweep.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
