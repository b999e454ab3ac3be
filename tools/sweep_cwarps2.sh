# smaller CTAs: 3 + 1 (4 CTAs/SM) and 2 + 1 (5 CTAs/SM) consumer + producer warps
set -u
O=${1:-gpurun_out/cw2}; mkdir -p $O
source tools/sweep.sh
for c in 1 2 3; do ARGS="--config $c"; ENVV="X=1" run "w4 c$c"; done > $O/sweep.txt 2>&1
for W in 3 2; do
  UHMV_NVCC_EXTRA="-DUHMV_CWARPS=$W" python -c "import __graft_entry__ as g; g.build()" > $O/build$W.log 2>&1
  N=$((W == 3 ? 4 : 5))
  UHMV_BULK_CTAS=$N UHMV_STAGE_ELEMS=1024 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_matches or bit_identical" > $O/pytest_w$W.log 2>&1; echo rc=$? >> $O/pytest_w$W.log
  for c in 1 2 3; do ARGS="--config $c"
    ENVV="UHMV_BULK_CTAS=$N UHMV_STAGE_ELEMS=1024" run "w$W x$N c$c st1024"
    ENVV="UHMV_BULK_CTAS=$N UHMV_STAGE_ELEMS=1024 UHMV_ROWS_PER_CHUNK=$((W*8))" run "w$W x$N c$c st1024 rpc$((W*8))"
    ENVV="UHMV_BULK_CTAS=$N" run "w$W x$N c$c st1408"
  done >> $O/sweep.txt 2>&1
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
