set -u
O=gpurun_out/j2; mkdir -p $O
source tools/sweep.sh
for c in 1 2; do ARGS="--config $c"; ENVV="X=1" run "w4 c$c base"; done > $O/sweep.txt 2>&1
ARGS="--config 3 --format sym"; ENVV="X=1" run "w4 sym3" >> $O/sweep.txt 2>&1
UHMV_NVCC_EXTRA="-DUHMV_CWARPS=8 -DUHMV_BULK_REGS=112" python -c "import __graft_entry__ as g; g.build()" > $O/build8.log 2>&1
UHMV_BULK_CTAS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "device_matches_reference or bit_identical" > $O/pytest_w8.log 2>&1; echo rc=$? >> $O/pytest_w8.log
for c in 1 2 3; do ARGS="--config $c"
  ENVV="UHMV_BULK_CTAS=2" run "w8 c$c rpc16"
  ENVV="UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=32" run "w8 c$c rpc32"
done >> $O/sweep.txt 2>&1
ARGS="--config 3 --format sym"; ENVV="UHMV_BULK_CTAS=2" run "w8 sym3" >> $O/sweep.txt 2>&1
ARGS="--config 4"; ENVV="UHMV_BULK_CTAS=2 UHMV_ROWS_PER_CHUNK=32" run "w8 c4 rpc32" >> $O/sweep.txt 2>&1
echo done
