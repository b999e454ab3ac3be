set -u
O=gpurun_out/d; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_symmetric.py -q -x > $O/pytest_sym.log 2>&1; echo rc=$? >> $O/pytest_sym.log
for c in 3 4 1; do timeout 300 python bench.py --config $c --format sym --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_sym_c$c.json 2> $O/bench_sym_c$c.err; done
source tools/sweep.sh
for c in 1 2; do
ARGS="--config $c"
ENVV="UHMV_ROWS_PER_CHUNK=32" run "c$c rpc32"
ENVV="UHMV_ROWS_PER_CHUNK=24" run "c$c rpc24"
ENVV="UHMV_ROWS_PER_CHUNK=40" run "c$c rpc40"
done > $O/sweep_rpc.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_sym -s 3 -c 1 -o $O/full_sym_cfg3 python bench.py --config 3 --format sym --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_s3.log 2>&1
echo done
