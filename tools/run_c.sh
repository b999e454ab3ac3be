set -u
O=gpurun_out/c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_symmetric.py -q -x > $O/pytest_sym.log 2>&1; echo rc=$? >> $O/pytest_sym.log
timeout 300 python bench.py --config 3 --format sym --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_sym_c3.json 2> $O/bench_sym_c3.err
timeout 300 python bench.py --config 1 --format sym --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_sym_c1.json 2> $O/bench_sym_c1.err
timeout 300 python bench.py --config 4 --format sym --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_sym_c4.json 2> $O/bench_sym_c4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 -o $O/full_bulk_cfg2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_sym -s 3 -c 1 -o $O/full_sym_cfg3 python bench.py --config 3 --format sym --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_s3.log 2>&1
echo done
