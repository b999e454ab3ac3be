set -u
O=gpurun_out/e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_guards.py -q -x > $O/pytest_sym_guard.log 2>&1; echo rc=$? >> $O/pytest_sym_guard.log
for c in 3 4 1; do timeout 300 python bench.py --config $c --format sym --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_sym_c$c.json 2> $O/bench_sym_c$c.err; done
timeout 900 python bench.py --config 3 --slice 2,4,8 --slice-exchange peer --no-cpu-baseline > $O/slice_peer_c3.json 2> $O/slice_peer_c3.err
timeout 900 python bench.py --config 4 --slice 2,4,8 --slice-exchange peer --no-cpu-baseline > $O/slice_peer_c4.json 2> $O/slice_peer_c4.err
echo done
