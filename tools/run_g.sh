set -u
O=gpurun_out/g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_guards.py -q -x -k "sym" > $O/pytest_sym.log 2>&1; echo rc=$? >> $O/pytest_sym.log
for c in 3 4 1; do timeout 300 python bench.py --config $c --format sym --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_sym_c$c.json 2> $O/bench_sym_c$c.err; done
UHMV_PROFILE=1 timeout 300 python bench.py --config 3 --format sym --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_sym_c3_prof.json 2> $O/bench_sym_c3_prof.err
timeout 300 python tools/timeline.py 3 fwd full sym > $O/timeline_sym_c3.txt 2>&1
echo done
