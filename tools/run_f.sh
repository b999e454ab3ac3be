set -u
O=gpurun_out/f; mkdir -p $O
timeout 300 python bench.py --config 3 --format sym --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_sym_c3.json 2> $O/bench_sym_c3.err
UHMV_PROFILE=1 timeout 300 python bench.py --config 3 --format sym --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_sym_c3_prof.json 2> $O/bench_sym_c3_prof.err
timeout 300 python tools/timeline.py 3 fwd full sym > $O/timeline_sym_c3.txt 2>&1
timeout 300 python tools/timeline.py 3 fwd full uh > $O/timeline_uh_c3.txt 2>&1
echo done
