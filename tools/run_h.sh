set -u
O=gpurun_out/h; mkdir -p $O
for iv in "0.2,0.1,0.3,0.4" "0.3,0.1,0.2,0.4" "0.2,0.1,0.2,0.5" "0.1,0.1,0.3,0.5"; do
  UHMV_SYM_INTERLEAVE=$iv timeout 300 python bench.py --config 3 --format sym --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_sym_c3_$iv.json 2> $O/bench_sym_c3_$iv.err
done
timeout 300 python tools/timeline.py 3 fwd full sym > $O/timeline_sym_c3.txt 2>&1
echo done
