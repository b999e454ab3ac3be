#!/bin/bash
# Round evidence on the GPU box: tests, smoke, bench lines, ncu launch list and full captures.
# usage (from the repo root, under gpurun):  bash tools/evidence.sh OUTDIR
set -u
O=${1:-gpurun_out/ev}
mkdir -p "$O"
timeout 1500 python -m pytest tests -q -m gpu > "$O/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$O/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$O/smoke.log" 2>&1
b() { local name=$1; shift; timeout 600 python bench.py "$@" > "$O/bench_$name.json" 2> "$O/bench_$name.err"; }
b cfg3 --steps 50 --warmup 5
b cfg1 --config 1 --steps 50 --warmup 5 --no-cpu-baseline
b cfg2 --config 2 --steps 50 --warmup 5 --no-cpu-baseline
b cfg4 --config 4 --steps 20 --warmup 5 --no-cpu-baseline
b cfg5 --config 5 --steps 20 --warmup 5
b cfg3_adj --config 3 --adjoint --steps 50 --warmup 5 --no-cpu-baseline
b cfg3_H --config 3 --format h --steps 20 --warmup 5 --no-cpu-baseline
b cfg3_peer_em2 --config 3 --emulate-ranks 2 --steps 30 --warmup 5 --no-cpu-baseline
b cfg3_peer_em4 --config 3 --emulate-ranks 4 --steps 30 --warmup 5 --no-cpu-baseline
b cfg3_peer_em8 --config 3 --emulate-ranks 8 --steps 30 --warmup 5 --no-cpu-baseline
b cfg4_peer_em8 --config 4 --emulate-ranks 8 --steps 20 --warmup 5 --no-cpu-baseline
b ref_cfg3 --impl reference --steps 2 --warmup 1
# ncu: launch list of the default command, then one full capture per engine (each only after
# its command ran clean above)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$O/launches_cfg3.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$O/ncu_l.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o "$O/full_bulk_cfg3" python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_b.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_mrtc -s 2 -c 1 \
  -o "$O/full_mrtc_cfg5" python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_m.log" 2>&1
timeout 900 ncu --set full --clock-control none -k regex:uhmv_bulk_peer -s 3 -c 1 \
  -o "$O/full_peer_em8_cfg3" python bench.py --config 3 --emulate-ranks 8 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_p.log" 2>&1
echo done
