#!/bin/bash
# Round-2 (final sessions) evidence on the GPU box: tests, smoke, bench lines, slice predictors, ncu launch list
# and full captures (each ncu only after its command ran clean).
# usage (repo root, under gpurun):  bash tools/evidence_r02.sh OUTDIR
set -u
O=${1:-gpurun_out/ev_b}
mkdir -p "$O"
timeout 1800 python -m pytest tests -q -m gpu > "$O/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$O/pytest_gpu.log"
cp gpurun_out/reference_suite.log "$O/" 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "rc=$?" >> "$O/smoke.log"
b() { local name=$1; shift; timeout 900 python bench.py "$@" > "$O/bench_$name.json" 2> "$O/bench_$name.err"; }
b cfg3 --steps 50 --warmup 5
b ref_cfg3 --impl reference --steps 3 --warmup 3
b cfg1 --config 1 --steps 100 --warmup 5 --no-cpu-baseline
b cfg1_l2hot --config 1 --l2 hot --steps 100 --warmup 5 --no-cpu-baseline
b cfg2 --config 2 --steps 100 --warmup 5 --no-cpu-baseline
b cfg4 --config 4 --steps 30 --warmup 5 --no-cpu-baseline
b cfg5 --config 5 --steps 20 --warmup 5
b cfg3_adj --config 3 --adjoint --steps 50 --warmup 5 --no-cpu-baseline
b cfg4_adj --config 4 --adjoint --steps 30 --warmup 5 --no-cpu-baseline
b cfg3_H --config 3 --format h --steps 30 --warmup 5 --no-cpu-baseline
b sym_cfg3 --config 3 --format sym --steps 50 --warmup 5 --no-cpu-baseline
b cfg3_peer_em8 --config 3 --emulate-ranks 8 --steps 30 --warmup 5 --no-cpu-baseline
b slice_cfg3 --config 3 --slice 2,4,8 --no-cpu-baseline
b slice_cfg4 --config 4 --slice 2,4,8 --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$O/launches_cfg3.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$O/ncu_l.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o "$O/full_bulk_cfg3" python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_b3.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o "$O/full_bulk_cfg1" python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_b1.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o "$O/full_bulk_cfg2" python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_b2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  --metrics smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  -k regex:uhmv_mrtc -s 2 -c 1 -o "$O/full_mrtc_cfg5" python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_m.log" 2>&1
echo done
