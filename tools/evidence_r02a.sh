#!/bin/bash
# Round-2 first GPU pass: tests (incl. the reference on the box), default bench, slice predictor,
# sanitizers.  usage (repo root, under gpurun):  bash tools/evidence_r02a.sh OUTDIR
set -u
O=${1:-gpurun_out/r02a}
mkdir -p "$O"
timeout 1500 python -m pytest tests -q -m gpu -x > "$O/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$O/pytest_gpu.log"
cp gpurun_out/reference_suite.log "$O/" 2>/dev/null
b() { local name=$1; shift; timeout 600 python bench.py "$@" > "$O/bench_$name.json" 2> "$O/bench_$name.err"; }
b cfg3 --steps 50 --warmup 5
b slice_cfg3 --config 3 --slice 2,4,8 --no-cpu-baseline
b slice_cfg4 --config 4 --slice 2,4,8 --no-cpu-baseline
for tool in memcheck synccheck racecheck; do
  for eng in bulk io peer mrtc fused; do
    timeout 400 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $eng > "$O/san_${tool}_${eng}.log" 2>&1
    echo "rc=$?" >> "$O/san_${tool}_${eng}.log"
  done
done
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize.py bulk --cfg1 > "$O/san_memcheck_bulk_cfg1.log" 2>&1; echo "rc=$?" >> "$O/san_memcheck_bulk_cfg1.log"
echo done
