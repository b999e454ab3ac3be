#!/bin/bash
# final check with the adjoint copy on by default: full GPU suite, smoke, adjoint + forward lines
O=gpurun_out/e19; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
b() { local name=$1; shift; timeout 900 python bench.py "$@" > "$O/bench_$name.json" 2> "$O/bench_$name.err"; }
b cfg3 --steps 50 --warmup 5
b cfg3_adj --config 3 --adjoint --steps 50 --warmup 5 --no-cpu-baseline
b cfg4 --config 4 --steps 30 --warmup 5 --no-cpu-baseline
b cfg4_adj --config 4 --adjoint --steps 30 --warmup 5 --no-cpu-baseline
b cfg2 --config 2 --steps 100 --warmup 5 --no-cpu-baseline
b cfg2_adj --config 2 --adjoint --steps 100 --warmup 5 --no-cpu-baseline
b cfg1 --config 1 --steps 100 --warmup 5 --no-cpu-baseline
b cfg1_adj --config 1 --adjoint --steps 100 --warmup 5 --no-cpu-baseline
b cfg5 --config 5 --steps 20 --warmup 5 --no-cpu-baseline
b cfg3_H --config 3 --format h --steps 30 --warmup 5 --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$O/launches_cfg3.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$O/ncu_l.log" 2>&1
echo done
