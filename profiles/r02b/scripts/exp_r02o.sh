#!/bin/bash
# confirmation of the config-1 nearfield shares (default now) + refreshed config-1 bench lines
O=gpurun_out/e13; mkdir -p $O
source tools/sweep.sh
{
ARGS="--config 1 --steps 100"
for r in 1 2 3; do
ENVV="X=1" run "c1 default r$r"
ENVV="UHMV_NEAR_INTERLEAVE=0.05,0.05,0.1,0.8" run "c1 old-shares r$r"
done
} > $O/exp.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py tests/test_gpu_reference.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config 1 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --config 1 --l2 hot --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1_l2hot.json 2> $O/bench_cfg1_l2hot.err
timeout 300 python bench.py --config 1 --adjoint --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1_adj.json 2> $O/bench_cfg1_adj.err
timeout 300 python bench.py --config 2 --adjoint --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg2_adj.json 2> $O/bench_cfg2_adj.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:uhmv_bulk_kernel -s 3 -c 1 \
  -o "$O/full_bulk_cfg1" python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > "$O/ncu_b1.log" 2>&1
echo done
