#!/bin/bash
# final lines of configs 1-2 (forward + adjoint) with the adjoint copy and its shares
O=gpurun_out/e17; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_stored_form.py tests/test_gpu_workloads.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in 1 2; do
timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg${c}.json 2> $O/bench_cfg${c}.err
timeout 300 python bench.py --config $c --adjoint --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg${c}_adj.json 2> $O/bench_cfg${c}_adj.err
done
timeout 300 python bench.py --config 1 --l2 hot --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg1_l2hot.json 2> $O/bench_cfg1_l2hot.err
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
echo done
