#!/bin/bash
# adjoint copy CT_t (operators under 1 GB): full GPU suite, then adjoint / forward lines of configs 1-2
O=gpurun_out/e16; mkdir -p $O
source tools/sweep.sh
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
{
for c in 2 1; do
ARGS="--config $c --steps 100 --adjoint"
ENVV="UHMV_ADJ_COPY=0" run "c$c adj no-copy"
ENVV="X=1" run "c$c adj copy"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.2,0.1,0.2,0.5" run "c$c adj copy .2.1.2.5"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.4,0.2,0.0,0.4" run "c$c adj copy .4.2.0.4"
ENVV="UHMV_NEAR_INTERLEAVE_ADJ=0.3,0.2,0.1,0.4" run "c$c adj copy .3.2.1.4"
ENVV="X=1" run "c$c adj copy again"
ARGS="--config $c --steps 100"
ENVV="X=1" run "c$c fwd"
done
} > $O/exp.txt 2>&1
for c in 1 2; do
timeout 300 python bench.py --config $c --adjoint --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg${c}_adj.json 2> $O/bench_cfg${c}_adj.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
echo done
