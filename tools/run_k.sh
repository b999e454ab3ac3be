set -u
O=gpurun_out/k; mkdir -p $O
source tools/sweep.sh
for c in 3 4 2; do ARGS="--config $c --adjoint"
  ENVV="X=1" run "adj c$c base"
  ENVV="UHMV_ADJ_NEAR_COLS=40" run "adj c$c cols40"
  ENVV="UHMV_ADJ_NEAR_COLS=27" run "adj c$c cols27"
  ENVV="UHMV_ADJ_NEAR_COLS=40 UHMV_NEAR_INTERLEAVE_ADJ=0.3,0.15,0.3,0.25" run "adj c$c cols40 il2"
done > $O/sweep.txt 2>&1
UHMV_ADJ_NEAR_COLS=40 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -q -x -k "device_matches or config_parity or host_io" > $O/pytest_adj40.log 2>&1; echo rc=$? >> $O/pytest_adj40.log
echo done
