set -u
O=gpurun_out/m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_workloads.py tests/test_hmatrix.py tests/test_abi.py -q -x -k "h_format or h_matvec or abi or library" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
source tools/sweep.sh
ARGS="--config 3 --format h"; ENVV="X=1" run "H3 xwin704" > $O/sweep.txt 2>&1
ENVV="UHMV_XWIN_H=0" run "H3 whole" >> $O/sweep.txt 2>&1
ENVV="UHMV_XWIN_H=1024" run "H3 xwin1024" >> $O/sweep.txt 2>&1
ARGS="--config 3 --format h --adjoint"; ENVV="X=1" run "H3adj xwin704" >> $O/sweep.txt 2>&1
ARGS="--config 2 --format h"; ENVV="X=1" run "H2 xwin704" >> $O/sweep.txt 2>&1
ENVV="UHMV_XWIN_H=0" run "H2 whole" >> $O/sweep.txt 2>&1
ARGS="--config 3"; ENVV="X=1" run "uh3" >> $O/sweep.txt 2>&1
