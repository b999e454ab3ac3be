#!/bin/bash
# consumer-instruction experiments at configs 1-3: single-slot N fast path (lib vs nacc0 lib),
# unsplit narrow N pieces, 16-row column panels
O=gpurun_out/e1; mkdir -p $O
source tools/sweep.sh
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $O/pytest_parity_knobs.log 2>&1; echo "rc=$?" >> $O/pytest_parity_knobs.log
L0=paper_2405_15573_b200/_build/libuhmv_nacc0.so
{
ARGS="--config 2"
ENVV="UHMV_LIB=$L0" run "c2 nacc0"
ENVV="X=1" run "c2 nacc1"
ENVV="UHMV_NOSPLIT=0.3" run "c2 nacc1 nosplit.3"
ENVV="UHMV_PANEL_ROWS=16" run "c2 nacc1 panel16"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3" run "c2 nacc1 panel16 nosplit.3"
ENVV="UHMV_PANEL_ROWS=8 UHMV_NOSPLIT=0.3" run "c2 nacc1 panel8 nosplit.3"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3 UHMV_WIDE_COLS=512" run "c2 nacc1 panel16 nosplit.3 wide512"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3 UHMV_STAGE_ELEMS=1200" run "c2 nacc1 panel16 nosplit.3 st1200"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3 UHMV_PROFILE=1" run "c2 nacc1 panel16 nosplit.3 prof"
ARGS="--config 1"
ENVV="UHMV_LIB=$L0" run "c1 nacc0"
ENVV="X=1" run "c1 nacc1"
ENVV="UHMV_NOSPLIT=0.3" run "c1 nacc1 nosplit.3"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3" run "c1 nacc1 panel16 nosplit.3"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3 UHMV_WIDE_COLS=512" run "c1 nacc1 panel16 nosplit.3 wide512"
ARGS="--config 3"
ENVV="X=1" run "c3 nacc1"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3" run "c3 nacc1 panel16 nosplit.3"
ARGS="--config 3 --adjoint"
ENVV="UHMV_PANEL_ROWS=16 UHMV_NOSPLIT=0.3" run "c3adj nacc1 panel16 nosplit.3"
} > $O/exp.txt 2>&1
echo done
