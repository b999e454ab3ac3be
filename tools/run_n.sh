mkdir -p gpurun_out/n
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_symmetric.py tests/test_gpu_reference.py -q -x -k "dropin or sym_golden or real_operator_installed or reference_suite" > gpurun_out/n/pytest.log 2>&1; echo rc=$? >> gpurun_out/n/pytest.log
timeout 600 python bench.py --config 3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/n/bench_cfg3.json 2> gpurun_out/n/bench_cfg3.err
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/n/bench_cfg1.json 2> gpurun_out/n/bench_cfg1.err
